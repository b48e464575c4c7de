"""Per-launch timeline of one K1 (+K3) call per config, from CUDA events the
library records between its launches (chp_debug_trace_*: diagnostics, not in
the header).  The events break the launches' programmatic overlap, so the sum
is a little above the bench's K1 time; read the shares.

    python tools/trace_k1.py [config ...] [--flags F]
"""
import ctypes
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1505_00914_b200.device import Context  # noqa: E402


def main():
    args = [a for a in sys.argv[1:]]
    flags = 0
    if "--flags" in args:
        i = args.index("--flags")
        flags = int(args[i + 1])
        del args[i:i + 2]
    configs = [int(a) for a in args] or [2, 4]
    ctx = Context(0)
    L = ctx.L
    L.chp_debug_trace_enable.argtypes = [ctypes.c_void_p, ctypes.c_int]
    L.chp_debug_trace_mark.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
    L.chp_debug_trace_read.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_float),
                                       ctypes.POINTER(ctypes.c_char_p), ctypes.c_int]
    for cfg in configs:
        n, p, seed, _ = bench.CONFIGS[cfg]
        xy = ctx.generate(cfg, seed, p, n)
        DL = ctx.empty_dl(p)
        bufs = {}
        for _ in range(5):
            ctx.reduce(xy, p, q=p, out=DL, flags=flags)
            ctx.compact(DL, p, chain=True, bufs=bufs)
        torch.cuda.synchronize()
        rows = {}
        for rep in range(5):
            L.chp_debug_trace_enable(ctx.h, 1)
            ctx._stream()
            L.chp_debug_trace_mark(ctx.h, b"k1:start")
            ctx.reduce(xy, p, q=p, out=DL, flags=flags)
            L.chp_debug_trace_mark(ctx.h, b"k3")
            ctx.compact(DL, p, chain=True, bufs=bufs)
            L.chp_debug_trace_mark(ctx.h, b"end")
            ms = (ctypes.c_float * 64)()
            lab = (ctypes.c_char_p * 64)()
            k = L.chp_debug_trace_read(ctx.h, ms, lab, 64)
            for i in range(k):
                rows.setdefault(i, (lab[i].decode(), []))[1].append(ms[i] * 1000)
            L.chp_debug_trace_enable(ctx.h, 0)
        tot = sum(min(v) for _, v in rows.values())
        print(f"config {cfg} ({ctx.variant}), n={n}, p={p}: min over 5 reps, us")
        for i in sorted(rows):
            name, v = rows[i]
            print(f"  {i:2d} {name:24s} {min(v):9.1f}  ({min(v) / tot * 100:4.1f}%)")
        print(f"  total {tot:.1f} us")
        del xy


if __name__ == "__main__":
    main()
