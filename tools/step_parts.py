"""Marginal cost of K3 inside the bench step: K steps of K1 alone vs K1+K3
(same stream, events only around the whole loop), per config.

    python tools/step_parts.py [config ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1505_00914_b200.device import Context  # noqa: E402


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(4_000_000)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1000


def main():
    configs = [int(a) for a in sys.argv[1:]] or [2, 4]
    ctx = Context(0)
    for cfg in configs:
        n, p, seed, _ = bench.CONFIGS[cfg]
        n = min(n, 1_000_000_000)
        xy = ctx.generate(cfg, seed, p, n)
        DL = ctx.empty_dl(p)
        bufs = {}
        reps = 20 if n >= 1e9 else 100
        k1 = timed(lambda: ctx.reduce(xy, p, q=p, out=DL), reps)
        k13 = timed(lambda: (ctx.reduce(xy, p, q=p, out=DL), ctx.compact(DL, p, chain=True, bufs=bufs)), reps)
        k3 = timed(lambda: ctx.compact(DL, p, chain=True, bufs=bufs), 100)
        print(f"config {cfg}: K1 {k1:.1f} us, K1+K3 {k13:.1f} us (K3 marginal {k13 - k1:.1f}), K3 alone {k3:.1f} us")
        del xy


if __name__ == "__main__":
    main()
