"""Diagnostic: C4's K1 time against where its buffers land (allocation
order and padding).  SEQ is a comma list of allocations, in order:
pad<MB>, xy, dl; then K1 is timed (median of 20 calls)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1505_00914_b200.device import Context  # noqa: E402

cfg = int(os.environ.get("CFG", "4"))
n, p, seed, _ = bench.CONFIGS[cfg]
ctx = Context(0)
if os.environ.get("STREAM") == "1":
    torch.cuda.set_stream(torch.cuda.Stream())
keep = []
xy = DL = None
for s in os.environ.get("SEQ", "xy,dl").split(","):
    if s.startswith("pad"):
        keep.append(torch.empty(int(s[3:]) << 20, dtype=torch.uint8, device="cuda"))
    elif s == "xy":
        xy = ctx.generate(cfg, seed, p, n)
    elif s == "dl":
        DL = ctx.empty_dl(p)
    elif s.startswith("dloff"):
        # DL at a chosen offset (MB) from a 32 MB-aligned virtual address
        words = ctx.empty_dl(p).numel()
        big = torch.empty((words * 4 + (64 << 20)) // 4, dtype=torch.int32, device="cuda")
        keep.append(big)
        base = (big.data_ptr() + (32 << 20) - 1) // (32 << 20) * (32 << 20)
        off = (base - big.data_ptr() + (int(s[5:]) << 20)) // 4
        DL = big[off:off + words]
K3 = os.environ.get("K3") == "1"
bufs = {}


def timed():
    for _ in range(5):
        ctx.reduce(xy, p, q=p, out=DL)
        if K3:
            ctx.compact(DL, p, chain=True, bufs=bufs)
    torch.cuda.synchronize()
    ev = []
    torch.cuda._sleep(4_000_000)
    for _ in range(20):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        ctx.reduce(xy, p, q=p, out=DL)
        b.record()
        ev.append((a, b))
        if K3:
            ctx.compact(DL, p, chain=True, bufs=bufs)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) * 1e3 / 20


r = [timed() for _ in range(3)]
print("%-16s K1 us (20 back to back) %s" % (os.environ.get("SEQ"), " ".join("%.1f" % v for v in r)),
      "xy %#x dl %#x" % (xy.data_ptr(), DL.data_ptr()), flush=True)
