"""Micro-timing of K3 alone (warm, back-to-back launches, CUDA events):
python tools/bench_compact.py [p] [iters]"""
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1505_00914_b200.device import Context  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
ctx = Context(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
xy = ctx.generate(2, 2, p, 100_000_000 if p == 65536 else 20 * p)
DL = ctx.empty_dl(p)
ctx.reduce(xy, p, q=p, out=DL)
bufs = {}
for _ in range(10):
    ctx.compact(DL, p, chain=True, bufs=bufs)
torch.cuda.synchronize()
for what in ("chain", "chain+lower+upper", "all"):
    kw = dict(chain=True)
    if what != "chain":
        kw.update(lower=True, upper=True)
    if what == "all":
        kw.update(occ=True, lpairs=True, upperd=True)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    ctx.compact(DL, p, bufs=bufs, **kw)
    a.record(st)
    for _ in range(iters):
        ctx.compact(DL, p, bufs=bufs, **kw)
    b.record(st)
    torch.cuda.synchronize()
    print(f"p={p} {what}: {a.elapsed_time(b) * 1e3 / iters:.2f} us/call")
