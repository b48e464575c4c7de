"""K4 alone: the hull of a config's reduced set, 10 calls back to back.
    python tools/hull_probe.py [config]   (CHP_HULL_LAUNCHES=1: the multi-launch form)"""
import sys, os, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_1505_00914_b200.device import Context
ctx = Context(0)
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n, p, seed, _ = bench.CONFIGS[cfg]
n = min(n, 300_000_000)
xy = ctx.generate(cfg, seed, p, n)
DL = ctx.reduce(xy, p, q=p)
comp = ctx.compact(DL, p, chain=False, lower=True, upper=True)
torch.cuda.synchronize()
for _ in range(3):
    ctx.hull(comp, p)
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    ctx.hull(comp, p)
b.record(); torch.cuda.synchronize()
print("hull ms", a.elapsed_time(b) / 10, "h", int(comp["_h"].item()) if "_h" in comp else None)
