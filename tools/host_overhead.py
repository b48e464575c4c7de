import time, torch, sys
sys.path.insert(0, '/root/repo')
from paper_1505_00914_b200.device import Context
ctx = Context(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
p = 65536
xy = ctx.generate(2, 2, p, 1_000_000)   # small input: GPU fast, host-bound
DL = ctx.empty_dl(p); bufs = {}
for _ in range(20):
    ctx.reduce(xy, p, q=p, out=DL); ctx.compact(DL, p, chain=True, bufs=bufs)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(500):
    ctx.reduce(xy, p, q=p, out=DL)
t1 = time.perf_counter()
for _ in range(500):
    ctx.compact(DL, p, chain=True, bufs=bufs)
t2 = time.perf_counter()
torch.cuda.synchronize()
print("host us/call: reduce %.1f compact %.1f" % ((t1 - t) / 500 * 1e6, (t2 - t1) / 500 * 1e6))
