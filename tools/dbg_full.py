import sys, time, os
sys.path.insert(0, '.')
import numpy as np, torch
import oracle, bench
from paper_1505_00914_b200.device import Context
orc = oracle.Oracle(); ctx = Context(0)
print("cpus", os.cpu_count(), os.sched_getaffinity(0).__len__())
os.system("free -g; nproc; lscpu | head -20")
for config in (3, 5):
    n, p, seed, _ = bench.CONFIGS[config]
    t = time.time()
    d = ctx.generate(config, seed, p, n); torch.cuda.synchronize()
    print("gen", time.time() - t, d.shape)
    acc = orc.accumulator(p, p)
    chunk = 1 << 27
    host = torch.empty((chunk, 2), dtype=torch.int32, pin_memory=True)
    tc = ta = 0
    for a in range(0, n, chunk):
        m = min(chunk, n - a)
        t = time.time(); host[:m].copy_(d[a:a + m]); tc += time.time() - t
        t = time.time(); acc.add(host[:m].numpy()); ta += time.time() - t
    print(config, "copy", tc, "add", ta, acc.points)
