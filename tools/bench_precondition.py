"""End-to-end time of the drop-in precondition (chp_precondition_host): bounds,
translation, K1, K3 from a host int32 buffer (pinned or pageable), chain back.
python tools/bench_precondition.py [n]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1505_00914_b200.device import Context, generate_host  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
ctx = Context(0)
xy = generate_host(2, 2, 65536, n)
xy[:, 0] -= 30000
xy[:, 1] += 123456
pin = torch.empty((n, 2), dtype=torch.int32, pin_memory=True)
pin.copy_(torch.from_numpy(xy))
for name, buf in (("pageable", xy), ("pinned", pin.numpy())):
    ctx.precondition_host(buf, chain=True)
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        out = ctx.precondition_host(buf, chain=True)
        ts.append(time.perf_counter() - t)
    t = min(ts)
    print(f"precondition {name}: {t * 1e3:.1f} ms  {n / t / 1e9:.2f} Gpts/s  h2d {ctx.last_h2d_bytes / 1e6:.0f} MB  "
          f"variant {ctx.variant}  s={len(out['chain'])}")
