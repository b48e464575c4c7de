"""K3 phase timeline per tile (instrumentation build: CHP_NVCC_EXTRA=-DCHP_K3_TIMING=1):
stamps at pdl_wait exit (0), after the local scan (1), after the look-back (2), after
the output stage (3); printed as distributions over the tiles of one call.

    CHP_NVCC_EXTRA=-DCHP_K3_TIMING=1 python tools/k3_phases.py [config]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1505_00914_b200 import _build  # noqa: E402

_build.build(force=True)
from paper_1505_00914_b200.device import Context  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    ctx = Context(0)
    n, p, seed, _ = bench.CONFIGS[cfg]
    n = min(n, 200_000_000)
    xy = ctx.generate(cfg, seed, p, n)
    DL = ctx.reduce(xy, p, q=p)
    bufs = {}
    for _ in range(10):
        ctx.compact(DL, p, chain=True, bufs=bufs)
    torch.cuda.synchronize()
    ctx.compact(DL, p, chain=True, bufs=bufs)
    torch.cuda.synchronize()
    buf = np.zeros((4096, 6), np.uint64)
    ctx.L.chp_debug_k3_phase.argtypes = [ctypes.c_void_p]
    assert ctx.L.chp_debug_k3_phase(buf.ctypes.data_as(ctypes.c_void_p)) == 0
    ntiles = int((buf[:, 0] > 0).sum())
    t = buf[:ntiles, :4].astype(np.int64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1000.0
    print(f"config {cfg}: {ntiles} tiles; us from the first tile's start")
    names = ["start", "scanned", "looked back", "written"]
    for k in range(4):
        v = rel[:, k]
        print(f"  {names[k]:12s} min {v.min():7.2f}  median {np.median(v):7.2f}  max {v.max():7.2f}")
    d = np.diff(rel, axis=1)
    for k, nm in enumerate(["load+scan", "look-back", "stage+write"]):
        print(f"  {nm:12s} per tile: median {np.median(d[:, k]):6.2f}  max {d[:, k].max():6.2f}")
    order = np.argsort(rel[:, 0])
    print("  start of tiles by index (every 64th):", [round(float(rel[i, 0]), 2) for i in range(0, ntiles, 64)])


if __name__ == "__main__":
    main()
