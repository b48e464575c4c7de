"""K3 (chp_compact) alone: the merged L of a config, then back-to-back
compactions timed with CUDA events (chain output only, as the bench step).

    python tools/k3_bench.py [config ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1505_00914_b200.device import Context  # noqa: E402


def main():
    configs = [int(a) for a in sys.argv[1:]] or [2, 4]
    ctx = Context(0)
    for cfg in configs:
        n, p, seed, _ = bench.CONFIGS[cfg]
        n = min(n, 200_000_000)
        xy = ctx.generate(cfg, seed, p, n)
        DL = ctx.reduce(xy, p, q=p)
        del xy
        bufs = {}
        for _ in range(20):
            ctx.compact(DL, p, chain=True, bufs=bufs)
        torch.cuda.synchronize()
        reps = 100
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)
        a.record()
        for _ in range(reps):
            ctx.compact(DL, p, chain=True, bufs=bufs)
        b.record()
        torch.cuda.synchronize()
        s = int(bufs["counts"][0].item())
        print(f"config {cfg}: p={p} s={s}: K3 {a.elapsed_time(b) / reps * 1000:.2f} us per call (back to back)")


if __name__ == "__main__":
    main()
