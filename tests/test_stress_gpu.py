"""Randomized stress of the device paths against the oracle: random widths
(1 .. 2^20), y windows (narrow, 16-bit, 2^20, unbounded), x offsets, sizes
around the chunk and vector boundaries, clustered or uniform points, a few
invalid points, pinned and pageable host buffers, and every forced K1
variant through the device API.  Seeded, so a failure reproduces."""
import os

import numpy as np
import pytest
import torch

from paper_1505_00914_b200 import _lib

pytestmark = pytest.mark.gpu
SEEDS = int(os.environ.get("CHP_STRESS_SEEDS", "40"))  # a one-off soak: CHP_STRESS_SEEDS=1000

FORCE = [0, _lib.REDUCE_FORCE_GLOBAL, _lib.REDUCE_FORCE_SMEM32, _lib.REDUCE_FORCE_SMEM16,
         _lib.REDUCE_FORCE_SAMPLED, _lib.REDUCE_FORCE_FILTER, _lib.REDUCE_FORCE_FILTER8,
         _lib.REDUCE_FORCE_GLOBAL | _lib.REDUCE_WARP_AGG, _lib.REDUCE_FORCE_FILTER | _lib.REDUCE_BLOCKED,
         _lib.REDUCE_FORCE_SAMPLED | _lib.REDUCE_SAMPLE_SPLIT, _lib.REDUCE_FORCE_FILTER | 128,
         _lib.REDUCE_FORCE_FILTER | 256 | 4096]


def draw_case(rng):
    width = int(rng.choice([1, 2, 7, 64, 257, 4096, 65536, 65537, 300_000, 1 << 20]))
    ywin = rng.choice(["tiny", "16", "20", "none"])
    q = {"tiny": int(rng.integers(1, 50)), "16": 65536, "20": 1 << 20, "none": None}[ywin]
    # (5 M: past the 4 Mi points where the group filter runs in phases)
    n = int(rng.choice([1, 2, 3, 15, 16, 17, 1000, 65_537, 1_000_003, 3_000_001, 5_000_001]))
    if rng.random() < 0.5:
        x = rng.integers(1, width + 1, n)
    else:  # a few hot clusters of columns
        centers = rng.integers(1, width + 1, 4)
        x = np.clip(centers[rng.integers(0, 4, n)] + rng.integers(-3, 4, n), 1, width)
    ymax = q if q is not None else 2**31 - 1
    if rng.random() < 0.5:
        y = rng.integers(1, min(ymax, 2**31 - 1) + 1, n)
    else:
        mid = rng.integers(1, min(ymax, 2**31 - 1) + 1)
        y = np.clip(mid + rng.integers(-100, 101, n), 1, ymax)
    xy = np.stack([x, y], 1).astype(np.int32)
    invalid = rng.random() < 0.15
    if invalid:
        k = int(rng.integers(0, n))
        xy[k] = rng.choice([(0, 1), (width + 1, 1), (1, 0)] + ([(1, q + 1)] if q is not None else []))
    return xy, width, q, invalid


@pytest.mark.parametrize("seed", range(SEEDS))
def test_stress_host_pipeline(ctx, orc, seed):
    rng = np.random.default_rng(1000 + seed)
    xy, width, q, invalid = draw_case(rng)
    if rng.random() < 0.5:
        t = torch.empty(xy.shape, dtype=torch.int32, pin_memory=True)
        t.copy_(torch.from_numpy(xy))
        xy = t.numpy()
    if invalid:
        with pytest.raises(ValueError):
            ctx.pipeline_host(xy, width, q)
        return
    out = ctx.pipeline_host(xy, width, q, L=True, chain=True)
    ref = orc.pipeline(xy, width, q)
    assert np.array_equal(out["L"], ref["L"])
    assert np.array_equal(out["chain"], ref["chain"])


@pytest.mark.parametrize("seed", range(SEEDS))
def test_stress_device_variants(ctx, orc, seed):
    rng = np.random.default_rng(5000 + seed)
    xy, width, q, invalid = draw_case(rng)
    flags = int(rng.choice(FORCE))
    d = torch.from_numpy(xy).cuda()
    DL = ctx.reduce(d, width, q=q, flags=flags)
    if invalid:
        with pytest.raises(ValueError):
            ctx.check(DL, width)
        return
    ctx.check(DL, width)
    comp = ctx.compact(DL, width, chain=True, lpairs=True)
    torch.cuda.synchronize()
    ref = orc.pipeline(xy, width, q)
    s = int(comp["counts"][0].item())
    assert np.array_equal(comp["lpairs"][:width].cpu().numpy(), ref["L"])
    assert s == ref["s"] and np.array_equal(comp["chain"][:s].cpu().numpy(), ref["chain"])


@pytest.mark.parametrize("seed", range(SEEDS // 2))
def test_stress_precondition(ctx, orc, seed):
    rng = np.random.default_rng(9000 + seed)
    n = int(rng.choice([1, 5, 1000, 200_001, 2_000_003]))
    span_x = int(rng.choice([1, 100, 65536, 1 << 20]))
    span_y = int(rng.choice([1, 300, 65536, 1 << 24]))
    ox = int(rng.integers(-2**31, 2**31 - span_x))
    oy = int(rng.integers(-2**31, 2**31 - span_y))
    xy = np.stack([ox + rng.integers(0, span_x, n), oy + rng.integers(0, span_y, n)], 1).astype(np.int32)
    out = ctx.precondition_host(xy, chain=True, hull=True)
    ref = orc.precondition(xy)
    assert out["bbox"] == ref["bbox"]
    assert np.array_equal(out["chain"], ref["chain"])
    assert np.array_equal(out["hull"], ref["hull"])
