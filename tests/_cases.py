"""Randomized point-set cases shaped like the reference's test fixtures
(/root/reference/proj/tests/test_util.hpp:13-59: dense, +-1000, sparse,
collinear along a random direction, duplicates of a handful of points,
single column).  numpy RNG, so the draws differ from mt19937_64, but every
case family is covered."""
from __future__ import annotations

import numpy as np


def random_points(rng: np.random.Generator, n: int, lo: int, hi: int) -> np.ndarray:
    return rng.integers(lo, hi + 1, size=(n, 2), dtype=np.int64)


def mixed_case(rng: np.random.Generator, n: int, sparse_extent: int = 50000) -> np.ndarray:
    which = int(rng.integers(0, 7))
    if which == 0:
        return random_points(rng, n, 1, 20)
    if which == 1:
        return random_points(rng, n, -1000, 1000)
    if which == 2:
        return random_points(rng, n, -sparse_extent, sparse_extent)
    if which == 3:
        dx, dy = (int(v) for v in rng.integers(-5, 6, size=2))
        if dx == 0 and dy == 0:
            dx = 1
        k = rng.integers(-100, 101, size=n)
        return np.stack([7 + k * dx, -3 + k * dy], axis=1)
    if which == 4:
        base = random_points(rng, 4, -50, 50)
        return base[rng.integers(0, 4, size=n)]
    if which == 5:
        return np.stack([np.full(n, 42), rng.integers(-500, 501, size=n)], axis=1)
    return random_points(rng, n, 1, 200)


def to_unit_box(pts: np.ndarray) -> tuple[np.ndarray, int]:
    """Translate so x is in [1, p] (the reduce() precondition); y untouched
    except shifted to >= 1."""
    pts = np.asarray(pts, dtype=np.int64)
    out = pts.copy()
    out[:, 0] -= pts[:, 0].min() - 1
    out[:, 1] -= pts[:, 1].min() - 1
    return out.astype(np.int32), int(out[:, 0].max())
