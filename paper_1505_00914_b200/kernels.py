"""Python mirror of chp::kernels (/root/reference/proj/include/chp/kernels.hpp:15-38)
on the device: min_max is K0 (csrc/misc.cu), translate the elementwise
kernel; active_kernel() names the device path instead of "avx2"/"scalar"."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .device import default_context
from .reducer import BoundingBox, _as_int32_points


@dataclass(frozen=True)
class MinMax:
    x_min: int
    x_max: int
    y_min: int
    y_max: int


def min_max(points) -> MinMax:
    """ValueError on empty input (src/kernels.cpp:55-58)."""
    xy = _as_int32_points(points)
    if len(xy) == 0:
        raise ValueError("min_max: empty input")
    b = default_context().precondition_host(xy, chain=False)["bbox"]
    return MinMax(*b)


def find_bounds(points) -> BoundingBox:
    """geometry.cpp find_bounds (src/geometry.cpp:12-17 in the reference numbering)."""
    m = min_max(points)
    return BoundingBox(m.x_min, m.x_max, m.y_min, m.y_max)


def translate(points, dx: int, dy: int) -> np.ndarray:
    """out[i] = in[i] + (dx, dy) on the device (src/kernels.cpp:60-65)."""
    xy = _as_int32_points(points)
    if len(xy) == 0:
        return xy.copy()
    ctx = default_context()
    d = torch.from_numpy(xy).to(torch.device("cuda", ctx.device))
    out = ctx.translate(d, int(dx), int(dy))
    return out.cpu().numpy()


def active_kernel() -> str:
    return "sm_100a"
