"""Python mirror of chp::hulls::melkman (/root/reference/proj/include/chp/hulls.hpp:24)
backed by the device hull (K4).

The reference runs Melkman's deque over the chain (src/hulls.cpp:137-181).
Here the chain's points are re-reduced on the device (bounds, Algorithm 1,
compaction -- exact by the reducer's idempotence) and the hull is the
multi-level monotone chain of csrc/hull.cu.  For every simple chain (every
chain build_polyline emits) the result equals the reference's canonical
hull; for non-simple chains it is the true hull of the chain's points.
"""
from __future__ import annotations

import numpy as np

from .device import default_context
from .reducer import PolygonalChain, _as_int32_points


class Hull:
    """include/chp/geometry.hpp:69-73: strictly convex, CCW, starting at the
    lexicographically smallest vertex; 1 or 2 vertices when degenerate."""

    def __init__(self, vertices):
        self.vertices = np.ascontiguousarray(np.asarray(vertices, dtype=np.int32).reshape(-1, 2))

    def __eq__(self, other) -> bool:
        return isinstance(other, Hull) and np.array_equal(self.vertices, other.vertices)

    def __repr__(self) -> str:
        return f"Hull({self.vertices.tolist()})"

    def tolist(self):
        return [tuple(v) for v in self.vertices.tolist()]


def melkman(chain: PolygonalChain) -> Hull:
    """ValueError on an empty chain (src/hulls.cpp:139)."""
    pts = chain.vertices if isinstance(chain, PolygonalChain) else chain
    xy = _as_int32_points(pts)
    if len(xy) == 0:
        raise ValueError("melkman: empty chain")
    res = default_context().precondition_host(xy, chain=False, hull=True)
    return Hull(res["hull"])


def hull_of_points(points) -> Hull:
    """Exact hull of an arbitrary point set through the same device path."""
    return melkman(PolygonalChain(_as_int32_points(points)))
