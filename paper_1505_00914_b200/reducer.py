"""Python mirror of chp::reducer (/root/reference/proj/include/chp/reducer.hpp)
backed by the B200 kernels.  Same names, argument meaning and error
behaviour: ValueError wherever the reference throws std::invalid_argument.

    arr   = reduce(points, width, q=None)        # reducer.hpp:65-67
    chain = build_polyline(arr)                  # reducer.hpp:76
    text  = serialize(arr)                       # reducer.hpp:79
    res   = precondition(points)                 # reducer.hpp:100-101
"""
from __future__ import annotations

import io
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from .device import default_context


class Kind(Enum):
    """occupancy::Kind (include/chp/occupancy.hpp:191).  Both kinds yield the
    same ordering; the device path keeps the array (bit words) form."""
    array = 0
    tree = 1


@dataclass(frozen=True)
class ColumnExtremes:
    """include/chp/reducer.hpp:19-25"""
    lo: int = 0
    hi: int = -1
    valid: bool = False


@dataclass(frozen=True)
class BoundingBox:
    """include/chp/geometry.hpp:51-61"""
    x_min: int = 0
    x_max: int = 0
    y_min: int = 0
    y_max: int = 0

    def width(self) -> int:
        return self.x_max - self.x_min + 1

    def height(self) -> int:
        return self.y_max - self.y_min + 1


@dataclass
class PolygonalChain:
    """include/chp/reducer.hpp:53-57; vertices as an (s,2) int array."""
    vertices: np.ndarray

    def __eq__(self, other) -> bool:
        return isinstance(other, PolygonalChain) and np.array_equal(self.vertices, other.vertices)

    def tolist(self):
        return [tuple(v) for v in self.vertices.tolist()]


class ExtremalArray:
    """include/chp/reducer.hpp:31-51.  `pairs` is L in serialize form:
    (lo, hi) per slot, empty slots (width+1, -1).  occ_words are the
    BlockedBitset<uint64_t> words."""

    def __init__(self, pairs: np.ndarray, occ_words: np.ndarray | None = None, major_offset: int = 0,
                 minor_offset: int = 0, axis_swapped: bool = False, occ_kind: Kind = Kind.array,
                 _chain: np.ndarray | None = None):
        self.pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
        self.major_offset = int(major_offset)
        self.minor_offset = int(minor_offset)
        self.axis_swapped = bool(axis_swapped)
        self.occ_kind = occ_kind
        self._occ = occ_words
        self._chain = _chain  # device-built Lemma-1 chain, valid while pairs are unchanged

    def width(self) -> int:
        return len(self.pairs)

    @property
    def valid(self) -> np.ndarray:
        return self.pairs[:, 0] <= self.pairs[:, 1]

    @property
    def entries(self) -> list[ColumnExtremes]:
        v = self.valid
        return [ColumnExtremes(int(a), int(b), True) if ok else ColumnExtremes()
                for (a, b), ok in zip(self.pairs.tolist(), v.tolist())]

    def occ_indices(self) -> list[int]:
        """1-based valid slots in increasing order (Index::indices)."""
        return (np.nonzero(self.valid)[0] + 1).tolist()

    def to_original(self, slot: int, value: int) -> tuple[int, int]:
        major = slot + self.major_offset
        minor = value + self.minor_offset
        return (minor, major) if self.axis_swapped else (major, minor)

    def _device_chain(self) -> np.ndarray:
        if self._chain is None:
            if not self.valid.any():
                return np.empty((0, 2), np.int32)
            self._chain = default_context().polyline_host(self.pairs, self.width(), self.major_offset,
                                                          self.minor_offset, self.axis_swapped)
        return self._chain

    def valid_count(self) -> int:
        """src/reducer.cpp:42-49"""
        return int(len(self._device_chain()))

    def valid_points(self) -> np.ndarray:
        """src/reducer.cpp:51-60 (slot order, lo before hi)."""
        return self._device_chain().copy()


def reduce(points, width: int, q: int | None = None, occ_kind: Kind = Kind.array) -> ExtremalArray:
    """Algorithm 1 on the device (src/reducer.cpp:69-79).  Raises
    ValueError for width < 1 or any coordinate outside x in [1,width],
    y >= 1 (y <= q when q is given)."""
    if int(width) < 1:
        raise ValueError("reduce: width must be >= 1")
    xy = _as_int32_points(points)
    ctx = default_context()
    out = ctx.pipeline_host(xy, int(width), q, L=True, occ=True, chain=True)
    return ExtremalArray(out["L"], out["occ"], occ_kind=occ_kind, _chain=out["chain"])


def build_polyline(arr: ExtremalArray) -> PolygonalChain:
    """Lemma-1 chain (src/reducer.cpp:108-119); ValueError when empty."""
    chain = arr._device_chain()
    if len(chain) == 0:
        raise ValueError("build_polyline: no valid points")
    return PolygonalChain(chain.copy())


def serialize(arr: ExtremalArray, os: io.TextIOBase | None = None) -> str:
    """One line per slot, "i lo hi", empty slots "i <width+1> -1"
    (src/reducer.cpp:121-130)."""
    lines = [f"{i} {lo} {hi}\n" for i, (lo, hi) in enumerate(arr.pairs.tolist(), start=1)]
    w1 = arr.width() + 1
    v = arr.valid.tolist()
    text = "".join(ln if ok else f"{i} {w1} -1\n" for i, (ln, ok) in enumerate(zip(lines, v), start=1))
    if os is not None:
        os.write(text)
    return text


@dataclass
class PreconditionOptions:
    """include/chp/reducer.hpp:81-85"""
    second_scan: bool = False
    auto_axis: bool = False
    occ_kind: Kind = Kind.array


@dataclass
class PreconditionResult:
    """include/chp/reducer.hpp:87-95"""
    array: ExtremalArray
    chain: PolygonalChain
    bbox: BoundingBox
    t_bounds: float = 0.0
    t_reduce: float = 0.0
    t_extract: float = 0.0

    def total(self) -> float:
        return self.t_bounds + self.t_reduce + self.t_extract


def precondition(points, options: PreconditionOptions | None = None) -> PreconditionResult:
    """Steps 1-3 on the device (src/reducer.cpp:132-178), x-only mode:
    bounds, fold with x_off = x_min - 1 and y untranslated, Lemma-1 chain."""
    import time

    options = options or PreconditionOptions()
    xy = _as_int32_points(points)
    if len(xy) == 0:
        raise ValueError("precondition: empty input")
    ctx = default_context()
    t0 = time.perf_counter()
    x_min, x_max, y_min, y_max = ctx.precondition_host(xy, chain=False)["bbox"]
    bbox = BoundingBox(x_min, x_max, y_min, y_max)
    full_bounds = options.second_scan or options.auto_axis
    swap = options.auto_axis and bbox.height() < bbox.width()  # bucket along the short side
    t1 = time.perf_counter()
    res = ctx.precondition_host(xy[:, ::-1].copy() if swap else xy, chain=True)
    # Device L stores untranslated minor values; translate them when the
    # reference does (full_bounds: src/reducer.cpp:156-158).
    minor_off = ((x_min if swap else y_min) - 1) if full_bounds else 0
    pairs = res["L"].astype(np.int64)
    valid = pairs[:, 0] <= pairs[:, 1]
    pairs[valid] -= minor_off
    major_off = (y_min if swap else x_min) - 1
    chain = res["chain"][:, ::-1].copy() if swap else res["chain"]
    arr = ExtremalArray(pairs.astype(np.int32), major_offset=major_off, minor_offset=minor_off, axis_swapped=swap,
                        occ_kind=options.occ_kind, _chain=chain)
    t2 = time.perf_counter()
    if options.second_scan:
        arr = second_scan(arr, options.occ_kind)
        chain = build_polyline(arr).vertices
    t3 = time.perf_counter()
    return PreconditionResult(arr, PolygonalChain(np.ascontiguousarray(chain)), bbox, t_bounds=t1 - t0,
                              t_reduce=t2 - t1, t_extract=t3 - t2)


def second_scan(arr: ExtremalArray, occ_kind: Kind = Kind.array) -> ExtremalArray:
    """Re-bucket the survivors along the other axis (src/reducer.cpp:81-106):
    the <= 2w survivors are re-reduced on the device with axes swapped."""
    pts = arr.valid_points().astype(np.int64)
    swapped = not arr.axis_swapped
    if len(pts) == 0:
        w = arr.width()
        return ExtremalArray(np.tile(np.array([[w + 1, -1]], np.int32), (w, 1)), axis_swapped=swapped,
                             occ_kind=occ_kind)
    major = pts[:, 1] if swapped else pts[:, 0]
    minor = pts[:, 0] if swapped else pts[:, 1]
    major_min, major_max, minor_min = int(major.min()), int(major.max()), int(minor.min())
    rebased = np.stack([major - (major_min - 1), minor - (minor_min - 1)], axis=1)
    out = reduce(rebased, major_max - major_min + 1, None, occ_kind)
    out.major_offset = major_min - 1
    out.minor_offset = minor_min - 1
    out.axis_swapped = swapped
    out._chain = None  # the cached chain was built without these offsets
    return out


def translate(points, bbox: BoundingBox) -> np.ndarray:
    """src/reducer.cpp:62-67 on the device."""
    from .kernels import translate as ktranslate

    xy = _as_int32_points(points)
    return ktranslate(xy, 1 - bbox.x_min, 1 - bbox.y_min)


def _as_int32_points(points) -> np.ndarray:
    a = np.asarray(points)
    if a.size == 0:
        return np.empty((0, 2), np.int32)
    a = a.reshape(-1, 2)
    if a.dtype != np.int32:
        if np.any(a > np.iinfo(np.int32).max) or np.any(a < np.iinfo(np.int32).min):
            raise ValueError("coordinates exceed the int32 range of the device path (DESIGN.md: narrowing)")
        a = a.astype(np.int32)
    return np.ascontiguousarray(a)
