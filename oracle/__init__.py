"""CPU checkers for the chp hot path -- TEST INFRASTRUCTURE ONLY.

`Oracle` wraps oracle/_build/liboracle.so (the plain-C restatement in
chp_oracle.c, every function citing the reference file:line it restates).
`Reference` wraps oracle/_ref/libchpref.so: the reference's own sources
compiled by oracle/Makefile, available wherever that .so was built (here,
and on the GPU box because built .so files travel with the snapshot).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this
package, and only as the checker / CPU baseline.  The product package
(paper_1505_00914_b200) never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import c_char_p, c_double, c_int, c_int64, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
GEN_SO = os.path.join(HERE, "_build", "libchpgen.so")
REF_SO = os.path.join(HERE, "_ref", "libchpref.so")
REF_SRC = "/root/reference/proj"


def build(ref: bool | None = None) -> None:
    """Compile the restatement and, when the reference tree is present, the
    reference itself (oracle/_ref)."""
    targets = [ORACLE_SO, GEN_SO]
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        targets.append("ref")
        # the reference's acceptance suite linked to the device drop-in
        # (needs the built library; tests/test_acceptance_gpu.py runs it)
        if os.path.exists(os.path.join(HERE, "..", "paper_1505_00914_b200", "lib", "libchp_b200.so")):
            targets.append("acceptance")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


_gen_lib = None


def generate(config: int, seed: int, p: int, n: int, offset: int = 0, threads: int = 0) -> np.ndarray:
    """Config 2-5 points on the host from oracle/_build/libchpgen.so (the
    product's generator header compiled for the host), for the CPU legs that
    must not load libchp_b200.so.  Same bytes as Context.generate."""
    global _gen_lib
    if _gen_lib is None:
        if not os.path.exists(GEN_SO):
            build(ref=False)
        _gen_lib = ctypes.CDLL(GEN_SO)
        _gen_lib.gen_points.restype = c_int
        _gen_lib.gen_points.argtypes = [c_int, c_uint64, c_int64, c_uint64, c_uint64, c_void_p, c_int]
    L = _gen_lib
    out = np.empty((n, 2), np.int32)
    if L.gen_points(int(config), int(seed), int(p), int(offset), int(n), _p(out), int(threads or os.cpu_count() or 1)):
        raise ValueError(f"generate: bad config {config} / p {p}")
    return out


def _p(a: np.ndarray) -> c_void_p:
    return a.ctypes.data_as(c_void_p)


def _xy(points) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(points, dtype=np.int32).reshape(-1, 2))
    return a


class Oracle:
    """The C restatement (chp_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = ctypes.CDLL(path)
        L.or_fnv1a64.restype = c_uint64
        L.or_fnv1a64.argtypes = [c_void_p, ctypes.c_size_t]
        L.or_gen_uniform_box.argtypes = [c_uint64, c_int64, c_uint64, c_void_p]
        L.or_reduce.restype = c_int
        L.or_reduce.argtypes = [c_void_p, c_uint64, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]
        L.or_bucket.argtypes = [c_void_p, c_uint64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]
        L.or_L_pairs.argtypes = [c_int64, c_void_p, c_void_p, c_void_p, c_void_p]
        L.or_serialize.restype = ctypes.c_size_t
        L.or_serialize.argtypes = [c_int64, c_void_p, c_void_p, c_void_p, c_char_p, ctypes.c_size_t]
        L.or_valid_count.restype = c_int64
        L.or_valid_count.argtypes = [c_int64, c_void_p, c_void_p, c_void_p]
        L.or_build_polyline.restype = c_int64
        L.or_build_polyline.argtypes = [c_int64, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int, c_void_p]
        L.or_ns_chain.restype = c_int64
        L.or_ns_chain.argtypes = [c_int64, c_void_p, c_void_p, c_void_p, c_int64, c_void_p]
        for fn in ("or_melkman", "or_canonicalize", "or_monotone_hull"):
            getattr(L, fn).restype = c_int64
            getattr(L, fn).argtypes = [c_void_p, c_int64, c_void_p]
        L.or_min_max.argtypes = [c_void_p, c_uint64, c_void_p]
        L.or_reduce_accumulate_mt.restype = c_int
        L.or_reduce_accumulate_mt.argtypes = [c_void_p, c_uint64, c_int64, c_int64, c_int, c_void_p, c_void_p,
                                              c_void_p]
        L.or_occ_from_valid.argtypes = [c_int64, c_void_p, c_void_p]
        self.L = L

    # -- inputs / digests
    def fnv(self, a: np.ndarray | bytes) -> str:
        if isinstance(a, (bytes, bytearray)):
            buf = ctypes.create_string_buffer(bytes(a), len(a))
            return f"{self.L.or_fnv1a64(buf, len(a)):016x}"
        a = np.ascontiguousarray(a)
        return f"{self.L.or_fnv1a64(_p(a), a.nbytes):016x}"

    def uniform_box(self, n: int, p: int, seed: int) -> np.ndarray:
        xy = np.empty((n, 2), dtype=np.int32)
        self.L.or_gen_uniform_box(n, p, seed, _p(xy))
        return xy

    # -- reduction
    def reduce(self, points, width: int, q: int | None = None):
        """reducer::reduce (src/reducer.cpp:69-79). Returns a dict with
        lo, hi, valid, occ; raises ValueError where the reference throws
        std::invalid_argument."""
        xy = _xy(points)
        w = max(int(width), 1)
        lo = np.zeros(w, np.int32)
        hi = np.zeros(w, np.int32)
        valid = np.zeros(w, np.uint8)
        occ = np.zeros((w + 63) // 64, np.uint64)
        rc = self.L.or_reduce(_p(xy), len(xy), int(width), -1 if q is None else int(q),
                              _p(lo), _p(hi), _p(valid), _p(occ))
        if rc != 0:
            raise ValueError("reduce: coordinate out of range")
        return {"width": int(width), "lo": lo, "hi": hi, "valid": valid, "occ": occ}

    def accumulator(self, width: int, q: int | None = None) -> "Accumulator":
        """SURVEY.md 8(c)'s chunked reduce for inputs beyond host RAM."""
        return Accumulator(self, width, q)

    def L_pairs(self, arr) -> np.ndarray:
        out = np.empty((arr["width"], 2), np.int32)
        self.L.or_L_pairs(arr["width"], _p(arr["lo"]), _p(arr["hi"]), _p(arr["valid"]), _p(out))
        return out

    def serialize(self, arr) -> str:
        n = self.L.or_serialize(arr["width"], _p(arr["lo"]), _p(arr["hi"]), _p(arr["valid"]), None, 0)
        buf = ctypes.create_string_buffer(n)
        self.L.or_serialize(arr["width"], _p(arr["lo"]), _p(arr["hi"]), _p(arr["valid"]), buf, n)
        return buf.raw[:n].decode()

    def valid_count(self, arr) -> int:
        return int(self.L.or_valid_count(arr["width"], _p(arr["lo"]), _p(arr["hi"]), _p(arr["occ"])))

    def build_polyline(self, arr, major_off: int = 0, minor_off: int = 0, swapped: bool = False):
        out = np.empty((2 * arr["width"] + 1, 2), np.int32)
        s = self.L.or_build_polyline(arr["width"], _p(arr["lo"]), _p(arr["hi"]), _p(arr["occ"]),
                                     major_off, minor_off, int(swapped), _p(out))
        if s < 0:
            raise ValueError("build_polyline: no valid points")
        return out[:s].copy()

    def ns_chain(self, arr, major_off: int = 0):
        out = np.empty((2 * arr["width"] + 1, 2), np.int32)
        s = self.L.or_ns_chain(arr["width"], _p(arr["lo"]), _p(arr["hi"]), _p(arr["occ"]), major_off, _p(out))
        if s < 0:
            raise ValueError("ns_chain: no valid points")
        return out[:s].copy()

    def _hull(self, fn, points) -> np.ndarray:
        xy = _xy(points)
        if len(xy) == 0:
            raise ValueError("empty input")
        out = np.empty((len(xy) + 2, 2), np.int32)
        h = fn(_p(xy), len(xy), _p(out))
        return out[:h].copy()

    def melkman(self, chain) -> np.ndarray:
        return self._hull(self.L.or_melkman, chain)

    def canonicalize(self, verts) -> np.ndarray:
        return self._hull(self.L.or_canonicalize, verts)

    def monotone_hull(self, points) -> np.ndarray:
        return self._hull(self.L.or_monotone_hull, points)

    def min_max(self, points):
        xy = _xy(points)
        out = np.zeros(4, np.int64)
        self.L.or_min_max(_p(xy), len(xy), _p(out))
        return tuple(int(v) for v in out)

    def precondition(self, points):
        """reducer::precondition, x-only mode (src/reducer.cpp:132-178):
        bounds, width = x_max - x_min + 1, bucket with x_off = x_min - 1 and
        y untranslated, Lemma-1 chain, Melkman hull."""
        xy = _xy(points)
        if len(xy) == 0:
            raise ValueError("precondition: empty input")
        xmin, xmax, ymin, ymax = self.min_max(xy)
        w = xmax - xmin + 1
        lo = np.zeros(w, np.int32)
        hi = np.zeros(w, np.int32)
        valid = np.zeros(w, np.uint8)
        occ = np.zeros((w + 63) // 64, np.uint64)
        self.L.or_bucket(_p(xy), len(xy), xmin - 1, _p(lo), _p(hi), _p(valid), _p(occ))
        arr = {"width": w, "lo": lo, "hi": hi, "valid": valid, "occ": occ}
        chain = self.build_polyline(arr, major_off=xmin - 1)
        return {"bbox": (xmin, xmax, ymin, ymax), "arr": arr, "chain": chain, "hull": self.melkman(chain)}

    def pipeline(self, points, width: int, q: int | None = None):
        """reduce -> L pairs, Lemma-1 chain, melkman hull (the reference
        pipeline of SURVEY.md section 3.3 plus section 3.1's hull)."""
        arr = self.reduce(points, width, q)
        L = self.L_pairs(arr)
        vc = self.valid_count(arr)
        if vc == 0:
            return {"arr": arr, "L": L, "chain": np.empty((0, 2), np.int32), "hull": None, "s": 0}
        chain = self.build_polyline(arr)
        return {"arr": arr, "L": L, "chain": chain, "hull": self.melkman(chain), "s": len(chain)}


class Accumulator:
    """reduce() over a stream of chunks: each chunk is
    reduced on host threads (src/reducer.cpp:69-79 per slice) and merged slot
    by slot; finish() rebuilds the exact ExtremalArray by reducing the
    survivors once more (idempotence, tests/test_reducer.cpp:113-127) and
    checks that it reproduces the merged L."""

    def __init__(self, orc: Oracle, width: int, q: int | None = None):
        self.orc, self.width, self.q = orc, int(width), q
        w = max(self.width, 1)
        self.lo = np.zeros(w, np.int32)
        self.hi = np.full(w, -1, np.int32)
        self.valid = np.zeros(w, np.uint8)
        self.points = 0

    def add(self, xy: np.ndarray, threads: int = 0) -> None:
        xy = np.ascontiguousarray(xy, dtype=np.int32).reshape(-1, 2)
        rc = self.orc.L.or_reduce_accumulate_mt(_p(xy), len(xy), self.width, -1 if self.q is None else int(self.q),
                                                int(threads or os.cpu_count() or 1), _p(self.lo), _p(self.hi),
                                                _p(self.valid))
        if rc != 0:
            raise ValueError("reduce: coordinate out of range")
        self.points += len(xy)

    def finish(self):
        w = self.width
        occ = np.zeros((w + 63) // 64, np.uint64)
        self.orc.L.or_occ_from_valid(w, _p(self.valid), _p(occ))
        merged = {"width": w, "lo": self.lo.copy(), "hi": self.hi.copy(), "valid": self.valid.copy(), "occ": occ}
        if self.orc.valid_count(merged) == 0:
            return merged
        survivors = self.orc.build_polyline(merged)
        arr = self.orc.reduce(survivors, w, self.q)
        v = arr["valid"].astype(bool)
        assert np.array_equal(v, self.valid.astype(bool)) and np.array_equal(arr["lo"][v], self.lo[v]) \
            and np.array_equal(arr["hi"][v], self.hi[v]) and np.array_equal(arr["occ"], occ), \
            "re-reducing the survivors did not reproduce the merged L"
        return arr


class Reference:
    """The reference library itself (oracle/_ref/libchpref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = ctypes.CDLL(path)
        L.ref_gen_uniform_box.argtypes = [c_uint64, c_int64, c_uint64, c_void_p]
        L.ref_pipeline.restype = c_int
        L.ref_pipeline.argtypes = [c_void_p, c_uint64, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_void_p]
        L.ref_serialize.restype = c_int64
        L.ref_serialize.argtypes = [c_void_p, c_uint64, c_int64, c_int64, c_char_p, c_int64]
        L.ref_precondition.restype = c_int
        L.ref_precondition.argtypes = [c_void_p, c_uint64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
        L.ref_melkman.restype = c_int64
        L.ref_melkman.argtypes = [c_void_p, c_int64, c_void_p]
        L.ref_graham.restype = c_int64
        L.ref_graham.argtypes = [c_void_p, c_int64, c_void_p]
        L.ref_time_reduce_compact.restype = c_double
        L.ref_time_reduce_compact.argtypes = [c_void_p, c_uint64, c_int64, c_int64, c_int, c_int, c_void_p]
        self.L = L

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def uniform_box(self, n: int, p: int, seed: int) -> np.ndarray:
        xy = np.empty((n, 2), dtype=np.int32)
        self.L.ref_gen_uniform_box(n, p, seed, _p(xy))
        return xy

    def pipeline(self, points, width: int, q: int | None = None):
        xy = _xy(points)
        w = int(width)
        Lp = np.empty((max(w, 1), 2), np.int32)
        chain = np.empty((2 * max(w, 1) + 1, 2), np.int32)
        hull = np.empty((2 * max(w, 1) + 3, 2), np.int32)
        s = np.zeros(1, np.int64)
        h = np.zeros(1, np.int64)
        vc = np.zeros(1, np.int64)
        rc = self.L.ref_pipeline(_p(xy), len(xy), w, -1 if q is None else int(q), _p(Lp), _p(chain),
                                 _p(s), _p(hull), _p(h), _p(vc))
        if rc == -1:
            raise ValueError("reduce: coordinate out of range")
        out = {"L": Lp[:w], "s": int(s[0]), "valid_count": int(vc[0])}
        out["chain"] = chain[: int(s[0])].copy()
        out["hull"] = hull[: int(h[0])].copy() if rc == 0 else None
        return out

    def serialize(self, points, width: int, q: int | None = None) -> str:
        xy = _xy(points)
        n = self.L.ref_serialize(_p(xy), len(xy), width, -1 if q is None else q, None, 0)
        if n < 0:
            raise ValueError("reduce: coordinate out of range")
        buf = ctypes.create_string_buffer(n)
        self.L.ref_serialize(_p(xy), len(xy), width, -1 if q is None else q, buf, n)
        return buf.raw[:n].decode()

    def precondition(self, points):
        xy = _xy(points)
        bbox = np.zeros(4, np.int64)
        offs = np.zeros(2, np.int64)
        cap = 2 * len(xy) + 2
        chain = np.empty((cap, 2), np.int32)
        hull = np.empty((cap, 2), np.int32)
        s = np.zeros(1, np.int64)
        h = np.zeros(1, np.int64)
        rc = self.L.ref_precondition(_p(xy), len(xy), _p(bbox), _p(offs), _p(chain), _p(s), _p(hull), _p(h))
        if rc != 0:
            raise ValueError("precondition: empty input")
        return {"bbox": tuple(int(v) for v in bbox), "major_offset": int(offs[0]),
                "minor_offset": int(offs[1]), "chain": chain[: int(s[0])].copy(),
                "hull": hull[: int(h[0])].copy()}

    def melkman(self, chain) -> np.ndarray:
        xy = _xy(chain)
        out = np.empty((len(xy) + 2, 2), np.int32)
        h = self.L.ref_melkman(_p(xy), len(xy), _p(out))
        if h < 0:
            raise ValueError("melkman: empty chain")
        return out[:h].copy()

    def graham(self, points) -> np.ndarray:
        xy = _xy(points)
        out = np.empty((len(xy) + 2, 2), np.int32)
        h = self.L.ref_graham(_p(xy), len(xy), _p(out))
        if h < 0:
            raise ValueError("graham_scan: empty input")
        return out[:h].copy()

    def time_reduce_compact(self, xy: np.ndarray, width: int, q: int, threads: int = 1, reps: int = 1):
        xy = _xy(xy)
        s = np.zeros(1, np.int64)
        t = self.L.ref_time_reduce_compact(_p(xy), len(xy), width, q, threads, reps, _p(s))
        return float(t), int(s[0])
