"""Device-resident API over the C ABI: torch tensors in HBM, CUDA streams.

torch is plumbing here (device memory, streams, events); every computation
is one of the sm_100a kernels in csrc/ reached through libchp_b200.so.

    ctx = Context(0)
    xy  = ctx.generate(config=2, seed=2, p=65536, n=100_000_000)   # (n,2) int32 on cuda:0
    DL  = ctx.reduce(xy, width=65536, q=65536)                      # Algorithm 1 (K1)
    out = ctx.compact(DL, 65536, chain=True, lower=True, upper=True)  # Lemma-1 chain (K3)
    hull = ctx.hull(out, 65536)                                     # exact hull (K4)
"""
from __future__ import annotations

import ctypes
from ctypes import byref, c_void_p

import numpy as np
import torch

from . import _lib
from ._lib import CHP_EINVAL, CHP_OK, ChpError


def _ptr(t: torch.Tensor | None):
    return None if t is None else c_void_p(t.data_ptr())


def _np_ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(c_void_p)


class Context:
    """One chp_ctx (one device, one stream).  By default every call runs on
    torch's current stream of that device, so torch.cuda.Event timing and
    tensor lifetimes follow the usual stream semantics."""

    def __init__(self, device: int = 0, follow_torch_stream: bool = True):
        self.L = _lib.load()
        self.device = int(device)
        self.follow = follow_torch_stream
        h = c_void_p()
        rc = self.L.chp_ctx_create(self.device, byref(h))
        if rc != CHP_OK:
            raise ChpError(f"chp_ctx_create({device}) failed (rc={rc}); is a CUDA device visible?")
        self.h = h
        self._dev = torch.device("cuda", self.device)

    def close(self):
        if getattr(self, "h", None):
            self.L.chp_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ plumbing
    def _stream(self):
        if self.follow:
            s = torch.cuda.current_stream(self._dev)
            self.L.chp_ctx_set_stream(self.h, c_void_p(s.cuda_stream))

    def _check(self, rc: int):
        if rc == CHP_OK:
            return
        msg = (self.L.chp_last_error(self.h) or b"").decode()
        if rc == CHP_EINVAL:
            raise ValueError(msg)
        raise ChpError(msg)

    @property
    def launches(self) -> int:
        return int(self.L.chp_launch_count(self.h))

    @property
    def variant(self) -> str:
        return self.L.chp_last_variant(self.h).decode()

    @property
    def last_h2d_bytes(self) -> int:
        """Host->device bytes of the last host-pipeline call (4/point when packed)."""
        return int(self.L.chp_last_h2d_bytes(self.h))

    def dl_len(self, width: int) -> int:
        return int(self.L.chp_dl_len(int(width)))

    def empty_dl(self, width: int) -> torch.Tensor:
        return torch.empty(self.dl_len(width), dtype=torch.int32, device=self._dev)

    @staticmethod
    def _xy(xy: torch.Tensor) -> torch.Tensor:
        if xy.dtype != torch.int32 or not xy.is_cuda:
            raise TypeError("points must be an int32 CUDA tensor of shape (n, 2)")
        if not xy.is_contiguous():
            raise ValueError("points must be contiguous")
        return xy

    # ------------------------------------------------------------------ K1
    def reduce(self, xy: torch.Tensor, width: int, q: int | None = None, x_off: int = 0,
               out: torch.Tensor | None = None, flags: int = 0) -> torch.Tensor:
        """Algorithm 1 into a device-form L (DL).  Asynchronous; call
        check(DL, width) to surface out-of-range input as ValueError."""
        xy = self._xy(xy)
        self._stream()
        DL = out if out is not None else self.empty_dl(width)
        n = xy.numel() // 2
        self._check(self.L.chp_reduce(self.h, _ptr(xy), n, int(width), -1 if q is None else int(q),
                                      int(x_off), _ptr(DL), int(flags)))
        return DL

    def dl_init(self, DL: torch.Tensor, width: int):
        self._stream()
        self._check(self.L.chp_dl_init(self.h, _ptr(DL), int(width)))

    def check(self, DL: torch.Tensor, width: int):
        self._stream()
        self._check(self.L.chp_check(self.h, _ptr(DL), int(width)))

    # ------------------------------------------------------------------ K3
    def compact(self, DL: torch.Tensor, width: int, major_off: int = 0, minor_off: int = 0,
                swapped: bool = False, chain: bool = True, occ: bool = False, lpairs: bool = False,
                lower: bool = False, upper: bool = False, upperd: bool = False, bufs: dict | None = None) -> dict:
        """Decoupled-look-back compaction.  Returns device tensors (sized for
        the worst case) plus `counts` = int64[4] {s, v, err, s-v} on device."""
        self._stream()
        w = int(width)
        d = self._dev
        b = bufs if bufs is not None else {}

        def buf(name, shape, dtype, want):
            if not want:
                return None
            t = b.get(name)
            if t is None:
                t = torch.empty(shape, dtype=dtype, device=d)
                b[name] = t
            return t

        r = {
            "chain": buf("chain", (2 * w, 2), torch.int32, chain),
            "occ": buf("occ", ((w + 63) // 64,), torch.int64, occ),
            "lpairs": buf("lpairs", (w, 2), torch.int32, lpairs),
            "lower": buf("lower", (w, 2), torch.int32, lower),
            "upper": buf("upper", (w, 2), torch.int32, upper),
            "upperd": buf("upperd", (w, 2), torch.int32, upperd),
            "counts": buf("counts", (8,), torch.int64, True),
        }
        self._check(self.L.chp_compact(self.h, _ptr(DL), w, int(major_off), int(minor_off), int(bool(swapped)),
                                       _ptr(r["chain"]), _ptr(r["occ"]), _ptr(r["lpairs"]), _ptr(r["lower"]),
                                       _ptr(r["upper"]), _ptr(r["upperd"]), _ptr(r["counts"])))
        return r

    def ns_chain(self, comp: dict, width: int) -> torch.Tensor:
        """The north_star order (minima ascending x, then maxima descending x)."""
        self._stream()
        w = int(width)
        ns = torch.empty((2 * w, 2), dtype=torch.int32, device=self._dev)
        self._check(self.L.chp_ns_chain(self.h, _ptr(comp["lower"]), _ptr(comp["upperd"]), _ptr(comp["counts"]),
                                        w, _ptr(ns)))
        return ns

    # ------------------------------------------------------------------ K4
    def hull(self, comp: dict, width: int, swapped: bool = False, out: torch.Tensor | None = None) -> dict:
        """Exact canonical hull from compact(..., lower=True, upper=True).
        Returns {'hull': (2w+2, 2) int32, 'h': int64[1]} on device."""
        self._stream()
        w = int(width)
        hull = out if out is not None else torch.empty((2 * w + 2, 2), dtype=torch.int32, device=self._dev)
        h = comp.get("_h")
        if h is None:
            h = torch.empty(1, dtype=torch.int64, device=self._dev)
            comp["_h"] = h
        self._check(self.L.chp_hull(self.h, _ptr(comp["lower"]), _ptr(comp["upper"]), _ptr(comp["counts"]), w,
                                    int(bool(swapped)), _ptr(hull), _ptr(h)))
        return {"hull": hull, "h": h}

    # --------------------------------------------------------- K0 and misc
    def bounds(self, xy: torch.Tensor) -> torch.Tensor:
        xy = self._xy(xy)
        self._stream()
        out = torch.empty(4, dtype=torch.int32, device=self._dev)
        self._check(self.L.chp_bounds(self.h, _ptr(xy), xy.numel() // 2, _ptr(out)))
        return out

    def translate(self, xy: torch.Tensor, dx: int, dy: int, out: torch.Tensor | None = None) -> torch.Tensor:
        xy = self._xy(xy)
        self._stream()
        out = out if out is not None else torch.empty_like(xy)
        self._check(self.L.chp_translate(self.h, _ptr(xy), xy.numel() // 2, int(dx), int(dy), _ptr(out)))
        return out

    def dl_from_pairs(self, lpairs: torch.Tensor, width: int) -> torch.Tensor:
        self._stream()
        DL = self.empty_dl(width)
        self._check(self.L.chp_dl_from_pairs(self.h, _ptr(lpairs), int(width), _ptr(DL)))
        return DL

    def generate(self, config: int, seed: int, p: int, n: int, offset: int = 0,
                 out: torch.Tensor | None = None) -> torch.Tensor:
        """Synthetic workload of BASELINE.json config 2-5 generated in HBM
        (byte-identical to generate_host)."""
        self._stream()
        out = out if out is not None else torch.empty((n, 2), dtype=torch.int32, device=self._dev)
        self._check(self.L.chp_generate(self.h, int(config), int(seed), int(p), int(offset), int(n), _ptr(out)))
        return out

    # ----------------------------------------------------- host pipelines
    def pipeline_host(self, xy: np.ndarray, width: int, q: int | None = None, L: bool = False,
                      occ: bool = False, chain: bool = True, hull: bool = False) -> dict:
        """reduce -> build_polyline (-> hull) from a HOST (n,2) int32 buffer
        (pinned or pageable), outputs back in host memory."""
        xy = np.ascontiguousarray(xy, dtype=np.int32)
        w = int(width)
        n = xy.size // 2
        Lp = np.empty((max(w, 1), 2), np.int32) if L else None
        oc = np.empty(((max(w, 1) + 63) // 64,), np.uint64) if occ else None
        ch = np.empty((2 * max(w, 1), 2), np.int32) if chain else None
        hl = np.empty((2 * max(w, 1) + 2, 2), np.int32) if hull else None
        s = np.zeros(1, np.int64)
        h = np.zeros(1, np.int64)
        self._check(self.L.chp_pipeline_host(self.h, _np_ptr(xy), n, w, -1 if q is None else int(q), _np_ptr(Lp),
                                             _np_ptr(oc), _np_ptr(ch), _np_ptr(s), _np_ptr(hl),
                                             _np_ptr(h) if hull else None))
        out = {"s": int(s[0])}
        if L:
            out["L"] = Lp[:w]
        if occ:
            out["occ"] = oc
        if chain:
            out["chain"] = ch[: int(s[0])]
        if hull:
            out["hull"] = hl[: int(h[0])]
        return out

    def pipeline_host_ptr(self, xy_ptr: int, n: int, width: int, q: int | None, chain_ptr: int | None,
                          s_out: np.ndarray) -> None:
        """Same as pipeline_host on raw host pointers (the bench's e2e leg:
        pinned input, pinned chain output, no Python-side copies)."""
        self._check(self.L.chp_pipeline_host(self.h, c_void_p(xy_ptr), int(n), int(width),
                                             -1 if q is None else int(q), None, None,
                                             None if chain_ptr is None else c_void_p(chain_ptr),
                                             _np_ptr(s_out), None, None))

    def reduce_host_ptr(self, xy_ptr: int, n: int, width: int, q: int | None, DL: torch.Tensor) -> None:
        """chp_reduce_host: HOST points (raw pointer; pinned is fastest) into a
        device DL, initialised here; the error word stays in DL (combine
        partials first, then finish_host raises)."""
        self._stream()
        self._check(self.L.chp_reduce_host(self.h, c_void_p(xy_ptr), int(n), int(width), -1 if q is None else int(q),
                                           _ptr(DL)))

    def reduce_host(self, xy: np.ndarray, width: int, q: int | None = None,
                    out: torch.Tensor | None = None) -> torch.Tensor:
        xy = np.ascontiguousarray(xy, dtype=np.int32)
        DL = out if out is not None else self.empty_dl(width)
        self.reduce_host_ptr(xy.ctypes.data, xy.size // 2, width, q, DL)
        return DL

    def finish_host_ptr(self, DL: torch.Tensor, width: int, chain_ptr: int | None, s_out: np.ndarray) -> None:
        """chp_finish_host: K3 of a device DL, chain to a host pointer."""
        self._stream()
        self._check(self.L.chp_finish_host(self.h, _ptr(DL), int(width), None, None,
                                           None if chain_ptr is None else c_void_p(chain_ptr), _np_ptr(s_out),
                                           None, None))

    def finish_host(self, DL: torch.Tensor, width: int, L: bool = False, chain: bool = True,
                    hull: bool = False) -> dict:
        """K3 (+K4) of a device DL, outputs in host memory (ValueError when
        DL's error word is set, as pipeline_host)."""
        self._stream()
        w = int(width)
        Lp = np.empty((w, 2), np.int32) if L else None
        ch = np.empty((2 * w, 2), np.int32) if chain else None
        hl = np.empty((2 * w + 2, 2), np.int32) if hull else None
        s = np.zeros(1, np.int64)
        h = np.zeros(1, np.int64)
        self._check(self.L.chp_finish_host(self.h, _ptr(DL), w, _np_ptr(Lp), None, _np_ptr(ch), _np_ptr(s),
                                           _np_ptr(hl), _np_ptr(h) if hull else None))
        out = {"s": int(s[0])}
        if L:
            out["L"] = Lp
        if chain:
            out["chain"] = ch[: int(s[0])]
        if hull:
            out["hull"] = hl[: int(h[0])]
        return out

    def polyline_host(self, lpairs: np.ndarray, width: int, major_off: int = 0, minor_off: int = 0,
                      swapped: bool = False) -> np.ndarray:
        lp = np.ascontiguousarray(lpairs, dtype=np.int32)
        w = int(width)
        ch = np.empty((2 * w, 2), np.int32)
        s = np.zeros(1, np.int64)
        self._check(self.L.chp_polyline_host(self.h, _np_ptr(lp), w, int(major_off), int(minor_off),
                                             int(bool(swapped)), _np_ptr(ch), _np_ptr(s)))
        return ch[: int(s[0])]

    def precondition_host(self, xy: np.ndarray, chain: bool = True, hull: bool = False) -> dict:
        """chp::reducer::precondition from a host buffer in one pass over the
        input (chp_precondition_run), outputs fetched once the width is known."""
        xy = np.ascontiguousarray(xy, dtype=np.int32)
        n = xy.size // 2
        bbox = np.zeros(4, np.int64)
        if not chain and not hull:
            self._check(self.L.chp_precondition_host(self.h, _np_ptr(xy), n, _np_ptr(bbox), None, None, None, None,
                                                     None))
            return {"bbox": tuple(int(v) for v in bbox)}
        w = np.zeros(1, np.int64)
        s = np.zeros(1, np.int64)
        h = np.zeros(1, np.int64)
        self._check(self.L.chp_precondition_run(self.h, _np_ptr(xy), n, int(bool(hull)), _np_ptr(bbox), _np_ptr(w),
                                                _np_ptr(s), _np_ptr(h)))
        w, s, h = int(w[0]), int(s[0]), int(h[0])
        Lp = np.empty((w, 2), np.int32)
        ch = np.empty((s, 2), np.int32)
        hl = np.empty((max(h, 1), 2), np.int32) if hull else None
        self._check(self.L.chp_last_outputs(self.h, _np_ptr(Lp), _np_ptr(ch), _np_ptr(hl) if hull else None))
        out = {"bbox": tuple(int(v) for v in bbox), "width": w, "major_offset": int(bbox[0]) - 1,
               "L": Lp, "chain": ch, "s": s}
        if hull:
            out["hull"] = hl[:h]
        return out


class Group:
    """A shard group (include/chp_b200.h chp_group_*): reduce over G devices
    of this box in one process, partial Ls merged by ONE element-wise MIN --
    ncclAllReduce (combine="nccl", distinct devices), one peer-memory
    kernel on device 0 (combine="peer"; devices may repeat), or no combine
    step at all: every shard's K1 folds straight into device 0's DL over
    peer memory (combine="fused"; only DL 0 is used)."""

    def __init__(self, devices, combine: str = "nccl"):
        self.L = _lib.load()
        devs = (ctypes.c_int * len(devices))(*[int(d) for d in devices])
        mode = {"nccl": _lib.COMBINE_NCCL, "peer": _lib.COMBINE_PEER, "fused": _lib.COMBINE_FUSED}[combine]
        h = c_void_p()
        rc = self.L.chp_group_create(devs, len(devices), mode, byref(h))
        if rc != CHP_OK:
            raise (ValueError if rc == CHP_EINVAL else ChpError)(
                f"chp_group_create({list(devices)}, {combine}) failed (rc={rc})")
        self.h = h
        self.devices = [int(d) for d in devices]
        self.combine = combine

    def close(self):
        if getattr(self, "h", None):
            self.L.chp_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def size(self) -> int:
        return int(self.L.chp_group_size(self.h))

    @property
    def last_h2d_bytes(self) -> int:
        return int(self.L.chp_group_last_h2d_bytes(self.h))

    @property
    def launches(self) -> int:
        return sum(int(self.L.chp_launch_count(self.L.chp_group_ctx(self.h, k))) for k in range(self.size))

    def _check(self, rc: int):
        if rc == CHP_OK:
            return
        msg = (self.L.chp_group_last_error(self.h) or b"").decode()
        if rc == CHP_EINVAL:
            raise ValueError(msg)
        raise ChpError(msg)

    def reduce_sharded(self, shards, width: int, q: int | None = None, outs=None, sync: bool = True):
        """Device-resident shards (one (n_k, 2) int32 CUDA tensor per group
        device).  Returns the per-shard DLs; DL 0 holds the merged L (NCCL:
        every DL does).  Runs on each shard context's own stream; sync=False
        returns without waiting for them (chp_reduce_sharded orders later
        group calls after the combine)."""
        G = self.size
        if len(shards) != G:
            raise ValueError(f"{len(shards)} shards for a group of {G}")
        outs = outs if outs is not None else [
            torch.empty(int(self.L.chp_dl_len(int(width))), dtype=torch.int32, device=t.device) for t in shards]
        for t in shards:
            Context._xy(t)
        # the shard contexts run on their own streams: order them after the
        # producers of the inputs / outputs on torch's current streams
        for k, t in enumerate(shards):
            torch.cuda.current_stream(t.device).synchronize()
        xs = (c_void_p * G)(*[t.data_ptr() for t in shards])
        ns = (ctypes.c_uint64 * G)(*[t.numel() // 2 for t in shards])
        ds = (c_void_p * G)(*[d.data_ptr() for d in outs])
        self._check(self.L.chp_reduce_sharded(self.h, xs, ns, int(width), -1 if q is None else int(q), ds))
        if sync:
            self.sync()
        return outs

    def sync(self):
        for k in range(self.size):
            self.L.chp_ctx_sync(self.L.chp_group_ctx(self.h, k))

    def pipeline_host(self, xy: np.ndarray, width: int, q: int | None = None, L: bool = False, occ: bool = False,
                      chain: bool = True, hull: bool = False) -> dict:
        """chp_pipeline_host_sharded: the host input split over the group."""
        xy = np.ascontiguousarray(xy, dtype=np.int32)
        w = int(width)
        n = xy.size // 2
        Lp = np.empty((max(w, 1), 2), np.int32) if L else None
        oc = np.empty(((max(w, 1) + 63) // 64,), np.uint64) if occ else None
        ch = np.empty((2 * max(w, 1), 2), np.int32) if chain else None
        hl = np.empty((2 * max(w, 1) + 2, 2), np.int32) if hull else None
        s = np.zeros(1, np.int64)
        h = np.zeros(1, np.int64)
        self._check(self.L.chp_pipeline_host_sharded(self.h, _np_ptr(xy), n, w, -1 if q is None else int(q),
                                                     _np_ptr(Lp), _np_ptr(oc), _np_ptr(ch), _np_ptr(s), _np_ptr(hl),
                                                     _np_ptr(h) if hull else None))
        out = {"s": int(s[0])}
        if L:
            out["L"] = Lp[:w]
        if occ:
            out["occ"] = oc
        if chain:
            out["chain"] = ch[: int(s[0])]
        if hull:
            out["hull"] = hl[: int(h[0])]
        return out


def generate_host(config: int, seed: int, p: int, n: int, offset: int = 0, threads: int = 0) -> np.ndarray:
    """Host copy of the config 2-5 generators (same bytes as Context.generate)."""
    import os

    L = _lib.load()
    out = np.empty((n, 2), np.int32)
    rc = L.chp_generate_host(int(config), int(seed), int(p), int(offset), int(n), _np_ptr(out),
                             int(threads or os.cpu_count() or 1))
    if rc != CHP_OK:
        raise ValueError(f"generate_host: bad config {config} / p {p}")
    return out


_default: dict[int, Context] = {}


def default_context(device: int | None = None) -> Context:
    """Process-wide context per device (the drop-in API uses it)."""
    if device is None:
        device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    ctx = _default.get(device)
    if ctx is None:
        ctx = Context(device)
        _default[device] = ctx
    return ctx
