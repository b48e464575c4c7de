"""ctypes binding of include/chp_b200.h (the C ABI of libchp_b200.so).

There is no fallback: if the library is missing the import fails loudly,
and every compute entry point runs the sm_100a kernels.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_int, c_int32, c_int64, c_uint32, c_uint64, c_void_p

from ._build import LIB

CHP_OK, CHP_EINVAL, CHP_EDEVICE = 0, 1, 2
COMBINE_NCCL, COMBINE_PEER, COMBINE_FUSED = 0, 1, 2
REDUCE_ACCUMULATE = 1
REDUCE_NO_VALIDATE = 2
REDUCE_FORCE_GLOBAL = 4
REDUCE_FORCE_SMEM32 = 8
REDUCE_FORCE_FILTER = 16
REDUCE_FORCE_FILTER8 = 32
REDUCE_FORCE_SMEM16 = 64
REDUCE_FORCE_SAMPLED = 8192
REDUCE_FUSED = 16384
REDUCE_SAMPLE_SPLIT = 1 << 25
REDUCE_BLOCKED = 1 << 26
REDUCE_SAMPLE_PREFIX = 1 << 27
REDUCE_WARP_AGG = 1 << 28

_lib = None


class ChpError(RuntimeError):
    """CHP_EDEVICE: a CUDA failure (std::runtime_error in the C++ drop-in)."""


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        raise ImportError(
            f"{LIB} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB)
    vp = c_void_p
    sig = {
        "chp_ctx_create": (c_int, [c_int, POINTER(c_void_p)]),
        "chp_ctx_destroy": (None, [vp]),
        "chp_last_error": (c_char_p, [vp]),
        "chp_ctx_set_stream": (c_int, [vp, vp]),
        "chp_ctx_use_own_stream": (c_int, [vp]),
        "chp_ctx_stream": (vp, [vp]),
        "chp_ctx_sync": (c_int, [vp]),
        "chp_launch_count": (c_uint64, [vp]),
        "chp_last_variant": (c_char_p, [vp]),
        "chp_last_h2d_bytes": (c_uint64, [vp]),
        "chp_dl_len": (c_uint64, [c_int64]),
        "chp_reduce": (c_int, [vp, vp, c_uint64, c_int64, c_int64, c_int64, vp, c_uint32]),
        "chp_dl_init": (c_int, [vp, vp, c_int64]),
        "chp_check": (c_int, [vp, vp, c_int64]),
        "chp_dl_from_pairs": (c_int, [vp, vp, c_int64, vp]),
        "chp_polyline_host": (c_int, [vp, vp, c_int64, c_int64, c_int64, c_int, vp, vp]),
        "chp_compact": (c_int, [vp, vp, c_int64, c_int64, c_int64, c_int, vp, vp, vp, vp, vp, vp, vp]),
        "chp_ns_chain": (c_int, [vp, vp, vp, vp, c_int64, vp]),
        "chp_hull": (c_int, [vp, vp, vp, vp, c_int64, c_int, vp, vp]),
        "chp_bounds": (c_int, [vp, vp, c_uint64, vp]),
        "chp_translate": (c_int, [vp, vp, c_uint64, c_int32, c_int32, vp]),
        "chp_translate_host": (c_int, [vp, vp, c_uint64, c_int32, c_int32, vp]),
        "chp_pipeline_host": (c_int, [vp, vp, c_uint64, c_int64, c_int64, vp, vp, vp, vp, vp, vp]),
        "chp_precondition_host": (c_int, [vp, vp, c_uint64, vp, vp, vp, vp, vp, vp]),
        "chp_precondition_run": (c_int, [vp, vp, c_uint64, c_int, vp, vp, vp, vp]),
        "chp_last_outputs": (c_int, [vp, vp, vp, vp]),
        "chp_pipeline_host64": (c_int, [vp, vp, c_uint64, c_int64, c_int64, vp, vp, vp, vp, vp, vp]),
        "chp_precondition_run64": (c_int, [vp, vp, c_uint64, c_int, c_int, vp, vp, vp, vp]),
        "chp_bounds_host64": (c_int, [vp, vp, c_uint64, vp]),
        "chp_reduce_host": (c_int, [vp, vp, c_uint64, c_int64, c_int64, vp]),
        "chp_reduce_host64": (c_int, [vp, vp, c_uint64, c_int64, c_int64, vp]),
        "chp_finish_host": (c_int, [vp, vp, c_int64, vp, vp, vp, vp, vp, vp]),
        "chp_group_create": (c_int, [vp, c_int, c_int, POINTER(c_void_p)]),
        "chp_group_destroy": (None, [vp]),
        "chp_group_ctx": (vp, [vp, c_int]),
        "chp_group_size": (c_int, [vp]),
        "chp_group_last_error": (c_char_p, [vp]),
        "chp_group_last_h2d_bytes": (c_uint64, [vp]),
        "chp_reduce_sharded": (c_int, [vp, vp, vp, c_int64, c_int64, vp]),
        "chp_pipeline_host_sharded": (c_int, [vp, vp, c_uint64, c_int64, c_int64, vp, vp, vp, vp, vp, vp]),
        "chp_pipeline_host64_sharded": (c_int, [vp, vp, c_uint64, c_int64, c_int64, vp, vp, vp, vp, vp, vp]),
        "chp_generate": (c_int, [vp, c_int, c_uint64, c_int64, c_uint64, c_uint64, vp]),
        "chp_generate_host": (c_int, [c_int, c_uint64, c_int64, c_uint64, c_uint64, vp, c_int]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


# Every symbol include/chp_b200.h declares (checked by tests without a GPU).
ABI_SYMBOLS = (
    "chp_ctx_create", "chp_ctx_destroy", "chp_last_error", "chp_ctx_set_stream", "chp_ctx_use_own_stream", "chp_ctx_stream",
    "chp_ctx_sync", "chp_launch_count", "chp_last_variant", "chp_last_h2d_bytes", "chp_dl_len", "chp_reduce", "chp_dl_init",
    "chp_check", "chp_dl_from_pairs", "chp_polyline_host", "chp_compact", "chp_ns_chain", "chp_hull", "chp_bounds", "chp_translate", "chp_translate_host",
    "chp_pipeline_host", "chp_precondition_host", "chp_precondition_run", "chp_last_outputs", "chp_pipeline_host64", "chp_precondition_run64",
    "chp_bounds_host64", "chp_reduce_host", "chp_reduce_host64", "chp_finish_host", "chp_group_create",
    "chp_group_destroy", "chp_group_ctx", "chp_group_size", "chp_group_last_error", "chp_group_last_h2d_bytes",
    "chp_reduce_sharded", "chp_pipeline_host_sharded", "chp_pipeline_host64_sharded", "chp_generate",
    "chp_generate_host",
)
