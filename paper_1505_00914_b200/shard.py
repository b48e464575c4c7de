"""Multi-GPU combine of partial L.

Min and max are associative, commutative and exact on integers, so any
partition of the points gives the same L.  Each rank reduces its own points
into a device-form L (DL: pairs (lo, ~hi), empty = INT32_MAX, then the error
word); storing ~hi makes every word a MIN, so ONE element-wise MIN merges
the partials -- NCCL over NVLink/NVSwitch on the GPU box (torch.distributed,
backend "nccl"), gloo in the CPU tests: an all-reduce when every rank needs
the merged L (allreduce_dl), a reduce onto one rank when only that rank
compacts it (reduce_dl; bench.py, rank 0).

The host helpers pack/unpack the same DL layout (tests, host-side merges).
"""
from __future__ import annotations

import numpy as np

INT32_MAX = np.iinfo(np.int32).max


def shard_bounds(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous equal slices: rank r owns [r*n/W, (r+1)*n/W)."""
    lo = n_total * rank // world
    hi = n_total * (rank + 1) // world
    return lo, hi - lo


def allreduce_dl(DL, group=None):
    """Element-wise MIN all-reduce of a device-form L (torch tensor, in place)."""
    import torch.distributed as dist

    if DL.is_cuda and dist.get_backend(group) == "gloo":  # CPU test path
        host = DL.cpu()
        dist.all_reduce(host, op=dist.ReduceOp.MIN, group=group)
        DL.copy_(host)
        return DL
    dist.all_reduce(DL, op=dist.ReduceOp.MIN, group=group)
    return DL


def reduce_dl(DL, dst: int = 0, group=None):
    """Element-wise MIN of the partial DLs onto rank `dst` only (K3 runs
    there; the other ranks' DL stays partial): half the traffic of the
    all-reduce for the same merged L."""
    import torch.distributed as dist

    if DL.is_cuda and dist.get_backend(group) == "gloo":  # CPU test path
        host = DL.cpu()
        dist.reduce(host, dst=dst, op=dist.ReduceOp.MIN, group=group)
        if dist.get_rank(group) == dst:
            DL.copy_(host)
        return DL
    dist.reduce(DL, dst=dst, op=dist.ReduceOp.MIN, group=group)
    return DL


def dl_pack_host(lo: np.ndarray, hi: np.ndarray, valid: np.ndarray, err: int = 0) -> np.ndarray:
    """Host copy of the DL layout of include/chp_b200.h."""
    w = len(lo)
    out = np.empty(2 * w + 2, np.int32)
    v = valid.astype(bool)
    out[0:2 * w:2] = np.where(v, lo, INT32_MAX)
    out[1:2 * w:2] = np.where(v, ~hi.astype(np.int32), INT32_MAX)
    out[2 * w] = -1 if err else 0
    out[2 * w + 1] = 0
    return out


def dl_unpack_host(DL: np.ndarray):
    """(lo, hi, valid, err) from a DL."""
    DL = np.asarray(DL, np.int32)
    w = (len(DL) - 2) // 2
    lo = DL[0:2 * w:2].copy()
    hi = ~DL[1:2 * w:2]
    valid = lo <= hi
    return lo, hi, valid, int(DL[2 * w])
