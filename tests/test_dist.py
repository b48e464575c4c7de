"""Multi-rank combine on CPU (gloo, world size 2): the host-side logic of the
N>1 path.  Each rank reduces its shard (the oracle stands in for K1 here,
there is no GPU), packs the device-form L, and the ranks merge with the same
element-wise MIN all-reduce bench.py runs over NCCL; the result must equal
the single-process L, chain and error flag bit for bit."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1505_00914_b200.shard import dl_pack_host, dl_unpack_host, shard_bounds


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, xy, p, q, out, op="allreduce"):
    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = oracle.Oracle()
    start, count = shard_bounds(len(xy), rank, world)
    part = xy[start:start + count]
    # K1 stand-in: per-shard reduce; out-of-range points set the error word
    ok = (part[:, 0] >= 1) & (part[:, 0] <= p) & (part[:, 1] >= 1) & ((q is None) | (part[:, 1] <= (q or 0)))
    arr = orc.reduce(part[ok], p, q)
    DL = torch.from_numpy(dl_pack_host(arr["lo"], arr["hi"], arr["valid"], err=int((~ok).any())))
    if op == "allreduce":
        dist.all_reduce(DL, op=dist.ReduceOp.MIN)
    else:
        from paper_1505_00914_b200.shard import reduce_dl

        reduce_dl(DL, dst=0)
    if rank == 0:
        out.put(DL.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def _run(xy, p, q, world=2, op="allreduce"):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, xy, p, q, out, op)) for r in range(world)]
    for pr in procs:
        pr.start()
    DL = out.get(timeout=120)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    return DL


def test_shard_bounds_cover_exactly():
    for n in (0, 1, 7, 1000, 4_000_000_000):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, r, world) for r in range(world)]
            assert spans[0][0] == 0
            assert sum(c for _, c in spans) == n
            for (a, c), (b, _) in zip(spans, spans[1:]):
                assert a + c == b


def test_dl_pack_roundtrip(orc):
    rng = np.random.default_rng(1)
    xy = rng.integers(1, 50, size=(300, 2)).astype(np.int32)
    arr = orc.reduce(xy, 60)
    lo, hi, valid, err = dl_unpack_host(dl_pack_host(arr["lo"], arr["hi"], arr["valid"]))
    assert err == 0
    assert np.array_equal(valid, arr["valid"].astype(bool))
    assert np.array_equal(lo[valid], arr["lo"][valid]) and np.array_equal(hi[valid], arr["hi"][valid])


def test_two_rank_min_allreduce_equals_single_process(orc):
    from paper_1505_00914_b200.device import generate_host

    p = 4096
    xy = generate_host(5, 5, p, 400_000)
    DL = _run(xy, p, p)
    lo, hi, valid, err = dl_unpack_host(DL)
    arr = orc.reduce(xy, p, p)
    assert err == 0
    L = np.stack([np.where(valid, lo, p + 1), np.where(valid, hi, -1)], axis=1)
    assert np.array_equal(L, orc.L_pairs(arr))


def test_two_rank_error_word_propagates(orc):
    xy = np.array([[1, 1], [2, 2], [3, 3], [9, 1]], np.int32)  # x=9 > p=5 on rank 1's shard
    DL = _run(xy, 5, 5)
    assert dl_unpack_host(DL)[3] == -1


def test_two_rank_min_reduce_onto_rank0(orc):
    """bench.py's combine: the MIN reduce onto rank 0 (shard.reduce_dl)."""
    from paper_1505_00914_b200.device import generate_host

    p = 65536
    xy = generate_host(2, 2, p, 300_000)
    DL = _run(xy, p, p, op="reduce")
    lo, hi, valid, err = dl_unpack_host(DL)
    arr = orc.reduce(xy, p, p)
    assert err == 0
    L = np.stack([np.where(valid, lo, p + 1), np.where(valid, hi, -1)], axis=1)
    assert np.array_equal(L, orc.L_pairs(arr))
