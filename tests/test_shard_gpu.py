"""Multi-GPU sharding on the device, checked against the
oracle: the C-ABI shard groups (chp_group_*, one process, NCCL or a
peer-memory combine) and bench.py's multi-rank path (one process per rank,
the partial Ls merged by the torch.distributed MIN all-reduce).

The test box has one GPU, so G > 1 groups place every shard on device 0
with the peer combine (the same code path as distinct devices: the combine
kernel reads the partial DLs through their device pointers), the NCCL group
runs at G = 1 (the communicator, the group call and the all-reduce are
real), and the multi-rank bench runs two ranks on one GPU over gloo.  A
G > 1 NCCL group runs when the box has more than one GPU."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

from paper_1505_00914_b200.device import Group, generate_host
from paper_1505_00914_b200.shard import dl_unpack_host

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def oracle_result(orc, xy, p, q):
    arr = orc.reduce(xy, p, q)
    chain = orc.build_polyline(arr)
    return orc.L_pairs(arr), chain, orc.melkman(chain)


@pytest.mark.parametrize("G", [1, 2, 3, 4])
@pytest.mark.parametrize("config,p,n", [(2, 65536, 5_000_003), (4, 1 << 20, 6_000_001), (5, 256, 4_000_000)])
@pytest.mark.parametrize("combine", ["peer", "fused"])
def test_peer_group_pipeline_host(orc, G, config, p, n, combine):
    xy = generate_host(config, config, p, n)
    g = Group([0] * G, combine=combine)
    got = g.pipeline_host(xy, p, p, L=True, chain=True, hull=True)
    L, chain, hull = oracle_result(orc, xy, p, p)
    assert np.array_equal(got["L"], L)
    assert got["s"] == len(chain) and np.array_equal(got["chain"], chain)
    assert np.array_equal(got["hull"], hull)
    assert g.last_h2d_bytes > 0
    g.close()


def test_nccl_group_single_device(orc):
    """G = 1 over NCCL: ncclCommInitAll, the group call and the MIN
    all-reduce run for real; the result is the oracle's."""
    g = Group([0], combine="nccl")
    xy = generate_host(5, 5, 256, 3_000_000)
    got = g.pipeline_host(xy, 256, 256, L=True, chain=True, hull=True)
    L, chain, hull = oracle_result(orc, xy, 256, 256)
    assert np.array_equal(got["L"], L) and np.array_equal(got["chain"], chain)
    assert np.array_equal(got["hull"], hull)
    d = torch.from_numpy(xy).cuda()
    DL = g.reduce_sharded([d], 256, 256)[0]
    from paper_1505_00914_b200.device import Context

    ctx = Context(0)
    comp = ctx.compact(DL, 256, chain=True, lpairs=True)
    torch.cuda.synchronize()
    assert np.array_equal(comp["lpairs"].cpu().numpy(), L)
    g.close()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_nccl_group_two_devices(orc):
    g = Group([0, 1], combine="nccl")
    xy = generate_host(2, 2, 65536, 8_000_000)
    got = g.pipeline_host(xy, 65536, 65536, L=True, chain=True)
    L, chain, _ = oracle_result(orc, xy, 65536, 65536)
    assert np.array_equal(got["L"], L) and np.array_equal(got["chain"], chain)
    g.close()


def test_nccl_group_rejects_repeated_device():
    with pytest.raises(ValueError):
        Group([0, 0], combine="nccl")


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("combine", ["peer", "fused"])
def test_peer_group_reduce_sharded_device_resident(ctx, orc, G, combine):
    p, n = 16384, 7_000_001
    xy = generate_host(3, 3, p, n)
    d = torch.from_numpy(xy).cuda()
    bounds = [(n * k // G, n * (k + 1) // G) for k in range(G)]
    shards = [d[a:b].contiguous() for a, b in bounds]
    g = Group([0] * G, combine=combine)
    DL = g.reduce_sharded(shards, p, p)[0]
    comp = ctx.compact(DL, p, chain=True, lpairs=True)
    torch.cuda.synchronize()
    L, chain, _ = oracle_result(orc, xy, p, p)
    assert np.array_equal(comp["lpairs"].cpu().numpy(), L)
    s = int(comp["counts"][0].item())
    assert s == len(chain) and np.array_equal(comp["chain"][:s].cpu().numpy(), chain)
    g.close()


@pytest.mark.parametrize("combine", ["peer", "fused"])
def test_peer_group_back_to_back_calls_share_partials(orc, combine):
    """Two chp_reduce_sharded calls without a sync between them, the shard
    partials (d_L[k], k > 0) shared: the second call's DL init on a shard
    stream must wait for the first call's combine to read that partial."""
    G, p = 4, 65536
    xs = [generate_host(2, 2, p, 4_000_000), generate_host(4, 4, p, 4_000_000)]
    g = Group([0] * G, combine=combine)
    shared = [torch.empty(int(g.L.chp_dl_len(p)), dtype=torch.int32, device="cuda") for _ in range(G - 1)]
    heads = [torch.empty(int(g.L.chp_dl_len(p)), dtype=torch.int32, device="cuda") for _ in range(2)]
    for _ in range(3):
        outs = []
        for xy, head in zip(xs, heads):
            d = torch.from_numpy(xy).cuda()
            n = len(xy)
            shards = [d[n * k // G:n * (k + 1) // G].contiguous() for k in range(G)]
            torch.cuda.synchronize()
            outs.append(g.reduce_sharded(shards, p, p, outs=[head] + shared, sync=False)[0])
        g.sync()
        for xy, DL in zip(xs, outs):
            arr = orc.reduce(xy, p, p)
            lo, hi, valid, err = dl_unpack_host(DL.cpu().numpy())
            assert err == 0
            L = np.stack([np.where(valid, lo, p + 1), np.where(valid, hi, -1)], axis=1)
            assert np.array_equal(L, orc.L_pairs(arr))
    g.close()


@pytest.mark.parametrize("combine", ["peer", "fused"])
def test_peer_group_error_in_one_shard(combine):
    """An invalid coordinate in the last shard sets that partial's error
    word; the MIN combine carries it, and the call raises like reduce()."""
    xy = generate_host(5, 5, 256, 1_000_000)
    xy[-3] = (300, 5)  # x > width
    g = Group([0, 0, 0], combine=combine)
    with pytest.raises(ValueError):
        g.pipeline_host(xy, 256, 256)
    xy[-3] = (3, 5)
    g.pipeline_host(xy, 256, 256)  # the group recovers
    g.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("config,n", [(2, 3_000_000), (5, 5_000_000)])
def test_bench_two_ranks_gloo_verified(config, n):
    """bench.py's N > 1 path -- each rank K1 on its slice, the MIN
    all-reduce, K3; the e2e leg with chp_reduce_host / chp_finish_host --
    run as two ranks on one GPU over gloo, the merged chain checked against
    the oracle over all n points (--verify)."""
    env = {**os.environ, "CHP_DIST_BACKEND": "gloo"}
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", "bench.py", "--gpus", "2",
           "--config", str(config), "--total-points", str(n), "--steps", "3", "--warmup", "3", "--e2e-steps", "2",
           "--no-cpu-baseline", "--verify"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["verified"] is True
    assert line["config"]["n_total"] == n and line["result"]["n_per_rank"] == n // 2
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0


@pytest.mark.parametrize("combine", ["peer", "fused"])
@pytest.mark.parametrize("config", [4, 5])
def test_full_size_sharded_vs_oracle(ctx, orc, combine, config):
    """BASELINE.json's full C4 (1e9 points) / C5 (4e9 points, "sharded over
    1/2/4/8 GPUs") as north_star (d) splits it: four contiguous equal
    shards, each reduced by its own group context, merged by the peer kernel
    or folded straight into shard 0's L; the merged L and chain against the
    chunked oracle over all n points (generated on the host, chunk by
    chunk, from the same counter-based generator)."""
    import bench

    n, p, seed, _ = bench.CONFIGS[config]
    free = torch.cuda.mem_get_info()[0]
    if n * 8 + (2 << 30) > free:
        pytest.skip("not enough device memory")
    G = 4
    bounds = [(n * k // G, n * (k + 1) // G) for k in range(G)]
    shards = [ctx.generate(config, seed, p, b - a, offset=a) for a, b in bounds]
    torch.cuda.synchronize()
    g = Group([0] * G, combine=combine)
    DL = g.reduce_sharded(shards, p, p)[0]
    comp = ctx.compact(DL, p, chain=True, lpairs=True)
    torch.cuda.synchronize()
    s = int(comp["counts"][0].item())
    assert int(comp["counts"][2].item()) == 0
    got_L, got_chain = comp["lpairs"].cpu().numpy(), comp["chain"][:s].cpu().numpy()
    del shards, comp
    g.close()
    acc = orc.accumulator(p, p)
    chunk = 1 << 26
    for a in range(0, n, chunk):
        acc.add(generate_host(config, seed, p, min(chunk, n - a), offset=a))
    arr = acc.finish()
    assert np.array_equal(got_L, orc.L_pairs(arr))
    assert np.array_equal(got_chain, orc.build_polyline(arr))
