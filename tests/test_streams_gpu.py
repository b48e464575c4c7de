"""A context's calls never overlap each other, whatever streams they are
issued on, and a refused cooperative launch leaves later calls intact.

The context's scratch (sampled-filter tables, the grid barrier of the two
cooperative kernels, the look-back status words, the hull buffers) is
shared by every call; chp_ctx_set_stream orders a new stream after the old
one, and the grid barrier returns to zero at the end of every launch."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from paper_1505_00914_b200.device import Context, generate_host

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [(2, 65536, 4_000_000), (3, 16384, 3_000_000), (4, 1 << 20, 5_000_000), (5, 256, 2_000_000)]


def test_alternating_torch_streams(orc):
    """Two torch streams, calls alternating between them with no host
    synchronisation: every result must still be the oracle's."""
    ctx = Context(0)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    inputs = []
    for config, p, n in CASES:
        xy = generate_host(config, config, p, n)
        inputs.append((xy, torch.from_numpy(xy).cuda(), p))
    torch.cuda.synchronize()
    outs = []
    for rep in range(3):
        for i, (_, d, p) in enumerate(inputs):
            s = streams[(i + rep) % 2]
            with torch.cuda.stream(s):
                d.record_stream(s)
                DL = ctx.reduce(d, p, q=p)
                comp = ctx.compact(DL, p, chain=True, lpairs=True, lower=True, upper=True)
                hull = ctx.hull(comp, p)
                outs.append((i, comp, hull))
    torch.cuda.synchronize()
    for i, comp, hull in outs:
        xy, _, p = inputs[i]
        arr = orc.reduce(xy, p, p)
        chain = orc.build_polyline(arr)
        s = int(comp["counts"][0].item())
        assert np.array_equal(comp["lpairs"].cpu().numpy(), orc.L_pairs(arr)), i
        assert s == len(chain) and np.array_equal(comp["chain"][:s].cpu().numpy(), chain), i
        h = int(hull["h"].item())
        assert np.array_equal(hull["hull"][:h].cpu().numpy(), orc.melkman(chain)), i


def test_refused_cooperative_launch_then_normal_calls():
    """CHP_TEST_COOP_REFUSE makes both cooperative kernels (the sampled
    filter's sample+merge and the one-kernel hull) ask for an oversized grid,
    which the runtime refuses; the split launches run instead.  A second
    context in the same process, and the same context after, stay exact."""
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import oracle
from paper_1505_00914_b200.device import Context, generate_host
orc = oracle.Oracle()
for _ in range(2):
    ctx = Context(0)
    for config, p, n in ((2, 65536, 3_000_000), (4, 1 << 20, 3_000_000), (2, 65536, 2_000_000)):
        xy = generate_host(config, config, p, n)
        DL = ctx.reduce(torch.from_numpy(xy).cuda(), p, q=p)
        comp = ctx.compact(DL, p, chain=True, lower=True, upper=True)
        hull = ctx.hull(comp, p)
        torch.cuda.synchronize()
        s = int(comp["counts"][0].item()); h = int(hull["h"].item())
        chain = orc.build_polyline(orc.reduce(xy, p, p))
        assert np.array_equal(comp["chain"][:s].cpu().numpy(), chain), config
        assert np.array_equal(hull["hull"][:h].cpu().numpy(), orc.melkman(chain)), config
print("ok")
""" % ROOT
    for env in ({"CHP_TEST_COOP_REFUSE": "1"}, {}):
        r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


def test_many_cooperative_launches_reuse_the_barrier(orc):
    """Hundreds of back-to-back cooperative launches (sampled K1 at p =
    2^16, hull) on one context: the barrier counter returns to zero after
    each, so none releases early or waits forever."""
    ctx = Context(0)
    p = 65536
    xy = generate_host(2, 2, p, 1_000_000)
    d = torch.from_numpy(xy).cuda()
    arr = orc.reduce(xy, p, p)
    chain = orc.build_polyline(arr)
    hull_ref = orc.melkman(chain)
    for _ in range(200):
        DL = ctx.reduce(d, p, q=p)
        comp = ctx.compact(DL, p, chain=True, lower=True, upper=True)
        hull = ctx.hull(comp, p)
    torch.cuda.synchronize()
    print(ctx.variant)
    s = int(comp["counts"][0].item())
    assert np.array_equal(comp["chain"][:s].cpu().numpy(), chain)
    h = int(hull["h"].item())
    assert np.array_equal(hull["hull"][:h].cpu().numpy(), hull_ref)


@pytest.mark.parametrize("config,p", [(2, 65536), (5, 256), (4, 1 << 20), (3, 16384)])
def test_reduce_own_chain_right_after_compact(ctx, orc, config, p):
    """Back-to-back calls where each consumes the previous one's output
    (the kernels that stream points before their programmatic wait must
    never overlap the kernel that wrote those points): reduce, compact,
    reduce the chain K3 just wrote (no copy), compact again -- idempotence,
    many times over without host synchronisation."""
    xy = generate_host(config, config, p, 4_000_000)
    d = torch.from_numpy(xy).cuda()
    arr = orc.reduce(xy, p, p)
    ref_chain = orc.build_polyline(arr)
    s = len(ref_chain)
    outs = []
    for _ in range(20):
        DL = ctx.reduce(d, p, q=p)
        comp = ctx.compact(DL, p, chain=True)
        DL2 = ctx.reduce(comp["chain"][:s], p, q=p)
        comp2 = ctx.compact(DL2, p, chain=True)
        outs.append(comp2)
    torch.cuda.synchronize()
    for comp2 in outs:
        assert int(comp2["counts"][0].item()) == s
        assert np.array_equal(comp2["chain"][:s].cpu().numpy(), ref_chain)
