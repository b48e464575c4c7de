"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Bit-exact for L (serialize form), the occupancy words, the Lemma-1 chain,
s = valid_count, the north_star chain and the canonical hull, for every K1
variant, on downscaled BASELINE.json configs, the reference's config-1
golden digests, edge cases (empty, odd n, unaligned
buffers, invalid coordinates) and randomized fixtures shaped like the
reference's (tests/test_util.hpp).
"""
import numpy as np
import pytest
import torch

from paper_1505_00914_b200 import _lib
from paper_1505_00914_b200.device import generate_host

from _cases import mixed_case, to_unit_box

pytestmark = pytest.mark.gpu

VARIANTS = {
    "auto": 0,
    "global": _lib.REDUCE_FORCE_GLOBAL,
    "global_agg": _lib.REDUCE_FORCE_GLOBAL | _lib.REDUCE_WARP_AGG,
    "smem32": _lib.REDUCE_FORCE_SMEM32,
    "filter": _lib.REDUCE_FORCE_FILTER,
    "filter8": _lib.REDUCE_FORCE_FILTER8,
    "smem16": _lib.REDUCE_FORCE_SMEM16,
    "sampled": _lib.REDUCE_FORCE_SAMPLED,
    "sampled_fused": _lib.REDUCE_FORCE_SAMPLED | 16384,
    "smem16_tma": _lib.REDUCE_FORCE_SMEM16 | 4096,
    # group filter: 32-bit words, RED-only and read-first misses, TMA ring
    "filter16": _lib.REDUCE_FORCE_FILTER | 512,
    "filter_red": _lib.REDUCE_FORCE_FILTER | 128,
    "filter_read_tma": _lib.REDUCE_FORCE_FILTER | 256 | 4096,
    "sampled_tma": _lib.REDUCE_FORCE_SAMPLED | 4096,
    "sampled_split": _lib.REDUCE_FORCE_SAMPLED | _lib.REDUCE_SAMPLE_SPLIT,
    "smem16_blocked": _lib.REDUCE_FORCE_SMEM16 | _lib.REDUCE_BLOCKED,
    "filter_blocked": _lib.REDUCE_FORCE_FILTER | _lib.REDUCE_BLOCKED,
    "sampled_prefix": _lib.REDUCE_FORCE_SAMPLED | _lib.REDUCE_SAMPLE_PREFIX,
    "sampled_split_prefix": _lib.REDUCE_FORCE_SAMPLED | _lib.REDUCE_SAMPLE_SPLIT | _lib.REDUCE_SAMPLE_PREFIX,
}


def run_device(ctx, xy_np, p, q, flags=0, offset_points=0):
    """H2D, K1, K3 (all outputs), K4, D2H.  offset_points > 0 places the
    input at an 8-byte (not 16-byte) aligned address."""
    n = len(xy_np)
    buf = torch.empty((n + offset_points, 2), dtype=torch.int32, device="cuda")
    buf[offset_points:] = torch.from_numpy(np.ascontiguousarray(xy_np))
    xy = buf[offset_points:]
    DL = ctx.reduce(xy, p, q=q, flags=flags)
    comp = ctx.compact(DL, p, chain=True, occ=True, lpairs=True, lower=True, upper=True, upperd=True)
    hull = ctx.hull(comp, p)
    ns = ctx.ns_chain(comp, p)
    torch.cuda.synchronize()
    c = comp["counts"].cpu().numpy()
    s, v = int(c[0]), int(c[1])
    h = int(hull["h"].item())
    return {
        "err": int(c[2]), "s": s, "v": v,
        "L": comp["lpairs"].cpu().numpy(),
        "occ": comp["occ"].cpu().numpy().view(np.uint64),
        "chain": comp["chain"][:s].cpu().numpy(),
        "ns": ns[:s].cpu().numpy(),
        "hull": hull["hull"][:h].cpu().numpy(),
    }


def check_against_oracle(orc, got, xy, p, q):
    arr = orc.reduce(xy, p, q)
    assert got["err"] == 0
    assert np.array_equal(got["L"], orc.L_pairs(arr)), "L mismatch"
    assert np.array_equal(got["occ"], arr["occ"]), "occupancy words mismatch"
    s = orc.valid_count(arr)
    assert got["s"] == s
    if s == 0:
        return
    chain = orc.build_polyline(arr)
    assert np.array_equal(got["chain"], chain), "Lemma-1 chain mismatch"
    assert np.array_equal(got["ns"], orc.ns_chain(arr)), "north_star chain mismatch"
    assert np.array_equal(got["hull"], orc.melkman(chain)), "hull mismatch"


DOWNSCALED = [  # (config, p, n)
    (2, 65536, 3_000_000),
    (2, 4096, 1_000_000),
    (3, 16384, 3_000_000),
    (4, 1 << 20, 3_000_000),
    (4, 8192, 1_000_000),
    (5, 256, 3_000_000),
    # >= 4 Mi points: the q-known group filter's phased mode (snapshot
    # rebuilds between phases of doubling length, csrc/reduce.cu plan_for)
    (4, 1 << 20, 10_000_000),
]


@pytest.mark.parametrize("config,p,n", DOWNSCALED)
@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_downscaled_configs(ctx, orc, config, p, n, variant):
    if variant == "smem32" and p * 8 > 200 * 1024:
        pytest.skip("table does not fit shared memory")
    xy = generate_host(config, config, p, n)
    got = run_device(ctx, xy, p, p, VARIANTS[variant])
    check_against_oracle(orc, got, xy, p, p)


def test_device_generator_matches_host(ctx):
    for config, p in ((2, 65536), (3, 16384), (4, 1 << 20), (5, 256)):
        n, off = 1_000_003, 123_456_789
        d = ctx.generate(config, config, p, n, offset=off).cpu().numpy()
        h = generate_host(config, config, p, n, offset=off)
        assert np.array_equal(d, h), f"config {config}: device and host generators disagree"


def test_config1_golden_digests(ctx, orc):
    """SURVEY.md Appendix A, produced by the reference itself."""
    xy = orc.uniform_box(1_000_000, 4096, 1)
    assert orc.fnv(xy) == "17239ebe0273b7d1"
    for flags in VARIANTS.values():
        got = run_device(ctx, xy, 4096, 4096, flags)
        assert orc.fnv(got["L"]) == "b5b55891aaae7596"
        assert got["s"] == 8192
        assert orc.fnv(got["chain"]) == "27d9354c9f73a66e"
        assert got["hull"].tolist() == [[1, 49], [2, 3], [15, 1], [4067, 1], [4093, 4], [4095, 7], [4096, 56],
                                        [4096, 4092], [4093, 4096], [21, 4096], [3, 4091], [1, 4071]]


@pytest.mark.parametrize("offset_points", [0, 1])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 31, 1001])
def test_alignment_and_ragged_sizes(ctx, orc, n, offset_points):
    rng = np.random.default_rng(n)
    xy = rng.integers(1, 41, size=(n, 2)).astype(np.int32)
    for flags in VARIANTS.values():
        got = run_device(ctx, xy, 40, None, flags, offset_points)
        check_against_oracle(orc, got, xy, 40, None)


def test_empty_input(ctx):
    xy = np.empty((0, 2), np.int32)
    got = run_device(ctx, xy, 5, None)
    assert got["s"] == 0 and got["v"] == 0 and got["err"] == 0
    assert got["L"].tolist() == [[6, -1]] * 5


@pytest.mark.parametrize("bad", [(6, 1), (0, 1), (1, 0), (1, 6), (-2147483648, 3), (3, -2147483648)])
def test_validation_flags_invalid_points(ctx, bad):
    xy = np.array([[1, 1], [2, 2], bad, [3, 3]], np.int32)
    d = torch.from_numpy(xy).cuda()
    for flags in VARIANTS.values():
        DL = ctx.reduce(d, 5, q=5, flags=flags)
        with pytest.raises(ValueError):
            ctx.check(DL, 5)


def test_large_y_without_q(ctx, orc):
    """No q: y may reach INT32_MAX (the ~y encoding keeps it exact)."""
    xy = np.array([[1, 2147483647], [1, 1], [2, 2147483647], [3, 5], [3, 2147483646]], np.int32)
    for flags in VARIANTS.values():
        got = run_device(ctx, xy, 3, None, flags)
        check_against_oracle(orc, got, xy, 3, None)


@pytest.mark.parametrize("p", [65536, 1 << 20])
@pytest.mark.parametrize("case", ["narrow_prefix", "sorted_desc", "gaussian"])
def test_q_unset_speculative_range(ctx, orc, case, p):
    """q unset with a width beyond the smem tables: the sampled filter
    (p = 2^16) or the group filter (p = 2^20) quantises the y range of the
    first 2^18 points; points outside it (both sides, far) must still be
    exact, and an invalid y must still fail."""
    rng = np.random.default_rng(77)
    n = 3_000_000 if p == 65536 else 6_000_000  # (the group filter phases start at 4 Mi points)
    x = rng.integers(1, p + 1, size=n)
    if case == "narrow_prefix":
        y = rng.integers(1000, 2000, size=n)
        tail = np.arange(n) >= (1 << 18)
        y[tail] = rng.integers(1, 2147483647, size=int(tail.sum()))
    elif case == "sorted_desc":
        y = np.sort(rng.integers(1, 1 << 30, size=n))[::-1].copy()
    else:
        y = np.clip(np.rint(rng.normal(p / 2, p / 8, size=n)), 1, p)
    xy = np.stack([x, y], axis=1).astype(np.int32)
    got = run_device(ctx, xy, p, None)
    assert ctx.variant.startswith("sampled" if p == 65536 else "filter") and ctx.variant.endswith("yspec"), \
        ctx.variant
    check_against_oracle(orc, got, xy, p, None)
    bad = xy.copy()
    bad[n - 5] = (7, 0)
    DL = ctx.reduce(torch.from_numpy(bad).cuda(), p)
    with pytest.raises(ValueError):
        ctx.check(DL, p)


def test_randomized_fixtures(ctx, orc):
    rng = np.random.default_rng(2026)
    for trial in range(300):
        n = int(rng.integers(1, 400)) if trial % 50 else 20000
        pts, p = to_unit_box(mixed_case(rng, n))
        for flags in (0, _lib.REDUCE_FORCE_GLOBAL):
            got = run_device(ctx, pts, p, None, flags)
            check_against_oracle(orc, got, pts, p, None)


def test_heavy_skew_single_column(ctx, orc):
    """Every point in one column (maximum contention), and two-point columns."""
    rng = np.random.default_rng(9)
    n = 2_000_000
    xy = np.stack([np.full(n, 7), rng.integers(1, 1 << 20, size=n)], axis=1).astype(np.int32)
    for flags in VARIANTS.values():
        got = run_device(ctx, xy, 1 << 10, 1 << 20, flags)
        check_against_oracle(orc, got, xy, 1 << 10, 1 << 20)


def test_full_size_config2_vs_oracle(ctx, orc):
    """BASELINE.json config 2 at full size (n = 1e8) against the oracle."""
    p, n = 65536, 100_000_000
    d = ctx.generate(2, 2, p, n)
    DL = ctx.reduce(d, p, q=p)
    comp = ctx.compact(DL, p, chain=True, lpairs=True, lower=True, upper=True)
    hull = ctx.hull(comp, p)
    torch.cuda.synchronize()
    xy = d.cpu().numpy()
    del d
    arr = orc.reduce(xy, p, p)
    c = comp["counts"].cpu().numpy()
    assert np.array_equal(comp["lpairs"].cpu().numpy(), orc.L_pairs(arr))
    chain = orc.build_polyline(arr)
    assert int(c[0]) == len(chain)
    assert np.array_equal(comp["chain"][: int(c[0])].cpu().numpy(), chain)
    h = int(hull["h"].item())
    assert np.array_equal(hull["hull"][:h].cpu().numpy(), orc.melkman(chain))


def _host_mem_available() -> int:
    with open("/proc/meminfo") as f:
        for line in f:
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    return 0


FULL_VARIANTS = ("auto", "global", "filter", "sampled", "smem16")


@pytest.mark.parametrize("config", [3, 4, 5])
def test_full_size_vs_oracle(ctx, orc, config):
    """BASELINE.json configs 3-5 at full size (1e9 / 1e9 / 4e9 points)
    against the oracle, bit for bit: L (serialize form), occupancy words,
    s, the Lemma-1 chain, the north_star chain and the hull, for the auto
    variant (q given and q unset) and every forced K1 variant.  The oracle reads the device's own
    input bytes back in 1 GB chunks and reduces them with SURVEY.md 8(c)'s
    chunked procedure (reduce per slice on host threads, slot-by-slot merge,
    then the survivors reduced once more), so nothing of 8-32 GB has to sit
    in host memory at once."""
    import bench

    n, p, seed, _ = bench.CONFIGS[config]
    need_host = (1 << 30) + 64 * 9 * p + (2 << 30)
    if _host_mem_available() < need_host:
        pytest.skip(f"needs ~{need_host / 2**30:.1f} GiB of available host RAM (1 GiB pinned chunk + oracle tables)")
    free = torch.cuda.mem_get_info()[0]
    if n * 8 + (1 << 30) > free:
        pytest.skip(f"needs {(n * 8 + (1 << 30)) / 2**30:.1f} GiB of free device memory")
    d = ctx.generate(config, seed, p, n)
    got = {}
    for name in FULL_VARIANTS + ("auto_q_unset",):
        # (q unset: the reference API's default; every y is valid here, so the
        # L is the same and the speculative-range variants must reproduce it)
        q = None if name == "auto_q_unset" else p
        DL = ctx.reduce(d, p, q=q, flags=VARIANTS.get(name, 0))
        comp = ctx.compact(DL, p, chain=True, occ=True, lpairs=True, lower=True, upper=True, upperd=True)
        hull = ctx.hull(comp, p)
        ns = ctx.ns_chain(comp, p)
        torch.cuda.synchronize()
        c = comp["counts"].cpu().numpy()
        s, h = int(c[0]), int(hull["h"].item())
        got[name] = {"variant": ctx.variant, "err": int(c[2]), "s": s, "L": comp["lpairs"].cpu().numpy(),
                     "occ": comp["occ"].cpu().numpy().view(np.uint64), "chain": comp["chain"][:s].cpu().numpy(),
                     "ns": ns[:s].cpu().numpy(), "hull": hull["hull"][:h].cpu().numpy()}
        del DL, comp, hull, ns
    acc = orc.accumulator(p, p)
    chunk = 1 << 27  # points (1 GiB)
    host = torch.empty((chunk, 2), dtype=torch.int32, pin_memory=True)
    for a in range(0, n, chunk):
        m = min(chunk, n - a)
        host[:m].copy_(d[a:a + m])
        acc.add(host[:m].numpy())
    assert acc.points == n
    del host, d
    arr = acc.finish()
    L = orc.L_pairs(arr)
    chain = orc.build_polyline(arr)
    ns = orc.ns_chain(arr)
    hull = orc.melkman(chain)
    for name, g in got.items():
        tag = f"config {config}, variant {name} ({g['variant']})"
        assert g["err"] == 0, tag
        assert np.array_equal(g["L"], L), "L mismatch: " + tag
        assert np.array_equal(g["occ"], arr["occ"]), "occupancy mismatch: " + tag
        assert g["s"] == len(chain), tag
        assert np.array_equal(g["chain"], chain), "Lemma-1 chain mismatch: " + tag
        assert np.array_equal(g["ns"], ns), "north_star chain mismatch: " + tag
        assert np.array_equal(g["hull"], hull), "hull mismatch: " + tag


@pytest.mark.parametrize("config", [3, 4, 5])
def test_full_size_properties(ctx, config):
    """Full BASELINE sizes (1e9 / 1e9 / 4e9 points): size-independent
    properties.  (1) every K1 variant yields the same L; (2) sharding the
    input and MIN-merging partial DLs (the multi-GPU combine) equals the
    one-shot L; (3) idempotence: reducing the chain reproduces L;
    (4) s <= 2p."""
    import bench

    n, p, seed, _ = bench.CONFIGS[config]
    free = torch.cuda.mem_get_info()[0]
    if n * 8 > free * 0.8:
        pytest.skip("not enough device memory")
    d = ctx.generate(config, seed, p, n)
    ref_dl = ctx.reduce(d, p, q=p).clone()
    for flags in (_lib.REDUCE_FORCE_GLOBAL, _lib.REDUCE_FORCE_FILTER, _lib.REDUCE_FORCE_SAMPLED):
        assert torch.equal(ctx.reduce(d, p, q=p, flags=flags), ref_dl)
    half = n // 2
    a = ctx.reduce(d[:half], p, q=p).clone()
    b = ctx.reduce(d[half:], p, q=p)
    assert torch.equal(torch.minimum(a, b), ref_dl)
    comp = ctx.compact(ref_dl, p, chain=True, lpairs=True)
    s = int(comp["counts"][0].item())
    assert 0 < s <= 2 * p
    again = ctx.reduce(comp["chain"][:s].contiguous(), p, q=p)
    assert torch.equal(again, ref_dl)


def test_hull_multi_launch_form():
    """K4 runs as one cooperative kernel when it can; the per-stage launch
    form (CHP_HULL_LAUNCHES=1, read once per process) must agree."""
    import os
    import subprocess
    import sys

    code = r"""
import numpy as np, torch, sys
sys.path.insert(0, %r)
import oracle
from paper_1505_00914_b200.device import Context, generate_host
orc = oracle.Oracle()
ctx = Context(0)
for config, p, n in ((2, 65536, 2_000_000), (3, 16384, 2_000_000), (4, 1 << 20, 2_000_000), (5, 256, 100_000)):
    xy = generate_host(config, config, p, n)
    DL = ctx.reduce(torch.from_numpy(xy).cuda(), p, q=p)
    comp = ctx.compact(DL, p, chain=True, lower=True, upper=True)
    hull = ctx.hull(comp, p)
    torch.cuda.synchronize()
    h = int(hull["h"].item())
    s = int(comp["counts"][0].item())
    chain = comp["chain"][:s].cpu().numpy()
    assert np.array_equal(hull["hull"][:h].cpu().numpy(), orc.melkman(chain)), config
print("ok")
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for env in ({"CHP_HULL_LAUNCHES": "1"}, {}):
        r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


@pytest.mark.parametrize("p", [(1 << 17) - 3, 1 << 17, (1 << 17) + 1, (1 << 17) + 2053, 3_000_001])
def test_compact_tile_forms(ctx, orc, p):
    """K3 takes 1024-slot tiles (256 threads x 4, striped) up to 2^17 slots
    and 4096-slot tiles (256 x 16) beyond; widths around the switch, ragged
    last tiles, partial occupancy words and sparse columns."""
    rng = np.random.default_rng(p)
    n = 400_000
    x = rng.integers(1, p + 1, size=n)
    x[:1000] = p  # the last slot
    x[1000:2000] = 1
    xy = np.stack([x, rng.integers(1, 1 << 20, size=n)], axis=1).astype(np.int32)
    got = run_device(ctx, xy, p, 1 << 20)
    check_against_oracle(orc, got, xy, p, 1 << 20)


def test_maximum_width(ctx, orc):
    """The device limit, width = 2^29 columns (31-bit look-back counters;
    SURVEY.md 8(b)): a sparse input over the whole width, the first and last
    slot included, through K1 (group filter), K3 and K4 against the oracle."""
    p = 1 << 29
    free = torch.cuda.mem_get_info()[0]
    if free < (100 << 30) or _host_mem_available() < (48 << 30):
        pytest.skip("needs ~100 GiB of free device memory and ~48 GiB of host RAM")
    rng = np.random.default_rng(29)
    n = 2_000_000
    xy = np.stack([rng.integers(1, p + 1, size=n), rng.integers(1, 1 << 30, size=n)], axis=1).astype(np.int32)
    xy[:5] = [[1, 7], [1, 9], [p, 3], [p, 1 << 29], [p // 2, 5]]
    got = run_device(ctx, xy, p, None)
    check_against_oracle(orc, got, xy, p, None)


def test_width_beyond_device_limit_rejected(ctx):
    """Beyond 2^29 columns the compaction and hull refuse (ValueError, the
    drop-in's std::invalid_argument) instead of overflowing their counters."""
    p = (1 << 29) + 1
    DL = torch.empty(2, dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):
        ctx.compact(DL, p, chain=False)
    with pytest.raises(ValueError):
        ctx.pipeline_host(np.array([[1, 1]], np.int32), p, 5)
