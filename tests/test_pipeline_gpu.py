"""The host-buffer pipelines (chp_pipeline_host / chp_precondition_host):
inputs larger than one 16 Mi-point chunk, pinned and pageable, so the
chunked H2D copy, the copy/compute overlap and the accumulating per-chunk
K1 launches are exercised.  Checked bit for bit against the oracle."""
import numpy as np
import pytest
import torch

from paper_1505_00914_b200.device import generate_host

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("config,p", [(2, 65536), (3, 16384), (5, 256)])
@pytest.mark.parametrize("pinned", [False, True])
def test_pipeline_host_multi_chunk(ctx, orc, config, p, pinned):
    n = 40_000_001  # three chunks, odd tail
    xy = generate_host(config, config, p, n)
    if pinned:
        t = torch.empty((n, 2), dtype=torch.int32, pin_memory=True)
        t.copy_(torch.from_numpy(xy))
        xy = t.numpy()
    out = ctx.pipeline_host(xy, p, p, L=True, occ=True, chain=True, hull=True)
    ref = orc.pipeline(xy, p, p)
    assert np.array_equal(out["L"], ref["L"])
    assert np.array_equal(out["occ"], ref["arr"]["occ"])
    assert np.array_equal(out["chain"], ref["chain"])
    assert np.array_equal(out["hull"], ref["hull"])


def test_precondition_host_large(ctx, orc):
    n = 20_000_000
    xy = generate_host(4, 4, 1 << 20, n)
    xy[:, 0] -= 12345  # untranslated input: precondition finds the offsets
    xy[:, 1] -= 777
    out = ctx.precondition_host(xy, chain=True, hull=True)
    ref = orc.precondition(xy)
    assert out["bbox"] == ref["bbox"]
    assert np.array_equal(out["chain"], ref["chain"])
    assert np.array_equal(out["hull"], ref["hull"])


def test_pipeline_host_invalid_point_raises(ctx):
    xy = generate_host(2, 2, 65536, 17_000_000)
    xy[16_777_300] = (65537, 5)  # in the second chunk
    with pytest.raises(ValueError):
        ctx.pipeline_host(xy, 65536, 65536)


# The packed transfer (slot | (y - 1) << 16 words, 4 bytes per point) is taken
# when width <= 2^16 and q <= 2^16; the int32 path otherwise.  Both must give
# the same answers and the same errors.
def _pinned(xy):
    t = torch.empty(xy.shape, dtype=torch.int32, pin_memory=True)
    t.copy_(torch.from_numpy(xy))
    return t.numpy()


@pytest.mark.parametrize("n", [1, 3, 4, 5, 1001, 16_777_216 + 7])
@pytest.mark.parametrize("pinned", [False, True])
def test_pipeline_host_packed_sizes(ctx, orc, n, pinned):
    # pinned input: the hybrid form (packed front + int32 chunks from the back)
    p = 4096
    xy = generate_host(2, 11, p, n)
    if pinned:
        xy = _pinned(xy)
    out = ctx.pipeline_host(xy, p, p, L=True, chain=True)
    if pinned:
        assert 4 * n <= ctx.last_h2d_bytes <= 8 * n
    else:
        assert ctx.last_h2d_bytes == 4 * n
    ref = orc.pipeline(xy, p, p)
    assert np.array_equal(out["L"], ref["L"])
    assert np.array_equal(out["chain"], ref["chain"])


def test_pipeline_host_unpacked_when_wide(ctx, orc):
    p = 65536
    xy = generate_host(2, 2, p, 100_000)
    xy[:, 1] = xy[:, 1] * 64  # y up to 2^22: q > 2^21 -> int32 transfer
    out = ctx.pipeline_host(xy, p, 64 * p, L=True, chain=True)
    assert ctx.last_h2d_bytes == 8 * len(xy)
    ref = orc.pipeline(xy, p, 64 * p)
    assert np.array_equal(out["L"], ref["L"])
    assert np.array_equal(out["chain"], ref["chain"])


# Known ranges up to 2^21 x 2^21 travel as 42-bit points, three per 16 bytes.
@pytest.mark.parametrize("n", [1, 2, 3, 4, 1001, 8_388_608 + 5, 20_000_001])
@pytest.mark.parametrize("pinned", [False, True])
def test_pipeline_host_packed42(ctx, orc, n, pinned):
    p = 1 << 20
    xy = generate_host(4, 4, p, n)
    if pinned:
        xy = _pinned(xy)
    out = ctx.pipeline_host(xy, p, p, L=True, chain=True, hull=True)
    if not pinned:  # (pinned input: part of it goes as int32 pairs from the end)
        assert ctx.last_h2d_bytes == (n + 2) // 3 * 16
    ref = orc.pipeline(xy, p, p)
    assert np.array_equal(out["L"], ref["L"])
    assert np.array_equal(out["chain"], ref["chain"])
    assert np.array_equal(out["hull"], ref["hull"])


def test_pipeline_host_packed42_extremes(ctx, orc):
    # the 21-bit fields at both ends, in every position of a 3-point word
    p, q = 1 << 21, 1 << 21
    base = np.array([[1, 1], [1, q], [p, 1], [p, q], [300, 7], [p - 1, q - 1], [2, 2]], np.int32)
    for shift in range(3):
        xy = np.concatenate([np.full((shift, 2), 5, np.int32), np.repeat(base, 301, axis=0)])
        out = ctx.pipeline_host(xy, p, q, L=True, chain=True)
        ref = orc.pipeline(xy, p, q)
        assert np.array_equal(out["L"], ref["L"])
        assert np.array_equal(out["chain"], ref["chain"])


@pytest.mark.parametrize("bad", [(0, 5), ((1 << 20) + 1, 5), (7, 0), (7, (1 << 20) + 1), (-2**31, 1)])
@pytest.mark.parametrize("where", [0, 1, 2, 999_999])
def test_pipeline_host_packed42_invalid_raises(ctx, bad, where):
    p = 1 << 20
    xy = generate_host(4, 4, p, 1_000_000)
    xy[where] = bad
    with pytest.raises(ValueError):
        ctx.pipeline_host(xy, p, p)


@pytest.mark.parametrize("bad", [(0, 5), (4097, 5), (7, 0), (7, 4097), (-2**31, 1), (2**31 - 1, 2**31 - 1)])
@pytest.mark.parametrize("where", [0, 2, 999_999])
@pytest.mark.parametrize("pinned", [False, True])
def test_pipeline_host_packed_invalid_raises(ctx, bad, where, pinned):
    p = 4096
    xy = generate_host(2, 2, p, 1_000_000)
    if pinned:
        xy = _pinned(xy)
    xy[where] = bad
    with pytest.raises(ValueError):
        ctx.pipeline_host(xy, p, p)
    xy[where] = (1, 1)  # and the context is still usable afterwards
    ctx.pipeline_host(xy, p, p)


def test_pipeline_host_packed_extremes(ctx, orc):
    # slots 0 and p-1, y = 1 and y = q: the 16-bit fields at both ends
    p = 65536
    xy = np.array([[1, 1], [1, 65536], [65536, 1], [65536, 65536], [300, 7]], np.int32)
    xy = np.repeat(xy, 1000, axis=0)
    out = ctx.pipeline_host(xy, p, p, L=True, chain=True)
    ref = orc.pipeline(xy, p, p)
    assert np.array_equal(out["L"], ref["L"])
    assert np.array_equal(out["chain"], ref["chain"])


# precondition runs K1 with the bounding box's y range as the valid range
# (ybase = ymin), so the filter variants and the 16-bit packing apply to
# untranslated inputs; a range of 2^32 - 1 values or more falls back.
@pytest.mark.parametrize("shift", [(-100_000, -50_000), (7, 1_000_000), (-2**31 + 5, -2**31 + 9)])
def test_precondition_host_y_range(ctx, orc, shift):
    xy = generate_host(2, 21, 65536, 2_000_000)
    xy[:, 0] += shift[0]
    xy[:, 1] += shift[1]
    out = ctx.precondition_host(xy, chain=True, hull=True)
    ref = orc.precondition(xy)
    assert out["bbox"] == ref["bbox"]
    assert np.array_equal(out["chain"], ref["chain"])
    assert np.array_equal(out["hull"], ref["hull"])


@pytest.mark.parametrize("ys", [(-2**31, 2**31 - 1), (-2**31 + 1, 2**31 - 1), (-2**31 + 1, 2**31 - 2), (0, 0)])
def test_precondition_host_extreme_y(ctx, orc, ys):
    xy = generate_host(3, 5, 1024, 300_000)
    xy[0, 1] = ys[0]
    xy[1, 1] = ys[1]
    out = ctx.precondition_host(xy, chain=True)
    ref = orc.precondition(xy)
    assert out["bbox"] == ref["bbox"]
    assert np.array_equal(out["chain"], ref["chain"])


def test_precondition_device_narrow_y_uses_fast_variant(ctx, orc):
    # y range of 300 values at a negative offset: smem16 with ybase != 1
    rng = np.random.default_rng(3)
    xy = np.stack([rng.integers(-5000, -4000, 1_000_000), rng.integers(-70_000, -69_700, 1_000_000)], 1)
    xy = xy.astype(np.int32)
    out = ctx.precondition_host(xy, chain=True, hull=True)
    assert ctx.variant in ("smem16", "smem16+tma")
    ref = orc.precondition(xy)
    assert out["bbox"] == ref["bbox"]
    assert np.array_equal(out["chain"], ref["chain"])
    assert np.array_equal(out["hull"], ref["hull"])


@pytest.mark.parametrize("shift", [(0, 0), (-100_000, -50_000), (3, 2**31 - 70_000)])
def test_precondition_host_streamed(ctx, orc, shift, monkeypatch):
    # the form taken when the input does not fit a quarter of free device
    # memory: bounds streamed, then K1 streamed (packed when the box fits 16 bits)
    monkeypatch.setenv("CHP_PRECONDITION_STREAM", "1")
    xy = generate_host(2, 22, 65536, 20_000_001)
    xy[:, 0] += shift[0]
    xy[:, 1] += shift[1]
    out = ctx.precondition_host(xy, chain=True, hull=True)
    assert ctx.last_h2d_bytes == 8 * len(xy) + 4 * len(xy)  # int32 bounds pass + packed K1 pass
    ref = orc.precondition(xy)
    assert out["bbox"] == ref["bbox"]
    assert np.array_equal(out["chain"], ref["chain"])
    assert np.array_equal(out["hull"], ref["hull"])


# q unset (the reference's default, y only >= 1): the host packs
# speculatively against a 2^16 window; a chunk holding a larger y goes as
# int32 pairs, and K1 validates it.
@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("big_y_at", [None, 5, 9_000_000, 17_999_999])
def test_pipeline_host_q_unset(ctx, orc, pinned, big_y_at):
    p = 65536
    xy = generate_host(2, 31, p, 18_000_000)
    if big_y_at is not None:
        xy[big_y_at, 1] = 2**31 - 1  # valid without q
    if pinned:
        xy = _pinned(xy)
    out = ctx.pipeline_host(xy, p, None, L=True, chain=True)
    assert 4 * len(xy) <= ctx.last_h2d_bytes <= 8 * len(xy)
    if not pinned:  # pageable: packed, except the one 8 Mi-point chunk holding the big y
        c = 8 << 20
        extra = 0 if big_y_at is None else 4 * min(c, len(xy) - (big_y_at // c) * c)
        assert ctx.last_h2d_bytes == 4 * len(xy) + extra
    ref = orc.pipeline(xy, p, None)
    assert np.array_equal(out["L"], ref["L"])
    assert np.array_equal(out["chain"], ref["chain"])


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("bad", [(7, 0), (0, 7), (65537, 7), (7, -5)])
def test_pipeline_host_q_unset_invalid(ctx, pinned, bad):
    p = 65536
    xy = generate_host(2, 32, p, 3_000_000)
    xy[2_500_000] = bad
    if pinned:
        xy = _pinned(xy)
    with pytest.raises(ValueError):
        ctx.pipeline_host(xy, p, None)


@pytest.mark.parametrize("pinned", [False, True])
def test_precondition_speculative_window(ctx, orc, pinned):
    # The packing window comes from the first 64 Ki points; later chunks that
    # leave it (here: x and y spread 4x wider after 9 M points) go as int32.
    rng = np.random.default_rng(77)
    n = 20_000_000
    xy = np.empty((n, 2), np.int32)
    xy[:9_000_000, 0] = rng.integers(-70_000, -50_000, 9_000_000)
    xy[:9_000_000, 1] = rng.integers(1000, 30_000, 9_000_000)
    xy[9_000_000:, 0] = rng.integers(-120_000, 10_000, n - 9_000_000)
    xy[9_000_000:, 1] = rng.integers(-50_000, 90_000, n - 9_000_000)
    if pinned:
        xy = _pinned(xy)
    out = ctx.precondition_host(xy, chain=True, hull=True)
    assert 4 * n < ctx.last_h2d_bytes <= 8 * n  # some chunks packed, some not
    ref = orc.precondition(xy)
    assert out["bbox"] == ref["bbox"]
    assert np.array_equal(out["chain"], ref["chain"])
    assert np.array_equal(out["hull"], ref["hull"])


@pytest.mark.parametrize("pinned", [False, True])
def test_precondition_speculative_window42(ctx, orc, pinned):
    # A prefix wider than 2^16 takes a 2^21 window and the 42-bit form; a later
    # chunk that leaves the window (a 2^24-wide spread after 12 M points) goes
    # as int32 pairs, and its points still count.
    rng = np.random.default_rng(78)
    n = 20_000_000
    xy = np.empty((n, 2), np.int32)
    xy[:12_000_000, 0] = rng.integers(-400_000, 300_000, 12_000_000)
    xy[:12_000_000, 1] = rng.integers(5, 900_000, 12_000_000)
    xy[12_000_000:, 0] = rng.integers(-(1 << 23), 1 << 23, n - 12_000_000)
    xy[12_000_000:, 1] = rng.integers(-(1 << 23), 1 << 23, n - 12_000_000)
    if pinned:
        xy = _pinned(xy)
    out = ctx.precondition_host(xy, chain=True, hull=True)
    assert 16 * n // 3 < ctx.last_h2d_bytes < 8 * n  # some chunks packed (42-bit), some not
    ref = orc.precondition(xy)
    assert out["bbox"] == ref["bbox"]
    assert np.array_equal(out["chain"], ref["chain"])
    assert np.array_equal(out["hull"], ref["hull"])


# Known ranges up to 2^8 x 2^8 (C5: 256 x 256) travel as 16-bit points,
# eight per 16 bytes (2 bytes per point instead of 8).
def _packed8_bytes(n, chunk=8 << 20):
    return sum((min(chunk, n - a) + 7) // 8 * 16 for a in range(0, n, chunk))


@pytest.mark.parametrize("n", [1, 7, 8, 9, 15, 16, 17, 1001, 8_388_608 + 13, 20_000_001])
@pytest.mark.parametrize("pinned", [False, True])
def test_pipeline_host_packed8(ctx, orc, n, pinned):
    p = 256
    xy = generate_host(5, 5, p, n)
    if pinned:
        xy = _pinned(xy)
    out = ctx.pipeline_host(xy, p, p, L=True, chain=True, hull=True)
    if pinned:  # (part of it goes as int32 pairs from the end)
        assert 2 * n <= ctx.last_h2d_bytes <= 8 * n + 16
    else:
        assert ctx.last_h2d_bytes == _packed8_bytes(n)
    ref = orc.pipeline(xy, p, p)
    assert np.array_equal(out["L"], ref["L"])
    assert np.array_equal(out["chain"], ref["chain"])
    assert np.array_equal(out["hull"], ref["hull"])


def test_pipeline_host_packed8_extremes(ctx, orc):
    # the 8-bit fields at both ends, in every position of a 16-point AVX2 step
    p, q = 256, 256
    base = np.array([[1, 1], [1, q], [p, 1], [p, q], [100, 7], [p - 1, q - 1], [2, 2]], np.int32)
    for shift in range(17):
        xy = np.concatenate([np.full((shift, 2), 5, np.int32), np.repeat(base, 37, axis=0)])
        out = ctx.pipeline_host(xy, p, q, L=True, chain=True)
        ref = orc.pipeline(xy, p, q)
        assert np.array_equal(out["L"], ref["L"])
        assert np.array_equal(out["chain"], ref["chain"])
    # a narrower box inside the 8-bit window (w = 100, q = 37)
    xy = np.stack([np.arange(1, 10_001) % 100 + 1, np.arange(10_000) % 37 + 1], axis=1).astype(np.int32)
    out = ctx.pipeline_host(xy, 100, 37, L=True, chain=True)
    ref = orc.pipeline(xy, 100, 37)
    assert np.array_equal(out["L"], ref["L"]) and np.array_equal(out["chain"], ref["chain"])


@pytest.mark.parametrize("bad", [(0, 5), (257, 5), (7, 0), (7, 257), (-2**31, 1), (2**31 - 1, 2**31 - 1)])
@pytest.mark.parametrize("where", [0, 15, 16, 999_999])
@pytest.mark.parametrize("pinned", [False, True])
def test_pipeline_host_packed8_invalid_raises(ctx, bad, where, pinned):
    p = 256
    xy = generate_host(5, 5, p, 1_000_000)
    if pinned:
        xy = _pinned(xy)
    xy[where] = bad
    with pytest.raises(ValueError):
        ctx.pipeline_host(xy, p, p)
    xy[where] = (1, 1)
    ctx.pipeline_host(xy, p, p)


@pytest.mark.parametrize("pinned", [False, True])
def test_precondition_speculative_window8(ctx, orc, pinned):
    # A prefix within 256 x 256 takes a 2^8 window and 2 bytes per point; a
    # later chunk that leaves it goes as int32 pairs, and its points count.
    rng = np.random.default_rng(79)
    n = 20_000_000
    xy = np.empty((n, 2), np.int32)
    xy[:, 0] = rng.integers(-5000, -4800, n)
    xy[:, 1] = rng.integers(70_000, 70_250, n)
    xy[17_000_000, 1] = 80_000  # outside the window: that chunk is sent unpacked
    if pinned:
        xy = _pinned(xy)
    out = ctx.precondition_host(xy, chain=True, hull=True)
    if not pinned:
        c = 8 << 20
        assert ctx.last_h2d_bytes == _packed8_bytes(n) - _packed8_bytes(min(c, n - 2 * c)) + 8 * (n - 2 * c)
    ref = orc.precondition(xy)
    assert out["bbox"] == ref["bbox"]
    assert np.array_equal(out["chain"], ref["chain"])
    assert np.array_equal(out["hull"], ref["hull"])


# The two halves of chp_pipeline_host (chp_reduce_host, chp_finish_host):
# partial DLs from separate host slices, merged by an element-wise MIN, give
# the one-call result; the error word survives the merge.
@pytest.mark.parametrize("config,p", [(2, 65536), (4, 1 << 20), (5, 256)])
@pytest.mark.parametrize("pinned", [False, True])
def test_reduce_host_finish_host_halves(ctx, orc, config, p, pinned):
    n = 20_000_003
    xy = generate_host(config, config, p, n)
    if pinned:
        xy = _pinned(xy)
    cut = 7_777_777
    a = ctx.reduce_host(xy[:cut], p, p)
    b = ctx.reduce_host(xy[cut:], p, p)
    merged = torch.minimum(a, b)
    out = ctx.finish_host(merged, p, L=True, chain=True, hull=True)
    ref = orc.pipeline(xy, p, p)
    assert np.array_equal(out["L"], ref["L"])
    assert out["s"] == ref["s"] and np.array_equal(out["chain"], ref["chain"])
    assert np.array_equal(out["hull"], ref["hull"])
    bad = np.array(xy[cut:cut + 1000])
    bad[500] = (p + 1, 1)
    c = ctx.reduce_host(bad, p, p)  # no raise here: the error word stays in the DL
    with pytest.raises(ValueError):
        ctx.finish_host(torch.minimum(a, c), p)


@pytest.mark.parametrize("config", [2, 3, 4, 5])
def test_full_size_host_pipeline_vs_oracle(ctx, orc, config):
    """bench.py's end-to-end paths at BASELINE.json size: the whole config
    (C2 1e8, C3 1e9, C4 1e9, C5 4e9 points) in pinned host memory through chp_pipeline_host
    (packed chunks from the host threads plus int32 chunks DMA'd from the
    input's end) and through chp_precondition_run, L, chain and hull against
    the chunked oracle over the same bytes."""
    import bench

    n, p, seed, _ = bench.CONFIGS[config]
    with open("/proc/meminfo") as f:
        avail = next(int(line.split()[1]) * 1024 for line in f if line.startswith("MemAvailable:"))
    if avail < n * 8 + (8 << 30):
        pytest.skip(f"needs {(n * 8 + (8 << 30)) / 2**30:.0f} GiB of available host RAM")
    host = torch.empty((n, 2), dtype=torch.int32, pin_memory=True)
    chunk = 1 << 27
    for a in range(0, n, chunk):  # the device generator, copied out chunk by chunk
        m = min(chunk, n - a)
        host[a:a + m].copy_(ctx.generate(config, seed, p, m, offset=a))
    hn = host.numpy()
    out = ctx.pipeline_host(hn, p, p, L=True, chain=True)
    acc = orc.accumulator(p, p)
    for a in range(0, n, chunk):
        acc.add(hn[a:a + chunk])
    arr = acc.finish()
    assert np.array_equal(out["L"], orc.L_pairs(arr))
    chain = orc.build_polyline(arr)
    assert np.array_equal(out["chain"], chain)
    # reducer::precondition (bounds unknown: one pass folds the bounds while
    # the chunks land) on the same pinned input: when the points fill their
    # p x p box its L and chain are reduce's and the hull the oracle's
    pre = ctx.precondition_host(hn, chain=True, hull=True)
    box = (int(hn[:, 0].min()), int(hn[:, 0].max()), int(hn[:, 1].min()), int(hn[:, 1].max()))
    assert pre["bbox"] == box
    if box == (1, p, 1, p):  # (else the translated L differs from reduce's; the bbox is still checked)
        assert pre["width"] == p
        assert np.array_equal(pre["chain"], chain)
        assert np.array_equal(pre["hull"], orc.melkman(chain))
