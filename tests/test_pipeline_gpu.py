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
