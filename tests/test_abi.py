"""The C-ABI library without a GPU: it loads, exports every symbol
include/chp_b200.h declares, rejects a context when no device is visible,
and its host-side generators are deterministic, offset-consistent and have
the BASELINE.json shapes."""
import os
import re

import numpy as np
import pytest
import torch

from paper_1505_00914_b200 import _lib
from paper_1505_00914_b200.device import generate_host

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "chp_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(chp_\w+)\s*\(", text)))


def test_header_symbols_all_exported(lib):
    declared = header_functions()
    assert len(declared) >= 20
    assert set(declared) == set(_lib.ABI_SYMBOLS)
    for name in declared:
        assert getattr(lib, name) is not None


def test_dl_len(lib):
    assert lib.chp_dl_len(5) == 12
    assert lib.chp_dl_len(65536) == 2 * 65536 + 2


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device path")
def test_context_without_device_fails_cleanly(lib):
    from ctypes import byref, c_void_p

    h = c_void_p()
    assert lib.chp_ctx_create(0, byref(h)) == _lib.CHP_EDEVICE
    assert not h.value


def test_no_cpu_fallback_without_device():
    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_1505_00914_b200 import reducer

    with pytest.raises(Exception):
        reducer.reduce([(1, 1)], 5)


@pytest.mark.parametrize("config,p", [(2, 65536), (3, 16384), (4, 1 << 20), (5, 256)])
def test_generator_shapes_and_determinism(config, p):
    a = generate_host(config, config, p, 200_000)
    b = generate_host(config, config, p, 200_000, threads=1)
    assert np.array_equal(a, b)
    tail = generate_host(config, config, p, 1000, offset=199_000)
    assert np.array_equal(a[199_000:], tail)
    assert a.min() >= 1 and a.max() <= p
    x, y = a[:, 0].astype(np.int64), a[:, 1].astype(np.int64)
    if config == 2:
        assert abs(x.mean() - p / 2) < p / 100 and abs(x.std() - p / 8) < p / 50
    if config == 3:
        r2 = (x - p / 2) ** 2 + (y - p / 2) ** 2
        assert r2.max() <= (p / 2 + 1) ** 2
    if config == 5:
        hot = (x >= p // 2 - 1) & (x <= p // 2 + 2)
        assert 0.89 < hot.mean() < 0.92


def test_generator_rejects_bad_config():
    with pytest.raises(ValueError):
        generate_host(1, 1, 4096, 10)
    with pytest.raises(ValueError):
        generate_host(2, 1, 0, 10)
