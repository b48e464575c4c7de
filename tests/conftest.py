import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


@pytest.fixture(scope="session")
def orc():
    import oracle

    if not os.path.exists(oracle.ORACLE_SO):
        oracle.build(ref=False)
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.Reference.available():
        if os.path.isdir(oracle.REF_SRC):
            oracle.build(ref=True)
        else:
            pytest.skip("oracle/_ref/libchpref.so not built and /root/reference absent")
    return oracle.Reference()


@pytest.fixture(scope="session")
def lib():
    from paper_1505_00914_b200 import _build, _lib

    if not os.path.exists(_build.LIB):
        _build.build()
    return _lib.load()


@pytest.fixture(scope="session")
def ctx(lib):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1505_00914_b200.device import Context

    return Context(0)
