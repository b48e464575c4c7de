"""The C++ drop-in (include/chp/*.hpp over libchp_b200.so) against the
reference's own known-answer tests, restated in tests/cpp/test_dropin.cpp."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
BIN = os.path.join(ROOT, "build", "test_dropin")


def build_driver(lib) -> str:
    from paper_1505_00914_b200._build import LIB

    if not os.path.exists(BIN) or os.path.getmtime(BIN) < max(os.path.getmtime(SRC), os.path.getmtime(LIB)):
        os.makedirs(os.path.dirname(BIN), exist_ok=True)
        subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-I" + os.path.join(ROOT, "include"), SRC,
                        "-L" + os.path.dirname(LIB), "-lchp_b200",
                        "-Wl,-rpath," + os.path.dirname(LIB), "-o", BIN], check=True)
    return BIN


def test_dropin_driver_builds(lib):
    """Compiles and links against the drop-in headers (no GPU needed)."""
    assert os.path.exists(build_driver(lib))


@pytest.mark.gpu
def test_dropin_reference_kats(ctx, lib):
    exe = build_driver(lib)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_dropin_reference_kats_fused_groups(ctx, lib):
    """The same, with the drop-in's multi-device reduce on fused shard
    groups (CHP_COMBINE=fused: the shards fold into the first device's L)."""
    exe = build_driver(lib)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600, env={**os.environ, "CHP_COMBINE": "fused"})
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout
