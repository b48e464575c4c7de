"""bench.py's reference arm on the CPU (no GPU needed): it prints the
contract's JSON line with the same `config` object as our arm, and the
process loads only oracle/ libraries -- never the product library (a
reference number measured with libchp_b200.so loaded would not be a clean
baseline)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import io, json, os, runpy, sys, contextlib
sys.argv = ["bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1", "--total-points", "200000",
            "--config", sys.argv[1]]
sys.path.insert(0, os.getcwd())
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    try:
        runpy.run_path("bench.py", run_name="__main__")
    except SystemExit:
        pass
libs = sorted({l.split()[-1] for l in open("/proc/self/maps") if l.rstrip().endswith(".so")
               and (os.getcwd() in l)})
print(json.dumps({"line": buf.getvalue().strip().splitlines()[-1], "libs": libs,
                  "torch": "torch" in sys.modules}))
"""


@pytest.fixture(scope="module")
def ref_built():
    import oracle

    if not oracle.Reference.available():
        if not os.path.isdir(oracle.REF_SRC):
            pytest.skip("oracle/_ref not built and /root/reference absent")
        oracle.build(ref=True)


@pytest.mark.parametrize("config", ["5", "2"])
def test_reference_arm_line_and_libraries(ref_built, config):
    r = subprocess.run([sys.executable, "-c", PROBE, config], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    line = json.loads(out["line"])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["kind"] == "reference"
    sys.path.insert(0, ROOT)
    import bench

    assert line["config"] == bench.config_dict(int(config), 200_000, 1)
    assert not any("libchp_b200" in lib for lib in out["libs"]), out["libs"]
    assert any("libchpref" in lib for lib in out["libs"]), out["libs"]
    assert not out["torch"]
