"""Per-phase timeline of the sampled K1.  Needs an instrumentation build:
  CHP_NVCC_EXTRA=-DCHP_PHASE_TIMING=1 python -c "import paper_1505_00914_b200._build as b; b.build(force=True)"
(rebuild without it afterwards).

Runs config 2's chp_reduce + compaction a few times, then prints, per phase boundary, the
median over CTAs of the globaltimer offset from the earliest CTA start (us).
usage: python tools/phase_timing.py [config] [flags]
"""
import ctypes
import statistics
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
from bench import CONFIGS  # noqa: E402
from paper_1505_00914_b200 import _lib  # noqa: E402
from paper_1505_00914_b200.device import Context  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n, p, seed, _ = CONFIGS[cfg]
ctx = Context(0)
xy = ctx.generate(cfg, seed, p, n)
DL = ctx.empty_dl(p)
L = _lib.load()
L.chp_debug_phase.argtypes = [ctypes.c_void_p]
names = ["start", "init", "fold", "dump", "bar1", "merge", "main_start", "main_end"]
for rep in range(6):
    ctx.reduce(xy, p, q=p, out=DL, flags=flags)
    ctx.compact(DL, p, chain=True)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (160 * 8))()
    assert L.chp_debug_phase(ctypes.addressof(buf)) == 0
    rows = [[buf[b * 8 + k] for k in range(8)] for b in range(148)]
    t0 = min(r[0] for r in rows)
    out = []
    for k in range(8):
        v = [(r[k] - t0) / 1000.0 for r in rows]
        out.append("%s %.1f/%.1f/%.1f" % (names[k], min(v), statistics.median(v), max(v)))
    print("rep", rep, " | ".join(out))

# per-CTA main-pass spans of the last rep: slowest / fastest CTAs
spans = sorted(((r[7] - r[6]) / 1000.0, b) for b, r in enumerate(rows))
print("main span min/med/max %.1f/%.1f/%.1f" % (spans[0][0], spans[74][0], spans[-1][0]))
print("slowest", [(b, round(t, 1)) for t, b in spans[-12:]])
print("fastest", [(b, round(t, 1)) for t, b in spans[:12]])
