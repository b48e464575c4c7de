"""Diagnostic: does one config's K1 time depend on what the same process /
context ran before it?  (bench.py's per_config runs configs back to back.)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = ["bench.py", "--steps", "20", "--warmup", "5"] + sys.argv[1:]
import torch  # noqa: E402

import bench  # noqa: E402

args = bench.parse()
arm = bench.Arm(args)
_gen, _edl = arm.ctx.generate, arm.ctx.empty_dl


def gen(*a, **k):
    t = _gen(*a, **k)
    print("  xy at %#x" % t.data_ptr(), end="", flush=True)
    return t


def edl(*a, **k):
    t = _edl(*a, **k)
    print("  dl at %#x" % t.data_ptr(), flush=True)
    return t


arm.ctx.generate, arm.ctx.empty_dl = gen, edl


def run(c, flags=0):
    arm.args.flags = flags
    r = arm.measure(c, bench.CONFIGS[c][0], e2e=False)
    return (c, flags, round(r["value"], 1), round(r["roofline"]["k1_ms"] * 1e3, 1), r["k1_variant"])


steps = [a for a in os.environ.get("SEQ", "4").split(",")]
pad = None
for s in steps:
    if s.startswith("pad"):
        pad = torch.empty(int(s[3:]) << 20, dtype=torch.uint8, device="cuda")
        print("pad", s[3:], "MB", flush=True)
    elif s == "free":
        pad = None
        torch.cuda.empty_cache()
    else:
        c, _, f = s.partition(":")
        print(run(int(c), int(f or 0)), flush=True)
