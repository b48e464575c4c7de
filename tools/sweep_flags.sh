#!/bin/bash
# Sweep chp_reduce flags for one config through bench.py (device-resident
# value and K1 roofline fraction only).  Usage: tools/sweep_flags.sh <config> <flags>...
c=$1; shift
for f in "$@"; do
  out=$(timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-per-config --no-cpu-baseline --flags $f 2>&1 | tail -1)
  python - "$f" "$out" <<'PY'
import json, sys
f, out = sys.argv[1], sys.argv[2]
try:
    d = json.loads(out)
    print(f"flags {int(f):>9} ({int(f):#x}): {d['value']:7.1f} Gpts/s  K1 {d['roofline']['k1_ms']*1e3:7.1f} us  frac {d['roofline']['frac']:.3f}  {d['k1_variant']}")
except Exception:
    print(f"flags {f}: FAILED {out[-300:]}")
PY
done
