#!/bin/bash
# Variant sweep: one bench line per (config, flags); prints value / K1 ms / variant.
out=${OUT:-gpurun_out}
for spec in "$@"; do
  c=${spec%%:*}; f=${spec##*:}
  timeout 300 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e --flags $f > $out/sw_${c}_${f}.json 2>$out/sw_${c}_${f}.err
  python - "$out/sw_${c}_${f}.json" "$c" "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print("config %s flags %s: %.1f Gpts/s  k1 %.3f ms  frac %.3f  %s  hull %.3f ms h=%d" % (sys.argv[2], sys.argv[3], d['value'], d['roofline']['k1_ms'], d['roofline']['frac'], d['config']['k1_variant'], d['hull_ms'], d['hull_vertices']))
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
