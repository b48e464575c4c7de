#!/bin/bash
# Round-end evidence refresh, run on the GPU box (tools/gpu.sh tools/refresh_profiles.sh r02).
# Per config: a short bench (must exit 0), then the ncu launch list of one bench step
# (-> profiles/<rnd>_launches_config<N>.json and k1_traffic_config<N>.json, which the bench
# reads into roofline.traffic), then the config's full bench line -> profiles/<rnd>_bench_config<N>.json.
# Then the driver's default command (config 5 + per_config) -> profiles/<rnd>_bench_default.json,
# and the reference arm -> profiles/<rnd>_bench_reference.json.  gpurun returns only
# gpurun_out/, so every file written under profiles/ is also copied to gpurun_out/profiles/
# (copy it back with: cp gpurun_out/profiles/* profiles/).
rnd=${1:-r02}
out=gpurun_out
declare -A N=([2]=100000000 [3]=1000000000 [4]=1000000000 [5]=4000000000)
B="--no-per-config --no-cpu-baseline --no-e2e"
for c in ${CONFIGS:-2 3 4 5}; do
  if timeout 600 python bench.py --config $c --steps 3 --warmup 3 $B > $out/pre_c$c.json 2> $out/pre_c$c.err; then
    timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_requests_srcunit_tex_op_red.sum,lts__t_requests_srcunit_tex_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum --clock-control none \
       -c 400 --csv --log-file $out/launches_c$c.csv \
       python bench.py --config $c --steps 1 --warmup 3 $B > $out/ncu_c$c.log 2>&1 \
       && python tools/launch_summary.py $out/launches_c$c.csv $c ${N[$c]} $rnd > /dev/null \
       || echo "ncu / summary config $c failed"
  else
    echo "short bench config $c failed"; tail -5 $out/pre_c$c.err
  fi
  timeout 900 python bench.py --config $c --no-per-config > $out/bench_c$c.json 2> $out/bench_c$c.err \
    && tail -n 1 $out/bench_c$c.json > profiles/${rnd}_bench_config$c.json \
    || { echo "bench config $c failed"; tail -5 $out/bench_c$c.err; }
done
if [ -z "${NO_DEFAULT:-}" ]; then
  timeout 1200 python bench.py > $out/bench_default.json 2> $out/bench_default.err \
    && tail -n 1 $out/bench_default.json > profiles/${rnd}_bench_default.json || echo "default bench failed"
fi
if [ -z "${NO_REF:-}" ]; then
  timeout 900 python bench.py --impl reference > $out/bench_ref.json 2> $out/bench_ref.err \
    && tail -n 1 $out/bench_ref.json > profiles/${rnd}_bench_reference.json || echo "reference arm failed"
fi
for c in ${CONFIGS:-2 3 4 5}; do python -c "
import json; d=json.load(open('profiles/${rnd}_bench_config$c.json'))
print($c, d['k1_variant'], round(d['value'],1), round(d['roofline']['frac'],3), d['roofline']['traffic'], d['e2e'] and round(d['e2e']['value'],2), d['cpu_baseline'] and d['cpu_baseline']['value'], d['clocks'])"; done
cat profiles/${rnd}_bench_reference.json
mkdir -p $out/profiles
cp profiles/${rnd}_bench_*.json profiles/${rnd}_launches_*.json profiles/k1_traffic_config*.json $out/profiles/ 2>/dev/null
