#!/bin/bash
# One `ncu --set full` capture per config of the K1 kernels of one chp_reduce call (after the
# same command has exited 0 without ncu), summarised to gpurun_out/ncu_full_c<N>.md.
# Run on the GPU box: tools/gpu.sh bash tools/ncu_full.sh
out=gpurun_out
declare -A K=([2]='k_sampled_fused|k_reduce_sampled' [3]='k_reduce_smem16' [4]='k_reduce_filter' [5]='k_reduce_smem16')
declare -A C=([2]=2 [3]=1 [4]=7 [5]=1)
for c in ${CONFIGS:-2 3 4 5}; do
  timeout 600 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-per-config > $out/nf_pre$c.log 2>&1 || { echo "config $c failed without ncu"; continue; }
  timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:${K[$c]}" -c ${C[$c]} \
    -o $out/full_c$c -f python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-per-config > $out/nf_c$c.log 2>&1 \
    && ncu -i $out/full_c$c.ncu-rep --page raw --csv > $out/full_c$c.csv \
    && python tools/ncu_summary.py $out/full_c$c.csv > $out/ncu_full_c$c.md && cat $out/ncu_full_c$c.md \
    || echo "ncu config $c failed"
done
