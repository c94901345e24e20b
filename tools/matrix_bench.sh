#!/bin/bash
# Bench (no CPU baseline) over (library variant, environment) pairs, R rounds interleaved.
# usage: R=2 tools/matrix_bench.sh "base HG_X=1" "U8 HG_X=1 HG_Y=2" ...
#   variant = paper_2311_13225_b200/libhg_gnn_<variant>.so, the rest = env assignments
R=${R:-2}
mkdir -p gpurun_out
L=paper_2311_13225_b200/libhg_gnn.so
CFGS=("$@")
for i in $(seq 1 $R); do
  for cfg in "${CFGS[@]}"; do
    v=${cfg%% *}; envs=""; [ "$cfg" != "$v" ] && envs=${cfg#* }
    cp paper_2311_13225_b200/libhg_gnn_$v.so $L
    tag=$(echo "$cfg" | tr ' =' '_-')
    env $envs timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/mx_$tag.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/mx_$tag.json')); r=d['roofline']
print('%-52s step %6.1f us  value %.3f M  agg %5.1f us  frac %.3f  e2e %.3f M' % ('$cfg', d['ms_per_step']*1e3, d['value']/1e6, r['avg_launch_ms']*1e3, r['frac'], d['e2e']['value']/1e6))"
  done
done
