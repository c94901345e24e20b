#!/bin/bash
# A/B of two prebuilt libraries (paper_2311_13225_b200/libhg_gnn_{A,B}.so), alternating, same box
# usage: VARS="A B C" tools/ab_bench.sh [rounds] [extra bench args...]
R=${1:-3}; shift
mkdir -p gpurun_out
L=paper_2311_13225_b200/libhg_gnn.so
for i in $(seq 1 $R); do
  for V in ${VARS:-A B}; do
    cp paper_2311_13225_b200/libhg_gnn_$V.so $L
    timeout 600 python bench.py --no-cpu-baseline "$@" > gpurun_out/ab_$V$i.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab_$V$i.json')); r=d['roofline']
print('$V$i step', round(d['ms_per_step']*1e3,1), 'us  value', round(d['value']/1e6,3), ' agg', round(r['avg_launch_ms']*1e3,1), ' e2e', round(d['e2e']['value']/1e6,3))"
  done
done
# (the last variant stays loaded)
