#!/bin/bash
# Bench (no CPU baseline) under several environment settings, R rounds interleaved.
# usage: R=2 tools/env_sweep.sh "HG_X=1 HG_Y=2" "HG_X=0" ...   ("-" = no extra env)
R=${R:-2}
mkdir -p gpurun_out
for i in $(seq 1 $R); do
  for cfg in "$@"; do
    envs=""; [ "$cfg" != "-" ] && envs="$cfg"
    tag=$(echo "$cfg" | tr ' =' '_-')
    env $envs timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/env_$tag.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/env_$tag.json')); r=d['roofline']
print('%-44s step %6.1f us  value %.3f M  agg %5.1f us  frac %.3f  e2e %.3f M' % ('$cfg', d['ms_per_step']*1e3, d['value']/1e6, r['avg_launch_ms']*1e3, r['frac'], d['e2e']['value']/1e6))"
  done
done
