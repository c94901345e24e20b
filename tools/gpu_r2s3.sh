#!/bin/bash
# L2 persisting-window size vs the bottom aggregation and the whole step (C2 bench)
mkdir -p gpurun_out
for MB in 0 16 32 48 64 80; do
  HG_L2_PERSIST_MB=$MB timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_l2_$MB.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_l2_$MB.json')); r=d['roofline']
print('window $MB MB: step', round(d['ms_per_step']*1e3,1), 'us  agg', round(r['avg_launch_ms']*1e3,1), 'us  frac', round(r['frac'],3), ' e2e', round(d['e2e']['value']/1e6,3))"
done
