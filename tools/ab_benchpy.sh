#!/bin/bash
# A/B of two bench.py versions x HG_AGG_CTAS_PER_SM, interleaved; make the old one with
#   git show <rev>:bench.py > tools/bench_prev_tmp.py  (and ROOT = parents[1] in it)
R=${R:-2}
for i in $(seq 1 $R); do
  for c in ${CTAS:-5 4 3}; do
    for b in tools/bench_prev_tmp.py bench.py; do
      HG_AGG_CTAS_PER_SM=$c timeout 600 python $b --no-cpu-baseline > gpurun_out/abpy.json 2>/dev/null
      python -c "
import json; d=json.load(open('gpurun_out/abpy.json')); r=d['roofline']
print('%-28s ctas %s  step %6.1f us  value %.3f M  agg %5.1f us  e2e %.3f M' % ('$b', '$c', d['ms_per_step']*1e3, d['value']/1e6, r['avg_launch_ms']*1e3, d['e2e']['value']/1e6))"
    done
  done
done
