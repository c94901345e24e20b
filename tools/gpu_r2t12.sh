#!/bin/bash
# sampler CTAs per SM under the split-row gather
mkdir -p gpurun_out; rm -f gpurun_out/sctas.txt
summ() { python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
print(sys.argv[2], 'value %.3fM e2e %.3fM ms %.4f agg_us %.2f frac %.3f' % (d['value']/1e6, d['e2e']['value']/1e6, d['ms_per_step'], r['avg_launch_ms']*1e3, r['frac']))" $1 "$2"; }
for r in 1 2; do
for cfg in "HG_X=0" "HG_SAMPLE_CTAS_PER_SM=4" "HG_SAMPLE_CTAS_PER_SM=6" "HG_SAMPLE_CTAS_PER_SM=2"; do
  env $cfg timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "$cfg failed"; continue; }
  summ gpurun_out/ab.json "$cfg" | tee -a gpurun_out/sctas.txt
done; done
