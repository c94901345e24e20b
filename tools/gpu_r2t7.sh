#!/bin/bash
# C3 (602-float rows): row stride 604 (16-byte) vs 608 floats (whole 128-byte lines: 19 per row instead of 19.75 on average)
mkdir -p gpurun_out; rm -f gpurun_out/c3_align.txt
summ() { python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
print(sys.argv[2], 'value %.3fM e2e %.3fM ms %.4f agg_us %.2f frac %.3f loss %.5f' % (d['value']/1e6, d['e2e']['value']/1e6, d['ms_per_step'], r['avg_launch_ms']*1e3, r['frac'], d['final_loss']))" $1 "$2"; }
for cfg in "HG_FEAT_ALIGN=4" "HG_FEAT_ALIGN=32" "HG_FEAT_ALIGN=4" "HG_FEAT_ALIGN=32"; do
  env $cfg timeout 400 python bench.py --workload c3 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "$cfg failed"; tail -3 gpurun_out/ab.err; continue; }
  summ gpurun_out/ab.json "$cfg" | tee -a gpurun_out/c3_align.txt
done
