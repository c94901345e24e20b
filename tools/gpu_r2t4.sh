#!/bin/bash
# source-range bucketed bottom gather: tests, then A/B over HG_AGG_RANGES
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_split_rows.py -q -x -p no:cacheprovider > gpurun_out/pytest_rng.txt 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_rng.txt
summ() { python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
print(sys.argv[2], 'value %.3fM e2e %.3fM ms %.4f agg_us %.2f frac %.3f loss %.5f' % (d['value']/1e6, d['e2e']['value']/1e6, d['ms_per_step'], r['avg_launch_ms']*1e3, r['frac'], d['final_loss']))" $1 "$2"; }
for cfg in "HG_AGG_RANGES=1" "HG_AGG_RANGES=2" "HG_AGG_RANGES=4" "HG_AGG_RANGES=8" "HG_AGG_RANGES=16" "HG_AGG_RANGES=1" "HG_AGG_RANGES=4" "HG_AGG_RANGES=8"; do
  env $cfg timeout 240 python bench.py --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "$cfg failed"; tail -3 gpurun_out/ab.err; continue; }
  summ gpurun_out/ab.json "$cfg" | tee -a gpurun_out/rng_ab.txt
done
