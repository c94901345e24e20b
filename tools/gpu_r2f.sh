#!/bin/bash
# round-2 pass f: GPU suite after pruning the measured-negative alternates; e2e vs sample-set count
mkdir -p gpurun_out; rm -f gpurun_out/parity_metrics.jsonl
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider > gpurun_out/pytest_f.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/pytest_f.log
for S in 2 3 4; do
  HG_SETS=$S timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_sets$S.json 2> gpurun_out/bench_sets$S.err; echo "sets=$S rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_sets$S.json')); print('sets=$S value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), 'e2e ms', round(d['e2e']['ms_per_step_device_events'],4), 'agg ms', round(d['roofline']['avg_launch_ms'],4))"
done
