#!/bin/bash
# train-private stage copy: full GPU suite + bench (e2e) + timeline
mkdir -p gpurun_out; rm -f gpurun_out/parity_metrics.jsonl
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider > gpurun_out/pytest_n.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/pytest_n.log
for r in 1 2; do
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_n$r.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_n$r.json')); print('value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), 'e2e ms', round(d['e2e']['ms_per_step_device_events'],4), 'agg ms', round(d['roofline']['avg_launch_ms'],4))"
done
