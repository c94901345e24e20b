#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_train.py -q -rf --timeout 600 -p no:cacheprovider > gpurun_out/pytest_p.log 2>&1; echo "train tests rc=$?"; tail -2 gpurun_out/pytest_p.log
for r in 1 2; do
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_p$r.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_p$r.json')); print('value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), 'e2e ms', round(d['e2e']['ms_per_step_device_events'],4), 'agg ms', round(d['roofline']['avg_launch_ms'],4))"
done
