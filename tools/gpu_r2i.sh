#!/bin/bash
# phased bottom aggregation: kernel + C2 parity tests, bench sweep over the phase count
mkdir -p gpurun_out; rm -f gpurun_out/parity_metrics.jsonl
timeout 900 python -m pytest tests/test_gpu_kernels.py -k "phased" tests/test_gpu_configs.py -q -rf --timeout 600 -p no:cacheprovider -k "phased or c2_training" > gpurun_out/pytest_i.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/pytest_i.log
grep c2 gpurun_out/parity_metrics.jsonl
for P in 0 4 8 16; do
  HG_AGG_PHASES=$P timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_ph$P.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_ph$P.json')); r=d['roofline']; print('phases=$P value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), 'e2e ms', round(d['e2e']['ms_per_step_device_events'],4), 'agg ms', round(r['avg_launch_ms'],4), 'frac', round(r['frac'],3))"
done
