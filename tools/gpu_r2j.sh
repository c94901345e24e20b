#!/bin/bash
# native driver test + e2e fixed-overhead check (200 vs 600 steps)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_train.py -q -rf --timeout 600 -p no:cacheprovider -k "native" > gpurun_out/pytest_j.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_j.log
for K in 200 600; do
  timeout 600 python bench.py --steps $K --warmup 10 --no-cpu-baseline > gpurun_out/bench_k$K.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_k$K.json')); print('K=$K value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), d['e2e'])"
done
