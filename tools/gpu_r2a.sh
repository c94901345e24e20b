#!/bin/bash
# round-2 first GPU pass: new parity tests, then the whole GPU suite, then a short bench
mkdir -p gpurun_out; rm -f gpurun_out/parity_metrics.jsonl
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_store.py tests/test_gpu_dist.py -q -rf --timeout 900 -p no:cacheprovider > gpurun_out/pytest_new.log 2>&1; echo "new rc=$?"; tail -25 gpurun_out/pytest_new.log
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider --deselect tests/test_gpu_configs.py --deselect tests/test_gpu_store.py --deselect tests/test_gpu_dist.py > gpurun_out/pytest_old.log 2>&1; echo "old rc=$?"; tail -15 gpurun_out/pytest_old.log
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo "bench rc=$?"; cut -c1-600 gpurun_out/bench_r2a.json
