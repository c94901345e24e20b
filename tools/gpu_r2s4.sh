#!/bin/bash
# GEMM epilogue change: microbench, GPU tests, bench
mkdir -p gpurun_out
python tools/gemm_bench.py 2>&1 | head -5
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_s4.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_s4.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_s4.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_s4.json')); r=d['roofline']
print('step', round(d['ms_per_step']*1e3,1), 'us  value', round(d['value']/1e6,3), 'agg', round(r['avg_launch_ms']*1e3,1), 'us  frac', round(r['frac'],3), ' e2e', round(d['e2e']['value']/1e6,3))"
