#!/bin/bash
# round-2 pass g: GPU suite + default bench (native driver packs each batch right before its launches)
mkdir -p gpurun_out; rm -f gpurun_out/parity_metrics.jsonl
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider > gpurun_out/pytest_g.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/pytest_g.log
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_g.json')); print('value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), d['e2e'], 'agg ms', round(d['roofline']['avg_launch_ms'],4))"
