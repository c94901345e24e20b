#!/bin/bash
# kernel-node stage copy (bench x2) + C3 wide-row NV A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_train.py -q -rf --timeout 600 -p no:cacheprovider > gpurun_out/pytest_o.log 2>&1; echo "train tests rc=$?"; tail -2 gpurun_out/pytest_o.log
for r in 1 2; do
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_o$r.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_o$r.json')); print('value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), 'e2e ms', round(d['e2e']['ms_per_step_device_events'],4), 'agg ms', round(d['roofline']['avg_launch_ms'],4))"
done
for T in 0 1; do
HG_AGG_TIGHT_NV=$T timeout 600 python bench.py --workload c3 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3_nv$T.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_c3_nv$T.json')); r=d['roofline']; print('c3 tight=$T value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'agg ms', round(r['avg_launch_ms'],4), 'frac', round(r['frac'],3))"
done
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_configs.py -q -rf --timeout 600 -p no:cacheprovider -k "wide or c3" > gpurun_out/pytest_o2.log 2>&1; echo "wide/c3 tests rc=$?"; tail -2 gpurun_out/pytest_o2.log
