#!/bin/bash
# session-3 validation after the aggregation occupancy change: GPU suite, smoke, bench (+CPU baseline),
# C3 line, ncu --set full of the bottom aggregation (traffic per launch)
TAG=${1:-r02s}
mkdir -p gpurun_out; rm -f gpurun_out/parity_metrics.jsonl
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/bench_$TAG.json
timeout 900 python bench.py --workload c3 --steps 50 --warmup 5 > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.err; echo "c3 rc=$?"; cut -c1-300 gpurun_out/bench_c3_$TAG.json
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_agg_fwd -c 1 \
  -o gpurun_out/agg_$TAG -f python tools/profile_step.py > /dev/null 2>&1; echo "ncu agg rc=$?"
