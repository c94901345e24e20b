#!/bin/bash
# final check on HEAD: GPU suite, smoke, default bench (+CPU baseline), reference arm, C3 line, launch list
TAG=r02tf
mkdir -p gpurun_out; rm -f gpurun_out/parity_metrics.jsonl
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/pytest_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; cut -c1-250 gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"; cut -c1-200 gpurun_out/bench_ref_$TAG.json
timeout 600 python bench.py --workload c3 --steps 100 --warmup 5 > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.err; echo "c3 rc=$?"; cut -c1-250 gpurun_out/bench_c3_$TAG.json
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py > /dev/null 2>&1; echo "launches rc=$?"
