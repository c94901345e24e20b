#!/bin/bash
# tests + bench + hot-config epochs + launch list (usage: tools/gpu_b.sh TAG [epoch specs...])
TAG=${1:-x}; shift
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_$TAG.log
timeout 900 python bench.py --phases --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
: > gpurun_out/epochs_$TAG.jsonl
for spec in "$@"; do timeout 900 python bench.py --epoch-mode "$spec" >> gpurun_out/epochs_$TAG.jsonl 2>> gpurun_out/epochs_$TAG.err; echo "$spec rc=$?"; done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py > gpurun_out/launches_$TAG.log 2>&1; echo "ncu launches rc=$?"
