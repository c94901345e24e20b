#!/bin/bash
# One GPU-box pass: gpu tests, smoke, default bench, launch list, ncu full of the top kernels.
# usage: tools/gpu_round.sh [tag]
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py --phases > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; cat gpurun_out/bench_$TAG.json
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py > gpurun_out/launches_$TAG.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:'k_agg_fwd|k_gemm_tc|k_wgrad_tc|k_sample_seg|k_agg_bwd' -c 8 \
  -o gpurun_out/full_$TAG -f python tools/profile_step.py > gpurun_out/full_$TAG.log 2>&1; echo "ncu full rc=$?"
