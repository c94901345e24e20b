#!/bin/bash
# Round-end evidence: default bench (with CPU baseline), reference arm, smoke, launch list, ncu full, epoch sweep.
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; cat gpurun_out/bench_$TAG.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"; cat gpurun_out/bench_ref_$TAG.json
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:'k_agg_fwd|k_gemm_tma|k_wgrad_tma|k_sample_seg|k_markscan|k_bwd_scatter|k_bwd_finish' -c 12 \
  -o gpurun_out/full_$TAG -f python tools/profile_step.py > /dev/null 2>&1; echo "ncu full rc=$?"
bash tools/configs_sweep.sh $TAG
