#!/bin/bash
# ncu captures of the current hot kernels (one eager C2 step) -> gpurun_out/prof_<tag>_*.ncu-rep
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:'k_agg_fwd|k_gemm_tma|k_wgrad_tma|k_sample_seg|k_markscan|k_bwd_scatter|k_bwd_finish|k_relabel' -c 14 \
  -o gpurun_out/prof_$TAG -f python tools/profile_step.py > gpurun_out/prof_$TAG.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py > /dev/null 2>&1; echo "ncu launches rc=$?"
