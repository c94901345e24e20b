#!/bin/bash
# session-3 evidence: launch list + ncu --set full of one C2 step (every kernel), current code
TAG=${1:-r02s}
mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py > /dev/null 2>&1; echo "launches rc=$?"
python tools/launch_summary.py gpurun_out/launches_$TAG.csv 2>&1 | head -30
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -o gpurun_out/full_$TAG -f python tools/profile_step.py > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full_$TAG.log
