#!/bin/bash
# round-2 pass e: compute-sanitizer (memcheck/racecheck/synccheck) over a small C2-shaped + GCN run,
# launch list of one C2 step, ncu --set full of every kernel of one step (no cap), C3 bottom agg ncu
TAG=${1:-r02}
mkdir -p gpurun_out
for T in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_step.py > gpurun_out/sanitize_${T}_$TAG.log 2>&1; echo "sanitizer $T rc=$?"; tail -4 gpurun_out/sanitize_${T}_$TAG.log
done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py > /dev/null 2>&1; echo "launches rc=$?"
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -o gpurun_out/full_$TAG -f python tools/profile_step.py > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full_$TAG.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_agg_fwd \
  -o gpurun_out/c3agg_$TAG -f python tools/profile_step.py c3 > /dev/null 2>&1; echo "ncu c3 rc=$?"
