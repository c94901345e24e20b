#!/bin/bash
# launch lists (C2, C3) and ncu --set full of every kernel of one C2 step, current code
mkdir -p gpurun_out
for W in c2 c3; do
  timeout 600 python -c "from paper_2311_13225_b200.datagen import make_dataset; make_dataset('$W', cache_dir='/tmp/hg_bench_cache')"
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$W.csv python tools/profile_step.py $W > /dev/null 2>&1; echo "launches $W rc=$?"
done
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -o gpurun_out/full_c2 -f python tools/profile_step.py c2 > gpurun_out/full_c2.log 2>&1; rc=$?; echo "ncu full rc=$rc"
if [ $rc -ne 0 ]; then  # --import-source has crashed C2 captures on some boxes
  timeout 1500 ncu --profile-from-start off --set full --clock-control none \
    -o gpurun_out/full_c2 -f python tools/profile_step.py c2 > gpurun_out/full_c2.log 2>&1; echo "ncu full (no source) rc=$?"
fi
