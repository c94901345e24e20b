#!/bin/bash
# ncu of the bottom aggregation for the C2 and C3 bench workloads (traffic per launch for bench.py's
# roofline.traffic) + the C3 step's launch list
mkdir -p gpurun_out
for W in c2 c3; do
  # build the dataset cache outside ncu first (the generator segfaulted under the profiler)
  timeout 600 python -c "from paper_2311_13225_b200.datagen import make_dataset; make_dataset('$W', cache_dir='/tmp/hg_bench_cache')"
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_agg_fwd -c 1 \
      -f -o gpurun_out/agg_$W python tools/profile_step.py $W > gpurun_out/agg_$W.log 2>&1; echo "$W agg rc=$?"
done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c3.csv python tools/profile_step.py c3 > gpurun_out/launches_c3.log 2>&1; echo "c3 launches rc=$?"
