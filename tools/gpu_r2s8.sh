#!/bin/bash
# GPU tests, ncu of the bottom aggregation per bench workload (no --import-source: it crashed the C2
# capture), C2 and C3 bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.txt
for W in c2 c3; do
  timeout 600 python -c "from paper_2311_13225_b200.datagen import make_dataset; make_dataset('$W', cache_dir='/tmp/hg_bench_cache')"
  timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:k_agg_fwd -c 1 \
      -f -o gpurun_out/agg_$W python tools/profile_step.py $W > gpurun_out/agg_$W.log 2>&1; echo "$W agg rc=$?"
done
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 bench rc=$?"
timeout 900 python bench.py --workload c3 --steps 100 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 bench rc=$?"
