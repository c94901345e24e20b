#!/bin/bash
# GPU suite + C3 bench line + C3 launch list with 128-byte-line rows for wide features; C2 bench line unchanged
TAG=r02t
mkdir -p gpurun_out; rm -f gpurun_out/parity_metrics.jsonl
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 -p no:cacheprovider > gpurun_out/pytest_t8.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest_t8.log
timeout 600 python bench.py --workload c3 --steps 50 --warmup 5 > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.err; echo "c3 rc=$?"; cut -c1-300 gpurun_out/bench_c3_$TAG.json
timeout 600 python -c "from paper_2311_13225_b200.datagen import make_dataset; make_dataset('c3', cache_dir='/tmp/hg_bench_cache')"
timeout 600 ncu --profile-from-start off --set full --clock-control none -k regex:k_agg_fwd -c 1 \
    -f -o gpurun_out/agg_c3_$TAG python tools/profile_step.py c3 > gpurun_out/agg_c3_$TAG.log 2>&1; echo "ncu c3 agg rc=$?"
