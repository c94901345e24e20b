#!/bin/bash
# split-row bottom gather: parity tests, A/B bench (split off / on, L2 window sizes), ncu of the split agg kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_split_rows.py tests/test_gpu_configs.py tests/test_gpu_train.py -q -x -p no:cacheprovider > gpurun_out/pytest_split.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_split.txt
summ() { python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
print(sys.argv[2], 'value %.3fM e2e %.3fM ms %.4f agg_us %.2f frac %.3f' % (d['value']/1e6, d['e2e']['value']/1e6, d['ms_per_step'], r['avg_launch_ms']*1e3, r['frac']))" $1 "$2"; }
for cfg in "HG_SPLIT_ROWS=0" "HG_SPLIT_ROWS=1" "HG_SPLIT_ROWS=1 HG_L2_PERSIST_MB=64" "HG_SPLIT_ROWS=1 HG_L2_PERSIST_MB=80" "HG_SPLIT_ROWS=1 HG_L2_PERSIST_MB=40" "HG_SPLIT_ROWS=0" "HG_SPLIT_ROWS=1"; do
  env $cfg timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "$cfg failed"; tail -3 gpurun_out/ab.err; continue; }
  summ gpurun_out/ab.json "$cfg" | tee -a gpurun_out/split_ab.txt
done
timeout 600 python -c "from paper_2311_13225_b200.datagen import make_dataset; make_dataset('c2', cache_dir='/tmp/hg_bench_cache')"
timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:k_agg_fwd -c 1 \
    -f -o gpurun_out/agg_split_c2 python tools/profile_step.py c2 > gpurun_out/agg_split_c2.log 2>&1; echo "ncu split rc=$?"
