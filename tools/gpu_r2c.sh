#!/bin/bash
# round-2 pass c: whole GPU suite, compute-sanitizer, NCCL path at N=1, bulk-stage sweep at C3
mkdir -p gpurun_out; rm -f gpurun_out/parity_metrics.jsonl
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider > gpurun_out/pytest_c.log 2>&1; echo "tests rc=$?"; tail -6 gpurun_out/pytest_c.log
for T in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_step.py > gpurun_out/sanitize_$T.log 2>&1; echo "sanitizer $T rc=$?"; tail -4 gpurun_out/sanitize_$T.log
done
HG_FORCE_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_dist_n1.json 2> gpurun_out/bench_dist_n1.err; echo "dist n1 rc=$?"; cut -c1-300 gpurun_out/bench_dist_n1.json
HG_FORCE_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --steps 50 --warmup 5 --no-cpu-baseline --scaling strong > gpurun_out/bench_dist_n1_strong.json 2> gpurun_out/bench_dist_n1_strong.err; echo "dist n1 strong rc=$?"; cut -c1-300 gpurun_out/bench_dist_n1_strong.json
for S in 4 16 32; do
  HG_AGG_BULK=1 HG_BULK_STAGES=$S timeout 600 python bench.py --workload c3 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3_bulkS$S.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_c3_bulkS$S.json')); r=d['roofline']; print('S=$S value', round(d['value']), 'agg_ms', round(r['avg_launch_ms'],4), 'frac', round(r['frac'],3))"
done
