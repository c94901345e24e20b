#!/bin/bash
# round-2 pass b: fixed tests, wide-row bulk gather, C3 bench lines (bulk on/off), ncu of the C3 bottom aggregation
mkdir -p gpurun_out; rm -f gpurun_out/parity_metrics.jsonl
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_store.py tests/test_gpu_dist.py tests/test_gpu_kernels.py -q -rf --timeout 900 -p no:cacheprovider > gpurun_out/pytest_b.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/pytest_b.log
for B in 1 0; do
  HG_AGG_BULK=$B timeout 900 python bench.py --workload c3 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3_bulk$B.json 2> gpurun_out/bench_c3_bulk$B.err; echo "c3 bulk=$B rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_c3_bulk$B.json')); r=d['roofline']; print('value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'agg_ms', round(r['avg_launch_ms'],4), 'frac', round(r['frac'],3), 'alg MB', round(r['alg_bytes_per_launch']/1e6,1), r['block0'])"
done
for B in 1 0; do
  HG_AGG_BULK=$B timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_agg_fwd python tools/profile_step.py c3 > gpurun_out/ncu_c3_agg_bulk$B.txt 2>&1; echo "ncu bulk=$B rc=$?"; grep -E "k_agg_fwd|duration|bytes|hit_rate|throughput" gpurun_out/ncu_c3_agg_bulk$B.txt | head -12
done
