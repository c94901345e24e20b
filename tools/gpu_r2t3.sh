#!/bin/bash
# round-2 re-entry final evidence with the split-row gather: knob sweep, GPU suite, smoke, bench (+CPU baseline),
# reference arm, C3 line, launch list, ncu --set full of one C2 step
TAG=${1:-r02t}
mkdir -p gpurun_out; rm -f gpurun_out/parity_metrics.jsonl
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
summ() { python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
print(sys.argv[2], 'value %.3fM e2e %.3fM ms %.4f agg_us %.2f frac %.3f' % (d['value']/1e6, d['e2e']['value']/1e6, d['ms_per_step'], r['avg_launch_ms']*1e3, r['frac']))" $1 "$2"; }
for cfg in "HG_SPLIT_ROWS=1" "HG_AGG_CTAS_PER_SM=4" "HG_AGG_CTAS_PER_SM=6" "HG_L2_PERSIST_MB=44" "HG_L2_PERSIST_MB=56" "HG_SPLIT_ROWS=0" "HG_SPLIT_ROWS=1"; do
  env $cfg timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "$cfg failed"; tail -3 gpurun_out/ab.err; continue; }
  summ gpurun_out/ab.json "$cfg" | tee -a gpurun_out/knobs_$TAG.txt
done
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider --durations=10 > gpurun_out/pytest_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/bench_$TAG.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"; cut -c1-300 gpurun_out/bench_ref_$TAG.json
timeout 900 python bench.py --workload c3 --steps 50 --warmup 5 > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.err; echo "c3 rc=$?"; cut -c1-300 gpurun_out/bench_c3_$TAG.json
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py > /dev/null 2>&1; echo "launches rc=$?"
timeout 1200 ncu --profile-from-start off --set full --clock-control none \
  -o gpurun_out/full_$TAG -f python tools/profile_step.py > /dev/null 2>&1; echo "ncu full rc=$?"
