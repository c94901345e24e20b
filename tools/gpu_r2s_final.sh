#!/bin/bash
# round-2 final evidence (current code): GPU suite, smoke, default bench (+CPU baseline), reference arm,
# C3 line, launch list + ncu --set full of every kernel of one C2 step, C3 hot-reuse epochs
TAG=${1:-r02f}
mkdir -p gpurun_out; rm -f gpurun_out/parity_metrics.jsonl
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider --durations=10 > gpurun_out/pytest_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/bench_$TAG.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"; cut -c1-300 gpurun_out/bench_ref_$TAG.json
timeout 900 python bench.py --workload c3 --steps 50 --warmup 5 > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.err; echo "c3 rc=$?"; cut -c1-300 gpurun_out/bench_c3_$TAG.json
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py > /dev/null 2>&1; echo "launches rc=$?"
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -o gpurun_out/full_$TAG -f python tools/profile_step.py > /dev/null 2>&1; echo "ncu full rc=$?"
for spec in "c3:gcn:hot=0.2:n=4:fan=10,25:epochs=2" "c3:gcn:hot=0:fan=10,25:epochs=2" "c3:gcn:hot=0.2:n=4:fan=4,4:bs=10000:epochs=2" "c2:sage:hot=0.2:n=4:epochs=2" "c2:sage:hot=0:epochs=2"; do
  timeout 900 python bench.py --epoch-mode "$spec" >> gpurun_out/epochs_$TAG.jsonl 2>/dev/null; echo "epoch $spec rc=$?"
done
