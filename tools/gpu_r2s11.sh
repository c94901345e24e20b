#!/bin/bash
# whole GPU suite + compute-sanitizer memcheck/racecheck/synccheck over the small C2-shaped + GCN run
# (after the row prefetch, the grid clamp and the reduction width change)
mkdir -p gpurun_out; rm -f gpurun_out/parity_metrics.jsonl
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider > gpurun_out/pytest_final.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest_final.log
for T in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_step.py > gpurun_out/sanitize_$T.log 2>&1; echo "sanitizer $T rc=$?"; tail -2 gpurun_out/sanitize_$T.log
done
