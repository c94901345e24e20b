#!/bin/bash
# GPU suite after routing the hot-embedding producer through the split-row gather; C2 hot-reuse epochs A/B
mkdir -p gpurun_out; rm -f gpurun_out/parity_metrics.jsonl gpurun_out/epochs_t5.jsonl
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 -p no:cacheprovider > gpurun_out/pytest_t5.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest_t5.log
for cfg in "HG_SPLIT_ROWS=0" "HG_SPLIT_ROWS=1"; do
  for spec in "c2:sage:hot=0.2:n=4:epochs=2" "c2:sage:hot=0:epochs=2"; do
    env $cfg timeout 400 python bench.py --epoch-mode "$spec" > gpurun_out/ep.json 2>/dev/null; echo "$cfg $spec rc=$?"
    python -c "import json,sys; d=json.loads(open('gpurun_out/ep.json').read().strip().splitlines()[-1]); d['env']='$cfg'; print(json.dumps(d))" >> gpurun_out/epochs_t5.jsonl
    tail -1 gpurun_out/epochs_t5.jsonl | cut -c1-330
  done
done
