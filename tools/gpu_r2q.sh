#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/parity_metrics.jsonl
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_q.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
