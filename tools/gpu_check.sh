#!/bin/bash
# Quick GPU check: full gpu test suite, pipeline probe, bench headline + phases, launch list.
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_h.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_h.log
timeout 600 python tools/overlap_probe.py 2>/dev/null | head -3
timeout 600 python bench.py --no-cpu-baseline --phases > gpurun_out/b_h.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b_h.json')); print(round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']), {k: round(v*1000,1) for k,v in d['phases_ms'].items()})"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_h.csv python tools/profile_step.py > /dev/null 2>&1
