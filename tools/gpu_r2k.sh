#!/bin/bash
timeout 600 python tools/timeline_probe.py 200 seg > gpurun_out/timeline_seg.txt 2>&1; echo "rc=$?"; grep -v Warn gpurun_out/timeline_seg.txt | grep -v "x\[:"
for A in 2 4; do HG_AGG_CTAS_PER_SM=$A timeout 600 python tools/timeline_probe.py 200 > gpurun_out/timeline_agg$A.txt 2>&1; echo "agg ctas/SM $A"; grep -E "period|half|gap" gpurun_out/timeline_agg$A.txt; done
