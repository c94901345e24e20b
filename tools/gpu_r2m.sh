#!/bin/bash
run() {
  env $1 timeout 300 python tools/timeline_probe.py 200 $2 > gpurun_out/tl.txt 2>&1
  echo "[$1 $2] $(grep -E 'period' gpurun_out/tl.txt) | $(grep -E 'sample half' gpurun_out/tl.txt)"; grep -E "^  k=2[01]" gpurun_out/tl.txt
}
run "HG_SETS=2"
run "HG_SETS=3" 2ss
run "HG_SETS=4" 2ss
