#!/bin/bash
# spatial partitioning experiment: bottom aggregation on G SMs (1024-thread CTAs), tensor-core kernels on TC CTAs
run() {
  env $1 timeout 300 python tools/timeline_probe.py 200 > gpurun_out/tl.txt 2>&1
  echo "[$1] $(grep -E 'period' gpurun_out/tl.txt) | $(grep -E 'sample half' gpurun_out/tl.txt)"
}
run "HG_X=0"
run "HG_AGG_THREADS=1024"
run "HG_AGG_THREADS=1024 HG_AGG_GRID=148 HG_TC_CTAS=148"
run "HG_AGG_THREADS=1024 HG_AGG_GRID=128 HG_TC_CTAS=148"
run "HG_AGG_THREADS=1024 HG_AGG_GRID=120 HG_TC_CTAS=28"
run "HG_AGG_THREADS=1024 HG_AGG_GRID=100 HG_TC_CTAS=48"
run "HG_AGG_THREADS=1024 HG_AGG_GRID=74 HG_TC_CTAS=74"
run "HG_AGG_THREADS=1024 HG_AGG_GRID=100 HG_TC_CTAS=148"
run "HG_TC_CTAS=100"
run "HG_TC_CTAS=74"
