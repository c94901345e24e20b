#!/bin/bash
# Whole-epoch measurements of the non-headline configs (C2 hot reuse, C3 GCN Reddit-shape, C5 sweep).
TAG=${1:-r01}
mkdir -p gpurun_out
OUT=gpurun_out/epochs_$TAG.jsonl
: > $OUT
run() { timeout 900 python bench.py --epoch-mode "$1" >> $OUT 2>> gpurun_out/epochs_$TAG.err; echo "$1 rc=$?"; }
run "c3:gcn:hot=0.2:n=4:fan=4,4:bs=10000"
run "c3:gcn:hot=0.2:n=4:fan=10,25"
run "c3:gcn:hot=0:fan=10,25"
for n in 1 2 4; do for h in 0.1 0.2 0.3; do run "c2:sage:hot=$h:n=$n"; done; done
run "c2:sage:hot=0"
