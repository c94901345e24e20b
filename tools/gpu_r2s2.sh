#!/bin/bash
# split-row gather probe on the real C2 bottom fetch list
mkdir -p gpurun_out
python tools/order_probe.py
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/split_probe tools/split_probe.cu
./tools/split_probe tools/fetch_list.i32 > gpurun_out/split_probe.txt 2>&1; cat gpurun_out/split_probe.txt
