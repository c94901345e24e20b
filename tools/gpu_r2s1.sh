#!/bin/bash
# session-3 probes: random-row gather cost vs row size / stride; GEMM stage breakdown at the C2 bottom shape
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_probe tools/gather_probe.cu
for fl in "32 32" "64 64" "100 100" "100 104" "100 128" "128 128" "200 200" "256 256"; do ./tools/gather_probe $fl | sed -n '1p;5p;8p'; done > gpurun_out/gather_rowsize.txt 2>&1
cat gpurun_out/gather_rowsize.txt
python tools/gemm_bench.py > gpurun_out/gemm_bench.txt 2>&1; cat gpurun_out/gemm_bench.txt
python tools/gemm_timeline.py fwd > gpurun_out/gemm_tl_fwd.txt 2>&1; head -30 gpurun_out/gemm_tl_fwd.txt
python tools/gemm_timeline.py wgrad > gpurun_out/gemm_tl_wg.txt 2>&1; head -30 gpurun_out/gemm_tl_wg.txt
