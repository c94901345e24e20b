#!/bin/bash
# NCCL data-parallel path at N=1 (torchrun, one rank; the all-reduce is captured in the step graph)
mkdir -p gpurun_out
HG_FORCE_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_dist.json 2> gpurun_out/bench_dist.err
echo "dist rc=$?"; cat gpurun_out/bench_dist.json; grep -v Warning gpurun_out/bench_dist.err | tail -5
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29518 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/bench_ref_tr.json 2> gpurun_out/bench_ref_tr.err
echo "ref rc=$?"; cat gpurun_out/bench_ref_tr.json
