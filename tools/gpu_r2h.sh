#!/bin/bash
# e2e experiment: H2D on a copy stream (0), on the sample stream (1), none (2); plus the gather-order probe
for M in 0 1 2; do
  HG_PIPE_COPY=$M timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_copy$M.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_copy$M.json')); print('copy=$M value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), 'e2e ms', round(d['e2e']['ms_per_step_device_events'],4), 'enq', round(d['e2e']['ms_per_step_host_enqueue'],4))"
done
./tools/order_probe tools/fetch_list.i32 > gpurun_out/order_probe.txt 2>&1; cat gpurun_out/order_probe.txt
