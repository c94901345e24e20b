#!/bin/bash
# C5: staleness bound / hot-ratio sweep on the learnable products-shaped graph (c2learn: 240K vertices,
# class means + noise), 3 epochs x 30 batches, SGD lr 0.5 (the learnable goldens' config), GPU epochs
# with the reference path (oracle port, fp64) run beside each point on the host cores: throughput,
# max staleness gap, reuse hits, test accuracy of both.
TAG=${1:-r02}
mkdir -p gpurun_out
OUT=gpurun_out/c5_$TAG.jsonl
: > $OUT
run() { timeout 1200 python bench.py --epoch-mode "$1" >> $OUT 2>> gpurun_out/c5_$TAG.err; echo "$1 rc=$?"; }
B="c2learn:sage:lr=0.5:epochs=3:limit=30720:cpu=1"
run "$B:hot=0"
for n in 1 2 4; do for h in 0.1 0.2 0.3; do run "$B:hot=$h:n=$n"; done; done
python - <<'PY'
import json
for l in open("gpurun_out/c5_${TAG}.jsonl".replace("${TAG}", __import__("os").environ.get("TAG","r02"))):
    d = json.loads(l); c = d["config"]; cpu = d["cpu_reference"] or {}
    e = d["epochs"]
    print(f"hot {c['hot_ratio']:.1f} n {c['super_batch_n']}: gpu {max(x['seeds_per_s'] for x in e)/1e6:.2f} M seeds/s, "
          f"max gap {max(x['max_gap'] for x in e)}, reuse {sum(x['reuse_hits'] for x in e)}, "
          f"test acc gpu {d['test_accuracy']:.4f} cpu {cpu.get('test_accuracy', float('nan')):.4f}, "
          f"cpu {cpu.get('seeds_per_s_incl_presampling', 0):.0f} seeds/s")
PY
