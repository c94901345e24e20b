#!/usr/bin/env python3
"""Run exactly one eager (non-graph) training step of a bench workload (c2 default, c3) inside
cudaProfilerStart/Stop, for `ncu --profile-from-start off`:

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/launches.csv python tools/profile_step.py
"""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2311_13225_b200 import runplan  # noqa: E402
from paper_2311_13225_b200.datagen import make_dataset  # noqa: E402
from paper_2311_13225_b200.orchestrator import TrainConfig, Trainer  # noqa: E402


def main():
    workload = sys.argv[1] if len(sys.argv) > 1 else "c2"
    from bench import WORKLOADS
    wl = WORKLOADS[workload]["config"]
    ds = make_dataset(workload, cache_dir="/tmp/hg_bench_cache")
    cfg = TrainConfig(model=wl["model"], layers=wl["layers"], fanouts=tuple(wl["fanouts"]), hidden_dim=wl["hidden"],
                      batch_size=1024, lr=wl["lr"], strategy="case1", hot_ratio=0.0, use_graph=False,
                      report_transfers=False)
    tr = Trainer(ds, cfg)
    order = runplan.shuffle_epoch(ds.train_ids(), 0, 0)
    batches = runplan.split_batches(order, 1024)
    for b in range(3):
        tr.train_step(batches[b], runplan.batch_sample_seed(0, 0, b))()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    tr.train_step(batches[3], runplan.batch_sample_seed(0, 0, 3))()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profiled one step; loss ok", np.isfinite(tr.engine.d_loss.item()))


if __name__ == "__main__":
    main()
