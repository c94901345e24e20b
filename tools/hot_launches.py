#!/usr/bin/env python3
"""One epoch of C2 (training mask cut to LIMIT vertices) with the hot-embedding
schedule (hot 0.2, n 4) inside cudaProfilerStart/Stop, for an ncu launch list:
which kernels the producer / store / injection add per batch.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \\
        --log-file gpurun_out/hot_launches.csv python tools/hot_launches.py [limit] [hot]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_13225_b200.datagen import limit_train, make_dataset  # noqa: E402
from paper_2311_13225_b200.orchestrator import TrainConfig, Trainer  # noqa: E402


def main():
    limit = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    hot = float(sys.argv[2]) if len(sys.argv) > 2 else 0.2
    ds = limit_train(make_dataset("c2", cache_dir="/tmp/hg_bench_cache"), limit)
    cfg = TrainConfig(model="sage", layers=3, fanouts=(15, 10, 5), hidden_dim=64, batch_size=1024, lr=0.01,
                      strategy="layer-based" if hot > 0 else "case1", hot_ratio=hot, super_batch_n=4,
                      presample_rounds=2, execution="pipelined", seed=0, epochs=2, use_graph=True,
                      report_transfers=False)
    tr = Trainer(ds, cfg)
    plan = tr.build_epoch_plan(0, 0)
    tr.run_epoch(plan)  # warm (graphs captured, producer buffers sized)
    plan = tr.build_epoch_plan(1, len(plan.batches))
    print("queue sizes", plan.queue_sizes)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    rep = tr.run_epoch(plan)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("batches", len(plan.batches), "reuse hits", rep.reuse_hits)


if __name__ == "__main__":
    main()
