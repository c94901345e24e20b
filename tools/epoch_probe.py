#!/usr/bin/env python3
"""Where does an epoch of Trainer.run_epoch spend its time?  Runs the C2 graph
(training mask cut to LIMIT vertices) with and without the hot-embedding
schedule, reports wall / GPU time per batch, and a cProfile of the host side of
run_epoch (host-bound if the time is in launches and Python, GPU-bound if it is
in synchronisation / event waits).

    python tools/epoch_probe.py [limit=61440] [hot=0.2] [n=4]
"""
import cProfile
import io
import pstats
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_13225_b200.datagen import limit_train, make_dataset  # noqa: E402
from paper_2311_13225_b200.orchestrator import TrainConfig, Trainer  # noqa: E402


def main():
    opts = dict(a.split("=", 1) for a in sys.argv[1:] if "=" in a)
    limit = int(opts.get("limit", 61440))
    hots = [float(h) for h in opts.get("hot", "0,0.2").split(",")]
    n = int(opts.get("n", 4))
    ds = limit_train(make_dataset("c2", cache_dir="/tmp/hg_bench_cache"), limit)
    for hot in hots:
        cfg = TrainConfig(model="sage", layers=3, fanouts=(15, 10, 5), hidden_dim=64, batch_size=1024, lr=0.01,
                          strategy="layer-based" if hot > 0 else "case1", hot_ratio=hot, super_batch_n=n,
                          presample_rounds=2, execution="pipelined", seed=0, epochs=2, use_graph=True,
                          report_transfers=False)
        tr = Trainer(ds, cfg)
        for epoch in range(2):
            plan = tr.build_epoch_plan(epoch, epoch * 1000)
            torch.cuda.synchronize()
            prof = cProfile.Profile() if epoch == 1 else None
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            w0 = time.perf_counter()
            ev0.record()
            if prof:
                prof.enable()
            rep = tr.run_epoch(plan)
            if prof:
                prof.disable()
            ev1.record()
            torch.cuda.synchronize()
            wall = time.perf_counter() - w0
            nb = len(plan.batches)
            print(f"hot={hot} n={n} epoch {epoch}: {nb} batches, wall {wall * 1e6 / nb:.1f} us/batch, "
                  f"gpu {ev0.elapsed_time(ev1) * 1e3 / nb:.1f} us/batch, {1024 * nb / wall / 1e6:.2f} M seeds/s, "
                  f"reuse hits {rep.reuse_hits}")
            if prof:
                s = io.StringIO()
                pstats.Stats(prof, stream=s).sort_stats("tottime").print_stats(14)
                print("\n".join(s.getvalue().splitlines()[:34]))


if __name__ == "__main__":
    main()
