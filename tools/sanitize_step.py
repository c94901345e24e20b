#!/usr/bin/env python3
"""A few training steps for compute-sanitizer (memcheck / racecheck / synccheck):
C2-shaped graph at 5 % scale, SAGE 3L [15,10,5] and GCN 2L [10,25], eager AND
captured-graph replay with PDL on, the two-stream pipeline and the hot-embedding
producer/consumer (layer-based, hot 0.2, n=2), so every kernel of the step —
sampling, dedup/relabel, fused gather, TMA/tcgen05 GEMMs, fused top layer,
fixed-point scatter, store put/lookup/inject, fused SGD — runs under the tool.

    compute-sanitizer --tool memcheck python tools/sanitize_step.py
"""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2311_13225_b200.datagen import limit_train, make_dataset  # noqa: E402
from paper_2311_13225_b200.orchestrator import TrainConfig, Trainer  # noqa: E402


def main():
    ds = limit_train(make_dataset("c2", scale=0.05), 6 * 512)
    for model, fan, hid in (("sage", (15, 10, 5), 64), ("gcn", (10, 25), 64)):
        for use_graph in (False, True):
            cfg = TrainConfig(model=model, layers=len(fan), fanouts=fan, hidden_dim=hid, batch_size=512, lr=0.05,
                              seed=1, strategy="layer-based", hot_ratio=0.2, super_batch_n=2, presample_rounds=1,
                              execution="pipelined", use_graph=use_graph)
            tr = Trainer(ds, cfg)
            plan = tr.build_epoch_plan(0, 0)
            rep = tr.run_epoch(plan)
            torch.cuda.synchronize()
            assert np.all(np.isfinite(rep.losses))
            print(model, "graph" if use_graph else "eager", "batches", len(rep.losses), "reuse", rep.reuse_hits,
                  flush=True)
    print("sanitize step ok")


if __name__ == "__main__":
    main()
