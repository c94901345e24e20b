#!/usr/bin/env python3
"""Where does the pipelined C2 step go?  Times K steps of (a) sample graphs
alone, (b) train graphs alone (on already-sampled sets), (c) the two-stream
pipeline, all with CUDA events on the default stream."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2311_13225_b200.datagen import make_dataset  # noqa: E402
from paper_2311_13225_b200.orchestrator import TrainConfig, Trainer  # noqa: E402


def install_skips(spec):
    """HG_WHATIF_SKIP="name[:k],...": drop the k-th (every, without :k) call of an
    entry point within each captured half — results become garbage, only the
    timing of the remaining work is meaningful.  Float-output kernels only."""
    from paper_2311_13225_b200 import _lib, engine
    rules = [(r.split(":")[0], int(r.split(":")[1]) if ":" in r else None) for r in spec.split(",") if r]
    counts = {}
    real = _lib.call

    def call(name, *args):
        k = counts.get(name, 0)
        counts[name] = k + 1
        for n, idx in rules:
            if n == name and (idx is None or idx == k):
                return 0
        return real(name, *args)

    _lib.call = call
    for half in ("enqueue_sample_part", "enqueue_train_part"):
        f = getattr(engine.TrainEngine, half)

        def wrapped(self, *a, _f=f, **kw):
            counts.clear()
            return _f(self, *a, **kw)

        setattr(engine.TrainEngine, half, wrapped)


def main():
    import os
    if os.environ.get("HG_WHATIF_SKIP"):
        install_skips(os.environ["HG_WHATIF_SKIP"])
    K = 100
    workload = os.environ.get("HG_PROBE_WORKLOAD", "c2")
    wl = bench.WORKLOADS[workload]["config"]
    ds = make_dataset(workload, cache_dir=bench.CACHE)
    cfg = TrainConfig(model=wl["model"], layers=wl["layers"], fanouts=tuple(wl["fanouts"]), hidden_dim=wl["hidden"],
                      batch_size=1024, lr=wl["lr"], strategy="case1", hot_ratio=0.0, use_graph=True, seed=0,
                      report_transfers=False)
    tr = Trainer(ds, cfg)
    e = tr.engine
    batches, rseeds = bench.epoch_batches(ds, K + 4)
    dev = e.device
    d_seeds = torch.as_tensor(np.stack(batches).astype(np.int32), device=dev)
    bp = np.zeros((K + 4, 8), dtype=np.int64)
    for i in range(K + 4):
        bp[i, 0] = np.array([rseeds[i] & 0xFFFFFFFFFFFFFFFF], np.uint64).view(np.int64)[0]
        bp[i, 1], bp[i, 2], bp[i, 3], bp[i, 4] = 1024, i, 0, -1
    d_bp = torch.as_tensor(bp, device=dev)
    d_counts = torch.tensor([1024, 1024], dtype=torch.int32, device=dev)

    def feed(k, i):
        s = e.sets[k]
        s.seeds.copy_(d_seeds[i])
        s.bp.copy_(d_bp[i])
        s.counts_in.copy_(d_counts)

    def timed(fn):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / K

    def sample_only():
        for i in range(K):
            feed(i % 2, i)
            e.g_sample[i % 2].replay()

    for k in range(2):
        feed(k, k)
        e.g_sample[k].replay()

    def train_only():
        for i in range(K):
            e.g_train[i % 2].replay()

    sample_only()
    print(f"sample graphs alone : {timed(sample_only):.4f} ms/step")
    for k in range(2):
        feed(k, k)
        e.g_sample[k].replay()
    train_only()
    print(f"train graphs alone  : {timed(train_only):.4f} ms/step")
    pipe = tr.pipeline

    def piped():
        pipe.sample(0, lambda st: feed(st, 0))
        for i in range(K):
            if i + 1 < K:
                pipe.sample(i + 1, lambda st, i=i: feed(st, i + 1))
            pipe.train(i)
        pipe.drain()

    piped()
    print(f"two-stream pipeline : {timed(piped):.4f} ms/step")
    lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
    print("priority range", lo, hi)
    for name, ps, pt in (("train high", 0, -1), ("sample high", -1, 0), ("train max", 0, -5)):
        pipe.ss = torch.cuda.Stream(device=dev, priority=ps)
        pipe.st = torch.cuda.Stream(device=dev, priority=pt)
        piped()
        print(f"pipeline {name:12s}: {timed(piped):.4f} ms/step (ss {pipe.ss.priority}, st {pipe.st.priority})")


if __name__ == "__main__":
    main()
