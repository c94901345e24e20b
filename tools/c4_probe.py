#!/usr/bin/env python3
"""C4 shape on ONE B200: GraphSAGE 3-layer [15,10,5], batch 1024, on an
ogbn-papers100M-shaped synthetic graph (111 M vertices, 3.23 B CSR entries =
1.6 B undirected edges, 128-dim fp32 features, 172 classes) held entirely in
this GPU's HBM (~75 GB: 57 GB features + 13 GB targets + tables).

BASELINE.json's C4 is 8 GPUs with NVLink-sharded features; every box this round
has one GPU, so this measures the replicated layout at full size instead.  The
graph is generated ON the device (a Zipf expected-degree sequence, hubs at low
ids, Zipf-weighted random targets — the shape of datagen's Chung-Lu generator
without its host-side sort, which would need ~80 GB of host RAM at this size).
Prints one JSON line: train seeds/s device-resident (two-stream pipeline,
CUDA events) and end to end through Trainer.train_batches.
"""
import json
import sys
import time
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_13225_b200.device import DeviceGraph, FirstOccurrenceTable  # noqa: E402
from paper_2311_13225_b200.orchestrator import TrainConfig, Trainer  # noqa: E402

V, ENTRIES, F, C = 111_059_956, 3_231_371_744, 128, 172
N_TRAIN = 1_207_179  # ogbn-papers100M training vertices


def make_graph(dev, seed=7, exponent=2.5, max_deg=200_000, chunk=1 << 27):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    w = (torch.arange(V, device=dev, dtype=torch.float64) + 1.0) ** (-1.0 / (exponent - 1.0))
    for _ in range(8):  # rescale to the target mass, cap hubs, renormalise the rest
        w *= ENTRIES / w.sum()
        w.clamp_(max=max_deg)
    deg = torch.floor(w)
    deg += (torch.rand(V, generator=g, device=dev, dtype=torch.float64) < (w - deg)).to(torch.float64)
    offsets = torch.zeros(V + 1, dtype=torch.int64, device=dev)
    torch.cumsum(deg.to(torch.int64), 0, out=offsets[1:])
    del deg
    E = int(offsets[-1].item())
    cdf = torch.cumsum(w, 0)
    cdf /= cdf[-1].clone()
    del w
    targets = torch.empty(E, dtype=torch.int32, device=dev)
    for s in range(0, E, chunk):
        n = min(chunk, E - s)
        r = torch.rand(n, generator=g, device=dev, dtype=torch.float64)
        targets[s:s + n] = torch.searchsorted(cdf, r, right=True).clamp_(max=V - 1).to(torch.int32)
        del r
    del cdf
    feats = torch.empty((V, F), dtype=torch.float32, device=dev)
    rows = chunk // F
    for s in range(0, V, rows):
        feats[s:s + rows].normal_(generator=g)
    labels = torch.randint(0, C, (V,), generator=g, device=dev, dtype=torch.int32)
    dg = DeviceGraph.__new__(DeviceGraph)
    dg.device, dg.offsets, dg.targets = dev, offsets, targets
    dg.num_vertices, dg.num_edges = V, E
    dg.feat_dim, dg.feat_ld, dg.features, dg.labels = F, F, feats, labels
    dg.minpos = FirstOccurrenceTable(V, dev)
    return dg


def main():
    K, W = 200, 10
    dev = torch.device("cuda:0")
    t0 = time.perf_counter()
    dg = make_graph(dev)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    rng = np.random.default_rng(0)
    train = np.zeros(V, bool)
    train[rng.choice(V, N_TRAIN, replace=False)] = True
    ds = SimpleNamespace(device_graph=dg, train_mask=train, labels=np.array([0, C - 1]))
    cfg = TrainConfig(model="sage", layers=3, fanouts=(15, 10, 5), hidden_dim=64, batch_size=1024, lr=0.01,
                      strategy="case1", hot_ratio=0.0, use_graph=True, seed=0, report_transfers=False)
    tr = Trainer(ds, cfg)
    e = tr.engine
    ids = np.flatnonzero(train)
    batches = [rng.choice(ids, 1024, replace=False) for _ in range(W + K)]
    rseeds = [int(x) for x in rng.integers(0, 1 << 62, size=W + K)]
    d_seeds = torch.as_tensor(np.stack(batches).astype(np.int32), device=dev)
    bp = np.zeros((W + K, 8), dtype=np.int64)
    for i in range(W + K):
        bp[i, 0], bp[i, 1], bp[i, 2], bp[i, 3], bp[i, 4] = rseeds[i], 1024, i, 0, -1
    d_bp = torch.as_tensor(bp, device=dev)
    d_counts = torch.tensor([1024, 1024], dtype=torch.int32, device=dev)
    pipe = tr.pipeline

    def feed(k, i):
        s = e.sets[k]
        s.seeds.copy_(d_seeds[i], non_blocking=True)
        s.bp.copy_(d_bp[i], non_blocking=True)
        s.counts_in.copy_(d_counts, non_blocking=True)

    def piped(lo, hi):
        pipe.sample(lo, lambda st: feed(st, lo))
        for i in range(lo, hi):
            if i + 1 < hi:
                pipe.sample(i + 1, lambda st, i=i: feed(st, i + 1))
            pipe.train(i)
        pipe.drain()

    piped(0, W)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    piped(W, W + K)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / K
    host = [(bt.astype(np.int64), rs) for bt, rs in zip(batches, rseeds)]
    [h() for h in tr.train_batches(host[:3])]
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    losses = [h() for h in tr.train_batches(host[W:W + K])]
    e2e_ms = (time.perf_counter() - w0) * 1000.0 / K
    if not np.all(np.isfinite(losses)):
        raise SystemExit("non-finite loss")
    print(json.dumps({
        "metric": "train seeds/sec (GraphSAGE papers100M-shape, 1 GPU, replicated)", "value": 1024 / (ms / 1e3),
        "unit": "seeds/s", "ms_per_step": ms, "steps": K, "warmup": W,
        "e2e": {"value": 1024 / (e2e_ms / 1e3), "ms_per_step": e2e_ms},
        "config": {"workload": "c4-papers100m-shape", "vertices": V, "csr_entries": dg.num_edges, "feat_dim": F,
                   "classes": C, "train_vertices": N_TRAIN, "fanouts": [15, 10, 5], "hidden": 64,
                   "batch_size": 1024, "model": "sage", "dtype": "fp32", "gpus": 1,
                   "layout": "graph + features replicated in one GPU's HBM"},
        "hbm_allocated_gb": torch.cuda.max_memory_allocated() / 1e9, "generate_s": gen_s,
        "loss_first_last": [losses[0], losses[-1]]}))


if __name__ == "__main__":
    main()
