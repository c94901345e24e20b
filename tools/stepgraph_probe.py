#!/usr/bin/env python3
"""One CUDA graph per pipelined step (sample half of batch k+1 || train half of
batch k as two branches of one graph) vs the two-stream pipeline of two graphs
per step.  Same dependency structure; one graph launch and no cross-stream
events per step."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2311_13225_b200.datagen import make_dataset  # noqa: E402
from paper_2311_13225_b200.orchestrator import TrainConfig, Trainer  # noqa: E402


def main():
    K = 200
    ds = make_dataset("c2", cache_dir=bench.CACHE)
    cfg = TrainConfig(model="sage", layers=3, fanouts=(15, 10, 5), hidden_dim=64, batch_size=1024, lr=0.01,
                      strategy="case1", hot_ratio=0.0, use_graph=True, seed=0, report_transfers=False)
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
        s.seeds.copy_(d_seeds[i], non_blocking=True)
        s.bp.copy_(d_bp[i], non_blocking=True)
        s.counts_in.copy_(d_counts, non_blocking=True)

    # step graphs: G[j] = sample half of set (j+1)%2 || train half of set j%2
    cap = torch.cuda.Stream(device=dev)
    sa, sb = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    G = []
    for j in range(2):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            sa.wait_stream(cap)
            sb.wait_stream(cap)
            e.cur = (j + 1) % 2
            e.enqueue_sample_part(sa)
            e.cur = j % 2
            e.enqueue_train_part(sb)
            e.cur = 0
            cap.wait_stream(sa)
            cap.wait_stream(sb)
        G.append(g)
    torch.cuda.synchronize()
    st = torch.cuda.Stream(device=dev)

    def stepgraphs():
        with torch.cuda.stream(st):
            feed(0, 0)
            e.g_sample[0].replay()
            for i in range(K):
                if i + 1 < K:
                    feed((i + 1) % 2, i + 1)  # set (i+1)%2 is free: train(i-1) finished in the previous graph
                    G[i % 2].replay()
                else:
                    e.g_train[i % 2].replay()
        torch.cuda.current_stream().wait_stream(st)

    pipe = tr.pipeline

    def piped():
        pipe.sample(0, lambda s: feed(s, 0))
        for i in range(K):
            if i + 1 < K:
                pipe.sample(i + 1, lambda s, i=i: feed(s, i + 1))
            pipe.train(i)
        pipe.drain()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / K

    for _ in range(2):
        print(f"two-stream pipeline {timed(piped):.4f} ms/step   one graph per step {timed(stepgraphs):.4f} ms/step")


if __name__ == "__main__":
    main()
