#!/usr/bin/env python3
"""Three-stage pipeline probe (HG_SETS=3): sampling of batch k+2 | bottom
aggregation of batch k+1 | training of batch k on three streams, vs the
two-stage pipeline (sample half incl. aggregation | train half)."""
import os
import sys
from pathlib import Path

os.environ.setdefault("HG_SETS", "3")
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2311_13225_b200.datagen import make_dataset  # noqa: E402
from paper_2311_13225_b200.orchestrator import TrainConfig, Trainer  # noqa: E402


def main():
    K = 100
    ds = make_dataset("c2", cache_dir=bench.CACHE)
    cfg = TrainConfig(model="sage", layers=3, fanouts=(15, 10, 5), hidden_dim=64, batch_size=1024, lr=0.01,
                      strategy="case1", hot_ratio=0.0, use_graph=True, seed=0, report_transfers=False)
    tr = Trainer(ds, cfg)
    e = tr.engine
    nset = len(e.sets)
    batches, rseeds = bench.epoch_batches(ds, K + 4)
    dev = e.device
    d_seeds = torch.as_tensor(np.stack(batches).astype(np.int32), device=dev)
    bp = np.zeros((K + 4, 8), dtype=np.int64)
    for i in range(K + 4):
        bp[i, 0] = np.array([rseeds[i] & 0xFFFFFFFFFFFFFFFF], np.uint64).view(np.int64)[0]
        bp[i, 1], bp[i, 2], bp[i, 3], bp[i, 4] = 1024, i, 0, -1
    d_bp = torch.as_tensor(bp, device=dev)
    d_counts = torch.tensor([1024, 1024], dtype=torch.int32, device=dev)
    parts = [e.capture_segments(split_at=("sample_agg0",), set_index=k) for k in range(nset)]
    gsamp = [p[0][0][1] for p in parts]
    gagg = [p[0][1][1] for p in parts]
    gtrain = [p[1][0][1] for p in parts]
    s1, s2, st = (torch.cuda.Stream(device=dev) for _ in range(3))
    sampled = [torch.cuda.Event() for _ in range(nset)]
    agged = [torch.cuda.Event() for _ in range(nset)]
    trained = [None] * nset

    def feed(k, i):
        s = e.sets[k]
        s.seeds.copy_(d_seeds[i], non_blocking=True)
        s.bp.copy_(d_bp[i], non_blocking=True)
        s.counts_in.copy_(d_counts, non_blocking=True)

    def samp(i):
        k = i % nset
        if trained[k] is not None:
            s1.wait_event(trained[k])
        with torch.cuda.stream(s1):
            feed(k, i)
            gsamp[k].replay()
            sampled[k].record(s1)

    def agg(i):
        k = i % nset
        s2.wait_event(sampled[k])
        with torch.cuda.stream(s2):
            gagg[k].replay()
            agged[k].record(s2)

    def train(i):
        k = i % nset
        st.wait_event(agged[k])
        with torch.cuda.stream(st):
            gtrain[k].replay()
            ev = torch.cuda.Event()
            ev.record(st)
            trained[k] = ev

    def three_stage():
        cur = torch.cuda.current_stream()
        for s in (s1, s2, st):
            s.wait_stream(cur)
        samp(0)
        samp(1)
        agg(0)
        for i in range(K):
            if i + 2 < K:
                samp(i + 2)
            if i + 1 < K:
                agg(i + 1)
            train(i)
        for s in (s1, s2, st):
            cur.wait_stream(s)

    def two_stage():
        cur = torch.cuda.current_stream()
        for s in (s1, s2, st):
            s.wait_stream(cur)

        def sample2(i):
            samp(i)
            k = i % nset
            s1.wait_event(sampled[k])
            with torch.cuda.stream(s1):
                gagg[k].replay()
                agged[k].record(s1)
        sample2(0)
        for i in range(K):
            if i + 1 < K:
                sample2(i + 1)
            train(i)
        for s in (s1, s2, st):
            cur.wait_stream(s)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / K

    print(f"sets {nset}: two-stage {timed(two_stage):.4f} ms/step, three-stage {timed(three_stage):.4f} ms/step")
    print(f"again:  two-stage {timed(two_stage):.4f} ms/step, three-stage {timed(three_stage):.4f} ms/step")


if __name__ == "__main__":
    main()
