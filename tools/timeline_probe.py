#!/usr/bin/env python3
"""Timeline of the two-stream pipelined C2 step: CUDA events (timing) recorded on
each stream right before and after every sample-half and train-half graph, so the
contended duration of each half, the overlap and the waits are visible.

    python tools/timeline_probe.py            # 200 steps, prints a summary
    python tools/timeline_probe.py 200 seg    # halves split into segments (events between them)
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2311_13225_b200.datagen import make_dataset  # noqa: E402
from paper_2311_13225_b200.orchestrator import TrainConfig, Trainer  # noqa: E402


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seg = len(sys.argv) > 2 and sys.argv[2] == "seg"
    two = len(sys.argv) > 2 and sys.argv[2] == "2ss"  # alternate two sample streams (needs >= 3 sets)
    native = len(sys.argv) > 2 and sys.argv[2] == "native"  # inputs by pinned H2D on a copy stream, as
    # hg_pipeline_run does (gated by the set's previous sample half)
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
    ns = len(e.sets)
    ss, st = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    ss2 = torch.cuda.Stream(device=dev)
    ss_main = ss
    cp = torch.cuda.Stream(device=dev)
    from paper_2311_13225_b200.engine import STAGE_SEEDS
    slot = STAGE_SEEDS + 4 * e.batch_cap
    pinned = torch.zeros((K + 4, slot), dtype=torch.uint8).pin_memory()
    for i in range(K + 4):  # the same inputs the device-resident loop copies, packed per step
        row = pinned[i]
        row[:64].view(torch.int64).copy_(d_bp[i].cpu())
        row[64:72].view(torch.int32).copy_(d_counts.cpu())
        row[STAGE_SEEDS:STAGE_SEEDS + 4096].view(torch.int32).copy_(d_seeds[i].cpu())
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    SPLIT = ("sample_l1", "sample_l0", "sample_agg0", "fwd0_gemm", "fwd_upper", "loss", "bwd", "update")
    parts = [e.capture_segments(split_at=SPLIT, set_index=k) for k in range(ns)] if seg else None
    segev = []  # per step: [(stream, name, event)]

    def run(record):
        marks = {"s0": [], "s1": [], "t0": [], "t1": []}
        trained = [None] * ns
        sampled = [torch.cuda.Event() for _ in range(ns)]
        cur = torch.cuda.current_stream(dev)
        ss.wait_stream(cur)
        ss2.wait_stream(cur)
        st.wait_stream(cur)

        sampled_prev = [None] * ns

        def sample(i):
            k = i % ns
            ss = ss2 if (two and i % 2) else ss_main
            if native:
                if sampled_prev[k] is not None:
                    cp.wait_event(sampled_prev[k])
                with torch.cuda.stream(cp):
                    e.sets[k].stage.copy_(pinned[i], non_blocking=True)
                    cpd = torch.cuda.Event(); cpd.record(cp)
                ss.wait_event(cpd)
            if trained[k] is not None:
                ss.wait_event(trained[k])
            with torch.cuda.stream(ss):
                s = e.sets[k]
                if not native:
                    s.seeds.copy_(d_seeds[i])
                    s.bp.copy_(d_bp[i])
                    s.counts_in.copy_(d_counts)
                if record:
                    a = ev(); a.record(ss); marks["s0"].append(a)
                if seg:
                    for name, g in parts[k][0]:
                        x = ev(); x.record(ss)
                        if record:
                            segev.append(("s", i, name, x))
                        g.replay()
                else:
                    e.g_sample[k].replay()
                if record:
                    b = ev(); b.record(ss); marks["s1"].append(b)
                sampled[k].record(ss)
                sp = torch.cuda.Event(); sp.record(ss); sampled_prev[k] = sp

        def train(i):
            k = i % ns
            st.wait_event(sampled[k])
            with torch.cuda.stream(st):
                if record:
                    a = ev(); a.record(st); marks["t0"].append(a)
                if seg:
                    for name, g in parts[k][1]:
                        x = ev(); x.record(st)
                        if record:
                            segev.append(("t", i, name, x))
                        g.replay()
                else:
                    e.g_train[k].replay()
                if record:
                    b = ev(); b.record(st); marks["t1"].append(b)
                x = torch.cuda.Event(); x.record(st)
                trained[k] = x

        origin = ev()
        origin.record(cur)
        sample(0)
        for i in range(K):
            if i + 1 < K:
                sample(i + 1)
            train(i)
        cur.wait_stream(ss_main)
        cur.wait_stream(ss2)
        cur.wait_stream(st)
        torch.cuda.synchronize()
        return origin, marks

    run(False)
    segev.clear()
    origin, m = run(True)
    t = {k: np.array([origin.elapsed_time(x) * 1000.0 for x in v]) for k, v in m.items()}  # us
    s0, s1, t0, t1 = t["s0"], t["s1"], t["t0"], t["t1"]
    sl = slice(10, K - 10)
    period = np.diff(t1)[sl]
    sdur = (s1 - s0)[sl]
    tdur = (t1 - t0)[sl]
    # train k waits for: its sample half (s1[k]) and the previous train (t1[k-1])
    tw_sample = (t0[1:] - t1[:-1])[sl]          # gap on the train stream between trains
    s_after_t = (s0[2:] - t1[:-2])              # sample k starts after train k-2 (set recycling)
    both = []
    for k in range(10, K - 10):
        ov = max(0.0, min(s1[k + 1], t1[k]) - max(s0[k + 1], t0[k]))
        both.append(ov)
    print(f"steps {K}: period {np.median(period):.1f} us (mean {period.mean():.1f})")
    print(f"sample half (contended): median {np.median(sdur):.1f} us; train half: median {np.median(tdur):.1f} us")
    print(f"train-stream gap between trains: median {np.median(tw_sample):.1f} us (waiting for the sample half)")
    print(f"sample start - end of train k-2: median {np.median(s_after_t[sl]):.1f} us")
    print(f"overlap of sample k+1 with train k: median {np.median(both):.1f} us")
    for k in range(20, 24):
        print(f"  k={k}: sample {s0[k]:.0f}-{s1[k]:.0f}  train {t0[k]:.0f}-{t1[k]:.0f}")
    if seg:  # per segment: median start offset inside its half and median duration
        import collections
        ends = {"s": s1, "t": t1}
        rows = collections.defaultdict(list)
        by = collections.defaultdict(list)
        for half, i, name, x in segev:
            by[(half, i)].append((name, origin.elapsed_time(x) * 1000.0))
        for (half, i), lst in by.items():
            if not 10 <= i < K - 10:
                continue
            for j, (name, t0_) in enumerate(lst):
                t1_ = lst[j + 1][1] if j + 1 < len(lst) else ends[half][i]
                rows[(half, j, name)].append(t1_ - t0_)
        for (half, j, name), v in sorted(rows.items()):
            print(f"  {'sample' if half == 's' else 'train '} seg {j} {name:12s} median {np.median(v):7.1f} us")


if __name__ == "__main__":
    main()
