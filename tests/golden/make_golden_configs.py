#!/usr/bin/env python3
"""Golden vectors at the BASELINE.json configurations, made by running the REAL
reference (hetgnn, numba backend) in-process on the graphs of our generator.

Run in the build container only (the reference tree does not exist on the GPU
box); ``configs.npz`` / ``configs.json`` are committed next to this script:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_configs.py

Runs (``datagen.make_dataset`` graphs, fingerprints recorded; the training mask
cut with ``datagen.limit_train`` where a full epoch would take the reference
hours):

* ``c1``: C1 as named (SAGE 2L [10,25], 10K V, F=128), 2 whole epochs + evaluate.
* ``c2``: C2 at full scale (2.4M V, 64M entries, SAGE 3L [15,10,5], H=64,
  bs 1024 = the bench config), the first 8 batches: losses, max |dw|, batch-0
  logits, and sha256 of batch 0's reference blocks (incl. the >100K-degree
  hubs, which are put into batch 0's seeds).
* ``c3``: C3 at full scale (233K V, 114M entries, F=602, GCN 2L (10,25),
  H=256, hot 0.2, n=4), 12 batches = 3 super-batches: hot list, queues,
  losses, reuse hits, fallbacks, stage events, max gap, epsilon trace.
* ``learn_sgd`` / ``learn_hot``: the learnable C2-shaped graph (``c2learn``:
  class means + noise, 240K V, 24K test vertices), 3 epochs of 30 batches,
  SGD lr 0.5, without / with hot-embedding reuse: test/val accuracy.
* ``skiphot``: sample_khop_skip_hot flags (sampler.py:150-163).
* ``store``: scripted EmbeddingStore protocol traces (store.py:24-146) incl.
  the contract and staleness exceptions.

The reference's evaluate() (full-graph inference) is run where it is tractable
on CPU (c1, learn_*); c2/c3 use its epoch loop pieces (build_epoch_plan,
_run_epoch) without it.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(OUT.parents[1]))

from hetgnn import orchestrator as RO  # noqa: E402
from hetgnn.gnnmath import forward_batch, init_params  # noqa: E402
from hetgnn.graph import Graph, VertexData  # noqa: E402
from hetgnn.hotness import estimate_hotness, select_hot  # noqa: E402
from hetgnn.sampler import Fanouts, sample_khop, sample_khop_skip_hot  # noqa: E402
from hetgnn.store import EmbeddingStore, StalenessViolation, StoreContractError  # noqa: E402
from hetgnn.workloads import powerlaw_fixture  # noqa: E402

from paper_2311_13225_b200.datagen import limit_train, make_dataset  # noqa: E402

# name -> (dataset, scale, train limit, TrainConfig kwargs, batches to keep, evaluate)
RUNS = {
    "c1": ("c1", None, dict(model="sage", layers=2, fanouts=(10, 25), hidden_dim=64, batch_size=1024,
                            epochs=2, lr=0.1, seed=0, strategy="case1", hot_ratio=0.0), None, True),
    "c2": ("c2", 8 * 1024, dict(model="sage", layers=3, fanouts=(15, 10, 5), hidden_dim=64, batch_size=1024,
                                epochs=1, lr=0.01, seed=0, strategy="case1", hot_ratio=0.0), 8, False),
    "c3": ("c3", 12 * 1024, dict(model="gcn", layers=2, fanouts=(10, 25), hidden_dim=256, batch_size=1024,
                                 epochs=1, lr=0.01, seed=0, strategy="layer-based", hot_ratio=0.2,
                                 super_batch_n=4, presample_rounds=1), 12, False),
    "learn_sgd": ("c2learn", 30 * 1024, dict(model="sage", layers=3, fanouts=(15, 10, 5), hidden_dim=64,
                                             batch_size=1024, epochs=3, lr=0.5, seed=0, strategy="case1",
                                             hot_ratio=0.0), None, True),
    "learn_hot": ("c2learn", 30 * 1024, dict(model="sage", layers=3, fanouts=(15, 10, 5), hidden_dim=64,
                                             batch_size=1024, epochs=3, lr=0.5, seed=0, strategy="layer-based",
                                             hot_ratio=0.2, super_batch_n=2, presample_rounds=2), None, True),
}


def ref_graph(ds):
    return Graph(offsets=np.ascontiguousarray(ds.offsets, np.int64), targets=ds.targets.astype(np.int64))


def ref_data(ds):
    return VertexData(features=ds.features.astype(np.float64), labels=ds.labels.astype(np.int64),
                      train_mask=ds.train_mask.copy(), val_mask=ds.val_mask.copy(), test_mask=ds.test_mask.copy())


def stack_hash(stack) -> str:
    h = hashlib.sha256()
    for b in stack.blocks:
        for a in (b.dst_vertices, b.src_vertices, b.edge_src, b.edge_dst):
            h.update(np.ascontiguousarray(a, np.int64).tobytes())
    return h.hexdigest()


def hub_seeds(ds, k=1024):
    """1024 training vertices that include every train vertex of degree >= 100K
    (and the top-degree ones), so the block hash covers the hub code paths."""
    deg = np.diff(ds.offsets)
    tr = np.nonzero(ds.train_mask)[0]
    top = tr[np.argsort(-deg[tr], kind="stable")[:64]]
    rest = tr[~np.isin(tr, top)]
    pick = np.random.default_rng(5).choice(rest, k - top.size, replace=False)
    return np.concatenate([top, pick]).astype(np.int64)


def run_config(name, arrays, meta):
    dsname, limit, kw, keep, do_eval = RUNS[name]
    t0 = time.time()
    full = make_dataset(dsname)
    ds = limit_train(full, limit) if limit else full
    g, d = ref_graph(ds), ref_data(ds)
    cfg = RO.TrainConfig(simulate_costs=False, **kw)
    out = {"dataset": dsname, "train_limit": limit, "config": {k: (list(v) if isinstance(v, tuple) else v)
                                                               for k, v in kw.items()},
           "fingerprint": full.fingerprint(), "epochs": []}
    if name == "c2":
        # batch-0 style blocks with the hubs, and the first batch's logits at init
        seeds = hub_seeds(ds)
        st = sample_khop(g, seeds, Fanouts(kw["fanouts"]), 0xC2C2)
        arrays["c2_hub_seeds"] = seeds
        out["hub_stack_sha256"] = stack_hash(st)
        out["hub_stack_sizes"] = [[int(b.n_dst), int(b.n_src), int(b.n_edges)] for b in st.blocks]
        out["hub_max_degree"] = int(np.diff(ds.offsets)[seeds].max())
    if do_eval:
        reps = RO.run_training(g, d, cfg)
        state = None
    else:
        dims = cfg.dims(d.feat_dim, d.num_classes)
        params = init_params(cfg.model, dims, cfg.seed)
        hot_list = np.empty(0, np.int64)
        if cfg.strategy == "layer-based" and cfg.hot_ratio > 0:
            tids = np.nonzero(d.train_mask)[0].astype(np.int64)
            tab = estimate_hotness(g, tids, Fanouts(tuple(cfg.fanouts)), cfg.presample_rounds, cfg.seed,
                                   batch_size=cfg.batch_size)
            hot_list = select_hot(tab, cfg.hot_ratio)
        store = EmbeddingStore(n=cfg.super_batch_n, emb_dim=cfg.hidden_dim) \
            if cfg.strategy == "layer-based" else None
        state = RO._RunState(params=params, store=store, hot_list=hot_list)
        plan = RO.build_epoch_plan(g, d, cfg, hot_list, 0, 0)
        assert len(plan.batches) == keep
        if name == "c2":
            b0 = plan.batches[0]
            st = sample_khop(g, b0, Fanouts(kw["fanouts"]), plan.batch_seeds[0])
            logits, _ = forward_batch(st, d.features[st.blocks[0].src_vertices],
                                      init_params(cfg.model, dims, cfg.seed))
            arrays["c2_logits0"] = logits
            out["batch0_stack_sha256"] = stack_hash(st)
        for gi, q in plan.queues.items():
            arrays[f"{name}_q{gi}"] = np.asarray(q, np.int64)
        out["queue_groups"] = sorted(int(k) for k in plan.queues)
        arrays[f"{name}_hot"] = np.asarray(hot_list, np.int64)
        rep = RO._run_epoch(g, d, cfg, state, plan, False)
        reps = [rep]
    for r in reps:
        out["epochs"].append({
            "losses": r.losses, "max_weight_deltas": r.max_weight_deltas,
            "reuse_hits": [row["reuse_hits"] for row in r.batch_rows],
            "fallbacks": [row["fallbacks"] for row in r.batch_rows],
            "stage_events": [list(e) for e in r.stage_events],
            "max_gap": r.max_gap, "max_gap_batch": r.max_gap_batch, "warmup_computed": r.warmup_computed,
            "epsilon_trace": r.epsilon_trace,
            "val_accuracy": r.val_accuracy if do_eval else None,
            "test_accuracy": r.test_accuracy if do_eval else None})
    out["seconds"] = time.time() - t0
    meta[name] = out
    print(name, f"{out['seconds']:.1f}s", out["epochs"][-1]["losses"][-3:],
          out["epochs"][-1]["test_accuracy"], flush=True)


def skiphot(arrays, meta):
    pl_g, _ = powerlaw_fixture()
    rng = np.random.default_rng(0)
    cases = []
    for k in range(4):
        hot = rng.choice(pl_g.num_vertices, size=int(rng.integers(1, 300)), replace=False).astype(np.int64)
        seeds = rng.choice(pl_g.num_vertices, size=16, replace=False).astype(np.int64)
        fan = (6, 4) if k < 3 else (5, 5, 5)
        st = sample_khop_skip_hot(pl_g, seeds, Fanouts(fan), hot, 1000 + k)
        arrays[f"skiphot{k}_hot"], arrays[f"skiphot{k}_seeds"] = hot, seeds
        arrays[f"skiphot{k}_flags"] = st.hot_flags
        arrays[f"skiphot{k}_src"] = st.blocks[0].src_vertices
        cases.append([list(fan), 1000 + k])
    meta["skiphot"] = cases


def store_traces(meta):
    """Random protocol-legal and illegal op sequences against the reference
    store; every op's outcome is recorded (value, None, or exception name)."""
    rng = np.random.default_rng(11)
    traces = []
    for t in range(40):
        n = int(rng.choice([1, 2, 4, 8]))
        s = EmbeddingStore(n=n, emb_dim=3)
        ops = []
        window = (0, n)
        for _ in range(int(rng.integers(20, 60))):
            kind = rng.choice(["put", "put", "get", "get", "get", "advance", "reset", "count"])
            rec = {"op": str(kind)}
            try:
                if kind == "put":
                    v = int(rng.integers(0, 12))
                    tgt = s.current_super_batch + (1 if rng.random() < 0.85 else int(rng.choice([0, 2])))
                    ver = int(window[0] + rng.integers(-2 * n - 2, n))
                    emb = (rng.integers(-1000, 1000, 3) / 8.0).tolist()
                    rec.update(v=v, target=tgt, version=ver, emb=emb)
                    s.put(v, np.array(emb), ver, tgt)
                    rec["out"] = "ok"
                elif kind == "get":
                    v = int(rng.integers(0, 12))
                    rb = int(window[0] + rng.integers(-1 if rng.random() < 0.1 else 0, window[1] + 1))
                    rec.update(v=v, reading_batch=rb)
                    e = s.get(v, rb)
                    rec["out"] = None if e is None else [float(x) for x in e]
                elif kind == "advance":
                    ln = int(rng.integers(1, n + 1)) if rng.random() < 0.9 else n + 1
                    ws = window[0] + window[1]
                    rec.update(window_start=ws, window_len=ln)
                    s.advance_super_batch(ws, ln)
                    window = (ws, ln)
                    rec["out"] = "ok"
                elif kind == "reset":
                    ws = window[0] + window[1] + int(rng.integers(0, 3))
                    rec.update(window_start=ws)
                    s.reset_epoch(ws)
                    window = (ws, n)
                    rec["out"] = "ok"
                else:
                    rec["out"] = [s.staged_count(), s.live_entries(), s.memory_bytes(), s.hits, s.misses, s.puts,
                                  s.max_observed_gap, s.max_gap_batch, s.max_gap_super_batch,
                                  s.current_super_batch]
            except (StoreContractError, StalenessViolation) as exc:
                rec["out"] = type(exc).__name__
                if kind == "advance":  # the reference advanced before validating the length
                    window = (rec["window_start"], rec["window_len"])
            ops.append(rec)
        traces.append({"n": n, "ops": ops})
    meta["store"] = traces


def main():
    only = sys.argv[1:]  # regenerate only these runs, keeping the rest of the committed fixtures
    arrays, meta = {}, {}
    if only:
        old = np.load(OUT / "configs.npz")
        arrays = {k: old[k] for k in old.files if not any(k.startswith(n + "_") for n in only)}
        meta = {k: v for k, v in json.loads((OUT / "configs.json").read_text()).items() if k not in only}
    else:
        skiphot(arrays, meta)
        store_traces(meta)
    for name in (only or RUNS):
        run_config(name, arrays, meta)
    np.savez_compressed(OUT / "configs.npz", **arrays)
    (OUT / "configs.json").write_text(json.dumps(meta, indent=1))
    print("wrote", OUT / "configs.npz", sum(a.nbytes for a in arrays.values()), "bytes raw")


if __name__ == "__main__":
    main()
