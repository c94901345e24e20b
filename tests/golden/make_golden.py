#!/usr/bin/env python3
"""Generate golden vectors by running the REAL reference (hetgnn) in-process.

Run in the build container only (the reference tree does not exist on the GPU
box); the .npz/.json outputs are committed next to this script:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Everything here goes through the reference's public API (hetgnn.kernels,
hetgnn.sampler, hetgnn.gnnmath, hetgnn.orchestrator, hetgnn.hotness); the
fixtures pin both the oracle restatement (oracle/oracle.py) and the CUDA path.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(OUT.parents[1]))  # repo root, for the scalable generator

from hetgnn import kernels  # noqa: E402
from hetgnn.gnnmath import (backward_batch, forward_batch, init_params,  # noqa: E402
                            loss_and_grad)
from hetgnn.graph import build_csr  # noqa: E402
from hetgnn.hotness import estimate_hotness, select_hot  # noqa: E402
from hetgnn.orchestrator import TrainConfig, build_epoch_plan, run_training  # noqa: E402
from hetgnn.sampler import Fanouts, sample_khop, sample_one_hop_hot  # noqa: E402
from hetgnn.workloads import powerlaw_fixture, sbm_fixture  # noqa: E402

from paper_2311_13225_b200.datagen import make_dataset  # noqa: E402


def graph_arrays(prefix, graph, data=None):
    d = {f"{prefix}_offsets": graph.offsets, f"{prefix}_targets": graph.targets.astype(np.int32)}
    if data is not None:
        d[f"{prefix}_features"] = data.features
        d[f"{prefix}_labels"] = data.labels.astype(np.int32)
        d[f"{prefix}_train"] = data.train_mask
        d[f"{prefix}_val"] = data.val_mask
        d[f"{prefix}_test"] = data.test_mask
    return d


def stack_arrays(prefix, stack):
    d = {f"{prefix}_L": np.int64(len(stack.blocks))}
    for l, b in enumerate(stack.blocks):
        d[f"{prefix}_b{l}_dst"] = b.dst_vertices
        d[f"{prefix}_b{l}_src"] = b.src_vertices
        d[f"{prefix}_b{l}_es"] = b.edge_src
        d[f"{prefix}_b{l}_ed"] = b.edge_dst
    return d


def main():
    assert kernels.backend_name() in ("numba", "numpy")
    kats = {
        "mix64": {str(x): int(kernels._mix64(np.uint64(x))) for x in
                  (0, 1, 0x9E3779B97F4A7C15, 982451653, 2**63 + 12345, 2**64 - 1)},
        "derive_seed": [[s, list(p), kernels.derive_seed(s, *p)] for s, p in
                        [(0, ()), (42, (0x5A, 0)), (0, (0x22, 0, 0)), (7, (7, 1, 0)),
                         (2**64 - 1, (1, 2, 3)), (123456789, (0x44, 3, 17)),
                         (5, (0x70, 2, 9))]],
    }

    arrays = {}
    # --- fixture graphs (reference generators; small) ---------------------
    star = build_csr(np.zeros(5, np.int64), np.arange(1, 6, dtype=np.int64), 6,
                     symmetrize=True, add_self_loops=True)
    pl_g, pl_d = powerlaw_fixture()
    sbm_g, sbm_d = sbm_fixture()
    arrays.update(graph_arrays("star", star))
    arrays.update(graph_arrays("pl", pl_g, pl_d))
    arrays.update(graph_arrays("sbm", sbm_g, sbm_d))

    # --- sample_layer (R2) ------------------------------------------------
    cases = [
        ("star", star, np.arange(6), 3, 777),
        ("pl", pl_g, np.array([0, 5, 17, 400, 999]), 4, 42),
        ("pl", pl_g, np.arange(0, 1000, 7), 5, 1234),
        ("pl", pl_g, np.arange(1000), 25, 99),
        ("pl", pl_g, np.arange(1000)[::-1].copy(), 1, 2**64 - 5),
        ("pl", pl_g, np.array([0, 0, 1, 1, 0]), 10, 3),
        ("pl", pl_g, np.array([0, 1, 2, 3]), 40, 8),   # fanout > 32 path
        ("sbm", sbm_g, np.arange(1000), 15, 5),
    ]
    meta_sl = []
    for k, (gname, g, dst, f, s) in enumerate(cases):
        dst = np.asarray(dst, np.int64)
        ed, es = kernels.sample_layer(g.offsets, g.targets, dst, f, s)
        arrays[f"sl{k}_dst"], arrays[f"sl{k}_ed"], arrays[f"sl{k}_es"] = dst, ed, es
        meta_sl.append([gname, int(f), int(s)])

    # --- stable_unique (R3) -----------------------------------------------
    rng = np.random.default_rng(0)
    su_cases = [np.array([7, 3, 7, 1, 3, 9]), rng.integers(0, 50, 300),
                rng.integers(0, 10**12, 500), np.array([5]), np.arange(100)[::-1].copy()]
    for k, v in enumerate(su_cases):
        u, inv = kernels.stable_unique(np.asarray(v, np.int64))
        arrays[f"su{k}_in"], arrays[f"su{k}_u"], arrays[f"su{k}_inv"] = v, u, inv

    # --- sample_khop stacks (R4/R5/R7) --------------------------------------
    kh_cases = [
        ("pl", pl_g, np.arange(8), (3, 2), 9),
        ("pl", pl_g, np.random.default_rng(1).permutation(1000)[:64], (5, 5, 5), 123),
        ("sbm", sbm_g, np.random.default_rng(2).permutation(1000)[:128], (10, 25), 77),
        ("pl", pl_g, np.random.default_rng(3).permutation(1000)[:200], (15, 10, 5), 2**40 + 3),
        ("pl", pl_g, np.array([3, 3, 5]), (4, 4), 11),  # duplicate seeds
    ]
    meta_kh = []
    for k, (gname, g, seeds, fan, s) in enumerate(kh_cases):
        st = sample_khop(g, seeds, Fanouts(fan), s)
        arrays[f"kh{k}_seeds"] = np.asarray(seeds, np.int64)
        arrays.update(stack_arrays(f"kh{k}", st))
        meta_kh.append([gname, list(fan), int(s)])
    blk = sample_one_hop_hot(pl_g, np.array([0, 10, 3, 999, 500]), 6, 31337, layer=0)
    arrays.update(stack_arrays("oh0", type("S", (), {"blocks": [blk]})))

    # --- larger graph from the scalable generator (C1-shaped) -------------
    c1 = make_dataset("c1", scale=1.0)
    arrays["c1_fingerprint"] = np.frombuffer(bytes.fromhex(c1.fingerprint()), np.uint8)
    seeds_c1 = np.nonzero(c1.train_mask)[0][:1024]
    from hetgnn.graph import Graph
    c1g = Graph(offsets=c1.offsets.copy(), targets=c1.targets.astype(np.int64))
    st = sample_khop(c1g, seeds_c1, Fanouts((10, 25)), 4242)
    arrays["c1kh_seeds"] = seeds_c1
    arrays.update(stack_arrays("c1kh", st))

    # --- layer math (A/F rows) on sbm1k -------------------------------------
    meta_gm = []
    st = sample_khop(sbm_g, np.arange(0, 1000, 13), Fanouts((5, 4, 3)), 55)
    arrays.update(stack_arrays("gm_stack", st))
    inputs = sbm_d.features[st.blocks[0].src_vertices]
    labels = sbm_d.labels[st.seeds]
    for model in ("gcn", "sage"):
        for inj in (False, True):
            params = init_params(model, [32, 16, 16, 4], 3)
            inject = None
            if inj:
                idx = np.arange(0, st.blocks[0].n_dst, 3)
                vals = np.random.default_rng(4).standard_normal((idx.size, 16))
                inject = (idx, vals)
                arrays[f"gm_{model}_inj_idx"], arrays[f"gm_{model}_inj_val"] = idx, vals
            logits, caches = forward_batch(st, inputs.copy(), params, inject=inject)
            loss, dl = loss_and_grad(logits, labels)
            grads = backward_batch(caches, dl, params)
            tag = f"gm_{model}_{int(inj)}"
            arrays[f"{tag}_logits"] = logits
            arrays[f"{tag}_loss"] = np.float64(loss)
            for l, lg in enumerate(grads):
                for m, g in enumerate(lg):
                    arrays[f"{tag}_g{l}_{m}"] = g
            for l, lw in enumerate(params.weights):
                for m, w in enumerate(lw):
                    arrays[f"gm_{model}_w{l}_{m}"] = w
            meta_gm.append(tag)

    # --- hotness (f1) ------------------------------------------------------
    train_ids = np.nonzero(pl_d.train_mask)[0].astype(np.int64)
    table = estimate_hotness(pl_g, train_ids, Fanouts((5, 5)), 3, 5, batch_size=100)
    arrays["hot_counts"], arrays["hot_rank"] = table.counts, table.rank
    arrays["hot_sel"] = select_hot(table, 0.2)

    # --- end-to-end training (S rows, F5) -----------------------------------
    runs = {
        "sbm_gcn_hot": dict(model="gcn", layers=3, fanouts=(5, 5, 5), batch_size=64,
                            hidden_dim=32, epochs=2, lr=0.005, seed=7, super_batch_n=4,
                            hot_ratio=0.2, presample_rounds=2),
        "sbm_sage_hot": dict(model="sage", layers=3, fanouts=(5, 5, 5), batch_size=64,
                             hidden_dim=32, epochs=2, lr=0.05, seed=1, super_batch_n=4,
                             hot_ratio=0.2, presample_rounds=2),
        "sbm_sage_plain": dict(model="sage", layers=2, fanouts=(10, 25), batch_size=128,
                               hidden_dim=64, epochs=2, lr=0.1, seed=2, super_batch_n=4,
                               hot_ratio=0.0, strategy="case1"),
        "pl_gcn_adam": dict(model="gcn", layers=2, fanouts=(4, 4), batch_size=100,
                            hidden_dim=16, epochs=1, lr=0.01, seed=3, super_batch_n=2,
                            hot_ratio=0.3, presample_rounds=1, optimizer="adam"),
        "sbm_sage_n1": dict(model="sage", layers=3, fanouts=(5, 5, 5), batch_size=64,
                            hidden_dim=32, epochs=1, lr=0.05, seed=4, super_batch_n=1,
                            hot_ratio=0.2, presample_rounds=1),
    }
    meta_runs = {}
    for name, kw in runs.items():
        g, d = (sbm_g, sbm_d) if name.startswith("sbm") else (pl_g, pl_d)
        cfg = TrainConfig(simulate_costs=False, **kw)
        reps = run_training(g, d, cfg)
        out = {"config": kw, "epochs": []}
        for r in reps:
            out["epochs"].append({
                "losses": r.losses,
                "max_weight_deltas": r.max_weight_deltas,
                "reuse_hits": [row["reuse_hits"] for row in r.batch_rows],
                "fallbacks": [row["fallbacks"] for row in r.batch_rows],
                # transfer-accounting columns of the per-batch CSV (reporting.py:23-27)
                "raw_rows": [row["raw_rows"] for row in r.batch_rows],
                "cache_hit_rows": [row["cache_hit_rows"] for row in r.batch_rows],
                "raw_elems": [row["raw_elems"] for row in r.batch_rows],
                "emb_elems": [row["emb_elems"] for row in r.batch_rows],
                "aux_elems": [row["aux_elems"] for row in r.batch_rows],
                "grad_elems": [row["grad_elems"] for row in r.batch_rows],
                "stage_events": [list(e) for e in r.stage_events],
                "max_gap": r.max_gap, "max_gap_batch": r.max_gap_batch,
                "warmup_computed": r.warmup_computed,
                "epsilon_trace": r.epsilon_trace,
                "val_accuracy": r.val_accuracy, "test_accuracy": r.test_accuracy,
            })
        # the epoch-0 plan queues (build_epoch_plan replay)
        hot_list = np.empty(0, np.int64)
        if kw.get("hot_ratio", 0) > 0:
            tids = np.nonzero(d.train_mask)[0].astype(np.int64)
            tab = estimate_hotness(g, tids, Fanouts(kw["fanouts"]), kw["presample_rounds"],
                                   kw["seed"], batch_size=kw["batch_size"])
            hot_list = select_hot(tab, kw["hot_ratio"])
            plan = build_epoch_plan(g, d, cfg, hot_list, 0, 0)
            for gi, q in plan.queues.items():
                arrays[f"run_{name}_q{gi}"] = q
            out["queue_groups"] = sorted(int(k) for k in plan.queues)
        arrays[f"run_{name}_hot"] = hot_list
        meta_runs[name] = out

    meta = {"kats": kats, "sample_layer": meta_sl, "khop": meta_kh, "gnnmath": meta_gm,
            "runs": meta_runs, "backend": kernels.backend_name(),
            "numpy": np.__version__}
    np.savez_compressed(OUT / "golden.npz", **arrays)
    (OUT / "golden.json").write_text(json.dumps(meta, indent=1))
    print("wrote", OUT / "golden.npz", sum(a.nbytes for a in arrays.values()), "bytes raw")


if __name__ == "__main__":
    main()
