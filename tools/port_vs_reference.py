#!/usr/bin/env python3
"""Cross-check of the reference arm (bench.py --impl reference, the oracle port) against
the REAL reference (`hetgnn`, imported from /root/reference; numba backend) on the same
C2 graph bytes and batch seeds: per-batch losses must agree bit for bit and the two
per-batch times are printed side by side.  Runs in the build container only (the
reference does not travel to the GPU box); output committed as
profiles/r02_port_vs_reference.txt.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tools/port_vs_reference.py [n_batches]
"""
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    import bench
    from oracle import oracle as O
    from paper_2311_13225_b200.datagen import make_dataset
    from hetgnn import gnnmath, kernels, sampler
    from hetgnn.graph import Graph, VertexData

    ds = make_dataset("c2", cache_dir=bench.CACHE)
    batches, rseeds = bench.epoch_batches(ds, n + 1)
    wl = bench.WORKLOADS["c2"]["config"]
    dims = [ds.feat_dim] + [wl["hidden"]] * (wl["layers"] - 1) + [int(ds.labels.max()) + 1]
    fan = tuple(wl["fanouts"])
    # the port (bench.py --impl reference)
    g = O.Graph(offsets=ds.offsets, targets=ds.targets.astype(np.int64))
    feats64 = ds.features.astype(np.float64)
    od = O.VertexData(features=feats64, labels=ds.labels, train_mask=ds.train_mask, val_mask=ds.val_mask,
                      test_mask=ds.test_mask)
    cfg = dict(O.DEFAULT_CFG, model="sage", layers=3, fanouts=fan, hidden_dim=wl["hidden"], batch_size=1024,
               lr=wl["lr"], strategy="case1", hot_ratio=0.0)
    W = O.init_params("sage", dims, 0)
    port_l, port_t = [], []
    for i in range(n + 1):
        t0 = time.perf_counter()
        st = O.sample_khop(g, batches[i], fan, rseeds[i])
        loss, _, _ = O.train_batch(cfg, od, W, st, ds.labels[batches[i]], None, O.Adam())
        port_t.append(time.perf_counter() - t0)
        port_l.append(loss)
    # the real reference: sampler.sample_khop + orchestrator._train_batch's body (orchestrator.py:236-256)
    rg = Graph(offsets=ds.offsets.astype(np.int64), targets=ds.targets.astype(np.int64))
    rd = VertexData(features=feats64, labels=ds.labels.astype(np.int64), train_mask=ds.train_mask,
                    val_mask=ds.val_mask, test_mask=ds.test_mask)
    P = gnnmath.init_params("sage", dims, 0)
    ref_l, ref_t = [], []
    for i in range(n + 1):
        t0 = time.perf_counter()
        st = sampler.sample_khop(rg, batches[i], sampler.Fanouts(fan), rseeds[i])
        inputs = rd.features[st.bottom_src()]
        logits, caches = gnnmath.forward_batch(st, inputs, P)
        loss, dl = gnnmath.loss_and_grad(logits, rd.labels[batches[i]])
        grads = gnnmath.backward_batch(caches, dl, P)
        old = [[w.copy() for w in layer] for layer in P.weights]  # orchestrator.py:246-255 (epsilon monitor)
        gnnmath.sgd_step(P, grads, wl["lr"])
        max(float(np.max(np.abs(wn - wo))) for lo, ln in zip(old, P.weights) for wo, wn in zip(lo, ln))
        ref_t.append(time.perf_counter() - t0)
        ref_l.append(loss)
    same = [a == b for a, b in zip(port_l, ref_l)]
    print(f"C2 bench config, {n} timed batches after 1 warm-up, {os.cpu_count()} host cores, "
          f"kernels backend {kernels.backend_name()}")
    for i in range(n + 1):
        print(f"batch {i}: loss port {port_l[i]!r} hetgnn {ref_l[i]!r} equal={same[i]}  "
              f"time port {port_t[i]:.3f}s hetgnn {ref_t[i]:.3f}s")
    pt, rt = sum(port_t[1:]), sum(ref_t[1:])
    print(f"losses bit-identical: {all(same)}")
    print(f"seeds/s: port {1024 * n / pt:.0f}  hetgnn {1024 * n / rt:.0f}  (port/hetgnn {rt / pt:.2f}x)")


if __name__ == "__main__":
    main()
