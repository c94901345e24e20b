"""The data-parallel PRODUCT path at world size 2: two processes,
each a Trainer(dist=DistContext) on the same B200 (one box has one GPU), the
gradient all-reduce over gloo on CUDA tensors (NCCL cannot run two ranks on
one device), eager steps (gloo cannot be captured in a CUDA graph; the NCCL
path captures its all-reduce inside the step graph).

* SAGE: rank r trains shard r of every global batch with dlogits scaled by
  1/|global batch|; after the epoch the weights equal the single-process union
  run's to fp32 rounding (the sharded step IS the union step).
* GCN: block-local out-degrees make a shard's step differ from the union's
  (gnnmath.py:96); the weights equal the oracle's per-shard emulation (each
  shard sampled with the batch seed, gradients scaled by 1/|global| and summed).
"""

import os
import socket

import numpy as np
import pytest

from conftest import has_cuda

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_cuda(), reason="needs CUDA")]

CFG = dict(layers=2, fanouts=(5, 4), hidden_dim=16, batch_size=96, epochs=1, lr=0.1, seed=5, strategy="case1",
           use_graph=False)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, model, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK="0")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2311_13225_b200.datagen import make_dataset
    from paper_2311_13225_b200.orchestrator import TrainConfig, Trainer
    from paper_2311_13225_b200.parallel import DistContext
    ctx = DistContext()
    ds = make_dataset("tiny")
    tr = Trainer(ds, TrainConfig(model=model, **CFG), dist=ctx)
    plan = tr.build_epoch_plan(0, 0)
    rep = tr.run_epoch(plan)
    out[rank] = (tr.engine.params.flat.cpu().numpy().copy(), list(rep.losses), len(plan.batches))
    dist.barrier()
    dist.destroy_process_group()


def _run_world2(model):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(2, _free_port(), model, out), nprocs=2, join=True, start_method="spawn")
    return dict(out)


def test_world2_sage_equals_union_run():
    from paper_2311_13225_b200.datagen import make_dataset
    from paper_2311_13225_b200.orchestrator import TrainConfig, Trainer
    res = _run_world2("sage")
    w0, l0, nb = res[0]
    w1, l1, _ = res[1]
    assert np.array_equal(w0, w1)  # identical updates on both ranks
    assert l0 == l1  # the union batch's mean loss on every rank
    tr = Trainer(make_dataset("tiny"), TrainConfig(model="sage", **CFG))
    rep = tr.run_epoch(tr.build_epoch_plan(0, 0))
    union = tr.engine.params.flat.cpu().numpy()
    assert nb == len(rep.losses) > 3
    rel = np.max(np.abs(w0 - union)) / np.max(np.abs(union))
    assert rel < 1e-5, rel
    np.testing.assert_allclose(l0, rep.losses, rtol=1e-5)


def test_world2_gcn_equals_per_shard_oracle():
    from oracle import oracle as O
    from paper_2311_13225_b200 import runplan
    from paper_2311_13225_b200.datagen import make_dataset
    from paper_2311_13225_b200.parallel import shard
    res = _run_world2("gcn")
    w0 = res[0][0]
    assert np.array_equal(w0, res[1][0])
    ds = make_dataset("tiny")
    g = O.Graph(ds.offsets, ds.targets.astype(np.int64))
    feats = ds.features.astype(np.float64)
    dims = [ds.feat_dim, CFG["hidden_dim"], ds.num_classes]
    W = O.init_params("gcn", dims, CFG["seed"])
    order = runplan.shuffle_epoch(ds.train_ids(), CFG["seed"], 0)
    for b, batch in enumerate(runplan.split_batches(order, CFG["batch_size"])):
        rs = runplan.batch_sample_seed(CFG["seed"], 0, b)
        total = None
        for r in range(2):
            mine = shard(batch, 2, r)
            st = O.sample_khop(g, mine, CFG["fanouts"], rs)
            logits, caches = O.forward_batch("gcn", st, feats[st.blocks[0].src_vertices], W)
            e = np.exp(logits - logits.max(1, keepdims=True))
            p = e / e.sum(1, keepdims=True)
            p[np.arange(mine.shape[0]), ds.labels[mine]] -= 1.0
            grads = O.backward_batch("gcn", caches, p / batch.shape[0], W)
            total = grads if total is None else [[a + c for a, c in zip(x, y)] for x, y in zip(total, grads)]
        O.sgd_step(W, total, CFG["lr"])
    ref = np.concatenate([w.ravel() for lw in W for w in lw])
    rel = np.max(np.abs(w0 - ref)) / np.max(np.abs(ref))
    assert rel < 1e-4, rel
