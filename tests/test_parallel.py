"""Data-parallel decomposition on CPU with torch.distributed/gloo,
world_size 2: seed shards sampled with the same batch seed + gradients scaled by
1/|global batch| + SUM all-reduce == the single-process union step (SAGE)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2311_13225_b200.parallel import shard, shard_bounds


def test_shard_bounds_cover():
    for n in (0, 1, 7, 1024, 1025):
        for w in (1, 2, 3, 8):
            spans = [shard_bounds(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _grads(model, seeds, n_total, seed_rng, g, data, W):
    from oracle import oracle as O
    st = O.sample_khop(g, seeds, (5, 4), seed_rng)
    logits, caches = O.forward_batch(model, st, data.features[st.blocks[0].src_vertices], W)
    e = np.exp(logits - logits.max(1, keepdims=True))
    p = e / e.sum(1, keepdims=True)
    p[np.arange(len(seeds)), data.labels[seeds]] -= 1.0
    dl = p / n_total  # scaled by the GLOBAL batch size (hg_softmax_xent d_div)
    grads = O.backward_batch(model, caches, dl, W)
    return np.concatenate([gm.ravel() for gl in grads for gm in gl]), logits


def _worker(rank, world, port, model, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2311_13225_b200.datagen import make_dataset
    ds = make_dataset("tiny")
    g = O.Graph(ds.offsets, ds.targets.astype(np.int64))
    data = O.VertexData(ds.features.astype(np.float64), ds.labels, ds.train_mask, ds.val_mask, ds.test_mask)
    W = O.init_params(model, [ds.feat_dim, 16, ds.num_classes], 5)
    batch = ds.train_ids()[:200]
    mine = shard(batch, world, rank)
    gl, _ = _grads(model, mine, batch.shape[0], 777, g, data, W)
    t = torch.as_tensor(gl)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    if rank == 0:
        union, _ = _grads(model, batch, batch.shape[0], 777, g, data, W)
        out[model] = float(np.abs(t.numpy() - union).max() / np.abs(union).max())
    dist.destroy_process_group()


@pytest.mark.parametrize("model", ["sage", "gcn"])
def test_sharded_step_equals_union_step_gloo(model):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), model, out), nprocs=2, join=True)
    if model == "sage":
        assert out["sage"] < 1e-12  # SAGE: sharded == union
    else:
        assert out["gcn"] > 1e-6   # GCN: block-local out-degree differs per shard (gnnmath.py:96)


def _ctx_worker(rank, world, port, out):
    """The product's DistContext host logic at world 2 on gloo: gradient all-reduce,
    global-batch divisor, max over ranks, barrier, teardown."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_2311_13225_b200.parallel import DistContext
    ctx = DistContext("gloo")
    g = torch.full((4,), float(rank + 1), dtype=torch.float32)
    ctx.allreduce(g)
    local = shard(np.arange(1000), ctx.world, ctx.rank)
    gb = ctx.global_batch(local)
    ctx.set_global_batch(1000)
    gb_strong = ctx.global_batch(local)
    mx = ctx.max_over_ranks(float(rank) * 2.5)
    ctx.barrier()
    ctx.close()
    out[rank] = (g.tolist(), int(local.shape[0]), gb, gb_strong, mx, torch.distributed.is_initialized())


def test_dist_context_world2_gloo():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_ctx_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in range(2):
        g, n_local, gb, gb_strong, mx, still = out[r]
        assert g == [3.0] * 4                 # sum over ranks
        assert n_local == 500 and gb == 1000  # weak: world x local
        assert gb_strong == 1000              # strong: the fixed global batch
        assert mx == 2.5                      # max over ranks
        assert not still                      # process group torn down
