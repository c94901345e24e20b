"""GPU parity of the plug-in kernels and the sampler against the golden vectors
(produced by the reference) and the CPU oracle.  Integer outputs: bit-exact.
segment_weighted_rows (fp64): bit-exact."""

import numpy as np
import pytest

from conftest import golden_stack, has_cuda

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_cuda(), reason="needs CUDA")]


@pytest.fixture(scope="module")
def K():
    from paper_2311_13225_b200 import kernels
    return kernels


@pytest.fixture(scope="module")
def S():
    from paper_2311_13225_b200 import sampler
    return sampler


def test_sample_layer_golden(K, golden, golden_meta, ggraphs):
    for k, (gname, f, s) in enumerate(golden_meta["sample_layer"]):
        g = ggraphs[gname].graph
        ed, es = K.sample_layer(g.offsets, g.targets, golden[f"sl{k}_dst"], f, s)
        assert np.array_equal(ed, golden[f"sl{k}_ed"]), (k, gname, f)
        assert np.array_equal(es, golden[f"sl{k}_es"]), (k, gname, f)


def test_sample_layer_appendix_a(K, ggraphs):
    star = ggraphs["star"].graph
    ed, es = K.sample_layer(star.offsets, star.targets, np.arange(6), 3, 777)
    assert ed.tolist() == [0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5]
    assert es.tolist() == [5, 3, 1, 0, 1, 0, 2, 0, 3, 0, 4, 0, 5]


def test_stable_unique_golden(K, golden):
    for k in range(5):
        u, inv = K.stable_unique(golden[f"su{k}_in"])
        assert np.array_equal(u, golden[f"su{k}_u"])
        assert np.array_equal(inv, golden[f"su{k}_inv"])


def test_stable_unique_sentinel_and_negative(K):
    from oracle import oracle as O
    v = np.array([-1, 5, -1, 2**63 - 1, -(2**63), 5, 0, -1], dtype=np.int64)
    u, inv = K.stable_unique(v)
    ru, rinv = O.stable_unique(v)
    assert np.array_equal(u, ru) and np.array_equal(inv, rinv)


def _cmp(st, ref):
    assert len(st.blocks) == len(ref)
    for b, r in zip(st.blocks, ref):
        assert np.array_equal(b.dst_vertices, r["dst"])
        assert np.array_equal(b.src_vertices, r["src"])
        assert np.array_equal(b.edge_src, r["es"])
        assert np.array_equal(b.edge_dst, r["ed"])


def test_sample_khop_golden(S, golden, golden_meta, ggraphs):
    for k, (gname, fan, s) in enumerate(golden_meta["khop"]):
        st = S.sample_khop(ggraphs[gname].graph, golden[f"kh{k}_seeds"], S.Fanouts(tuple(fan)), s)
        _cmp(st, golden_stack(golden, f"kh{k}"))
    blk = S.sample_one_hop_hot(ggraphs["pl"].graph, np.array([0, 10, 3, 999, 500]), 6, 31337)
    _cmp(S.SampledBlockStack(blocks=[blk], seeds=None), golden_stack(golden, "oh0"))


def test_sample_khop_c1(S, golden):
    from paper_2311_13225_b200.datagen import make_dataset
    ds = make_dataset("c1")
    st = S.sample_khop(ds, golden["c1kh_seeds"], (10, 25), 4242)
    _cmp(st, golden_stack(golden, "c1kh"))


@pytest.mark.parametrize("fan", [(15, 10, 5), (10, 25), (4, 4), (40, 3)])
def test_sample_khop_vs_oracle_c2_shape(S, fan):
    """Full-size products-shaped batch, oracle on the same graph bytes."""
    from oracle import oracle as O
    from paper_2311_13225_b200.datagen import make_dataset
    ds = make_dataset("c2", scale=0.1)
    seeds = ds.train_ids()[:1024]
    st = S.sample_khop(ds, seeds, fan, 0x1234567)
    ref = O.sample_khop(O.Graph(ds.offsets, ds.targets.astype(np.int64)), seeds, fan, 0x1234567)
    _cmp(st, [dict(dst=b.dst_vertices, src=b.src_vertices, es=b.edge_src, ed=b.edge_dst) for b in ref.blocks])


def test_sampling_uniformity_five_sigma(K, ggraphs):
    """test_kernels.py:92-107 on the GPU draw kernel."""
    star = ggraphs["star"].graph
    hits = np.zeros(6, np.int64)
    reps = 3000
    for seed in range(reps):
        _, srcs = K.sample_layer(star.offsets, star.targets, np.array([0]), 3, seed)
        assert len(set(srcs.tolist())) == 3
        hits[srcs] += 1
    assert np.all(np.abs(hits - reps * 0.5) <= 5 * np.sqrt(reps * 0.25)), hits


def test_segment_weighted_rows_bitexact(K):
    from oracle import oracle as O
    rng = np.random.default_rng(3)
    for n_e, n_src, n_out, d in [(400, 50, 30, 6), (5000, 300, 200, 37), (1, 1, 1, 1), (0, 5, 4, 3)]:
        es = rng.integers(0, n_src, n_e)
        ed = rng.integers(0, n_out, n_e)
        w = rng.standard_normal(n_e)
        rows = rng.standard_normal((n_src, d))
        got = K.segment_weighted_rows(es, ed, w, rows, n_out)
        want = np.zeros((n_out, d))
        np.add.at(want, ed, w[:, None] * rows[es])
        assert np.array_equal(got, want)
        assert np.array_equal(got, O.segment_weighted_rows(es, ed, w, rows, n_out))


def test_count_into(K):
    c = np.zeros(10, np.int64)
    K.count_into(c, np.array([1, 1, 3, 9, 1]))
    assert c.tolist() == [0, 3, 0, 1, 0, 0, 0, 0, 0, 1]


def test_sampler_errors(S, ggraphs):
    g = ggraphs["pl"].graph
    with pytest.raises(S.SamplerError):
        S.sample_khop(g, np.array([], np.int64), (2,), 1)
    with pytest.raises(S.SamplerError):
        S.sample_khop(g, np.array([5000]), (2,), 1)
    with pytest.raises(S.SamplerError):
        S.sample_one_hop_hot(g, np.array([1, 1]), 2, 1)
    with pytest.raises(S.SamplerError):
        S.Fanouts(())


def test_layer_sampler_varying_chunk_sizes(S):
    """One LayerSampler reused with growing and shrinking size overrides (the
    hot producer's queue chunks, orchestrator.py:259-271): every block equals the
    oracle's sample_one_hop_hot block on the same graph bytes."""
    import torch
    from oracle import oracle as O
    from paper_2311_13225_b200.datagen import make_dataset
    from paper_2311_13225_b200.device import DeviceGraph, u64_tensor
    ds = make_dataset("c2", scale=0.1)
    dg = DeviceGraph.from_dataset(ds)
    og = O.Graph(ds.offsets, ds.targets.astype(np.int64))
    smp = S.LayerSampler(dg, 60000, 15, minpos=dg.minpos.like())
    rng = np.random.default_rng(5)
    for c in (60000, 1200, 45000, 7, 60000, 31000):
        ids = rng.choice(ds.num_vertices, size=c, replace=False)
        seed = int(rng.integers(1 << 62))
        smp.run(torch.as_tensor(ids.astype(np.int32), device="cuda"), None, u64_tensor(seed, "cuda"), 0, cap_dst=c)
        got = smp.to_block(ids)
        ref = O.sample_one_hop_hot(og, ids, 15, seed)
        assert np.array_equal(got.src_vertices, ref.src_vertices), c
        assert np.array_equal(got.edge_src, ref.edge_src), c
        assert np.array_equal(got.edge_dst, ref.edge_dst), c


def test_draws_only_matches_full_block(S):
    """hg_sample_layer_draws (the SAGE bottom block of the training step) yields the
    same per-destination draws and non-self counts as the full draw + dedup +
    relabel pass (whose slots are the same draws re-ordered by local source id)."""
    import torch
    from paper_2311_13225_b200.datagen import make_dataset
    from paper_2311_13225_b200.device import DeviceGraph, u64_tensor
    ds = make_dataset("c2", scale=0.1)
    dg = DeviceGraph.from_dataset(ds)
    rng = np.random.default_rng(11)
    ids = torch.as_tensor(rng.choice(ds.num_vertices, size=20000, replace=False).astype(np.int32), device="cuda")
    seed = u64_tensor(0xABCDEF, "cuda")
    full = S.LayerSampler(dg, 20000, 15, need_nself=True, minpos=dg.minpos.like()).run(ids, None, seed, 0)
    draws = S.LayerSampler(dg, 20000, 15, need_nself=True).run(ids, None, seed, 0, dedup=False)
    torch.cuda.synchronize()
    assert torch.equal(full.counts, draws.counts)
    assert torch.equal(full.nself, draws.nself)
    f = 15
    a = full.slots.view(-1, f).cpu().numpy()
    b = draws.slots.view(-1, f).cpu().numpy()
    cnt = full.counts.cpu().numpy()
    for i in range(0, 20000, 97):
        assert sorted(a[i, :cnt[i]].tolist()) == sorted(b[i, :cnt[i]].tolist()), i


@pytest.mark.parametrize("model,F", [("gcn", 602), ("sage", 602), ("sage", 200), ("gcn", 1000)])
def test_wide_row_bulk_gather_bitexact(model, F):
    """Wide rows (F > 128): the TMA bulk-copy staged aggregation (tuning key 12)
    and the per-lane LDG loop (default) compute the same items in the same FMA
    order: whole training runs (bottom gather by global id, upper layers by local
    id, hot-embedding injection skipping rows) are bit-identical, and both match
    the fp64 oracle."""
    import dataclasses
    from oracle import oracle as O
    from paper_2311_13225_b200 import _lib
    from paper_2311_13225_b200.datagen import make_dataset
    from paper_2311_13225_b200.orchestrator import TrainConfig, run_training
    base = make_dataset("tiny")
    feats = np.random.default_rng(3).standard_normal((base.num_vertices, F)).astype(np.float32)
    ds = dataclasses.replace(base, features=feats)
    kw = dict(model=model, layers=2, fanouts=(10, 25) if model == "gcn" else (7, 5), hidden_dim=64,
              batch_size=128, epochs=1, lr=0.05, seed=4, super_batch_n=2, hot_ratio=0.2, presample_rounds=1)
    lib = _lib.load()
    out = {}
    try:
        for bulk in (1, 0):
            lib.hg_set_tuning(12, bulk)
            out[bulk] = run_training(ds, None, TrainConfig(**kw))[0].losses
    finally:
        lib.hg_set_tuning(12, 0)
    assert out[1] == out[0]
    og = O.Graph(ds.offsets, ds.targets.astype(np.int64))
    od = O.VertexData(ds.features.astype(np.float64), ds.labels, ds.train_mask, ds.val_mask, ds.test_mask)
    ref, _, _ = O.run_training(og, od, kw, evaluate_each_epoch=False)
    np.testing.assert_allclose(out[1], ref[0]["losses"], rtol=1e-4)
