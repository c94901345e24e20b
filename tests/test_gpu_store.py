"""The historical-embedding store, its staleness / contract / fallback error
paths, the skip-hot flags, and the numerics guard, on the GPU.

* ``store.EmbeddingStore`` runs the reference's own store tests
  (/root/reference/pkg/tests/test_store.py:15-190, restated) and replays 40
  recorded protocol traces of the reference store op for op
  (tests/golden/configs.json "store": every get's value / miss, every
  exception, the counters) — exact.
* The training engine's device store: a forced gap-bound violation raises
  StalenessViolation and injects nothing; a dropped producer exhausts the
  fallback budget (FallbackBudgetExceeded, orchestrator.py:581-589).
* sample_khop_skip_hot's device flags (hg_member_flags) vs the reference's.
* The two-word fixed-point transposed aggregation across 24 decades of gradient
  scale vs an fp64 reference, and its range / non-finite flags.
"""

import json
import threading

import numpy as np
import pytest

from conftest import GOLDEN_DIR, has_cuda
from _metrics import record

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_cuda(), reason="needs CUDA")]


@pytest.fixture(scope="module")
def S():
    from paper_2311_13225_b200 import store
    return store


def _emb(v, version, dim=4):
    return np.full(dim, v * 1000.0 + version)


# ---- test_store.py:15-190 ---------------------------------------------------
def test_put_accepts_next_super_batch_only(S):
    st = S.EmbeddingStore(n=4, emb_dim=4)
    st.put(7, _emb(7, 2), version=2, target_super_batch=1)
    for bad in (0, 2):
        with pytest.raises(S.StoreContractError):
            st.put(7, _emb(7, 2), version=2, target_super_batch=bad)


def test_put_twice_last_write_wins(S):
    st = S.EmbeddingStore(n=2, emb_dim=4)
    st.put(3, _emb(3, 0), version=0, target_super_batch=1)
    st.put(3, _emb(3, 1), version=1, target_super_batch=1)
    st.advance_super_batch(window_start=2)
    assert np.array_equal(st.get(3, reading_batch=2), _emb(3, 1))


def test_put_many_duplicates_last_write_wins(S):
    st = S.EmbeddingStore(n=2, emb_dim=4)
    st.put_many(np.array([5, 6, 5]), np.stack([_emb(5, 0), _emb(6, 0), _emb(5, 1)]), 1, 1)
    assert st.staged_count() == 2 and st.puts == 3
    st.advance_super_batch(window_start=2)
    assert np.array_equal(st.get(5, 2), _emb(5, 1))


def test_gap_exactly_2n_minus_1_is_a_hit(S):
    st = S.EmbeddingStore(n=4, emb_dim=4)
    st.put(1, _emb(1, 0), version=0, target_super_batch=1)
    st.advance_super_batch(window_start=4)
    assert st.get(1, reading_batch=7) is not None
    assert st.max_observed_gap == 7


def test_boundary_eviction_returns_miss(S):
    st = S.EmbeddingStore(n=4, emb_dim=4)
    st.put(1, _emb(1, 0), version=0, target_super_batch=1)
    st.advance_super_batch(window_start=4)
    st.advance_super_batch(window_start=8)
    assert st.get(1, reading_batch=8) is None


def test_gap_violation_raises(S):
    st = S.EmbeddingStore(n=2, emb_dim=4)
    st.put(5, _emb(5, 0), version=-10, target_super_batch=1)
    st.advance_super_batch(window_start=2)
    with pytest.raises(S.StalenessViolation):
        st.get(5, reading_batch=3)


def test_read_outside_window_rejected(S):
    st = S.EmbeddingStore(n=2, emb_dim=4)
    st.advance_super_batch(window_start=2)
    with pytest.raises(S.StoreContractError):
        st.get(0, reading_batch=9)


def test_advance_with_empty_staging_all_miss(S):
    st = S.EmbeddingStore(n=3, emb_dim=4)
    st.advance_super_batch(window_start=3)
    assert all(st.get(v, reading_batch=3) is None for v in range(5))


def test_stage_k_then_advance_k_hits(S):
    st = S.EmbeddingStore(n=3, emb_dim=4)
    for v in range(7):
        st.put(v, _emb(v, 1), version=1, target_super_batch=1)
    st.advance_super_batch(window_start=3)
    assert sum(st.get(v, reading_batch=4) is not None for v in range(7)) == 7


def test_memory_accounting_matches_live_entries(S):
    st = S.EmbeddingStore(n=2, emb_dim=8)
    for v in range(5):
        st.put(v, np.zeros(8), version=0, target_super_batch=1)
    st.advance_super_batch(window_start=2)
    for v in range(3):
        st.put(v + 100, np.zeros(8), version=2, target_super_batch=2)
    assert st.live_entries() == 8 and st.memory_bytes() == 8 * 8 * 8
    st.advance_super_batch(window_start=4)
    assert st.live_entries() == 3 and st.memory_bytes() == 3 * 8 * 8


def test_reset_epoch_clears_everything(S):
    st = S.EmbeddingStore(n=2, emb_dim=4)
    st.put(1, _emb(1, 0), version=0, target_super_batch=1)
    st.advance_super_batch(window_start=2)
    st.reset_epoch(window_start=10)
    assert st.get(1, reading_batch=10) is None
    assert st.current_super_batch == 0


def test_schedule_fuzz_gap_bound_never_violated(S):
    rng = np.random.default_rng(42)
    trials = 0
    while trials < 200:
        for n in (1, 2, 4, 8):
            trials += 1
            st = S.EmbeddingStore(n=n, emb_dim=2)
            for sb in range(int(rng.integers(2, 5))):
                first = sb * n
                if sb > 0:
                    st.advance_super_batch(window_start=first)
                ops = [("get", first + j) for j in range(n)]
                ops += [("put", v, sb * n + int(rng.integers(0, n))) for v in range(int(rng.integers(0, 6)))]
                for k in rng.permutation(len(ops)):
                    op = ops[k]
                    if op[0] == "put":
                        st.put(op[1], np.zeros(2), version=op[2], target_super_batch=sb + 1)
                    else:
                        for v in range(6):
                            if st.get(v, reading_batch=op[1]) is not None:
                                assert st.max_observed_gap <= 2 * n - 1
            assert st.max_observed_gap <= 2 * n - 1


def test_concurrent_put_get_advance_linearizable(S):
    st = S.EmbeddingStore(n=2, emb_dim=16)
    stop = threading.Event()
    errors = []

    def writer():
        version = 0
        try:
            while not stop.is_set():
                for v in range(8):
                    st.put(v, np.full(16, v * 1e6 + version), version=version,
                           target_super_batch=st.current_super_batch + 1)
                version += 1
        except S.StoreContractError:
            pass
        except Exception as exc:  # pragma: no cover
            errors.append(exc)

    def reader():
        try:
            while not stop.is_set():
                start = st._window_start
                for v in range(8):
                    try:
                        got = st.get(v, reading_batch=start)
                    except (S.StoreContractError, S.StalenessViolation):
                        continue
                    if got is not None and not np.all(got == got[0]):
                        errors.append(AssertionError(f"torn value for {v}"))
        except Exception as exc:  # pragma: no cover
            errors.append(exc)

    threads = [threading.Thread(target=writer), threading.Thread(target=reader)]
    for t in threads:
        t.start()
    for i in range(50):
        st.advance_super_batch(window_start=(i + 1) * 2)
    stop.set()
    for t in threads:
        t.join()
    assert not errors, errors[:3]


def test_invalid_n_rejected(S):
    with pytest.raises(S.StoreContractError):
        S.EmbeddingStore(n=0, emb_dim=4)


# ---- recorded reference traces --------------------------------------------------
def test_store_replays_reference_traces(S):
    traces = json.loads((GOLDEN_DIR / "configs.json").read_text())["store"]
    n_ops = 0
    for t in traces:
        st = S.EmbeddingStore(n=t["n"], emb_dim=3)
        for rec in t["ops"]:
            op, want = rec["op"], rec["out"]
            try:
                if op == "put":
                    st.put(rec["v"], np.array(rec["emb"]), rec["version"], rec["target"])
                    got = "ok"
                elif op == "get":
                    e = st.get(rec["v"], rec["reading_batch"])
                    got = None if e is None else [float(x) for x in e]
                elif op == "advance":
                    st.advance_super_batch(rec["window_start"], rec["window_len"])
                    got = "ok"
                elif op == "reset":
                    st.reset_epoch(rec["window_start"])
                    got = "ok"
                else:
                    got = [st.staged_count(), st.live_entries(), st.memory_bytes(), st.hits, st.misses, st.puts,
                           st.max_observed_gap, st.max_gap_batch, st.max_gap_super_batch, st.current_super_batch]
            except (S.StoreContractError, S.StalenessViolation) as exc:
                got = type(exc).__name__
            assert got == want, (t["n"], rec)
            n_ops += 1
    assert n_ops > 1000


# ---- engine store: violations, fallbacks ---------------------------------------
def _hot_trainer(golden_meta, ggraphs, **over):
    from paper_2311_13225_b200.orchestrator import TrainConfig, Trainer, _Merged
    meta = golden_meta["runs"]["sbm_sage_hot"]
    kw = dict(meta["config"])
    kw.update(over)
    g = ggraphs["sbm"]
    return Trainer(_Merged(g.graph, g.data), TrainConfig(**kw))


@pytest.mark.parametrize("execution", ["serial", "pipelined"])
def test_forced_staleness_violation_raises_and_injects_nothing(golden_meta, ggraphs, execution):
    """A gap bound of 0 (every reuse is 'stale'): the device lookup counts the
    violations, injects no row, and run_epoch raises StalenessViolation."""
    from paper_2311_13225_b200.store import StalenessViolation
    tr = _hot_trainer(golden_meta, ggraphs, use_graph=False, execution=execution)
    tr.engine.hot.gap_bound = 0
    plan = tr.build_epoch_plan(0, 0)
    with pytest.raises(StalenessViolation):
        tr.run_epoch(plan)
    hot = tr.engine.hot
    assert int(hot.batch_hits.sum().item()) == 0
    assert int(hot.stats[1].item()) > 0


def test_dropped_producer_exceeds_fallback_budget(golden_meta, ggraphs, monkeypatch):
    from paper_2311_13225_b200 import orchestrator
    from paper_2311_13225_b200.store import FallbackBudgetExceeded
    monkeypatch.setattr(orchestrator.HotProducer, "run_chunk", lambda self, *a, **k: None)
    tr = _hot_trainer(golden_meta, ggraphs)
    with pytest.raises(FallbackBudgetExceeded):
        tr.run_epoch(tr.build_epoch_plan(0, 0))
    tr2 = _hot_trainer(golden_meta, ggraphs, max_fallback_frac=1.0)
    rep = tr2.run_epoch(tr2.build_epoch_plan(0, 0))
    assert rep.reuse_hits == 0 and rep.fallbacks > 0


# ---- skip-hot flags ---------------------------------------------------------------
def test_skip_hot_flags_match_reference(ggraphs):
    from paper_2311_13225_b200.sampler import sample_khop, sample_khop_skip_hot
    z = np.load(GOLDEN_DIR / "configs.npz")
    cases = json.loads((GOLDEN_DIR / "configs.json").read_text())["skiphot"]
    g = ggraphs["pl"].graph
    for k, (fan, s) in enumerate(cases):
        st = sample_khop_skip_hot(g, z[f"skiphot{k}_seeds"], tuple(fan), z[f"skiphot{k}_hot"], s)
        assert np.array_equal(st.blocks[0].src_vertices, z[f"skiphot{k}_src"])
        assert np.array_equal(st.hot_flags, z[f"skiphot{k}_flags"])
        plain = sample_khop(g, z[f"skiphot{k}_seeds"], tuple(fan), s)
        for a, b in zip(plain.blocks, st.blocks):  # flags only, never topology
            assert np.array_equal(a.src_vertices, b.src_vertices) and np.array_equal(a.edge_src, b.edge_src)
    seeds = np.arange(20)
    full = sample_khop_skip_hot(g, seeds, (5, 5), np.arange(g.num_vertices), 31)
    assert full.hot_flags.all()
    empty = sample_khop_skip_hot(g, seeds, (5, 5), np.array([], np.int64), 31)
    assert not empty.hot_flags.any()


# ---- fixed-point transposed aggregation ---------------------------------------------
def _scatter(dagg_np, counts, slot_local, slot_g, frontier, nself, outdeg, n_src, F):
    import torch
    from paper_2311_13225_b200 import _lib
    from paper_2311_13225_b200.device import ptr
    dev = "cuda"
    t = lambda a, dt=torch.int32: torch.as_tensor(np.asarray(a), dtype=dt, device=dev)  # noqa: E731
    n_dst, f = counts.shape[0], slot_local.shape[0] // counts.shape[0]
    dagg = t(dagg_np, torch.float32)
    acc = torch.zeros((n_src, 2 * F), dtype=torch.int64, device=dev)
    dx = torch.full((n_src, F), float("nan"), device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    ns = t([n_src])
    keep = [t(a) for a in (frontier, counts, slot_g, slot_local, nself, outdeg)]  # alive across the call
    fr_d, cnt_d, sg_d, sl_d, ns_d, od_d = keep
    _lib.call("hg_aggregate_bwd_scatter", 0, ptr(dagg), F, None, 0, F, ptr(fr_d), None, n_dst, f,
              ptr(cnt_d), ptr(sg_d), ptr(sl_d), ptr(ns_d), ptr(od_d), ptr(ns), n_src,
              None, 0, None, ptr(acc), ptr(dx), F, ptr(flags), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return dx.double().cpu().numpy(), int(flags.item()), int(acc.abs().sum().item())


def _random_block(rng, n_dst=300, n_src=900, f=12):
    counts = rng.integers(1, f + 1, n_dst)
    slot_local = np.zeros(n_dst * f, np.int64)
    for i in range(n_dst):  # distinct sources per destination, some shared hubs
        pool = np.concatenate([rng.integers(n_dst, n_src, counts[i] + 4), rng.integers(n_dst, n_dst + 8, 2)])
        slot_local[i * f:i * f + counts[i]] = np.unique(pool)[:counts[i]] if np.unique(pool).size >= counts[i] \
            else rng.choice(np.arange(n_dst, n_src), counts[i], replace=False)
    frontier = np.arange(n_dst) + 10_000
    slot_g = slot_local + 10_000
    outdeg = np.zeros(n_src, np.int64)
    for i in range(n_dst):
        np.add.at(outdeg, slot_local[i * f:i * f + counts[i]], 1)
    return counts, slot_local, slot_g, frontier, counts.copy(), outdeg


@pytest.mark.parametrize("scale", [1e-14, 1e-9, 1e-5, 1.0, 1e4, 1e9])
def test_fixed_point_scatter_exact_across_scales(scale):
    """SAGE transposed aggregation dx[s] = sum_e dagg[dst_e] / nself(dst_e) with
    gradients of magnitude `scale`, 1e-14 to 1e9: equal to the fp64 sum of the
    fp32 contributions to fp32 rounding (relative 1e-6) plus the accumulator's
    absolute resolution of 2^-61 per contribution (the two-word fixed point holds
    every contribution >= 2^-37 exactly)."""
    rng = np.random.default_rng(7)
    counts, sl, sg, fr, ns, od = _random_block(rng)
    F, n_dst, n_src, f = 16, counts.shape[0], 900, 12
    dagg = (rng.standard_normal((n_dst, F)) * scale).astype(np.float32)
    dx, flags, acc_left = _scatter(dagg, counts, sl, sg, fr, ns, od, n_src, F)
    want = np.zeros((n_src, F))
    for i in range(n_dst):
        w = np.float32(1.0) / np.float32(ns[i])
        for j in range(counts[i]):
            want[sl[i * f + j]] += (np.float32(w) * dagg[i]).astype(np.float64)
    mask = od > 0
    bound = 1e-6 * np.abs(want[mask]) + od[mask, None] * 2.0 ** -61
    excess = float(np.max(np.abs(dx[mask] - want[mask]) / bound))
    record(f"fixed_point.scale_{scale:g}.err_over_bound", excess, 1.0)
    assert flags == 0 and acc_left == 0
    assert excess <= 1.0, excess


def test_fixed_point_scatter_range_and_nonfinite_flags():
    rng = np.random.default_rng(8)
    counts, sl, sg, fr, ns, od = _random_block(rng)
    F = 16
    big = np.full((counts.shape[0], F), 1e14, np.float32)  # outdeg * |v| >= 2^42 for shared sources
    _, flags, _ = _scatter(big, counts, sl, sg, fr, ns, od, 900, F)
    assert flags & 2
    bad = np.zeros((counts.shape[0], F), np.float32)
    bad[5, 3] = np.inf
    _, flags, acc_left = _scatter(bad, counts, sl, sg, fr, ns, od, 900, F)
    assert flags & 1 and acc_left == 0
