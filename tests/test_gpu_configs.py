"""GPU parity at the BASELINE.json configurations against the REAL reference
(tests/golden/make_golden_configs.py ran hetgnn in-process on the same graph
bytes; the graphs are regenerated here by datagen and fingerprint-checked).

Tolerances (fp32 device arithmetic vs the reference's fp64), each the stated
bound with the achieved value recorded (tests/_metrics.py):
* sampled blocks, hot list, queues, reuse hits, fallbacks, stage events, max
  gap, staleness counters, batch-CSV row counts: bit-exact;
* first-batch logits: |d| <= 2e-4 * max(1, |ref|);
* per-batch losses at C1/C2/C3 (SGD, lr <= 0.1): relative 1e-4 (SURVEY §8(c)'s
  proposal; fp32 rounding of features and weights alone moves them ~1e-6);
* max |dw| per batch and the epsilon trace: relative 1e-3 (a max over 27K-165K
  weight steps, each an fp32 gradient x lr);
* the learnable dataset (SGD lr 0.5, 3 epochs x 30 batches): the first 10
  losses relative 1e-4, all losses 2e-2 (a large step amplifies fp32 rounding
  along the trajectory),
  test and val accuracy within 0.005 (0.5 points, north_star) on 24,000 test
  vertices.
"""

import json

import numpy as np
import pytest

from conftest import GOLDEN_DIR, has_cuda
from _metrics import record

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_cuda(), reason="needs CUDA")]

LOSS_RTOL = 1e-4
MD_RTOL = 1e-3
ACC_TOL = 0.005


@pytest.fixture(scope="module")
def cz():
    return np.load(GOLDEN_DIR / "configs.npz")


@pytest.fixture(scope="module")
def cmeta():
    return json.loads((GOLDEN_DIR / "configs.json").read_text())


_DS = {}


def dataset(name, meta=None):
    from paper_2311_13225_b200.datagen import make_dataset
    if name not in _DS:
        _DS[name] = make_dataset(name)
    ds = _DS[name]
    if meta is not None:
        assert ds.fingerprint() == meta["fingerprint"], f"{name}: generator output changed"
    return ds


def run_cfg(meta, **over):
    from paper_2311_13225_b200.orchestrator import TrainConfig
    kw = dict(meta["config"])
    kw["fanouts"] = tuple(kw["fanouts"])
    kw.update(over)
    return TrainConfig(**kw)


def limited(meta):
    from paper_2311_13225_b200.datagen import limit_train
    ds = dataset(meta["dataset"], meta)
    return limit_train(ds, meta["train_limit"]) if meta["train_limit"] else ds


def stack_hash(stack):
    import hashlib
    h = hashlib.sha256()
    for b in stack.blocks:
        for a in (b.dst_vertices, b.src_vertices, b.edge_src, b.edge_dst):
            h.update(np.ascontiguousarray(a, np.int64).tobytes())
    return h.hexdigest()


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-30)))


def check_epoch(name, rep, want, exact_hot=True):
    r_loss = rel(rep.losses, want["losses"])
    r_md = rel(rep.max_weight_deltas, want["max_weight_deltas"])
    r_eps = rel(rep.epsilon_trace, want["epsilon_trace"])
    record(f"{name}.loss_rel", r_loss, LOSS_RTOL)
    record(f"{name}.max_dw_rel", r_md, MD_RTOL)
    record(f"{name}.epsilon_rel", r_eps, MD_RTOL)
    assert len(rep.losses) == len(want["losses"])
    assert r_loss <= LOSS_RTOL, r_loss
    assert r_md <= MD_RTOL, r_md
    assert r_eps <= MD_RTOL, r_eps
    if exact_hot:
        assert [r["reuse_hits"] for r in rep.batch_rows] == want["reuse_hits"]
        assert [r["fallbacks"] for r in rep.batch_rows] == want["fallbacks"]
        assert [list(e) for e in rep.stage_events] == want["stage_events"]
        assert rep.max_gap == want["max_gap"]
        assert rep.max_gap_batch == want["max_gap_batch"]
        assert rep.warmup_computed == want["warmup_computed"]


# ---------------------------------------------------------------------------
# C2: the bench configuration at full scale (2.4M V, 64M entries)
# ---------------------------------------------------------------------------
def test_c2_hub_blocks_bitexact(cz, cmeta):
    """A 1024-seed batch holding the 64 highest-degree training vertices (max
    degree >= 100K): all three blocks bit-identical to the reference's."""
    from paper_2311_13225_b200.sampler import sample_khop
    meta = cmeta["c2"]
    ds = dataset("c2", meta)
    assert meta["hub_max_degree"] >= 100_000
    st = sample_khop(ds, cz["c2_hub_seeds"], (15, 10, 5), 0xC2C2)
    assert [[b.n_dst, b.n_src, b.n_edges] for b in st.blocks] == meta["hub_stack_sizes"]
    assert stack_hash(st) == meta["hub_stack_sha256"]


def test_c2_first_batch_blocks_and_logits(cz, cmeta):
    """Batch 0 of epoch 0 (the run's shuffle and batch seed): blocks bit-exact
    through the module API, and the training engine's logits at the initial
    weights (one captured step: sampling, fused gather, TMA/tcgen05 GEMMs, fused
    top layer) within 2e-4 of the reference's fp64 logits."""
    import torch
    from paper_2311_13225_b200.orchestrator import Trainer
    from paper_2311_13225_b200.sampler import sample_khop
    meta = cmeta["c2"]
    ds = limited(meta)
    cfg = run_cfg(meta)
    tr = Trainer(ds, cfg)
    plan = tr.build_epoch_plan(0, 0)
    b0, s0 = plan.batches[0], plan.batch_seeds[0]
    assert stack_hash(sample_khop(ds, b0, cfg.fanouts, s0)) == meta["batch0_stack_sha256"]
    loss = tr.train_step(b0, s0, 0)()
    e = tr.engine
    ref = cz["c2_logits0"]
    got = e.out[e.L - 1][:ref.shape[0], :ref.shape[1]].double().cpu().numpy()
    torch.cuda.synchronize()
    err = float(np.max(np.abs(got - ref) / np.maximum(1.0, np.abs(ref))))
    record("c2.logits0_err", err, 2e-4)
    assert err <= 2e-4, err
    assert abs(loss - meta["epochs"][0]["losses"][0]) <= LOSS_RTOL * abs(meta["epochs"][0]["losses"][0])


def test_c2_training_matches_reference(cmeta):
    """The bench configuration for 8 batches (one epoch of an 8,192-seed training
    mask on the full graph): per-batch losses, max |dw| and epsilon trace."""
    from paper_2311_13225_b200.orchestrator import Trainer
    meta = cmeta["c2"]
    tr = Trainer(limited(meta), run_cfg(meta))
    rep = tr.run_epoch(tr.build_epoch_plan(0, 0))
    check_epoch("c2", rep, meta["epochs"][0], exact_hot=False)


# ---------------------------------------------------------------------------
# C3: GCN on the Reddit-shaped graph (233K V, 114M entries, F=602, H=256)
# with hot-embedding reuse (hot 0.2, n=4)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("execution", ["serial", "pipelined"])
def test_c3_hot_reuse_matches_reference(cz, cmeta, execution):
    from paper_2311_13225_b200.orchestrator import Trainer
    meta = cmeta["c3"]
    tr = Trainer(limited(meta), run_cfg(meta, execution=execution))
    assert np.array_equal(tr.hot_list, cz["c3_hot"])
    plan = tr.build_epoch_plan(0, 0)
    assert sorted(plan.queue_sizes) == meta["queue_groups"]
    for g in plan.queue_sizes:
        got = plan.queues[g][:plan.queue_sizes[g]].cpu().numpy()
        assert np.array_equal(got, cz[f"c3_q{g}"]), g
    rep = tr.run_epoch(plan)
    check_epoch(f"c3_{execution}", rep, meta["epochs"][0])
    assert rep.reuse_hits > 0


# ---------------------------------------------------------------------------
# C1 and the learnable C2-shaped graph: whole runs incl. full-graph evaluate
# ---------------------------------------------------------------------------
def test_c1_two_epochs_match_reference(cmeta):
    from paper_2311_13225_b200.orchestrator import run_training
    meta = cmeta["c1"]
    reps = run_training(limited(meta), None, run_cfg(meta))
    for k, (rep, want) in enumerate(zip(reps, meta["epochs"])):
        check_epoch(f"c1_e{k}", rep, want, exact_hot=False)
        # random labels: chance-level accuracy; still within 0.5 points of the reference
        record(f"c1_e{k}.test_acc_diff", abs(rep.test_accuracy - want["test_accuracy"]), ACC_TOL)
        assert abs(rep.test_accuracy - want["test_accuracy"]) <= ACC_TOL
        assert abs(rep.val_accuracy - want["val_accuracy"]) <= ACC_TOL


@pytest.mark.parametrize("name", ["learn_sgd", "learn_hot"])
def test_learnable_accuracy_within_half_point(cmeta, name):
    """north_star: test accuracy within 0.5 points of the reference on a
    non-saturating task (24,000 test vertices), plus the losses of all 90 batches."""
    from paper_2311_13225_b200.orchestrator import run_training
    meta = cmeta[name]
    ds = limited(meta)
    assert int(np.asarray(ds.test_mask).sum()) >= 20_000
    reps = run_training(ds, None, run_cfg(meta, execution="pipelined"))
    for k, (rep, want) in enumerate(zip(reps, meta["epochs"])):
        # a large SGD step amplifies fp32 rounding along the trajectory: the first 10
        # batches agree to 1e-4, the rest of the run drifts (recorded) within 2e-2
        r_first = rel(rep.losses[:10], want["losses"][:10])
        r_loss = rel(rep.losses, want["losses"])
        if k == 0:
            record(f"{name}_e0.loss_rel_first10", r_first, 1e-4)
            assert r_first <= 1e-4, r_first
        record(f"{name}_e{k}.loss_rel", r_loss, 2e-2)
        assert r_loss <= 2e-2, r_loss
        for split in ("test", "val"):
            d = abs(getattr(rep, f"{split}_accuracy") - want[f"{split}_accuracy"])
            record(f"{name}_e{k}.{split}_acc_diff", d, ACC_TOL)
            assert d <= ACC_TOL, (split, d)
        if name == "learn_hot":
            assert [r["reuse_hits"] for r in rep.batch_rows] == want["reuse_hits"]
            assert rep.max_gap == want["max_gap"]
    assert 0.1 < reps[-1].test_accuracy < 0.9  # non-saturating
