"""The oracle (CPU restatement, test infrastructure) against the REAL
reference's outputs at the BASELINE.json configurations
(tests/golden/make_golden_configs.py): this pins the oracle — and with it the
bench's CPU reference arm (``kind: "port"``) — to hetgnn at the bench's own
configuration, and re-checks the generator's bytes (fingerprints).

* C1 (2 whole epochs) and C2 (the bench config, 8 batches on the full 2.4M-vertex
  graph): the oracle's per-batch losses equal the reference's to 1e-9 relative
  (both fp64; only BLAS summation order differs), max |dw| likewise.
* The skip-hot flags and the 40 recorded store traces: exact.
"""

import json

import numpy as np
import pytest

from conftest import GOLDEN_DIR


@pytest.fixture(scope="module")
def cz():
    return np.load(GOLDEN_DIR / "configs.npz")


@pytest.fixture(scope="module")
def cmeta():
    return json.loads((GOLDEN_DIR / "configs.json").read_text())


def _oracle_inputs(meta):
    from oracle import oracle as O
    from paper_2311_13225_b200.datagen import limit_train, make_dataset
    full = make_dataset(meta["dataset"])
    assert full.fingerprint() == meta["fingerprint"]
    ds = limit_train(full, meta["train_limit"]) if meta["train_limit"] else full
    g = O.Graph(ds.offsets, ds.targets.astype(np.int64))
    d = O.VertexData(ds.features.astype(np.float64), ds.labels, ds.train_mask, ds.val_mask, ds.test_mask)
    cfg = dict(meta["config"])
    cfg["fanouts"] = tuple(cfg["fanouts"])
    return O, g, d, cfg


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_oracle_matches_reference_at_config(cmeta, name):
    meta = cmeta[name]
    O, g, d, cfg = _oracle_inputs(meta)
    reps, _, _ = O.run_training(g, d, cfg, evaluate_each_epoch=(name == "c1"))
    for rep, want in zip(reps, meta["epochs"]):
        np.testing.assert_allclose(rep["losses"], want["losses"], rtol=1e-9)
        np.testing.assert_allclose(rep["max_deltas"], want["max_weight_deltas"], rtol=1e-7)
        if want["test_accuracy"] is not None:
            assert rep["test_accuracy"] == want["test_accuracy"]


def test_oracle_skip_hot_flags(cz, cmeta, ggraphs):
    from oracle import oracle as O
    g = ggraphs["pl"].graph
    for k, (fan, s) in enumerate(cmeta["skiphot"]):
        st = O.sample_khop_skip_hot(g, cz[f"skiphot{k}_seeds"], tuple(fan), cz[f"skiphot{k}_hot"], s)
        assert np.array_equal(st.blocks[0].src_vertices, cz[f"skiphot{k}_src"])
        assert np.array_equal(st.hot_flags, cz[f"skiphot{k}_flags"])


def test_oracle_store_replays_reference_traces(cmeta):
    from oracle import oracle as O
    errs = (O.StoreContractError, O.StalenessViolation)
    for t in cmeta["store"]:
        st = O.Store(t["n"], 3)
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
                    st.advance(rec["window_start"], rec["window_len"])
                    got = "ok"
                elif op == "reset":
                    st.reset_epoch(rec["window_start"])
                    got = "ok"
                else:
                    got = [st.staged_count(), st.live_entries(), st.memory_bytes(), st.hits, st.misses, st.puts,
                           st.max_gap, st.max_gap_batch, st.max_gap_sb, st.sb]
            except errs as exc:
                got = {"StoreContractError": "StoreContractError"}.get(type(exc).__name__, "StalenessViolation")
            assert got == want, (t["n"], rec)


def test_config_rejects_simulator_options():
    from paper_2311_13225_b200.orchestrator import ConfigError, TrainConfig
    with pytest.raises(ConfigError):
        TrainConfig(simulate_costs=True).validate()
    with pytest.raises(ConfigError):
        TrainConfig(preset="paper-like").validate()
    TrainConfig().validate()
