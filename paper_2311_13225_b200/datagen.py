"""Scalable deterministic synthetic datasets for the BASELINE.json configs (§8(f4)).

The reference's generators draw a dense V x V matrix (graph.py:331,363), so
they cannot produce products-shaped graphs.  This generator keeps their
conventions — incoming-neighbour CSR with symmetrised edges and self-loops,
rows sorted by source id, duplicate edges collapsed (graph.py:131-159), hubs at
low vertex ids (graph.py:357), 65/10/25 train/test/val split (graph.py:181-196),
features N(0,1) from a Philox stream keyed by derive_seed(seed, 101)
(graph.py:171-172) — but draws O(E) Chung–Lu endpoint pairs instead of O(V^2)
coin flips.  Both the CUDA path and the CPU reference arm load the same bytes
(optionally through the reference's HGNNBIN1 cache format, graph.py:375-418).

Features are stored as float32 values so the float64 CPU reference and the
fp32 GPU path start from identical inputs.
"""

from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .seeds import derive_seed

TRAIN_FRACTION = 0.65  # graph.py:23
TEST_FRACTION = 0.10  # graph.py:24

_GEN_TAG = 0xD47A

#: name -> generator parameters.  Shapes follow BASELINE.json `configs`.
SPECS = {
    # C1: 10K-vertex / ~200K-entry power-law graph, 128-dim features
    "c1": dict(V=10_000, avg_deg=20.0, exponent=2.5, max_deg=2_500, F=128, C=8),
    # C2: ogbn-products-shaped (2.4M V, ~62M directed entries, 100-dim, 47 classes)
    "c2": dict(V=2_400_000, avg_deg=26.0, exponent=2.5, max_deg=150_000, F=100, C=47),
    # C3: Reddit-shaped (233K V, ~114M entries, 602-dim, 41 classes)
    "c3": dict(V=233_000, avg_deg=489.0, exponent=2.5, max_deg=21_000, F=602, C=41),
    # learnable C2-shaped graph for accuracy parity (class means + noise, graph.py:336-340
    # style; the signal is weak enough that test accuracy does not saturate)
    "c2learn": dict(V=240_000, avg_deg=26.0, exponent=2.5, max_deg=47_000, F=100, C=47, signal=0.3),
    # small learnable variant for accuracy parity (weak signal; does not saturate)
    "learn": dict(V=20_000, avg_deg=12.0, exponent=2.5, max_deg=2_000, F=64, C=8,
                  signal=0.35),
    # tiny, for CPU tests / smoke
    "tiny": dict(V=2_000, avg_deg=10.0, exponent=2.5, max_deg=400, F=32, C=5),
}


@dataclass
class Dataset:
    """CSR graph (int64 offsets, int32 targets) + vertex data (float32 features)."""

    name: str
    offsets: np.ndarray
    targets: np.ndarray
    features: np.ndarray
    labels: np.ndarray
    train_mask: np.ndarray
    val_mask: np.ndarray
    test_mask: np.ndarray
    meta: dict = field(default_factory=dict)

    @property
    def num_vertices(self) -> int:
        return self.offsets.shape[0] - 1

    @property
    def num_edges(self) -> int:
        return self.targets.shape[0]

    @property
    def feat_dim(self) -> int:
        return self.features.shape[1]

    @property
    def num_classes(self) -> int:
        return int(self.labels.max()) + 1

    @property
    def degrees(self) -> np.ndarray:
        return np.diff(self.offsets)

    def train_ids(self) -> np.ndarray:
        return np.nonzero(self.train_mask)[0].astype(np.int64)

    def fingerprint(self) -> str:
        h = hashlib.sha256()
        h.update(self.offsets.tobytes())
        h.update(self.targets.astype(np.int64).tobytes())
        h.update(self.features.tobytes())
        h.update(self.labels.astype(np.int64).tobytes())
        return h.hexdigest()


def _philox(seed: int, *parts: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=derive_seed(seed, *parts)))


def split_masks(n: int, seed: int):
    """graph.py:181-196 semantics: permute, first 65% train, next 10% test, rest val."""
    order = _philox(seed, 103).permutation(n)
    n_tr, n_te = int(n * TRAIN_FRACTION), int(n * TEST_FRACTION)
    train = np.zeros(n, bool)
    val = np.zeros(n, bool)
    test = np.zeros(n, bool)
    train[order[:n_tr]] = True
    test[order[n_tr:n_tr + n_te]] = True
    val[order[n_tr + n_te:]] = True
    return train, val, test


def csr_from_pairs(u: np.ndarray, v: np.ndarray, n: int):
    """Symmetrise + self-loops + collapse duplicates -> incoming-neighbour CSR
    with rows sorted by source id (graph.py:131-159 conventions)."""
    keep = u != v
    u, v = u[keep], v[keep]
    ids = np.arange(n, dtype=np.int64)
    dst = np.concatenate([v, u, ids])
    src = np.concatenate([u, v, ids])
    keys = dst * np.int64(n) + src
    del dst, src
    keys.sort()
    if keys.size > 1:
        keys = keys[np.concatenate(([True], keys[1:] != keys[:-1]))]
    row = keys // n
    offsets = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(row, minlength=n), out=offsets[1:])
    targets = (keys - row * n).astype(np.int32)
    return offsets, targets


def chung_lu_pairs(V, avg_deg, exponent, max_deg, seed):
    """Expected-degree (Chung–Lu) endpoint pairs: zipf weights, rescaled so the
    expected degree of vertex i equals w_i, capped at max_deg, sorted so low ids
    are hubs.  Returns int64 endpoint arrays of V*avg_deg/2 draws."""
    gen = _philox(seed, _GEN_TAG, 1)
    w = gen.zipf(exponent, size=V).astype(np.float64)
    total = V * avg_deg
    for _ in range(8):  # cap, then renormalise the uncapped mass
        w *= total / w.sum()
        np.minimum(w, max_deg, out=w)
    w = np.sort(w)[::-1]
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    n_pairs = int(total // 2)
    g2 = _philox(seed, _GEN_TAG, 2)
    # sorted queries keep searchsorted cache-friendly; the independent
    # permutation of v keeps the pairs i.i.d.
    u = np.searchsorted(cdf, np.sort(g2.random(n_pairs)), side="right").astype(np.int64)
    v = np.searchsorted(cdf, np.sort(g2.random(n_pairs)), side="right").astype(np.int64)
    v = v[g2.permutation(n_pairs)]
    np.minimum(u, V - 1, out=u)
    np.minimum(v, V - 1, out=v)
    return u, v


def make_dataset(name: str, seed: int = 7, scale: float = 1.0,
                 cache_dir: str | os.PathLike | None = None) -> Dataset:
    """Build (or load from ``cache_dir``) the named synthetic dataset.

    ``scale`` shrinks V (and keeps avg degree) for quick tests.
    """
    spec = dict(SPECS[name])
    V = max(16, int(spec["V"] * scale))
    max_deg = max(4, int(spec["max_deg"] * min(1.0, scale ** 0.5)))
    cache = None
    if cache_dir is not None:
        cache = Path(cache_dir) / f"hg_{name}_s{seed}_x{scale:g}.hgnnbin"
        if cache.exists():
            from .graph import load_binary
            return load_binary(cache, name=name)
    u, v = chung_lu_pairs(V, spec["avg_deg"], spec["exponent"], max_deg, seed)
    offsets, targets = csr_from_pairs(u, v, V)
    del u, v
    F, C = spec["F"], spec["C"]
    labels = _philox(seed, 102).integers(0, C, size=V).astype(np.int64)
    feats = _philox(seed, 101).standard_normal((V, F), dtype=np.float32)
    if "signal" in spec:  # learnable: class means + noise (graph.py:336-340 style)
        means = _philox(seed, 2).standard_normal((C, F)).astype(np.float32)
        feats += np.float32(spec["signal"]) * means[labels]
    train, val, test = split_masks(V, seed)
    ds = Dataset(name=name, offsets=offsets, targets=targets, features=feats, labels=labels,
                 train_mask=train, val_mask=val, test_mask=test,
                 meta=dict(spec, V=V, max_deg_cap=max_deg, seed=seed, scale=scale))
    if cache is not None:
        from .graph import save_binary
        cache.parent.mkdir(parents=True, exist_ok=True)
        tmp = cache.with_suffix(".tmp%d" % os.getpid())
        save_binary(tmp, ds)
        os.replace(tmp, cache)
    return ds


def limit_train(ds: Dataset, n: int) -> Dataset:
    """The same graph and vertex data with the training mask cut to its first ``n``
    vertices in id order (bounded-size parity runs at full graph scale)."""
    ids = np.nonzero(ds.train_mask)[0][:int(n)]
    train = np.zeros_like(ds.train_mask)
    train[ids] = True
    return Dataset(name=f"{ds.name}-train{int(n)}", offsets=ds.offsets, targets=ds.targets,
                   features=ds.features, labels=ds.labels, train_mask=train, val_mask=ds.val_mask,
                   test_mask=ds.test_mask, meta=dict(ds.meta, train_limit=int(n)))
