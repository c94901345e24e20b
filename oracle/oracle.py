"""ORACLE — test infrastructure only (never imported by the product package).

A CPU restatement of the reference's sample-based training hot path
(`/root/reference/pkg/src/hetgnn`, "hetgnn" v0.1.0) in numpy plus the two
compiled loops in ``oracle/hg_oracle.c``.  Every function names the reference
file:line it restates.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
CPU legs of ``bench.py`` may import this module; it is the checker, never the
thing measured as the product.

Pinning: ``tests/test_oracle_golden.py`` checks this module against golden
vectors that ``tests/golden/make_golden.py`` produced by importing the real
reference in the build container (KATs, sampled blocks, layer math, training
losses, store/queue traces).  The arithmetic is float64 like the reference.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

MASK = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15  # kernels.py:21
MIX1 = 0xBF58476D1CE4E5B9  # kernels.py:22
MIX2 = 0x94D049BB133111EB  # kernels.py:23
PHI = 0x2545F4914F6CDD1D  # kernels.py:24

SAMPLE_TAG = 0x5A  # sampler.py:19
SHUFFLE_TAG, BATCH_TAG, HOT_TAG, QUEUE_TAG = 0x11, 0x22, 0x33, 0x44  # runplan.py:14-17
PRESAMPLE_TAG = 0x70  # hotness.py:19
TRAIN_FRACTION, TEST_FRACTION = 0.65, 0.10  # graph.py:23-24

_HERE = Path(__file__).resolve().parent
_LIB = None


def _lib():
    """Load (building on first use) oracle/libhg_oracle.so; None if no compiler."""
    global _LIB
    if _LIB is not None:
        return _LIB or None
    so = _HERE / "libhg_oracle.so"
    if not so.exists():
        try:
            subprocess.run(["make", "-C", str(_HERE)], check=True,
                           capture_output=True)
        except Exception:
            _LIB = False
            return None
    lib = ctypes.CDLL(str(so))
    i64p = ctypes.POINTER(ctypes.c_int64)
    f64p = ctypes.POINTER(ctypes.c_double)
    lib.oracle_mix64.restype = ctypes.c_uint64
    lib.oracle_mix64.argtypes = [ctypes.c_uint64]
    lib.oracle_sample_counts.restype = ctypes.c_int64
    lib.oracle_sample_counts.argtypes = [i64p, i64p, ctypes.c_int64, ctypes.c_int64, i64p]
    lib.oracle_sample_layer.restype = None
    lib.oracle_sample_layer.argtypes = [i64p, i64p, i64p, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_uint64, i64p, i64p]
    lib.oracle_segment_weighted_rows.restype = None
    lib.oracle_segment_weighted_rows.argtypes = [i64p, i64p, f64p, ctypes.c_int64, f64p,
                                                 ctypes.c_int64, f64p]
    _LIB = lib
    return lib


def _p(a, ct=ctypes.c_int64):
    return a.ctypes.data_as(ctypes.POINTER(ct))


# ---------------------------------------------------------------------------
# R1: splitmix64 streams — kernels.py:51-70
# ---------------------------------------------------------------------------

def mix64(x: int) -> int:
    """kernels.py:51-55."""
    x &= MASK
    x = ((x ^ (x >> 30)) * MIX1) & MASK
    x = ((x ^ (x >> 27)) * MIX2) & MASK
    return x ^ (x >> 31)


def derive_seed(seed: int, *parts: int) -> int:
    """kernels.py:61-70: chained finalisers over (seed, parts...)."""
    st = mix64((seed & MASK) + GOLDEN)
    for p in parts:
        st = mix64(((st + GOLDEN) & MASK) ^ (p & MASK))
    return st


# ---------------------------------------------------------------------------
# R2/R3/A1: the plug-in kernels — kernels.py:77-180
# ---------------------------------------------------------------------------

def sample_layer(offsets, targets, dst, fanout, stream_seed):
    """kernels.py:147-158 -> _sample_layer kernels.py:77-118.

    Returns (edge_dst_local, edge_src_global) in emission order.
    """
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    targets = np.ascontiguousarray(targets, dtype=np.int64)
    dst = np.ascontiguousarray(dst, dtype=np.int64)
    lib = _lib()
    if lib is not None:
        counts = np.empty(dst.shape[0], np.int64)
        total = lib.oracle_sample_counts(_p(offsets), _p(dst), dst.shape[0], int(fanout),
                                         _p(counts))
        ed = np.empty(total, np.int64)
        es = np.empty(total, np.int64)
        lib.oracle_sample_layer(_p(offsets), _p(targets), _p(dst), dst.shape[0],
                                int(fanout), int(stream_seed) & MASK, _p(ed), _p(es))
        return ed, es
    # pure-Python restatement (small inputs only)
    base = mix64((int(stream_seed) & MASK) + GOLDEN)
    out_d, out_s = [], []
    for i, v in enumerate(dst.tolist()):
        lo, hi = int(offsets[v]), int(offsets[v + 1])
        deg = hi - lo
        if deg <= fanout:
            out_d += [i] * deg
            out_s += targets[lo:hi].tolist()
            continue
        st = mix64(base ^ ((v * PHI) & MASK))
        perm = {}
        for j in range(fanout):
            st = (st + GOLDEN) & MASK
            pick = j + mix64(st) % (deg - j)
            a, b = perm.get(j, j), perm.get(pick, pick)
            perm[j], perm[pick] = b, a
            out_d.append(i)
            out_s.append(int(targets[lo + b]))
    return np.asarray(out_d, np.int64), np.asarray(out_s, np.int64)


def stable_unique(values):
    """kernels.py:166-180: first-occurrence dedup; uniq[inverse] == values."""
    values = np.asarray(values)
    _, first, inv = np.unique(values, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")
    rank = np.empty_like(order)
    rank[order] = np.arange(order.shape[0])
    return values[np.sort(first)], rank[inv.reshape(-1)]


def count_into(counter, ids):
    """kernels.py:161-163."""
    np.add.at(counter, ids, 1)


def segment_weighted_rows(edge_src, edge_dst, weights, rows, n_out):
    """kernels.py:121-129 (numba loop) == kernels.py:132-136 (np.add.at)."""
    rows = np.ascontiguousarray(rows, dtype=np.float64)
    out = np.zeros((n_out, rows.shape[1]), np.float64)
    es = np.ascontiguousarray(edge_src, dtype=np.int64)
    ed = np.ascontiguousarray(edge_dst, dtype=np.int64)
    w = np.ascontiguousarray(weights, dtype=np.float64)
    if es.shape[0] == 0:
        return out
    lib = _lib()
    if lib is not None:
        lib.oracle_segment_weighted_rows(_p(es), _p(ed), _p(w, ctypes.c_double), es.shape[0],
                                         _p(rows, ctypes.c_double), rows.shape[1],
                                         _p(out, ctypes.c_double))
    else:
        np.add.at(out, ed, w[:, None] * rows[es])
    return out


# ---------------------------------------------------------------------------
# data model + CSR helpers — graph.py:33-196
# ---------------------------------------------------------------------------

@dataclass
class Graph:
    """graph.py:33-77 (incoming-neighbour CSR, int64)."""
    offsets: np.ndarray
    targets: np.ndarray

    @property
    def num_vertices(self):
        return self.offsets.shape[0] - 1

    @property
    def num_edges(self):
        return self.targets.shape[0]

    @property
    def degrees(self):
        return np.diff(self.offsets)


@dataclass
class VertexData:
    """graph.py:81-124."""
    features: np.ndarray
    labels: np.ndarray
    train_mask: np.ndarray
    val_mask: np.ndarray
    test_mask: np.ndarray

    @property
    def feat_dim(self):
        return self.features.shape[1]

    @property
    def num_classes(self):
        return int(self.labels.max()) + 1 if self.labels.size else 0


def build_csr(src, dst, n, symmetrize=False, add_self_loops=False):
    """graph.py:131-159: unique (dst, src) keys -> row = dst, sorted by src."""
    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    if symmetrize:
        src, dst = np.concatenate([src, dst]), np.concatenate([dst, src])
    if add_self_loops:
        ids = np.arange(n, dtype=np.int64)
        src, dst = np.concatenate([src, ids]), np.concatenate([dst, ids])
    keys = np.unique(dst * np.int64(n) + src)
    offsets = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(keys // n, minlength=n), out=offsets[1:])
    return Graph(offsets=offsets, targets=keys % n)


def split_masks(n, seed):
    """graph.py:181-196: 65/10/25 train/test/val split."""
    gen = np.random.Generator(np.random.Philox(key=derive_seed(seed, 103)))
    order = gen.permutation(n)
    n_tr, n_te = int(n * TRAIN_FRACTION), int(n * TEST_FRACTION)
    masks = [np.zeros(n, bool) for _ in range(3)]
    masks[0][order[:n_tr]] = True
    masks[2][order[n_tr:n_tr + n_te]] = True
    masks[1][order[n_tr + n_te:]] = True
    return tuple(masks)  # train, val, test


# ---------------------------------------------------------------------------
# R4-R7: k-hop sampler — sampler.py:26-180
# ---------------------------------------------------------------------------

@dataclass
class Block:
    """sampler.py:46-78."""
    dst_vertices: np.ndarray
    src_vertices: np.ndarray
    edge_src: np.ndarray
    edge_dst: np.ndarray

    @property
    def n_dst(self):
        return self.dst_vertices.shape[0]

    @property
    def n_src(self):
        return self.src_vertices.shape[0]

    @property
    def n_edges(self):
        return self.edge_src.shape[0]


@dataclass
class Stack:
    """sampler.py:82-101."""
    blocks: list
    seeds: np.ndarray
    hot_flags: np.ndarray = None


def expand_frontier(graph, frontier, fanout, stream_seed):
    """sampler.py:104-118: draw -> first-occurrence dedup -> (dst, src) order."""
    ed, es_g = sample_layer(graph.offsets, graph.targets, frontier, fanout, stream_seed)
    src_vertices, inverse = stable_unique(np.concatenate([frontier, es_g]))
    es = inverse[frontier.shape[0]:]
    order = np.lexsort((es, ed))
    return Block(dst_vertices=np.asarray(frontier, np.int64), src_vertices=src_vertices,
                 edge_src=es[order], edge_dst=ed[order])


def sample_khop(graph, seeds, fanouts, rng_seed):
    """sampler.py:130-147: layers top (L-1) to bottom (0)."""
    seeds = np.asarray(seeds, np.int64)
    blocks = [None] * len(fanouts)
    frontier = seeds
    for layer in range(len(fanouts) - 1, -1, -1):
        blk = expand_frontier(graph, frontier, fanouts[layer],
                              derive_seed(rng_seed, SAMPLE_TAG, layer))
        blocks[layer] = blk
        frontier = blk.src_vertices
    return Stack(blocks=blocks, seeds=seeds)


def sample_khop_skip_hot(graph, seeds, fanouts, hot, rng_seed):
    """sampler.py:150-163: same topology, hot flags on the bottom frontier."""
    st = sample_khop(graph, seeds, fanouts, rng_seed)
    hot = np.asarray(list(hot), np.int64)
    st.hot_flags = (np.isin(st.blocks[0].src_vertices, hot) if hot.size
                    else np.zeros(st.blocks[0].n_src, bool))
    return st


def sample_one_hop_hot(graph, hot_vertices, fanout, rng_seed, layer=0):
    """sampler.py:166-180."""
    return expand_frontier(graph, np.asarray(hot_vertices, np.int64), fanout,
                           derive_seed(rng_seed, SAMPLE_TAG, layer))


# ---------------------------------------------------------------------------
# A2-A5, F1-F4: layer math in float64 — gnnmath.py:55-312
# ---------------------------------------------------------------------------

def init_params(model, dims, seed):
    """gnnmath.py:55-71: Glorot uniform, Philox key derive_seed(seed,7,l,m)."""
    weights = []
    for l in range(len(dims) - 1):
        fi, fo = dims[l], dims[l + 1]
        lim = np.sqrt(6.0 / (fi + fo))
        mats = []
        for m in range(1 if model == "gcn" else 2):
            g = np.random.Generator(np.random.Philox(key=derive_seed(seed, 7, l, m)))
            mats.append(g.uniform(-lim, lim, size=(fi, fo)))
        weights.append(mats)
    return weights


def gcn_norm(blk):
    """gnnmath.py:89-97: 1/sqrt(outdeg_blk(src) * indeg_blk(dst))."""
    indeg = np.bincount(blk.edge_dst, minlength=blk.n_dst).astype(np.float64)
    outdeg = np.bincount(blk.edge_src, minlength=blk.n_src).astype(np.float64)
    return 1.0 / np.sqrt(outdeg[blk.edge_src] * indeg[blk.edge_dst])


def sage_edges(blk):
    """gnnmath.py:145-154: non-self edges and 1/count weights."""
    keep = blk.src_vertices[blk.edge_src] != blk.dst_vertices[blk.edge_dst]
    es, ed = blk.edge_src[keep], blk.edge_dst[keep]
    cnt = np.bincount(ed, minlength=blk.n_dst).astype(np.float64)
    w = np.zeros(es.shape[0])
    c = cnt[ed]
    w[c > 0] = 1.0 / c[c > 0]
    return es, ed, w


def layer_forward(model, blk, h_in, W, act):
    """gnnmath.py:105-126 (gcn) / :157-179 (sage) via layer_forward :203-208."""
    if model == "gcn":
        nw = gcn_norm(blk)
        agg = segment_weighted_rows(blk.edge_src, blk.edge_dst, nw, h_in, blk.n_dst)
        z = agg @ W[0]
        cache = dict(blk=blk, h_in=h_in, agg=agg, z=z, act=act, nw=nw, inj=None)
    else:
        es, ed, w = sage_edges(blk)
        agg = segment_weighted_rows(es, ed, w, h_in, blk.n_dst)
        z = h_in[:blk.n_dst] @ W[0] + agg @ W[1]
        cache = dict(blk=blk, h_in=h_in, agg=agg, z=z, act=act, nw=w, ne=(es, ed), inj=None)
    h = np.maximum(z, 0.0) if act else z
    if not np.all(np.isfinite(h)):
        raise FloatingPointError("non-finite layer output")
    return h, cache


def layer_backward(model, c, d_out, W, need_dx):
    """gnnmath.py:129-142 (gcn) / :182-200 (sage)."""
    dz = d_out * (c["z"] > 0.0) if c["act"] else d_out
    if c["inj"] is not None and c["inj"].any():
        dz = dz.copy()
        dz[c["inj"]] = 0.0
    blk = c["blk"]
    if model == "gcn":
        grads = [c["agg"].T @ dz]
        dx = None
        if need_dx:
            dx = segment_weighted_rows(blk.edge_dst, blk.edge_src, c["nw"], dz @ W[0].T,
                                       blk.n_src)
        return grads, dx
    grads = [c["h_in"][:blk.n_dst].T @ dz, c["agg"].T @ dz]
    dx = None
    if need_dx:
        dx = np.zeros((blk.n_src, W[0].shape[0]))
        dx[:blk.n_dst] += dz @ W[0].T
        es, ed = c["ne"]
        dx += segment_weighted_rows(ed, es, c["nw"], dz @ W[1].T, blk.n_src)
    return grads, dx


def forward_batch(model, stack, inputs, weights, inject=None):
    """gnnmath.py:219-247: bottom-up; inject overwrites bottom OUTPUT rows."""
    caches = []
    h = inputs
    L = len(stack.blocks)
    for l, blk in enumerate(stack.blocks):
        h, c = layer_forward(model, blk, h, weights[l], l < L - 1)
        if l == 0 and inject is not None and len(inject[0]):
            h[inject[0]] = inject[1]
            m = np.zeros(h.shape[0], bool)
            m[inject[0]] = True
            c["inj"] = m
        caches.append(c)
    return h, caches


def backward_batch(model, caches, dlogits, weights):
    """gnnmath.py:250-260: need_dx only above the bottom layer."""
    grads = [None] * len(caches)
    d = dlogits
    for l in range(len(caches) - 1, -1, -1):
        grads[l], d = layer_backward(model, caches[l], d, weights[l], l > 0)
    return grads


def loss_and_grad(logits, labels):
    """gnnmath.py:263-274: max-shifted softmax CE (mean) and dlogits."""
    e = np.exp(logits - logits.max(axis=1, keepdims=True))
    p = e / e.sum(axis=1, keepdims=True)
    n = logits.shape[0]
    loss = float(-np.log(np.maximum(p[np.arange(n), labels], 1e-300)).mean())
    d = p.copy()
    d[np.arange(n), labels] -= 1.0
    return loss, d / n


def sgd_step(weights, grads, lr):
    """gnnmath.py:277-283 (version bump is the caller's)."""
    for lw, lg in zip(weights, grads):
        for w, g in zip(lw, lg):
            w -= lr * g


@dataclass
class Adam:
    """gnnmath.py:286-312."""
    m: list = field(default_factory=list)
    v: list = field(default_factory=list)
    t: int = 0

    def step(self, weights, grads, lr, b1=0.9, b2=0.999, eps=1e-8):
        if not self.m:
            self.m = [[np.zeros_like(w) for w in lw] for lw in weights]
            self.v = [[np.zeros_like(w) for w in lw] for lw in weights]
        self.t += 1
        for li, (lw, lg) in enumerate(zip(weights, grads)):
            for wi, (w, g) in enumerate(zip(lw, lg)):
                m, v = self.m[li][wi], self.v[li][wi]
                m *= b1
                m += (1 - b1) * g
                v *= b2
                v += (1 - b2) * g * g
                w -= lr * (m / (1 - b1 ** self.t)) / (np.sqrt(v / (1 - b2 ** self.t)) + eps)


# ---------------------------------------------------------------------------
# S1: versioned store — store.py:24-146
# ---------------------------------------------------------------------------

class StalenessViolation(RuntimeError):
    pass


class StoreContractError(ValueError):
    pass


class Store:
    """store.py:24-146 (double buffer, put only for current+1, gap <= 2n-1)."""

    def __init__(self, n, emb_dim):
        if n < 1:
            raise StoreContractError("n must be >= 1")
        self.n, self.emb_dim = n, emb_dim
        self.sb, self.w0, self.wlen = 0, 0, n
        self.cur, self.stg = {}, {}
        self.hits = self.misses = self.puts = 0
        self.max_gap, self.max_gap_batch, self.max_gap_sb = 0, -1, -1

    @property
    def gap_bound(self):
        return 2 * self.n - 1

    def put(self, v, emb, version, target):
        if target != self.sb + 1:
            raise StoreContractError("put must target current+1")
        self.stg[int(v)] = (np.array(emb, np.float64), int(version))
        self.puts += 1

    def get(self, v, reading_batch):
        if not (self.w0 <= reading_batch < self.w0 + self.wlen):
            raise StoreContractError("read outside window")
        e = self.cur.get(int(v))
        if e is None:
            self.misses += 1
            return None
        gap = reading_batch - e[1]
        if gap > self.gap_bound:
            raise StalenessViolation(f"gap {gap} > {self.gap_bound}")
        self.hits += 1
        if gap > self.max_gap:
            self.max_gap, self.max_gap_batch, self.max_gap_sb = gap, reading_batch, self.sb
        return e[0]

    def advance(self, window_start=None, window_len=None):
        self.cur, self.stg = self.stg, {}
        self.sb += 1
        self.w0 = int(self.w0 + self.wlen if window_start is None else window_start)
        self.wlen = int(window_len) if window_len else self.n
        if not 1 <= self.wlen <= self.n:
            raise StoreContractError("bad window length")

    def reset_epoch(self, window_start):
        self.cur, self.stg = {}, {}
        self.sb, self.w0, self.wlen = 0, int(window_start), self.n

    def staged_count(self):  # store.py:132-134
        return len(self.stg)

    def live_entries(self):  # store.py:136-138
        return len(self.cur) + len(self.stg)

    def memory_bytes(self):  # store.py:140-142
        return self.live_entries() * self.emb_dim * 8


# ---------------------------------------------------------------------------
# S4: planning — runplan.py:20-57, orchestrator.py:200-229
# ---------------------------------------------------------------------------

def shuffle_epoch(train_ids, seed, epoch):
    g = np.random.Generator(np.random.Philox(key=derive_seed(seed, SHUFFLE_TAG, epoch)))
    return train_ids[g.permutation(train_ids.shape[0])]


def split_batches(order, bs):
    return [order[i:i + bs] for i in range(0, order.shape[0], bs)]


def super_batch_groups(nb, n):
    return [list(range(i, min(i + n, nb))) for i in range(0, nb, n)]


def chunk_bounds(total, parts):
    """runplan.py:48-57."""
    base, extra = divmod(total, parts)
    out, s = [], 0
    for j in range(parts):
        k = base + (j < extra)
        out.append((s, s + k))
        s += k
    return out


def build_epoch_plan(graph, data, cfg, hot_list, epoch, first_global_batch):
    """orchestrator.py:200-229 (queue replay with the 0x44 stream)."""
    train_ids = np.nonzero(data.train_mask)[0].astype(np.int64)
    batches = split_batches(shuffle_epoch(train_ids, cfg["seed"], epoch), cfg["batch_size"])
    groups = super_batch_groups(len(batches), cfg["super_batch_n"])
    plan = dict(epoch=epoch, batches=batches, groups=groups, first=first_global_batch,
                seeds=[derive_seed(cfg["seed"], BATCH_TAG, epoch, b) for b in range(len(batches))],
                queues={}, hot_seeds={})
    if cfg["strategy"] == "layer-based" and hot_list.size and cfg["layers"] > 1:
        for g in range(1, len(groups)):
            reach = set()
            for b in groups[g]:
                st = sample_khop(graph, batches[b], cfg["fanouts"],
                                 derive_seed(cfg["seed"], QUEUE_TAG, epoch, g))
                reach.update(st.blocks[0].dst_vertices.tolist())
            q = np.array([v for v in hot_list.tolist() if v in reach], np.int64)
            if cfg.get("stage_budget_frac", 1.0) < 1.0 and q.size:
                q = q[:int(np.ceil(q.size * cfg["stage_budget_frac"]))]
            plan["queues"][g] = q
            plan["hot_seeds"][g] = derive_seed(cfg["seed"], HOT_TAG, epoch, g)
    return plan


# ---------------------------------------------------------------------------
# f1: hotness — hotness.py:28-108
# ---------------------------------------------------------------------------

def estimate_hotness(graph, train_set, fanouts, rounds, seed, batch_size=None):
    """hotness.py:70-100; returns (counts, rank)."""
    train_set = np.asarray(train_set, np.int64)
    bs = batch_size or train_set.shape[0]
    counts = np.zeros(graph.num_vertices, np.int64)
    for r in range(rounds):
        g = np.random.Generator(np.random.Philox(key=derive_seed(seed, PRESAMPLE_TAG, r)))
        order = train_set[g.permutation(train_set.shape[0])]
        for b, s in enumerate(range(0, order.shape[0], bs)):
            st = sample_khop(graph, order[s:s + bs], fanouts,
                             derive_seed(seed, PRESAMPLE_TAG, r, b))
            count_into(counts, st.blocks[0].src_vertices)
    rank = np.lexsort((np.arange(counts.shape[0]), -counts)).astype(np.int64)  # hotness.py:35-41
    return counts, rank


def select_hot(rank, ratio):
    """hotness.py:103-108."""
    return rank[:int(ratio * rank.shape[0])].copy()


# ---------------------------------------------------------------------------
# S2/S3/S5 + E1: training loop (serial; simulate_costs=False) —
# orchestrator.py:236-271, 330-618, 662-725
# ---------------------------------------------------------------------------

def full_graph_block(graph):
    """orchestrator.py:662-666."""
    ids = np.arange(graph.num_vertices, dtype=np.int64)
    return Block(dst_vertices=ids, src_vertices=ids, edge_src=graph.targets.astype(np.int64),
                 edge_dst=np.repeat(ids, graph.degrees))


def evaluate(graph, data, model, weights):
    """orchestrator.py:669-680: full-neighbour inference accuracy."""
    blk = full_graph_block(graph)
    h = data.features
    for l in range(len(weights)):
        h, _ = layer_forward(model, blk, h, weights[l], l < len(weights) - 1)
    pred = h.argmax(axis=1)
    out = {}
    for name, m in (("val", data.val_mask), ("test", data.test_mask)):
        out[name] = float((pred[m] == data.labels[m]).mean()) if m.any() else 0.0
    return out, h


DEFAULT_CFG = dict(model="gcn", layers=3, fanouts=(25, 10, 5), hidden_dim=64, batch_size=1024,
                   super_batch_n=4, hot_ratio=0.2, strategy="layer-based", lr=0.1, epochs=1,
                   seed=0, optimizer="sgd", presample_rounds=20, stage_budget_frac=1.0,
                   max_fallback_frac=0.5)


def train_batch(cfg, data, weights, stack, labels, inject, adam):
    """orchestrator.py:236-256: gather -> fwd -> CE -> bwd -> update -> max|dw|."""
    inputs = data.features[stack.blocks[0].src_vertices]
    logits, caches = forward_batch(cfg["model"], stack, inputs, weights, inject)
    loss, dl = loss_and_grad(logits, labels)
    grads = backward_batch(cfg["model"], caches, dl, weights)
    old = [[w.copy() for w in lw] for lw in weights]
    if cfg["optimizer"] == "sgd":
        sgd_step(weights, grads, cfg["lr"])
    else:
        adam.step(weights, grads, cfg["lr"])
    md = max(float(np.max(np.abs(wn - wo))) if wo.size else 0.0
             for lo, ln in zip(old, weights) for wo, wn in zip(lo, ln))
    return loss, md, logits


def run_training(graph, data, cfg=None, hot_list=None, evaluate_each_epoch=True):
    """orchestrator.py:683-725 with _run_epoch :330-618 (serial execution,
    simulate_costs=False => partition_hot keeps every queued vertex in
    cpu_compute, hotness.py:129).  Returns a list of per-epoch dicts."""
    cfg = dict(DEFAULT_CFG, **(cfg or {}))
    fan = tuple(cfg["fanouts"])
    cfg["fanouts"] = fan
    dims = [data.feat_dim] + [cfg["hidden_dim"]] * (cfg["layers"] - 1) + [data.num_classes]
    weights = init_params(cfg["model"], dims, cfg["seed"])
    layer_based = cfg["strategy"] == "layer-based"
    if hot_list is None:
        hot_list = np.empty(0, np.int64)
        if layer_based and cfg["hot_ratio"] > 0 and cfg["layers"] > 1:
            train_ids = np.nonzero(data.train_mask)[0].astype(np.int64)
            _, rank = estimate_hotness(graph, train_ids, fan, cfg["presample_rounds"],
                                       cfg["seed"], cfg["batch_size"])
            hot_list = select_hot(rank, cfg["hot_ratio"])
    emb_dim = cfg["hidden_dim"] if cfg["layers"] > 1 else data.num_classes
    store = Store(cfg["super_batch_n"], emb_dim) if layer_based else None
    adam = Adam()
    version = 0
    first = 0
    reports = []
    hot_global = set(hot_list.tolist())
    for epoch in range(cfg["epochs"]):
        plan = build_epoch_plan(graph, data, cfg, hot_list, epoch, first)
        rep = dict(epoch=epoch, losses=[], max_deltas=[], rows=[], stage_events=[],
                   warmup_computed=0, epsilon=[])
        if store is not None:
            store.reset_epoch(first)
        for g, group in enumerate(plan["groups"]):
            q_next = plan["queues"].get(g + 1)
            staged = q_next if (layer_based and q_next is not None and q_next.size) \
                else np.empty(0, np.int64)
            cpu_set = set(plan["queues"].get(g, np.empty(0, np.int64)).tolist()) \
                if layer_based else set()
            for j, b in enumerate(group):
                gb = first + b
                seeds = plan["batches"][b]
                stack = sample_khop(graph, seeds, fan, plan["seeds"][b])
                if staged.size:  # serial producer, orchestrator.py:471-478
                    lo, hi = chunk_bounds(staged.size, len(group))[j]
                    if hi > lo:
                        blk = sample_one_hop_hot(graph, staged[lo:hi], fan[0],
                                                 plan["hot_seeds"][g + 1], 0)
                        emb, _ = layer_forward(cfg["model"], blk,
                                               data.features[blk.src_vertices],
                                               [w.copy() for w in weights[0]],
                                               cfg["layers"] > 1)
                        for row, v in enumerate(blk.dst_vertices.tolist()):
                            store.put(v, emb[row], version, g + 1)
                        rep["stage_events"].append((g + 1, version, int(blk.n_dst)))
                idx, vals, fb = [], [], 0
                bdst = stack.blocks[0].dst_vertices
                if layer_based and cfg["layers"] > 1 and cpu_set and g > 0:
                    for i, v in enumerate(bdst.tolist()):
                        if v in cpu_set:
                            e = store.get(v, gb)
                            if e is None:
                                fb += 1
                            else:
                                idx.append(i)
                                vals.append(e)
                elif layer_based and g == 0 and hot_global:
                    rep["warmup_computed"] += sum(1 for v in bdst.tolist() if v in hot_global)
                inject = (np.array(idx, np.int64), np.stack(vals)) if idx else None
                loss, md, _ = train_batch(cfg, data, weights, stack, data.labels[seeds],
                                          inject, adam)
                version += 1
                rep["losses"].append(loss)
                rep["max_deltas"].append(md)
                rep["rows"].append(dict(batch=gb, super_batch=g, loss=loss, reuse_hits=len(idx),
                                        fallbacks=fb))
            rep["epsilon"].append(max(rep["max_deltas"][-len(group):]) * 2 * cfg["super_batch_n"])
            if store is not None and g + 1 < len(plan["groups"]):
                store.advance(first + plan["groups"][g + 1][0], len(plan["groups"][g + 1]))
        hits = sum(r["reuse_hits"] for r in rep["rows"])
        fbs = sum(r["fallbacks"] for r in rep["rows"])
        if hits + fbs > 0 and fbs / (hits + fbs) > cfg["max_fallback_frac"]:
            raise RuntimeError("fallback budget exceeded")
        if store is not None:
            rep["max_gap"], rep["max_gap_batch"] = store.max_gap, store.max_gap_batch
        if evaluate_each_epoch:
            accs, _ = evaluate(graph, data, cfg["model"], weights)
            rep["val_accuracy"], rep["test_accuracy"] = accs["val"], accs["test"]
        reports.append(rep)
        first += len(plan["batches"])
    return reports, weights, hot_list
