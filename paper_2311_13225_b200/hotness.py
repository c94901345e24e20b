"""Pre-sampling hotness estimation on the GPU (reference hotness.py:1-136).

``estimate_hotness`` replays R sampling epochs with the production sampler
(K1-K3) and counts bottom-frontier occurrences with device atomics
(count_into, kernels.py:161-163); the ranking "count desc, id asc"
(hotness.py:35-41) is a stable radix sort of (max - count) over ids in
ascending order.  The whole pre-pass is one captured graph replayed per batch.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .device import DeviceGraph, ptr, stream_ptr
from .seeds import derive_seed

PRESAMPLE_TAG = 0x70  # hotness.py:19
REAL_SIZE = 8


class HotnessError(ValueError):
    """hotness.py:23-24."""


@dataclass
class HotnessTable:
    """hotness.py:27-41."""

    counts: np.ndarray
    rounds: int
    rank: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.rank is None:
            self.rank = np.lexsort((np.arange(self.counts.shape[0]), -self.counts)).astype(np.int64)


@dataclass
class FeedbackSnapshot:
    """hotness.py:44-49."""

    observed_fast_idle_time: float
    free_fast_memory: float


@dataclass
class HotSetPartition:
    """hotness.py:52-67."""

    cpu_compute: np.ndarray
    gpu_cache: np.ndarray
    hot_ratio: float = 0.0

    def cache_set(self) -> set:
        return set(int(v) for v in self.gpu_cache)

    def compute_set(self) -> set:
        return set(int(v) for v in self.cpu_compute)

    def gpu_cache_bytes(self, feat_dim: int) -> int:
        return self.gpu_cache.shape[0] * feat_dim * REAL_SIZE


def _device_rank(counts_dev: torch.Tensor) -> np.ndarray:
    """Stable radix sort of ids by (max - count): count desc, id asc."""
    V = counts_dev.numel()
    mx = int(counts_dev.max().item()) if V else 0
    keys = (mx - counts_dev).to(torch.int32).contiguous()
    vals = torch.arange(V, dtype=torch.int32, device=counts_dev.device)
    k_alt = torch.empty_like(keys)
    v_alt = torch.empty_like(vals)
    ws = torch.empty(int(_lib.fn("hg_radix_ws_size")(V)), dtype=torch.int32, device=counts_dev.device)
    bits = max(1, int(mx).bit_length())
    import ctypes
    flag = ctypes.c_int32(0)
    _lib.call("hg_radix_sort_pairs", ptr(keys), ptr(vals), ptr(k_alt), ptr(v_alt), V, bits, ptr(ws),
              ctypes.addressof(flag), stream_ptr())
    out = v_alt if flag.value else vals
    return out.cpu().numpy().astype(np.int64)


def estimate_hotness(graph, train_set, fanouts, rounds: int, seed: int, batch_size: int | None = None,
                     engine=None) -> HotnessTable:
    """hotness.py:70-100 on the device.  ``graph`` may be a DeviceGraph or a
    host Graph/Dataset; ``engine`` (optional) lends its samplers."""
    from .sampler import Fanouts, as_device_graph
    if rounds < 1:
        raise HotnessError(f"presample rounds must be >= 1, got {rounds}")
    train_set = np.asarray(train_set, dtype=np.int64)
    if train_set.size == 0:
        raise HotnessError("train set must not be empty")
    if not isinstance(fanouts, Fanouts):
        fanouts = Fanouts(tuple(fanouts))
    bs = int(batch_size or train_set.shape[0])
    dg = graph if isinstance(graph, DeviceGraph) else as_device_graph(graph)
    sampler = engine if engine is not None else _SampleOnly(dg, list(fanouts.counts), bs)
    counts = torch.zeros(dg.num_vertices, dtype=torch.int64, device=dg.device)
    runner = _CountRunner(sampler, counts)
    for r in range(rounds):
        gen = np.random.Generator(np.random.Philox(key=derive_seed(seed, PRESAMPLE_TAG, r)))
        order = train_set[gen.permutation(train_set.shape[0])]
        for b, start in enumerate(range(0, order.shape[0], bs)):
            runner.run(order[start:start + bs], derive_seed(seed, PRESAMPLE_TAG, r, b))
    torch.cuda.synchronize(dg.device)
    table = HotnessTable(counts=counts.cpu().numpy(), rounds=rounds, rank=_device_rank(counts))
    return table


def select_hot(table: HotnessTable, hot_ratio: float) -> np.ndarray:
    """hotness.py:103-108."""
    if not (0.0 <= hot_ratio <= 1.0):
        raise HotnessError(f"hot ratio must be in [0, 1], got {hot_ratio}")
    k = int(hot_ratio * table.rank.shape[0])
    return table.rank[:k].copy()


def partition_hot(hot_list, feedback: FeedbackSnapshot, feat_dim: int, emb_dim: int,
                  est_slow_time_per_vertex: float = 0.0) -> HotSetPartition:
    """hotness.py:111-136 (host worklist; with no measured idle time every hot
    vertex stays in the embedding-reuse set)."""
    hot = np.asarray(hot_list, dtype=np.int64)
    if hot.size == 0:
        return HotSetPartition(cpu_compute=hot.copy(), gpu_cache=hot.copy())
    row_bytes = feat_dim * REAL_SIZE
    idle, mem = float(feedback.observed_fast_idle_time), float(feedback.free_fast_memory)
    moved = 0
    while moved < hot.shape[0] and idle > 0.0 and mem >= row_bytes:
        moved += 1
        mem -= row_bytes
        idle -= est_slow_time_per_vertex
    return HotSetPartition(cpu_compute=hot[moved:].copy(), gpu_cache=hot[:moved].copy())


class _SampleOnly:
    """Just the k-hop samplers (used when no training engine exists yet)."""

    def __init__(self, dg, fan, bs):
        from .engine import BP_SIZE
        from .sampler import LayerSampler
        self.dg, self.fan, self.L, self.batch_cap = dg, fan, len(fan), bs
        self.cap_dst = [0] * self.L
        self.cap_dst[-1] = bs
        for l in range(self.L - 1, 0, -1):
            self.cap_dst[l - 1] = int(min(dg.num_vertices, self.cap_dst[l] * (fan[l] + 1)))
        self.samplers = [LayerSampler(dg, self.cap_dst[l], fan[l], need_nself=False) for l in range(self.L)]
        self.seeds = torch.zeros(bs, dtype=torch.int32, device=dg.device)
        self.counts_in = torch.zeros(2, dtype=torch.int32, device=dg.device)
        self.bp = torch.zeros(BP_SIZE, dtype=torch.int64, device=dg.device)

    def frontier(self, l):
        if l == self.L - 1:
            return self.seeds, self.counts_in[0:1]
        return self.samplers[l + 1].src, self.samplers[l + 1].n_src

    def enqueue_sample(self, stream=None, seed_ptr=None, layers=None):
        sp = self.bp if seed_ptr is None else seed_ptr
        for l in (range(self.L - 1, -1, -1) if layers is None else layers):
            fr, n = self.frontier(l)
            self.samplers[l].run(fr, n, sp, l, stream)


class _CountRunner:
    """Graph-captured "sample k hops + count bottom sources" per batch."""

    def __init__(self, smp, counts):
        self.smp, self.counts = smp, counts
        self.pin_seeds = torch.zeros(smp.batch_cap, dtype=torch.int32).pin_memory()
        self.pin_meta = torch.zeros(2, dtype=torch.int64).pin_memory()
        self.graph = None
        self.ev = None
        self.warmed = False

    def _body(self):
        smp = self.smp
        smp.enqueue_sample()
        s0 = smp.samplers[0]
        _lib.call("hg_count_into", ptr(self.counts), ptr(s0.src), ptr(s0.n_src), s0.cap_src, stream_ptr())

    def run(self, seeds, rng_seed):
        smp = self.smp
        if self.ev is not None:
            self.ev.synchronize()
        n = seeds.shape[0]
        self.pin_seeds.numpy()[:n] = seeds
        self.pin_meta.numpy()[0] = np.array([int(rng_seed) & 0xFFFFFFFFFFFFFFFF], np.uint64).view(np.int64)[0]
        smp.seeds[:n].copy_(self.pin_seeds[:n], non_blocking=True)
        smp.counts_in[0:1].fill_(n)
        smp.bp[0:1].copy_(self.pin_meta[0:1], non_blocking=True)
        if self.graph is None and n == smp.batch_cap and self.warmed:
            st = torch.cuda.Stream()
            st.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                self._body()
            torch.cuda.current_stream().wait_stream(st)
            self.graph = g
        if self.graph is not None:
            self.graph.replay()
        else:
            self._body()  # eager first batch doubles as the pre-capture warm-up
            self.warmed = True
        self.ev = torch.cuda.Event()
        self.ev.record()
