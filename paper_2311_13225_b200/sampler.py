"""Fanout-bounded k-hop block sampling on the GPU (reference sampler.py:1-180).

Two faces:

* ``LayerSampler`` — the device-resident, graph-capturable block builder the
  training engine uses (frontier and counts stay in HBM; capacities are
  static upper bounds n_src <= n_dst * (f + 1)).
* ``sample_khop`` / ``sample_khop_skip_hot`` / ``sample_one_hop_hot`` — the
  reference's public API returning numpy ``Block``s, for drop-in use and the
  parity tests (one host sync per layer to size the next one exactly).
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .device import DeviceGraph, ptr, stream_ptr, u64_tensor
from .seeds import derive_seed

SAMPLE_TAG = 0x5A  # sampler.py:19


class SamplerError(ValueError):
    """sampler.py:22-23."""


@dataclass(frozen=True)
class Fanouts:
    """Per-layer neighbour caps, bottom layer first (sampler.py:26-42)."""

    counts: tuple

    def __post_init__(self):
        if not self.counts:
            raise SamplerError("fanouts must not be empty")
        if any(int(c) < 1 for c in self.counts):
            raise SamplerError(f"fanouts must all be >= 1, got {self.counts}")

    def __len__(self):
        return len(self.counts)

    def __getitem__(self, i):
        return self.counts[i]


@dataclass
class Block:
    """sampler.py:45-78: src_vertices starts with dst_vertices; edges sorted by (dst, src)."""

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

    def edge_src_global(self):
        return self.src_vertices[self.edge_src]

    def edge_dst_global(self):
        return self.dst_vertices[self.edge_dst]

    def sampled_in_degree(self):
        return np.bincount(self.edge_dst, minlength=self.n_dst).astype(np.int64)


@dataclass
class SampledBlockStack:
    """sampler.py:81-101."""

    blocks: list
    seeds: np.ndarray
    hot_flags: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.hot_flags is None:
            self.hot_flags = np.zeros(self.blocks[0].n_src, dtype=bool)

    @property
    def num_layers(self):
        return len(self.blocks)

    def bottom_src(self):
        return self.blocks[0].src_vertices

    def total_sampled_edges(self):
        return sum(b.n_edges for b in self.blocks)


def _as_stream(stream, device):
    return stream if stream is not None else torch.cuda.current_stream(device)


class LayerSampler:
    """Workspace + launches for one layer's block (draw -> dedup -> order).

    Buffers (int32): counts[cap_dst], slots/slot_local[cap_dst*f] (slot form),
    src[cap_src] with device count n_src; nself[cap_dst] (SAGE), outdeg[cap_src]
    (GCN; layers >= 1: the backward scatter's per-source edge counts).
    """

    def __init__(self, dg: DeviceGraph, cap_dst: int, fanout: int, need_nself=True, need_outdeg=False,
                 minpos=None):
        lib = _lib.load()
        dev = dg.device
        self.dg, self.f, self.cap_dst = dg, int(fanout), int(cap_dst)
        # first-occurrence table (device.FirstOccurrenceTable); samplers that may
        # run concurrently on different streams need their own
        self.minpos = dg.minpos if minpos is None else minpos
        self.cap_src = int(min(dg.num_vertices, self.cap_dst * (self.f + 1)))
        z = lambda n: torch.zeros(max(int(n), 1), dtype=torch.int32, device=dev)  # noqa: E731
        self.counts = z(cap_dst)
        self.slots = z(cap_dst * self.f)
        self.slot_local = z(cap_dst * self.f)
        self.src = z(self.cap_src)
        self.n_src = z(1)
        self.nself = z(cap_dst) if need_nself else None
        self.outdeg = z(self.cap_src) if need_outdeg else None
        self.ws = z(lib.hg_dedup_ws_size(self.cap_dst, self.f))
        self.scratch = z(cap_dst * 2 * self.f) if self.f > 32 else None

    def run(self, frontier, d_n_dst, d_seed, layer: int, stream=None, cap_dst: int | None = None,
            dedup: bool = True, relabel_stream=None):
        """Enqueue the block build for `frontier` (device int32, count *d_n_dst).
        ``relabel_stream``: the
        relabel half (segment order, slot_local, nself, outdeg) runs there after
        the draw + mark half on ``stream``; src / n_src are ready on ``stream``,
        the rest once ``relabel_stream`` is joined.  The next layer's sampler on
        ``stream`` must then use a different first-occurrence table."""
        cap = self.cap_dst if cap_dst is None else int(cap_dst)
        assert cap <= self.cap_dst
        if cap != self.cap_dst:
            # the dedup workspace (decoupled look-back status + generation counter)
            # is laid out for the sampler's static capacity: a smaller call keeps
            # that layout and passes its size as a device count instead
            if d_n_dst is not None:
                raise ValueError("cap_dst override needs d_n_dst=None (the count is the override)")
            if not hasattr(self, "_n_override"):
                self._n_override = torch.zeros(1, dtype=torch.int32, device=self.dg.device)
            with torch.cuda.stream(_as_stream(stream, self.dg.device)):
                self._n_override.fill_(cap)
            d_n_dst, cap = self._n_override, self.cap_dst
        cap_src = min(self.cap_src, self.dg.num_vertices, cap * (self.f + 1))
        s = stream_ptr(stream)
        g = self.dg
        if not dedup:  # draws + non-self counts only (sources consumed by global id)
            if self.nself is None:
                raise ValueError("draws-only sampling produces SAGE non-self counts: need_nself=True")
            _lib.call("hg_sample_layer_draws", ptr(g.offsets), ptr(g.targets), ptr(frontier), ptr(d_n_dst), cap,
                      self.f, ptr(d_seed), int(layer), ptr(self.counts), ptr(self.slots), ptr(self.nself),
                      ptr(self.scratch), s)
            return self
        if relabel_stream is not None:
            _lib.call("hg_sample_block_mark", ptr(g.offsets), ptr(g.targets), ptr(frontier), ptr(d_n_dst), cap,
                      self.f, ptr(d_seed), int(layer), ptr(self.counts), ptr(self.slots), ptr(self.minpos.table),
                      ptr(self.minpos.tag), ptr(self.src), ptr(self.n_src), ptr(self.outdeg), ptr(self.ws),
                      ptr(self.scratch), s)
            relabel_stream.wait_stream(_as_stream(stream, g.device))
            _lib.call("hg_block_relabel", ptr(frontier), ptr(d_n_dst), cap, self.f, ptr(self.counts),
                      ptr(self.slots), ptr(self.slot_local), ptr(self.minpos.table), ptr(self.minpos.tag),
                      ptr(self.nself), ptr(self.outdeg), ptr(self.ws), relabel_stream.cuda_stream)
            return self
        # draw + dedup + relabel
        _lib.call("hg_sample_block", ptr(g.offsets), ptr(g.targets), ptr(frontier), ptr(d_n_dst), cap, self.f,
                  ptr(d_seed), int(layer), ptr(self.counts), ptr(self.slots), ptr(self.slot_local),
                  ptr(self.minpos.table), ptr(self.minpos.tag), ptr(self.src), ptr(self.n_src), cap_src,
                  ptr(self.nself), ptr(self.outdeg), ptr(self.ws), ptr(self.scratch), s)
        return self

    # -- host views (sync) ---------------------------------------------------
    def to_block(self, frontier_np: np.ndarray, stream=None) -> Block:
        n_dst = int(frontier_np.shape[0])
        dev = self.dg.device
        lib = _lib.load()
        es = torch.zeros(max(n_dst * self.f, 1), dtype=torch.int32, device=dev)
        ed = torch.zeros_like(es)
        ne = torch.zeros(1, dtype=torch.int32, device=dev)
        ws = torch.zeros(max(int(lib.hg_block_edges_ws_size(n_dst)), 1), dtype=torch.int32, device=dev)
        _lib.call("hg_block_to_edges", None, n_dst, self.f, ptr(self.counts), ptr(self.slot_local), ptr(es),
                  ptr(ed), ptr(ne), ptr(ws), stream_ptr(stream))
        n_src = int(self.n_src.item())
        n_e = int(ne.item())
        return Block(dst_vertices=np.asarray(frontier_np, np.int64),
                     src_vertices=self.src[:n_src].cpu().numpy().astype(np.int64),
                     edge_src=es[:n_e].cpu().numpy().astype(np.int64),
                     edge_dst=ed[:n_e].cpu().numpy().astype(np.int64))


# ---------------------------------------------------------------------------
# reference-shaped API
# ---------------------------------------------------------------------------

_DG_CACHE: dict = {}


def as_device_graph(graph) -> DeviceGraph:
    """DeviceGraph for a reference-style Graph/Dataset (cached per offsets array)."""
    if isinstance(graph, DeviceGraph):
        return graph
    key = id(graph.offsets)
    hit = _DG_CACHE.get(key)
    if hit is not None and hit[0]() is graph.offsets:
        return hit[1]
    dg = DeviceGraph(graph.offsets, graph.targets)
    try:
        ref = weakref.ref(graph.offsets)
    except TypeError:
        ref = (lambda o=graph.offsets: o)
    _DG_CACHE[key] = (ref, dg)
    return dg


def _check_seeds(num_vertices, seeds):
    """sampler.py:121-127."""
    seeds = np.asarray(seeds, dtype=np.int64)
    if seeds.size == 0:
        raise SamplerError("seeds must not be empty")
    if seeds.min() < 0 or seeds.max() >= num_vertices:
        raise SamplerError("seed vertex id out of range")
    return seeds


def _expand(dg, frontier_np, fanout, stream_seed):
    dev = dg.device
    fr = torch.as_tensor(frontier_np.astype(np.int32), device=dev)
    n = torch.tensor([fr.numel()], dtype=torch.int32, device=dev)
    seed = u64_tensor(stream_seed, dev)
    ls = LayerSampler(dg, fr.numel(), fanout, need_nself=False, need_outdeg=False)
    ls.run(fr, n, seed, layer=-1)
    return ls.to_block(frontier_np)


def sample_khop(graph, seeds, fanouts, rng_seed: int) -> SampledBlockStack:
    """sampler.py:130-147 on the GPU; bit-identical blocks."""
    dg = as_device_graph(graph)
    if not isinstance(fanouts, Fanouts):
        fanouts = Fanouts(tuple(fanouts))
    seeds = _check_seeds(dg.num_vertices, seeds)
    blocks = [None] * len(fanouts)
    frontier = seeds
    for layer in range(len(fanouts) - 1, -1, -1):
        blk = _expand(dg, frontier, fanouts[layer], derive_seed(rng_seed, SAMPLE_TAG, layer))
        blocks[layer] = blk
        frontier = blk.src_vertices
    return SampledBlockStack(blocks=blocks, seeds=seeds)


def sample_khop_skip_hot(graph, seeds, fanouts, hot_set, rng_seed: int) -> SampledBlockStack:
    """sampler.py:150-163: identical topology, bottom-frontier hot flags."""
    stack = sample_khop(graph, seeds, fanouts, rng_seed)
    hot = np.asarray(list(hot_set) if isinstance(hot_set, set) else hot_set, dtype=np.int64)
    if hot.size:
        stack.hot_flags = hot_flags(as_device_graph(graph), stack.blocks[0].src_vertices, hot)
    return stack


def hot_flags(dg: DeviceGraph, values: np.ndarray, hot: np.ndarray) -> np.ndarray:
    """np.isin(values, hot) on the device (sampler.py:161-162): tag the hot ids in
    a vertex-indexed table, then one flag per value (hg_member_flags)."""
    dev = dg.device
    hot = hot[(hot >= 0) & (hot < dg.num_vertices)]  # ids outside the graph match nothing (np.isin)
    tag_of = torch.full((dg.num_vertices,), -1, dtype=torch.int32, device=dev)
    h = torch.as_tensor(hot.astype(np.int32), device=dev)
    v = torch.as_tensor(np.asarray(values).astype(np.int32), device=dev)
    flags = torch.zeros(max(v.numel(), 1), dtype=torch.uint8, device=dev)
    s = stream_ptr()
    _lib.call("hg_tag_vertices", ptr(h), None, h.numel(), ptr(tag_of), 1, s)
    _lib.call("hg_member_flags", ptr(v), None, v.numel(), ptr(tag_of), 1, ptr(flags), s)
    return flags[:v.numel()].cpu().numpy().astype(bool)


def sample_one_hop_hot(graph, hot_vertices, fanout: int, rng_seed: int, layer: int = 0) -> Block:
    """sampler.py:166-180."""
    dg = as_device_graph(graph)
    hot = np.asarray(hot_vertices, dtype=np.int64)
    if hot.size == 0:
        raise SamplerError("hot vertex list must not be empty")
    if np.unique(hot).shape[0] != hot.shape[0]:
        raise SamplerError("hot vertex list must be deduplicated")
    hot = hot[(hot >= 0) & (hot < dg.num_vertices)]  # ids outside the graph match nothing (np.isin)
    return _expand(dg, hot, fanout, derive_seed(rng_seed, SAMPLE_TAG, layer))
