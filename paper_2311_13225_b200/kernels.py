"""The reference's operator plug-in surface (hetgnn/kernels.py) on sm_100a.

Same function names, argument meaning and return shapes as the reference
(kernels.py:42-180); numpy in, numpy out.  Inside, every call runs one of the
library's CUDA kernels (include/hg_gnn.h) — there is no CPU fallback: without
a CUDA device or the built library these raise ``BackendUnavailable``.

The numpy-shaped entry points exist for drop-in use and parity tests; the
training engine keeps everything device-resident and calls the C ABI directly.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .device import ptr, require_cuda, stream_ptr, u64_tensor

_GOLDEN = 0x9E3779B97F4A7C15


def backend_name() -> str:
    """kernels.py:42-44 reports "numba"/"numpy"; this backend is "cuda"."""
    return "cuda"


def _mix64(x) -> int:
    """kernels.py:51-55 (host side of the library)."""
    return int(_lib.fn("hg_mix64_host")(int(x) & 0xFFFFFFFFFFFFFFFF))


def derive_seed(seed: int, *parts: int) -> int:
    """kernels.py:61-70."""
    arr = (ctypes.c_uint64 * max(len(parts), 1))(*[int(p) & 0xFFFFFFFFFFFFFFFF for p in parts])
    return int(_lib.fn("hg_derive_seed")(int(seed) & 0xFFFFFFFFFFFFFFFF, arr, len(parts)))


def sample_layer(offsets, targets, dst_globals, fanout, stream_seed):
    """kernels.py:147-158: (edge_dst_local, edge_src_global) in emission order."""
    from .device import DeviceGraph
    from .graph import Graph
    from .sampler import as_device_graph
    dg = offsets if isinstance(offsets, DeviceGraph) else as_device_graph(
        Graph(offsets=np.asarray(offsets, np.int64), targets=np.asarray(targets)))
    dev = dg.device
    dst = np.asarray(dst_globals, dtype=np.int64)
    n = int(dst.shape[0])
    f = int(fanout)
    if n == 0:
        return np.empty(0, np.int64), np.empty(0, np.int64)
    z = lambda k: torch.zeros(max(int(k), 1), dtype=torch.int32, device=dev)  # noqa: E731
    fr = torch.as_tensor(dst.astype(np.int32), device=dev)
    counts, slots = z(n), z(n * f)
    scratch = z(n * 2 * f) if f > 32 else None
    seed = u64_tensor(stream_seed, dev)
    s = stream_ptr()
    _lib.call("hg_sample_layer", ptr(dg.offsets), ptr(dg.targets), ptr(fr), None, n, f, ptr(seed), -1,
              ptr(counts), ptr(slots), ptr(dg.minpos.table), ptr(dg.minpos.tag), ptr(scratch), s)
    # this call does not dedup: retire the first-occurrence tag
    _lib.call("hg_first_occurrence_advance", ptr(dg.minpos.tag), s)
    ed, es, ne = z(n * f), z(n * f), z(1)
    ws = z(_lib.fn("hg_block_edges_ws_size")(n))
    _lib.call("hg_raw_edges", None, n, f, ptr(counts), ptr(slots), ptr(ed), ptr(es), ptr(ne), ptr(ws), s)
    k = int(ne.item())
    return ed[:k].cpu().numpy().astype(np.int64), es[:k].cpu().numpy().astype(np.int64)


def stable_unique(values):
    """kernels.py:166-180: first-occurrence dedup; uniq[inverse] == values."""
    dev = require_cuda()
    v = np.ascontiguousarray(np.asarray(values).reshape(-1), dtype=np.int64)
    n = v.shape[0]
    if n == 0:
        return v.copy(), np.empty(0, np.int64)
    dv = torch.as_tensor(v, device=dev)
    uniq = torch.empty(n, dtype=torch.int64, device=dev)
    inv = torch.empty(n, dtype=torch.int64, device=dev)
    nu = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(int(_lib.fn("hg_unique_ws_size")(n)), dtype=torch.int32, device=dev)
    _lib.call("hg_unique_first_i64", ptr(dv), n, ptr(uniq), ptr(inv), ptr(nu), ptr(ws), stream_ptr())
    k = int(nu.item())
    return uniq[:k].cpu().numpy().astype(np.asarray(values).dtype), inv.cpu().numpy()


def count_into(counter: np.ndarray, ids: np.ndarray) -> None:
    """kernels.py:161-163: counter[v] += 1 for every v in ids (in place)."""
    dev = require_cuda()
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    if ids.size == 0:
        return
    if isinstance(counter, torch.Tensor):
        _lib.call("hg_count_into_i64", ptr(counter), ptr(torch.as_tensor(ids, device=counter.device)), ids.size,
                  stream_ptr())
        return
    dc = torch.as_tensor(np.ascontiguousarray(counter, dtype=np.int64), device=dev)
    _lib.call("hg_count_into_i64", ptr(dc), ptr(torch.as_tensor(ids, device=dev)), ids.size, stream_ptr())
    counter[...] = dc.cpu().numpy().astype(counter.dtype)


def segment_weighted_rows(edge_src, edge_dst, weights, rows, n_out):
    """kernels.py:121-144: out[d] += w*rows[s] in edge order — fp64, bit-exact."""
    dev = require_cuda()
    rows = np.ascontiguousarray(rows, dtype=np.float64)
    es = np.ascontiguousarray(edge_src, dtype=np.int64)
    ed = np.ascontiguousarray(edge_dst, dtype=np.int64)
    w = np.ascontiguousarray(weights, dtype=np.float64)
    d = rows.shape[1]
    n_out = int(n_out)
    out = torch.zeros((max(n_out, 1), max(d, 1)), dtype=torch.float64, device=dev)
    if es.shape[0] and n_out and d:
        ws = torch.empty(int(_lib.fn("hg_swr_ws_size")(es.shape[0], n_out)), dtype=torch.int32, device=dev)
        t = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731
        des, ded, dw, dr = t(es), t(ed), t(w), t(rows)
        _lib.call("hg_segment_weighted_rows_f64", ptr(des), ptr(ded), ptr(dw), es.shape[0], ptr(dr), d, n_out,
                  ptr(out), ptr(ws), stream_ptr())
    return out[:n_out, :d].cpu().numpy()
