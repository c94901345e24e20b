"""Device plumbing: CUDA availability, raw pointers, HBM-resident graph.

torch is used only to own device memory and streams; every computation on
these buffers is one of the library's sm_100a kernels.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from ._lib import BackendUnavailable, load


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise BackendUnavailable("a CUDA device (B200, sm_100a) is required; there is no CPU fallback")
    load()
    dev = torch.device(device if device is not None else "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def ptr(t):
    """Raw device pointer of a tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def pad4(n: int) -> int:
    return (n + 3) // 4 * 4


def i32(x, device):
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.int32), device=device)


def i64(x, device):
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.int64), device=device)


def u64_tensor(values, device):
    """uint64 scalars stored bit-exactly in an int64 tensor (kernels read uint64_t*)."""
    arr = np.asarray([int(v) & 0xFFFFFFFFFFFFFFFF for v in np.atleast_1d(values)], dtype=np.uint64)
    return torch.as_tensor(arr.view(np.int64), device=device)


class FirstOccurrenceTable:
    """Dense per-vertex first-occurrence table of the dedup kernels.

    ``table`` holds uint64 keys ``(tag << 32) | position`` (all ~0 when
    allocated); ``tag`` is the device counter the relabel kernel bumps after
    each use, so stale keys always lose and the table is never reset.  Users
    that may run concurrently (different streams) need separate tables.
    """

    def __init__(self, num_vertices: int, device):
        self.table = torch.full((max(int(num_vertices), 1),), -1, dtype=torch.int64, device=device)
        self.tag = torch.zeros(1, dtype=torch.int32, device=device)

    def like(self):
        return FirstOccurrenceTable(self.table.numel(), self.table.device)

    def nbytes(self) -> int:
        return self.table.numel() * 8 + 4


class DeviceGraph:
    """HBM layout of one dataset (see graph.py docstring):
    offsets int64[V+1], targets int32[E], features fp32[V, F_pad], labels int32[V]."""

    def __init__(self, offsets, targets, features=None, labels=None, device=None):
        self.device = require_cuda(device)
        offsets = np.asarray(offsets)
        targets = np.asarray(targets)
        self.num_vertices = int(offsets.shape[0] - 1)
        self.num_edges = int(targets.shape[0])
        if self.num_vertices >= 2**31 - 1:
            raise ValueError("vertex ids must fit int32")
        self.offsets = i64(offsets, self.device)
        self.targets = i32(targets, self.device)
        self.feat_dim = 0
        self.feat_ld = 0
        self.features = None
        if features is not None:
            feats = np.asarray(features)
            V, F = feats.shape
            self.feat_dim = F
            # row stride: multiple of HG_FEAT_ALIGN floats.  Default: 4 (16-byte rows for
            # float4 loads) up to 128 features — narrower rows get the split-row copy
            # (split_rows) — and 32 (whole 128-byte lines) for wider rows: C3's 602
            # features as 608 floats touch 19 lines per row instead of 19.75 on average,
            # bottom aggregation 74.8 -> 73.4 us, step 259.5 -> 255.8 us
            # (profiles/r02t_c3_align.txt); the GEMMs pad K to 32 anyway.
            align = max(4, int(os.environ.get("HG_FEAT_ALIGN", "32" if F > 128 else "4")))
            self.feat_ld = (F + align - 1) // align * align
            x = torch.zeros((V, self.feat_ld), dtype=torch.float32, device=self.device)
            x[:, :F] = torch.as_tensor(np.ascontiguousarray(feats, dtype=np.float32), device=self.device)
            self.features = x
        self.labels = None if labels is None else i32(labels, self.device)
        # first-occurrence table for the dedup kernel (shared by sequential users)
        self.minpos = FirstOccurrenceTable(self.num_vertices, self.device)

    def persist_hot_rows(self, max_bytes: int | None = None, hit_ratio: float | None = None) -> int:
        """Pin the hottest contiguous block of feature rows in L2 (persisting
        access-policy window on the feature-gathering kernels).  Rows are chosen
        as the window of consecutive ids with the largest degree sum (sampled
        neighbours are drawn roughly in proportion to degree; the generators put
        hubs at low ids, graph.py:357).  Size: ``max_bytes`` or env
        HG_L2_PERSIST_MB (default 48 MB; 0/16/32/48/64/80 MB measured, §5), clamped to the device's persisting-L2
        limit; 0 disables.  Returns the window size in bytes."""
        from . import _lib
        lib = _lib.load()
        if self.features is None:
            return 0
        if max_bytes is None:
            max_bytes = int(float(os.environ.get("HG_L2_PERSIST_MB", "48")) * 2**20)
        if hit_ratio is None:  # fraction of the window's lines given the persisting property
            hit_ratio = float(os.environ.get("HG_L2_HIT", "1.0"))
        sp = self.split_rows()
        if sp is not None:  # window over [tail table | first body rows] (hubs at low ids, graph.py:357)
            nbytes = min(int(max_bytes), int(lib.hg_l2_persist_max()), sp["buf"].numel() * 4)
            if nbytes <= 0:
                _lib.call("hg_set_l2_persist", None, 0, 0.0)
                return 0
            hub_rows = max(0, nbytes - sp["tail_bytes"]) // (sp["body_cols"] * 4)
            self.l2_window = (0, hub_rows)
            _lib.call("hg_set_l2_persist", sp["buf"].data_ptr(), nbytes, float(hit_ratio))
            return nbytes
        row = self.feat_ld * 4
        nbytes = min(int(max_bytes), int(lib.hg_l2_persist_max()), self.num_vertices * row)
        rows = nbytes // row
        if rows <= 0:
            _lib.call("hg_set_l2_persist", None, 0, 0.0)
            return 0
        deg = torch.diff(self.offsets)
        cs = torch.cumsum(torch.nn.functional.pad(deg, (1, 0)), 0)
        start = int(torch.argmax(cs[rows:] - cs[:-rows]).item()) if rows < self.num_vertices else 0
        self.l2_window = (start, rows)
        _lib.call("hg_set_l2_persist", self.features[start].data_ptr(), rows * row, float(hit_ratio))
        return rows * row

    def split_rows(self):
        """Split-row copy of the feature table for the bottom gather
        (``hg_aggregate_fwd_split``), or None when it does not apply.

        A row of F_pad floats whose size is not a multiple of 128 bytes touches
        ceil-plus-one 128-byte lines (400-byte C2 rows: always 4), and the random
        gather's DRAM cost is per line touched (profiles/r02s_gather_rowsize.txt).
        The copy keeps columns [0, 32*floor(F_pad/32)) as whole lines of a body
        table and the last F_pad mod 32 (<= 8) columns in a tail table
        (V x 16 B for C2: 38 MB) placed in front of the body in one allocation, so
        the persisting L2 window covers the whole tail table plus the first (hub)
        body rows.  Off with HG_SPLIT_ROWS=0; never used for row-sharded tables, nor when
        the copy would take more than half of the free HBM (the plain table is then read)."""
        if hasattr(self, "_split"):
            return self._split
        self._split = None
        x = self.features
        if x is None or os.environ.get("HG_SPLIT_ROWS", "1") == "0" or getattr(self, "shards", None) is not None:
            return None
        V, ld = x.shape
        body_cols = ld // 32 * 32
        tail_cols = ld - body_cols
        if ld > 128 or body_cols == 0 or tail_cols == 0 or tail_cols > 8:
            return None
        tail_elems = (V * tail_cols + 31) // 32 * 32  # body starts 128-byte aligned
        need = (tail_elems + V * body_cols) * 4
        free, _ = torch.cuda.mem_get_info(self.device)
        if need > free // 2:  # a second copy of the table only while it leaves HBM to spare
            return None
        buf = torch.empty(tail_elems + V * body_cols, dtype=torch.float32, device=self.device)
        tail = buf[:V * tail_cols].view(V, tail_cols)
        body = buf[tail_elems:].view(V, body_cols)
        tail.copy_(x[:, body_cols:])
        body.copy_(x[:, :body_cols])
        self._split = dict(buf=buf, body=body, tail=tail, body_cols=body_cols, tail_cols=tail_cols,
                           tail_bytes=tail_elems * 4)
        return self._split

    @classmethod
    def from_dataset(cls, ds, device=None):
        return cls(ds.offsets, ds.targets, ds.features, ds.labels, device=device)

    def nbytes(self) -> int:
        n = self.offsets.numel() * 8 + self.targets.numel() * 4 + self.minpos.nbytes()
        if self.features is not None:
            n += self.features.numel() * 4
        if getattr(self, "_split", None) is not None:
            n += self._split["buf"].numel() * 4
        if self.labels is not None:
            n += self.labels.numel() * 4
        return n
