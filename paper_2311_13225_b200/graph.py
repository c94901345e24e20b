"""Graph data model and the HGNNBIN1 binary cache (reference graph.py:20-124, 375-418).

``Graph`` / ``VertexData`` keep the reference's host-side contract (int64 CSR
of incoming neighbours, read-only arrays; graph.py:33-124) and add
``DeviceGraph``: the HBM-resident copy the kernels read —

* ``offsets``  int64 [V+1]   (edge counts can exceed 2^31 for papers100M-shape)
* ``targets``  int32 [E]     (vertex ids < 2^31; halves the sampler's gather bytes)
* ``features`` fp32  [V, F_pad] row-major, F_pad = F rounded up to 4 so every
  row starts 16-byte aligned for 128-bit vector loads
* ``labels``   int32 [V]
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

_CACHE_MAGIC = b"HGNNBIN1"  # graph.py:20
_CACHE_VERSION = 1  # graph.py:21


class GraphFormatError(ValueError):
    """Malformed dataset input (graph.py:28-29)."""


@dataclass(frozen=True)
class Graph:
    """Immutable incoming-neighbour CSR (graph.py:33-77)."""

    offsets: np.ndarray
    targets: np.ndarray

    def __post_init__(self):
        if self.offsets.dtype != np.int64:
            raise GraphFormatError("CSR offsets must be int64")
        if self.offsets.shape[0] < 2:
            raise GraphFormatError("empty graph rejected: no vertices")
        if self.offsets[0] != 0 or self.offsets[-1] != self.targets.shape[0]:
            raise GraphFormatError("CSR offsets do not bracket the edge array")

    @property
    def num_vertices(self) -> int:
        return self.offsets.shape[0] - 1

    @property
    def num_edges(self) -> int:
        return self.targets.shape[0]

    @property
    def degrees(self) -> np.ndarray:
        return np.diff(self.offsets)

    def in_neighbors(self, v: int) -> np.ndarray:
        return self.targets[self.offsets[v]:self.offsets[v + 1]]


@dataclass(frozen=True)
class VertexData:
    """Per-vertex features, labels and masks (graph.py:81-124)."""

    features: np.ndarray
    labels: np.ndarray
    train_mask: np.ndarray
    val_mask: np.ndarray
    test_mask: np.ndarray

    @property
    def feat_dim(self) -> int:
        return self.features.shape[1]

    @property
    def num_classes(self) -> int:
        return int(self.labels.max()) + 1 if self.labels.size else 0


def split(ds) -> tuple[Graph, VertexData]:
    """A datagen.Dataset (or anything with the same fields) as (Graph, VertexData)."""
    return (Graph(offsets=ds.offsets, targets=ds.targets),
            VertexData(features=ds.features, labels=ds.labels, train_mask=ds.train_mask,
                       val_mask=ds.val_mask, test_mask=ds.test_mask))


def save_binary(path, ds) -> None:
    """Write the reference's HGNNBIN1 layout (graph.py:375-389): magic, version,
    array count, then per array (dtype str, ndim, shape, raw bytes).  CSR arrays
    are written as int64 so the reference's own ``load_binary`` accepts them."""
    arrays = [ds.offsets.astype(np.int64), ds.targets.astype(np.int64), ds.features,
              ds.labels.astype(np.int64), ds.train_mask, ds.val_mask, ds.test_mask]
    with open(path, "wb") as fh:
        fh.write(_CACHE_MAGIC)
        fh.write(struct.pack("<I", _CACHE_VERSION))
        fh.write(struct.pack("<I", len(arrays)))
        for arr in arrays:
            dt = arr.dtype.str.encode("ascii")
            fh.write(struct.pack("<I", len(dt)))
            fh.write(dt)
            fh.write(struct.pack("<I", arr.ndim))
            fh.write(struct.pack(f"<{arr.ndim}q", *arr.shape))
            fh.write(np.ascontiguousarray(arr).tobytes())


def load_binary(path, name: str = "hgnnbin"):
    """Read HGNNBIN1 (graph.py:392-418) into a datagen.Dataset (targets -> int32)."""
    from .datagen import Dataset
    with open(path, "rb") as fh:
        if fh.read(len(_CACHE_MAGIC)) != _CACHE_MAGIC:
            raise GraphFormatError(f"{path}: not a hetgnn binary cache (bad magic)")
        (version,) = struct.unpack("<I", fh.read(4))
        if version != _CACHE_VERSION:
            raise GraphFormatError(f"{path}: unsupported cache version {version}")
        (count,) = struct.unpack("<I", fh.read(4))
        arrays = []
        for _ in range(count):
            (dlen,) = struct.unpack("<I", fh.read(4))
            dt = np.dtype(fh.read(dlen).decode("ascii"))
            (ndim,) = struct.unpack("<I", fh.read(4))
            shape = struct.unpack(f"<{ndim}q", fh.read(8 * ndim))
            n = int(np.prod(shape)) if ndim else 1
            arrays.append(np.frombuffer(fh.read(n * dt.itemsize), dtype=dt).reshape(shape))
    offsets, targets, feats, labels, tr, va, te = arrays
    if targets.size and int(targets.max()) >= 2**31:
        raise GraphFormatError("vertex ids must fit int32 on device")
    return Dataset(name=name, offsets=offsets.astype(np.int64), targets=targets.astype(np.int32),
                   features=np.ascontiguousarray(feats), labels=labels.astype(np.int64),
                   train_mask=tr.astype(bool), val_mask=va.astype(bool),
                   test_mask=te.astype(bool), meta={"path": str(path)})


def load_reference_binary(path: str | Path):
    """Alias kept for symmetry with the reference's ``load_binary`` name."""
    return load_binary(path)
