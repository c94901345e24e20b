"""Seed-sharded data parallelism over NCCL (new — the reference
is single-process).

One process per GPU.  Each global batch is split into contiguous per-rank
shards; every rank samples its shard with the SAME batch rng seed, so (per-dst
RNG streams depend only on (stream, layer, vertex), kernels.py:105) every
vertex's draws equal the single-process draws.  Each rank's dlogits are
scaled by 1/|global batch| (hg_softmax_xent's d_div), so the sum of per-rank
gradients — one NCCL all-reduce of the flat gradient buffer, captured inside
the step's CUDA graph — equals the gradient of the union batch for SAGE
(GCN's block-local out-degree makes its sharded step differ, gnnmath.py:96).
"""

from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous split of n items, sizes within one (runplan.chunk_bounds rule)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard(seeds: np.ndarray, world: int, rank: int) -> np.ndarray:
    lo, hi = shard_bounds(seeds.shape[0], world, rank)
    return seeds[lo:hi]


class DistContext:
    """Rank/world plus the gradient all-reduce hook the engine calls."""

    def __init__(self, backend: str | None = None):
        if not dist.is_initialized():
            backend = backend or ("nccl" if torch.cuda.is_available() else "gloo")
            dist.init_process_group(backend=backend)
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.local_rank = int(os.environ.get("LOCAL_RANK", self.rank))
        self._global_n = None

    def allreduce(self, grad: torch.Tensor):
        dist.all_reduce(grad, op=dist.ReduceOp.SUM)

    def global_batch(self, local_seeds) -> int:
        """|global batch| used as the gradient divisor.  In weak scaling every rank
        holds a full local batch, so the global size is world * local."""
        if self._global_n is not None:
            return self._global_n
        return int(local_seeds.shape[0]) * self.world

    def set_global_batch(self, n: int | None):
        self._global_n = n

    def max_over_ranks(self, x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64,
                         device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier(self):
        if dist.get_backend() == "nccl" and torch.cuda.is_available():
            dist.barrier(device_ids=[torch.cuda.current_device()])
        else:
            dist.barrier()

    def close(self):
        """Tear the process group down (end of a run)."""
        if dist.is_initialized():
            dist.destroy_process_group()


class ShardedFeatures:
    """Feature table row-sharded over the ranks of one box (SURVEY §8(e), C4:
    features larger than one GPU's HBM).  Rank r keeps rows
    [r*rows_per_shard, (r+1)*rows_per_shard) in its own HBM, exports the shard
    through CUDA IPC, and opens every other rank's shard, so the bottom gather
    (hg_aggregate_fwd_sharded) reads remote rows in place over NVLink — no
    all-to-all exchange step.  ``all_gather`` is any list-gathering callable
    (torch.distributed.all_gather_object over gloo or NCCL).

    With world == 1 the shards may also be carved out of one local table
    (``local_slices``) — the same kernel, used by the single-GPU tests."""

    def __init__(self, features: np.ndarray, rank: int, world: int, all_gather=None, device=None,
                 local_slices: int = 0):
        import ctypes

        from . import _lib
        from .device import pad4
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        feats = np.asarray(features, dtype=np.float32)
        V, F = feats.shape
        self.num_vertices, self.feat_dim, self.ld = V, F, pad4(F)
        n_shards = local_slices if local_slices else world
        if not 1 <= n_shards <= 8:
            raise ValueError("1..8 feature shards")
        self.n_shards = n_shards
        self.rows_per_shard = (V + n_shards - 1) // n_shards
        self._opened = []
        lib = _lib.load()
        if local_slices:  # one table, n slices (single process)
            x = torch.zeros((n_shards * self.rows_per_shard, self.ld), dtype=torch.float32, device=self.device)
            x[:V, :F] = torch.as_tensor(feats, device=self.device)
            self.local = x
            ptrs = [x[k * self.rows_per_shard].data_ptr() for k in range(n_shards)]
        else:
            lo = rank * self.rows_per_shard
            hi = min(V, lo + self.rows_per_shard)
            x = torch.zeros((self.rows_per_shard, self.ld), dtype=torch.float32, device=self.device)
            if hi > lo:
                x[:hi - lo, :F] = torch.as_tensor(feats[lo:hi], device=self.device)
            self.local = x
            torch.cuda.synchronize(self.device)
            handle = (ctypes.c_uint8 * 64)()
            off = ctypes.c_int64(0)
            _lib.call("hg_ipc_get_handle", x.data_ptr(), handle, ctypes.byref(off))
            mine = (bytes(handle), int(off.value), int(self.device.index or 0))
            allh = all_gather(mine) if world > 1 else [mine]
            ptrs = []
            for r, (h, o, dev) in enumerate(allh):
                if r == rank:
                    ptrs.append(x.data_ptr())
                    continue
                if dev != (self.device.index or 0):
                    _lib.call("hg_enable_peer_access", dev)
                p = ctypes.c_void_p()
                buf = (ctypes.c_uint8 * 64).from_buffer_copy(h)
                _lib.call("hg_ipc_open_handle", buf, ctypes.byref(p))
                self._opened.append(p.value)
                ptrs.append(p.value + o)
        self.ptrs = (ctypes.c_void_p * n_shards)(*ptrs)
        self._lib = lib

    def close(self):
        for p in self._opened:
            self._lib.hg_ipc_close(p)
        self._opened = []
