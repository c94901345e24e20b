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
        dist.barrier()
