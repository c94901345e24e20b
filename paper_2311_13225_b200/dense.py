"""Dense layer transforms (K8) on the tcgen05 tensor cores (3xTF32, fp32-class).

Weights follow the flat layout of engine.DenseParams: per layer W_self then
W_neigh (SAGE) or W (GCN), each row-major [d_in, d_out], so the stacked
[W_self; W_neigh] is one contiguous [2*d_in, d_out] matrix.

The tensor-core GEMM consumes its B operand (the weights) as a prebuilt
swizzled hi/lo image (``BImage``); the engine rebuilds its images once per
step from the current weights, the functional API builds them on the fly.
"""

from __future__ import annotations

import torch

from . import _lib


class BImage:
    """Device buffer holding op(B)'s swizzled tf32 hi/lo tiles for hg_gemm_tc."""

    def __init__(self, K1: int, K2: int, N: int, trans_b: int, device):
        self.K1, self.K2, self.N, self.trans_b = int(K1), int(K2), int(N), int(trans_b)
        nbytes = int(_lib.fn("hg_gemm_tc_bimg_size")(self.K1, self.K2, self.N))
        self.buf = torch.empty(max(nbytes // 4, 4), dtype=torch.float32, device=device)

    def prep(self, W: int, ldb: int, s):
        _lib.call("hg_gemm_tc_prep_b", W, ldb, self.trans_b, self.K1, self.K2, self.N, self.buf.data_ptr(), s)


def fwd(A1, lda1, A2, lda2, K, W, N, C, ldc, d_M, cap, act, s, img: BImage | None = None, device=None):
    """C = act(A1 W[0:K] + A2 W[K:2K])  (A2 None: C = act(A1 W))."""
    if img is None:
        img = BImage(K, K if A2 is not None else 0, N, 1, device or torch.cuda.current_device())
        img.prep(W, N, s)
    _lib.call("hg_gemm_tc", A1, lda1, K, A2, lda2 if A2 else 0, K if A2 else 0, img.buf.data_ptr(), C, ldc, N,
              d_M, cap, act, s)


def dx(dZ, ldz, K, W, N, C, ldc, d_M, cap, s, img: BImage | None = None, device=None):
    """C[M x N] = dZ[M x K] W^T with W stored [N x K] (row-major, ld K)."""
    if img is None:
        img = BImage(K, 0, N, 0, device or torch.cuda.current_device())
        img.prep(W, K, s)
    _lib.call("hg_gemm_tc", dZ, ldz, K, None, 0, 0, img.buf.data_ptr(), C, ldc, N, d_M, cap, 0, s)


def wgrad_ws_size(K, N, cap, n_src) -> int:
    lib = _lib.load()
    return int(lib.hg_wgrad_tc_ws_size(K, N, cap, n_src))


def wgrad(A1, lda1, A2, lda2, K, G, ldg, N, d_M, cap, out1, out2, ws, s):
    """out1 = A1^T G, out2 = A2^T G (A2 optional)."""
    _lib.call("hg_wgrad_tc", A1, lda1, A2, lda2 if A2 else 0, K, G, ldg, N, d_M, cap, out1, out2, ws, s)
