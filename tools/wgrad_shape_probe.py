#!/usr/bin/env python3
"""Weight-gradient time at a given shape (single source): python tools/wgrad_shape_probe.py M K N..."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from gemm_bench import timeit  # noqa: E402
from paper_2311_13225_b200 import _lib  # noqa: E402
from paper_2311_13225_b200.device import ptr  # noqa: E402

lib = _lib.load()
M, K = int(sys.argv[1]), int(sys.argv[2])
for N in [int(x) for x in sys.argv[3:]]:
    R = 4
    LDA = (K + 3) // 4 * 4
    A = [torch.randn(M, LDA, device="cuda")[:, :K] for _ in range(R)]
    G = [torch.randn(M, N, device="cuda") for _ in range(R)]
    dM = torch.tensor([M], dtype=torch.int32, device="cuda")
    o = torch.empty(K, N, device="cuda")
    ws = torch.zeros(int(lib.hg_wgrad_tc_ws_size(K, N, M, 1)), device="cuda")
    g = lambda r: _lib.call("hg_wgrad_tc", ptr(A[r % R]), LDA, None, 0, K, ptr(G[r % R]), N, N, ptr(dM), M, ptr(o),  # noqa
                            None, ptr(ws), torch.cuda.current_stream().cuda_stream)
    us = timeit(g)
    g(0)
    torch.cuda.synchronize()
    err = (o - (A[0].double().T @ G[0].double()).float()).abs().max().item()
    print(f"wgrad M={M} K={K} N={N}: {us:.2f} us (max err {err:.2e})")
