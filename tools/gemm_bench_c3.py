#!/usr/bin/env python3
"""Microbenchmark of the dense-transform kernels at the C3 bottom-layer shape (GCN: one source,
M=22.5K rows, K=602, N=256): forward A W and the weight gradient A^T G, CUDA events over CUDA-graph
replays, inputs rotated (> L2 in total), with the kernels' profiling modes (hg_set_tuning key 9):
no MMA / no split / loads only, to see which stage paces each kernel.

    python tools/gemm_bench_c3.py [M] [K] [N]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_13225_b200 import _lib  # noqa: E402
from paper_2311_13225_b200.device import ptr  # noqa: E402
from tools.gemm_bench import timeit  # noqa: E402


def main():
    lib = _lib.load()
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 22500
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 602
    N = int(sys.argv[3]) if len(sys.argv) > 3 else 256
    LD = (K + 3) // 4 * 4
    R = 6
    A = [torch.randn(M, LD, device="cuda")[:, :K] for _ in range(R)]
    G = [torch.randn(M, N, device="cuda") for _ in range(R)]
    W = torch.randn(K, N, device="cuda")
    C = torch.empty(M, N, device="cuda")
    dM = torch.tensor([M], dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    img = torch.zeros(int(lib.hg_gemm_tc_bimg_size(K, 0, N)) // 4 + 4, device="cuda")
    _lib.call("hg_gemm_tc_prep_b", ptr(W), N, 1, K, 0, N, ptr(img), s)
    o1 = torch.empty(K, N, device="cuda")
    ws = torch.zeros(int(lib.hg_wgrad_tc_ws_size(K, N, M, 1)), device="cuda")
    flops = 2.0 * M * K * N * 3  # 3xTF32
    f = lambda r: _lib.call("hg_gemm_tc", ptr(A[r % R]), LD, K, None, 0, 0, ptr(img), ptr(C), N, N,  # noqa: E731
                            ptr(dM), M, 0, torch.cuda.current_stream().cuda_stream)
    g = lambda r: _lib.call("hg_wgrad_tc", ptr(A[r % R]), LD, None, 0, K, ptr(G[r % R]), N, N,  # noqa: E731
                            ptr(dM), M, ptr(o1), None, ptr(ws), torch.cuda.current_stream().cuda_stream)
    f(0)
    g(0)
    torch.cuda.synchronize()
    err = (C - (A[0].double() @ W.double()).float()).abs().max().item()
    werr = (o1 - (A[0].double().T @ G[0].double()).float()).abs().max().item()
    print(f"M={M} K={K} N={N}: max err fwd {err:.2e} wgrad {werr:.2e}")
    for dbg, what in ((0, "full"), (1, "no MMA"), (2, "no split"), (3, "loads only")):
        lib.hg_set_tuning(9, dbg)
        uf, ug = timeit(f), timeit(g)
        print(f"{what:12s} fwd {uf:7.2f} us ({flops / uf / 1e6:6.1f} TFLOP/s 3xTF32)   "
              f"wgrad+reduce {ug:7.2f} us ({flops / ug / 1e6:6.1f} TFLOP/s)")
    lib.hg_set_tuning(9, 0)


if __name__ == "__main__":
    main()
