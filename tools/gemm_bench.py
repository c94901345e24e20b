#!/usr/bin/env python3
"""Microbenchmark of the dense-transform kernels at the C2 bottom-layer shape:
forward [self | mean] [W_self; W_neigh] (M=51K, K=100+100, N=64) and the two
weight gradients, for each kernel form (hg_set_tuning keys 3/7/11), CUDA events,
inputs larger than L2 rotated between iterations."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_13225_b200 import _lib  # noqa: E402
from paper_2311_13225_b200.device import ptr  # noqa: E402


def timeit(fn, reps=24):
    """Launches captured in one CUDA graph (no host overhead in the timing)."""
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for r in range(reps):
            fn(r)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(4):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (4 * reps) * 1000.0


def main():
    lib = _lib.load()
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 51000
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 100  # per source
    N = 64
    LD = int(sys.argv[3]) if len(sys.argv) > 3 else K  # row stride of the activations (elements)
    print(f"M={M} K={K}+{K} N={N} ld={LD}")
    R = 6  # rotate 6 input sets (> L2 in total)
    A1 = [torch.randn(M, LD, device="cuda")[:, :K] for _ in range(R)]
    A2 = [torch.randn(M, LD, device="cuda")[:, :K] for _ in range(R)]
    G = [torch.randn(M, N, device="cuda") for _ in range(R)]
    W = torch.randn(2 * K, N, device="cuda")
    C = torch.empty(M, N, device="cuda")
    dM = torch.tensor([M], dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    img = torch.zeros(int(lib.hg_gemm_tc_bimg_size(K, K, N)) // 4 + 4, device="cuda")
    _lib.call("hg_gemm_tc_prep_b", ptr(W), N, 1, K, K, N, ptr(img), s)
    o1, o2 = torch.empty(K, N, device="cuda"), torch.empty(K, N, device="cuda")
    ws = torch.zeros(int(lib.hg_wgrad_tc_ws_size(K, N, M, 2)), device="cuda")
    ref = None
    fwd_bytes = M * 2 * K * 4 + M * N * 4
    wg_bytes = M * 2 * K * 4 + M * N * 4
    for name, form, pair, wts in (("tma SS", 0, 0, 1), ("tma TS", 1, 0, 1), ("tma TS paired", 1, 1, 1),
                                  ("paired, SS-form wgrad", 1, 1, 0)):
        lib.hg_set_tuning(11, wts)
        lib.hg_set_tuning(7, pair)
        lib.hg_set_tuning(3, form)
        f = lambda r: _lib.call("hg_gemm_tc", ptr(A1[r % R]), LD, K, ptr(A2[r % R]), LD, K, ptr(img), ptr(C), N, N,  # noqa
                                ptr(dM), M, 1, torch.cuda.current_stream().cuda_stream)
        us = timeit(f)
        f(0)
        torch.cuda.synchronize()
        out = C.clone()
        want = torch.relu(torch.cat([A1[0], A2[0]], 1).double() @ W.double()).float()
        err = (out - want).abs().max().item()
        g = lambda r: _lib.call("hg_wgrad_tc", ptr(A1[r % R]), LD, ptr(A2[r % R]), LD, K, ptr(G[r % R]), N, N,  # noqa
                                ptr(dM), M, ptr(o1), ptr(o2), ptr(ws), torch.cuda.current_stream().cuda_stream)
        us_w = timeit(g)
        g(0)
        torch.cuda.synchronize()
        werr = max((o1 - (A1[0].double().T @ G[0].double()).float()).abs().max().item(),
                   (o2 - (A2[0].double().T @ G[0].double()).float()).abs().max().item())
        print(f"{name:16s} fwd {us:7.2f} us ({fwd_bytes / us / 1e3:6.0f} GB/s, max err {err:.2e})   "
              f"wgrad {us_w:7.2f} us ({wg_bytes / us_w / 1e3:6.0f} GB/s, max err {werr:.2e})")
    lib.hg_set_tuning(3, 1)
    for dbg, what in ((1, "no MMA"), (2, "no split"), (3, "loads only"), (4, "no stores"), (7, "loads, no st")):
        lib.hg_set_tuning(9, dbg)
        f = lambda r: _lib.call("hg_gemm_tc", ptr(A1[r % R]), LD, K, ptr(A2[r % R]), LD, K, ptr(img), ptr(C), N, N,  # noqa
                                ptr(dM), M, 1, torch.cuda.current_stream().cuda_stream)
        print(f"fwd TS paired {what:12s} {timeit(f):7.2f} us")
    for dbg, what in ((1, "no MMA"), (2, "no split"), (3, "loads only")):
        lib.hg_set_tuning(9, dbg)
        g = lambda r: _lib.call("hg_wgrad_tc", ptr(A1[r % R]), LD, ptr(A2[r % R]), LD, K, ptr(G[r % R]), N, N,  # noqa
                                ptr(dM), M, ptr(o1), ptr(o2), ptr(ws), torch.cuda.current_stream().cuda_stream)
        print(f"wgrad tma {what:12s} {timeit(g):7.2f} us")
    lib.hg_set_tuning(9, 0)


if __name__ == "__main__":
    main()
