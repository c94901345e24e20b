#!/usr/bin/env python3
"""Pipeline timeline of CTA 0 of the TS tensor-core GEMM at the C2 bottom shape
(hg_set_tuning key 9 bit 3): per K iteration, producer issue -> data landed
(split start) -> split done -> MMA start -> MMA commit, in microseconds."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_13225_b200 import _lib  # noqa: E402
from paper_2311_13225_b200.device import ptr  # noqa: E402


def main():
    lib = _lib.load()
    M, K, N = 51000, 100, 64
    A1 = torch.randn(M, K, device="cuda")
    A2 = torch.randn(M, K, device="cuda")
    W = torch.randn(2 * K, N, device="cuda")
    C = torch.empty(M, N, device="cuda")
    dM = torch.tensor([M], dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    img = torch.zeros(int(lib.hg_gemm_tc_bimg_size(K, K, N)) // 4 + 4, device="cuda")
    _lib.call("hg_gemm_tc_prep_b", ptr(W), N, 1, K, K, N, ptr(img), s)
    G = torch.randn(M, N, device="cuda")
    o1, o2 = torch.empty(K, N, device="cuda"), torch.empty(K, N, device="cuda")
    ws = torch.zeros(int(lib.hg_wgrad_tc_ws_size(K, N, M, 2)), device="cuda")
    which = sys.argv[1] if len(sys.argv) > 1 else "fwd"
    for dbg in (8, 8 | 3):
        lib.hg_set_tuning(9, dbg)
        for _ in range(3):
            if which == "fwd":
                _lib.call("hg_gemm_tc", ptr(A1), K, K, ptr(A2), K, K, ptr(img), ptr(C), N, N, ptr(dM), M, 1, s)
            else:
                _lib.call("hg_wgrad_tc", ptr(A1), K, ptr(A2), K, K, ptr(G), N, N, ptr(dM), M, ptr(o1), ptr(o2),
                          ptr(ws), s)
        torch.cuda.synchronize()
        tl = np.zeros((8, 64), dtype=np.uint64)
        _lib.call("hg_debug_timeline", tl.ctypes.data)
        t0 = tl[0, 0]
        rel = (tl.astype(np.int64) - np.int64(t0)) / 1000.0
        print(f"dbg={dbg}: it  issue  landed  split_done  mma_start  mma_commit   (us from first issue)")
        for it in range(0, 24):
            print(f"  {it:2d} {rel[0, it]:7.2f} {rel[1, it]:7.2f} {rel[2, it]:7.2f} {rel[3, it]:7.2f} {rel[4, it]:7.2f}")
    lib.hg_set_tuning(9, 0)


if __name__ == "__main__":
    main()
