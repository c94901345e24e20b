"""Diagnostic: relative error of hg_wgrad_tc for both MN-major descriptor offset assignments."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_13225_b200 import _lib  # noqa: E402
from paper_2311_13225_b200.device import ptr  # noqa: E402


def run(M, K, N, swap):
    _lib.call("hg_set_tuning", 1, swap)
    rng = np.random.default_rng(0)
    A = rng.standard_normal((M, K)).astype(np.float32)
    G = rng.standard_normal((M, N)).astype(np.float32)
    ld = lambda k: (k + 3) // 4 * 4  # noqa: E731
    dA = torch.zeros((M, ld(K)), device="cuda"); dA[:, :K] = torch.as_tensor(A, device="cuda")
    dG = torch.zeros((M, ld(N)), device="cuda"); dG[:, :N] = torch.as_tensor(G, device="cuda")
    dM = torch.tensor([M], dtype=torch.int32, device="cuda")
    o = torch.zeros((K, N), device="cuda")
    ws = torch.zeros(int(_lib.fn("hg_wgrad_tc_ws_size")(K, N, M, 1)), device="cuda")
    _lib.call("hg_wgrad_tc", ptr(dA), ld(K), None, 0, K, ptr(dG), ld(N), N, ptr(dM), M, ptr(o), None, ptr(ws),
              torch.cuda.current_stream().cuda_stream)
    ref = A.astype(np.float64).T @ G.astype(np.float64)
    got = o.double().cpu().numpy()
    return np.abs(got - ref).max() / np.abs(ref).max()


for M, K, N in [(32, 128, 64), (8, 128, 64), (8, 32, 32), (256, 100, 64)]:
    print(M, K, N, "swap0", run(M, K, N, 0), "swap1", run(M, K, N, 1), flush=True)
