"""tcgen05 GEMMs (3xTF32) against a float64 numpy reference.

Tolerance: |C - C_ref| <= 2e-5 * (|A| |B|)_ij  (the product-magnitude bound; 3xTF32
lands ~1e-6 relative to it)."""

import numpy as np
import pytest

from conftest import has_cuda

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_cuda(), reason="needs CUDA")]


def _pad(x, ld):
    import torch
    t = torch.zeros((max(x.shape[0], 1), ld), dtype=torch.float32, device="cuda")
    t[:x.shape[0], :x.shape[1]] = torch.as_tensor(x.astype(np.float32), device="cuda")
    return t


def _ld(k):
    return (k + 3) // 4 * 4


@pytest.fixture(params=["tc", "tc_unpaired", "tc_wg_ss", "tc_wg_ss_unpaired", "tc_ss_fwd"])
def path(request):
    """hg_gemm_tc / hg_wgrad_tc kernel forms: default (paired MMAs, A through TMEM,
    wgrad with A^T through TMEM), unpaired MMAs (hg_set_tuning key 7), the
    shared-memory wgrad form (key 11), the shared-memory forward form (key 3)."""
    from paper_2311_13225_b200 import _lib
    lib = _lib.load()
    lib.hg_set_tuning(7, 0 if request.param.endswith("unpaired") else 1)
    lib.hg_set_tuning(11, 0 if request.param.startswith("tc_wg_ss") else 1)
    lib.hg_set_tuning(3, 0 if request.param == "tc_ss_fwd" else 1)
    yield request.param
    lib.hg_set_tuning(7, 1)
    lib.hg_set_tuning(11, 1)
    lib.hg_set_tuning(3, 1)


@pytest.mark.parametrize("M,K1,K2,N,trans,act", [
    (300, 100, 100, 64, 1, 1), (1000, 64, 64, 47, 1, 0), (129, 32, 0, 16, 1, 0), (5000, 47, 0, 64, 0, 0),
    (777, 602, 0, 256, 1, 1), (1024, 128, 0, 172, 1, 0), (1, 3, 5, 9, 1, 0), (200, 64, 0, 300, 0, 0),
    (5700, 64, 64, 64, 1, 1), (1024, 64, 0, 128, 0, 0), (3000, 128, 128, 128, 1, 0), (6000, 47, 0, 64, 0, 0),
])
def test_gemm(M, K1, K2, N, trans, act, path):
    import torch
    from paper_2311_13225_b200 import _lib
    from paper_2311_13225_b200.device import ptr
    rng = np.random.default_rng(M + K1 + N)
    A1 = rng.standard_normal((M, K1))
    A2 = rng.standard_normal((M, K2)) if K2 else None
    Ktot = K1 + K2
    W = rng.standard_normal((Ktot, N)) if trans else rng.standard_normal((N, Ktot))
    Wf = W.astype(np.float32).astype(np.float64)
    a1 = A1.astype(np.float32).astype(np.float64)
    ref = a1 @ (Wf[:K1] if trans else Wf[:, :K1].T)
    mag = np.abs(a1) @ np.abs(Wf[:K1] if trans else Wf[:, :K1].T)
    if K2:
        a2 = A2.astype(np.float32).astype(np.float64)
        ref = ref + a2 @ (Wf[K1:] if trans else Wf[:, K1:].T)
        mag = mag + np.abs(a2) @ np.abs(Wf[K1:] if trans else Wf[:, K1:].T)
    if act:
        ref = np.maximum(ref, 0)
    dA1, dA2 = _pad(A1, _ld(K1)), (_pad(A2, _ld(K2)) if K2 else None)
    dW = torch.as_tensor(W.astype(np.float32), device="cuda").contiguous()
    ldb = N if trans else Ktot
    ldc = _ld(N)
    C = torch.full((M, ldc), 7.0, dtype=torch.float32, device="cuda")
    dM = torch.tensor([M], dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    img = torch.zeros(int(_lib.fn("hg_gemm_tc_bimg_size")(K1, K2, N)) // 4 + 4, dtype=torch.float32, device="cuda")
    _lib.call("hg_gemm_tc_prep_b", ptr(dW), ldb, trans, K1, K2, N, ptr(img), s)
    _lib.call("hg_gemm_tc", ptr(dA1), _ld(K1), K1, ptr(dA2), _ld(K2) if K2 else 0, K2, ptr(img), ptr(C), ldc, N,
              ptr(dM), M + 5, act, s)
    got = C[:M, :N].double().cpu().numpy()
    err = np.abs(got - ref)
    assert np.all(err <= 2e-5 * mag + 1e-6), (err.max(), (err / (mag + 1e-9)).max())
    if ldc > N:  # padding columns untouched
        assert np.all(C[:M, N:].cpu().numpy() == 7.0)


@pytest.mark.parametrize("M,K,N,two", [(51000, 100, 64, True), (1000, 64, 47, False), (37, 602, 256, False),
                                       (5, 3, 7, True), (70000, 64, 64, True), (0, 16, 16, False),
                                       (5700, 64, 64, True), (1024, 64, 47, True), (3000, 128, 128, False),
                                       (100, 47, 128, True)])
def test_wgrad_tc(M, K, N, two, path):
    import torch
    from paper_2311_13225_b200 import _lib
    from paper_2311_13225_b200.device import ptr
    rng = np.random.default_rng(K * N + M)
    A1 = rng.standard_normal((M, K))
    A2 = rng.standard_normal((M, K)) if two else None
    G = rng.standard_normal((M, N))
    cap = M + 100
    dA1 = _pad(np.vstack([A1, np.zeros((cap - M, K))]), _ld(K))
    dA2 = _pad(np.vstack([A2, np.zeros((cap - M, K))]), _ld(K)) if two else None
    dG = _pad(np.vstack([G, np.zeros((cap - M, N))]), _ld(N))
    dM = torch.tensor([M], dtype=torch.int32, device="cuda")
    o1 = torch.zeros((K, N), dtype=torch.float32, device="cuda")
    o2 = torch.zeros((K, N), dtype=torch.float32, device="cuda")
    ws = torch.zeros(int(_lib.fn("hg_wgrad_tc_ws_size")(K, N, cap, 2 if two else 1)), dtype=torch.float32,
                     device="cuda")
    _lib.call("hg_wgrad_tc", ptr(dA1), _ld(K), ptr(dA2), _ld(K), K, ptr(dG), _ld(N), N, ptr(dM), cap, ptr(o1),
              ptr(o2) if two else None, ptr(ws), torch.cuda.current_stream().cuda_stream)
    g32 = G.astype(np.float32).astype(np.float64)
    for A, o in ((A1, o1), (A2, o2)) if two else ((A1, o1),):
        a32 = A.astype(np.float32).astype(np.float64)
        ref = a32.T @ g32
        mag = np.abs(a32).T @ np.abs(g32)
        err = np.abs(o.double().cpu().numpy() - ref)
        assert np.all(err <= 2e-5 * mag + 1e-6), (err.max(), (err / (mag + 1e-9)).max())
