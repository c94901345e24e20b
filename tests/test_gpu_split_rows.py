"""Split-row feature copy (DeviceGraph.split_rows, hg_aggregate_fwd_split): the
bottom gather over [line-aligned body | L2-held tail] is bit-identical to the
gather over the plain table (orchestrator.py:239 + gnnmath.py:145-154 / 89-97),
for SAGE and GCN, with injected (skipped) destinations, and the C-ABI rejects
bad geometry."""

import numpy as np
import pytest

from conftest import has_cuda

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_cuda(), reason="needs CUDA")]


def _run(dg, ids, smp, model, inj, split):
    import torch
    from paper_2311_13225_b200 import _lib
    from paper_2311_13225_b200.device import ptr
    n, ld = ids.shape[0], dg.feat_ld
    self_out = torch.full((n, ld), 7.0, device="cuda")
    agg = torch.full((n, ld), 7.0, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    common = (ptr(ids), None, n, smp.f, ptr(smp.counts), ptr(smp.slots), ptr(smp.slot_local), ptr(smp.nself),
              ptr(smp.outdeg), ptr(inj), ptr(self_out), ld, ptr(agg), ld, s)
    if split is None:
        _lib.call("hg_aggregate_fwd", model, 1, ptr(dg.features), ld, ld, *common)
    else:
        _lib.call("hg_aggregate_fwd_split", model, ptr(split["body"]), split["body_cols"], ptr(split["tail"]),
                  split["tail_cols"], split["body_cols"], ld, *common)
    torch.cuda.synchronize()
    return self_out.cpu().numpy(), agg.cpu().numpy()


@pytest.mark.parametrize("model", [0, 1])
def test_split_gather_bitexact(model, monkeypatch):
    import torch
    from paper_2311_13225_b200.datagen import make_dataset
    from paper_2311_13225_b200.device import DeviceGraph, u64_tensor
    from paper_2311_13225_b200.sampler import LayerSampler
    monkeypatch.delenv("HG_SPLIT_ROWS", raising=False)
    ds = make_dataset("c2learn", scale=0.1)  # F = 100: 400-byte rows, body 96 + tail 4
    dg = DeviceGraph.from_dataset(ds)
    sp = dg.split_rows()
    assert sp is not None and sp["body_cols"] == 96 and sp["tail_cols"] == 4
    assert sp["body"].data_ptr() % 128 == 0
    assert torch.equal(torch.cat([sp["body"], sp["tail"]], 1), dg.features)
    rng = np.random.default_rng(11 + model)
    n = 5000
    ids = torch.as_tensor(rng.choice(ds.num_vertices, size=n, replace=False).astype(np.int32), device="cuda")
    smp = LayerSampler(dg, n, 15, need_nself=model == 0, need_outdeg=model == 1)
    smp.run(ids, None, u64_tensor(5, "cuda"), 0, dedup=model == 1)
    inj = torch.as_tensor((rng.random(n) < 0.2).astype(np.uint8), device="cuda")
    for m in (None, inj):
        a = _run(dg, ids, smp, model, m, None)
        b = _run(dg, ids, smp, model, m, sp)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert not np.all(a[1] == 0)


def test_split_rows_geometry(monkeypatch):
    from paper_2311_13225_b200 import _lib
    from paper_2311_13225_b200.datagen import make_dataset
    from paper_2311_13225_b200.device import DeviceGraph
    ds = make_dataset("c1")  # F = 128: whole lines already, no split copy
    assert DeviceGraph.from_dataset(ds).split_rows() is None
    monkeypatch.setenv("HG_SPLIT_ROWS", "0")
    assert DeviceGraph.from_dataset(make_dataset("c2learn", scale=0.02)).split_rows() is None
    with pytest.raises(Exception):  # tail columns not covered by ld_tail
        _lib.call("hg_aggregate_fwd_split", 0, 16, 96, 32, 2, 96, 100, 16, None, 1, 15, 16, 16, 16, 16, None,
                  None, None, 100, 16, 100, None)
