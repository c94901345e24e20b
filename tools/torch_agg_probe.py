#!/usr/bin/env python3
"""The bottom aggregation of one C2 block written with stock torch ops (the
baseline a PyTorch user would write) next to the repo's fused kernel:
index_select of the source rows + index_add_ of the weighted rows into the
destinations (float atomics: not deterministic), self rows by index_select.
Same block (oracle sample_khop of the bench's first batch), CUDA events, L2
flushed by a 512 MB memset between repetitions."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle as O  # noqa: E402  (test infrastructure: the block only)
from paper_2311_13225_b200 import runplan  # noqa: E402
from paper_2311_13225_b200.datagen import make_dataset  # noqa: E402

ds = make_dataset("c2", cache_dir="/tmp/hg_bench_cache")
g = O.Graph(ds.offsets, ds.targets.astype(np.int64))
seeds = runplan.shuffle_epoch(ds.train_ids(), 0, 0)[:1024]
st = O.sample_khop(g, seeds, (15, 10, 5), runplan.batch_sample_seed(0, 0, 0))
b = st.blocks[0]
src_g = b.src_vertices[b.edge_src]
dst_g = b.dst_vertices[b.edge_dst]
keep = src_g != dst_g  # SAGE drops self edges
es, ed = src_g[keep], b.edge_dst[keep]
cnt = np.bincount(ed, minlength=b.n_dst).astype(np.float32)
w = (1.0 / np.maximum(cnt, 1))[ed].astype(np.float32)
dev = torch.device("cuda")
X = torch.as_tensor(ds.features, device=dev)
t_es = torch.as_tensor(es, device=dev)
t_ed = torch.as_tensor(ed, device=dev)
t_w = torch.as_tensor(w, device=dev).unsqueeze(1)
t_dst = torch.as_tensor(b.dst_vertices, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def torch_agg():
    self_rows = X.index_select(0, t_dst)
    rows = X.index_select(0, t_es) * t_w
    mean = torch.zeros(b.n_dst, X.shape[1], device=dev).index_add_(0, t_ed, rows)
    return self_rows, mean


best = 1e9
for r in range(6):
    flush.fill_(r)
    a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    torch_agg()
    c.record()
    torch.cuda.synchronize()
    if r:
        best = min(best, a.elapsed_time(c) * 1e3)
alg = (len(np.unique(np.concatenate([b.dst_vertices, es]))) + b.n_dst) * X.shape[1] * 4 + es.size * 8
print(f"C2 bottom block: {b.n_dst} dsts, {es.size} non-self edges; torch index_select + index_add_: {best:.1f} us "
      f"({alg / best / 1e3:.0f} GB/s of the §8(d) algorithmic bytes)")
