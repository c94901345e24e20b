"""Write the C2 bottom block's row-fetch list (self row + drawn neighbours per
destination, destination order) for tools/order_probe.cu."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle as O  # noqa: E402  (test infrastructure: the fetch list only)
from paper_2311_13225_b200 import runplan  # noqa: E402
from paper_2311_13225_b200.datagen import make_dataset  # noqa: E402

ds = make_dataset("c2")
g = O.Graph(ds.offsets, ds.targets.astype(np.int64))
seeds = runplan.shuffle_epoch(ds.train_ids(), 0, 0)[:1024]
st = O.sample_khop(g, seeds, (15, 10, 5), runplan.batch_sample_seed(0, 0, 0))
b = st.blocks[0]
src = b.src_vertices[b.edge_src]
starts = np.searchsorted(b.edge_dst, np.arange(b.n_dst))
ends = np.searchsorted(b.edge_dst, np.arange(b.n_dst), side="right")
out = []
for i in range(b.n_dst):
    out.append(b.dst_vertices[i:i + 1])
    out.append(src[starts[i]:ends[i]])
lst = np.concatenate(out).astype(np.int32)
lst.tofile(Path(__file__).resolve().parent / "fetch_list.i32")
print(lst.size, np.unique(lst).size)
