"""Batch / accuracy CSV schemas match the reference's (reporting.py:17-79):
same header, same formatting, byte-identical output for equal rows."""

import csv
from types import SimpleNamespace


def test_batch_csv_schema_and_format(tmp_path):
    from paper_2311_13225_b200 import reporting as R
    row = dict(epoch=0, batch=3, super_batch=1, loss=0.123456789012345, reuse_hits=5, fallbacks=0, raw_rows=992,
               cache_hit_rows=0, raw_elems=992 * 16, emb_elems=0, aux_elems=0, grad_elems=2048,
               max_weight_delta=1e-3)
    rep = SimpleNamespace(batch_rows=[row], losses=[0.5, 0.25], epoch=0, val_accuracy=0.5, test_accuracy=0.25)
    p = tmp_path / "b.csv"
    R.write_batch_csv(p, [rep])
    rows = list(csv.reader(open(p)))
    assert rows[0] == ["schema_version", "epoch", "batch", "super_batch", "loss", "reuse_hits", "fallbacks",
                       "raw_rows", "cache_hit_rows", "raw_elems", "emb_elems", "aux_elems", "grad_elems",
                       "max_weight_delta"]
    assert rows[1] == ["1", "0", "3", "1", "0.123456789012", "5", "0", "992", "0", "15872", "0", "0", "2048",
                       "0.001"]
    q = tmp_path / "b2.csv"
    R.write_batch_csv(q, [rep])
    assert p.read_bytes() == q.read_bytes()
    a = tmp_path / "a.csv"
    R.write_accuracy_csv(a, [rep])
    assert list(csv.reader(open(a)))[1] == ["1", "0", "0.5", "0.25", "0.375"]
    m = tmp_path / "m.json"
    R.RunManifest(config={"model": "sage"}, seed=3).write(m)
    assert '"seed": 3' in m.read_text()
