#!/usr/bin/env python3
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel totals and shares."""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.OrderedDict(), collections.Counter()
    for r in data:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        tot[name] = tot.get(name, 0.0) + v
        cnt[name] += 1
    s = sum(tot.values())
    print(f"launches {sum(cnt.values())}  total {s:.1f} us (serialised, cold-cache)")
    for n, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        print(f"{v:9.1f} us {100 * v / s:5.1f}%  x{cnt[n]:<3d} {n}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
