#!/usr/bin/env python3
"""One markdown row per kernel launch of an `ncu --set full` report (for profiles/):

    python tools/ncu_table.py gpurun_out/full_r02.ncu-rep > profiles/r02_ncu_full.md
"""
import csv
import io
import subprocess
import sys

COLS = [("gpu__time_duration.sum", "us", 1e-3), ("dram__bytes_read.sum", "DRAM rd MB", 1e-6),
        ("dram__bytes_write.sum", "DRAM wr MB", 1e-6),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %", 1),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor %", 1),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %", 1),
        ("lts__t_sector_hit_rate.pct", "L2 hit %", 1), ("launch__grid_size", "grid", 1),
        ("launch__registers_per_thread", "regs", 1)]
SCALE = {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "byte": 1, "Kbyte": 1e3,
         "Mbyte": 1e6, "Gbyte": 1e9}


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    ki = h.index("Kernel Name")
    print("| # | kernel | " + " | ".join(c[1] for c in COLS) + " |")
    print("|---|---|" + "---|" * len(COLS))
    for n, r in enumerate(rows[2:]):
        name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        cells = []
        for key, _, mul in COLS:
            if key not in h:
                cells.append("-")
                continue
            i = h.index(key)
            try:
                v = float(r[i].replace(",", "")) * SCALE.get(u[i], 1) * mul
                cells.append(f"{v:.0f}" if key.startswith("launch__") or v >= 1e4 else f"{v:.1f}")
            except ValueError:
                cells.append(r[i])
        print(f"| {n} | `{name}` | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
