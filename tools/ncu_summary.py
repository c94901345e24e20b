#!/usr/bin/env python3
"""Key metrics of an `ncu --set full` report as text (for profiles/):

    python tools/ncu_summary.py gpurun_out/prof_k_agg_fwd.ncu-rep [alg_bytes]
"""
import csv
import io
import subprocess
import sys

WANT = [
    ("Kernel Name", "kernel"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % (occupancy)"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall long scoreboard"),
]


def main(path, alg_bytes=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        vals = {}
        for key, label in WANT:
            if key in h:
                i = h.index(key)
                vals[key] = (v[i], u[i])
                print(f"{label:32s} {v[i]} {u[i]}".rstrip())
        if alg_bytes and "dram__bytes_read.sum" in vals:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            r = float(vals["dram__bytes_read.sum"][0]) * scale.get(vals["dram__bytes_read.sum"][1], 1)
            w = float(vals["dram__bytes_write.sum"][0]) * scale.get(vals["dram__bytes_write.sum"][1], 1)
            print(f"{'traffic / algorithmic bytes':32s} {(r + w) / float(alg_bytes):.3f}")
        print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
