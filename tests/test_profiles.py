"""The committed measurement records bench.py reads at run time: each bench workload's dominant-kernel
DRAM traffic must come from that workload's own ncu capture (profiles/ncu_traffic.json), so the
roofline.traffic of a C3 line can never carry C2's bytes."""
import json
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_ncu_traffic_per_workload():
    import bench
    rec = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())
    for wl in ("c2", "c3"):
        assert wl in bench.WORKLOADS
        r = rec[wl]
        assert r["kernel"].startswith("k_agg_fwd<")
        assert r["traffic_bytes_per_launch"] == r["dram_read_bytes"] + r["dram_write_bytes"]
        assert 0 < r["gpu_time_us_cold"] < 1000
        assert wl.upper() in r["kernel"]
    # the two captures are different kernels (C2: one float4 per lane, C3: five)
    assert rec["c2"]["kernel"].split(" (")[0] != rec["c3"]["kernel"].split(" (")[0]


@pytest.mark.parametrize("name", ["r02s_bench_default.json", "r02s_bench_c3.json"])
def test_committed_bench_lines_keep_the_contract(name):
    d = json.loads((ROOT / "profiles" / name).read_text())
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    r = d["roofline"]
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert r["traffic"] is not None and r["traffic"] > r["alg_bytes_per_launch"] * 0.5
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert not set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
