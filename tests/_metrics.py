"""Achieved parity numbers of the GPU tests, appended to
gpurun_out/parity_metrics.jsonl (when that directory exists) so each stated
tolerance can be reported next to the value actually reached."""

import json
import os
from pathlib import Path

OUT = Path(__file__).resolve().parents[1] / "gpurun_out"


def record(name: str, value: float, bound: float) -> None:
    if not OUT.is_dir():
        return
    with open(OUT / "parity_metrics.jsonl", "a") as f:
        f.write(json.dumps({"test": os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0], "name": name,
                            "value": float(value), "bound": float(bound)}) + "\n")
