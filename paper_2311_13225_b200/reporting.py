"""Run manifest and the per-batch / accuracy CSV emitters with the reference's
versioned schemas (reporting.py:17-79), so runs can be diffed row for row
against the reference's own CSVs.  Per-batch rows carry no
wall-clock values: reruns with equal manifests are byte-identical."""

from __future__ import annotations

import csv
import json
from dataclasses import dataclass, field
from pathlib import Path

BATCH_SCHEMA_VERSION = 1     # reporting.py:18
ACCURACY_SCHEMA_VERSION = 1  # reporting.py:19

BATCH_COLUMNS = [            # reporting.py:23-27
    "schema_version", "epoch", "batch", "super_batch", "loss", "reuse_hits",
    "fallbacks", "raw_rows", "cache_hit_rows", "raw_elems", "emb_elems",
    "aux_elems", "grad_elems", "max_weight_delta",
]


@dataclass
class RunManifest:
    """reporting.py:30-50."""

    config: dict
    seed: int
    code_version: str = "paper_2311_13225_b200"
    dataset_fingerprint: str = ""
    outputs: list = field(default_factory=list)

    def to_dict(self) -> dict:
        return {"config": self.config, "seed": self.seed, "code_version": self.code_version,
                "dataset_fingerprint": self.dataset_fingerprint, "outputs": list(self.outputs)}

    def write(self, path: str | Path) -> None:
        with open(path, "w", encoding="ascii") as fh:
            json.dump(self.to_dict(), fh, indent=2, sort_keys=True)
            fh.write("\n")


def _fmt(value) -> str:
    """reporting.py:53-56 (floats with 12 significant digits)."""
    if isinstance(value, float):
        return f"{value:.12g}"
    return str(value)


def write_batch_csv(path: str | Path, reports) -> None:
    """reporting.py:59-67: one row per training batch of every epoch report."""
    with open(path, "w", newline="", encoding="ascii") as fh:
        writer = csv.writer(fh)
        writer.writerow(BATCH_COLUMNS)
        for report in reports:
            for row in report.batch_rows:
                writer.writerow([_fmt(BATCH_SCHEMA_VERSION)] + [_fmt(row[c]) for c in BATCH_COLUMNS[1:]])


def write_accuracy_csv(path: str | Path, reports) -> None:
    """reporting.py:70-79: epoch -> accuracy series."""
    with open(path, "w", newline="", encoding="ascii") as fh:
        writer = csv.writer(fh)
        writer.writerow(["schema_version", "epoch", "val_accuracy", "test_accuracy", "mean_loss"])
        for r in reports:
            mean_loss = sum(r.losses) / len(r.losses) if r.losses else 0.0
            writer.writerow([ACCURACY_SCHEMA_VERSION, r.epoch, _fmt(r.val_accuracy), _fmt(r.test_accuracy),
                             _fmt(mean_loss)])
