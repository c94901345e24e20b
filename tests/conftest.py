import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN_DIR = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN_DIR / "golden.npz")


@pytest.fixture(scope="session")
def golden_meta():
    return json.loads((GOLDEN_DIR / "golden.json").read_text())


class GG:
    """A golden fixture graph with the oracle's containers."""

    def __init__(self, z, prefix):
        from oracle import oracle as O
        self.graph = O.Graph(offsets=z[f"{prefix}_offsets"],
                             targets=z[f"{prefix}_targets"].astype(np.int64))
        self.data = None
        if f"{prefix}_features" in z:
            self.data = O.VertexData(features=z[f"{prefix}_features"],
                                     labels=z[f"{prefix}_labels"].astype(np.int64),
                                     train_mask=z[f"{prefix}_train"],
                                     val_mask=z[f"{prefix}_val"],
                                     test_mask=z[f"{prefix}_test"])


@pytest.fixture(scope="session")
def ggraphs(golden):
    return {p: GG(golden, p) for p in ("star", "pl", "sbm")}


def golden_stack(z, prefix):
    L = int(z[f"{prefix}_L"])
    return [dict(dst=z[f"{prefix}_b{l}_dst"], src=z[f"{prefix}_b{l}_src"],
                 es=z[f"{prefix}_b{l}_es"], ed=z[f"{prefix}_b{l}_ed"]) for l in range(L)]


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
