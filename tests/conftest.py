import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full-size configuration checks")


def cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container (run with -m gpu on a B200)")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


class Golden:
    """Accessor over a golden .npz written by tests/golden/make_golden.py."""

    def __init__(self, path):
        self._z = np.load(path)
        self.files = set(self._z.files)

    def __getitem__(self, k):
        return self._z[k]

    def __contains__(self, k):
        return k in self.files

    def knots(self, key):
        flat, m = self._z[key + ".knots"], self._z[key + ".m"]
        out, off = [], 0
        for mk in m:
            out.append(flat[off:off + mk])
            off += mk
        return out

    def keys(self, prefix):
        return sorted({k[len(prefix):].split(".")[0] for k in self.files if k.startswith(prefix)})


@pytest.fixture(scope="session")
def small_golden():
    return Golden(GOLDEN / "small.npz")


@pytest.fixture(scope="session")
def cfg_meta():
    p = GOLDEN / "configs.json"
    return json.loads(p.read_text()) if p.exists() else {}


def cfg_golden(name):
    p = GOLDEN / f"{name}.npz"
    return Golden(p) if p.exists() else None


@pytest.fixture(scope="session")
def oracle():
    import oracle as orc

    orc.build()
    return orc
