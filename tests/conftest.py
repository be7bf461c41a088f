"""Shared fixtures.  `-m gpu` tests need a B200 (run through gpurun); everything
else runs on the CPU build container."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(ROOT))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: large-shape test")


def load_golden(name):
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden():
    return {n: load_golden(n) for n in ("calibrate", "stats", "accel", "normalize", "datalink", "fec", "air")}


@pytest.fixture
def rng():
    # same seed as the reference suite (pkg/tests/conftest.py:31-33)
    return np.random.default_rng(20240901)


def case_names(store, suffix):
    return sorted({k.split("/")[0] for k in store if k.endswith("/" + suffix)})
