"""Shared test setup.

Markers: ``gpu`` tests need a CUDA device and call the product through the
libsrt C ABI; everything else runs on CPU (oracle vs golden fixtures, host
logic, ABI exports, multi-process gloo).  The oracle (``oracle/``) is used
only as the checker.
"""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"
TMAX = float(np.finfo(np.float64).max)
CUTOFF = 2.0 * np.sqrt(2.0)
S2 = CUTOFF * CUTOFF


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libsrt.so")
    config.addinivalue_line("markers", "slow: long-running statistical check")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(GOLDEN / f"{name}.npz")

    return load


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.build()
    return O


def random_rays(rng, n, box=3.0):
    origins = rng.uniform(-box, box, size=(n, 3))
    dirs = rng.normal(size=(n, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    return origins, dirs


def axis_rays(rng, n, lateral=0.4):
    """Rays along +z from z = 0 at jittered lateral offsets (validate.py:36-43 style)."""
    origins = np.zeros((n, 3))
    origins[:, 0] = rng.uniform(-lateral, lateral, n)
    origins[:, 1] = rng.uniform(-lateral, lateral, n)
    dirs = np.tile([0.0, 0.0, 1.0], (n, 1))
    return origins, dirs


REFERENCE_SRC = Path("/root/reference/pkg/src")
HAVE_REFERENCE = REFERENCE_SRC.exists() and os.environ.get("SRT_NO_REFERENCE") != "1"
