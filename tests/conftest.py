"""Shared fixtures.  `-m gpu` tests need a B200 and libpsell.so; `-m "not gpu"`
tests run on the CPU build box (oracle vs golden fixtures, host logic, ABI)."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device and libpsell.so")
    config.addinivalue_line("markers", "slow: long-running full-size case")


@pytest.fixture(scope="session")
def golden_build():
    z = np.load(os.path.join(GOLDEN, "build_golden.npz"))
    with open(os.path.join(GOLDEN, "build_golden.json")) as f:
        meta = json.load(f)
    return z, meta


@pytest.fixture(scope="session")
def golden_codec():
    return np.load(os.path.join(GOLDEN, "codec_golden.npz"))


@pytest.fixture(scope="session")
def golden_errors():
    with open(os.path.join(GOLDEN, "errors_golden.json")) as f:
        return {e["name"]: e for e in json.load(f)}


@pytest.fixture(scope="session")
def golden_solver():
    z = np.load(os.path.join(GOLDEN, "solver_golden.npz"))
    with open(os.path.join(GOLDEN, "solver_golden.json")) as f:
        return z, json.load(f)


def golden_x(case: int, n_cols: int, dt) -> np.ndarray:
    """Same as tests/golden/make_golden.py:golden_x."""
    return np.random.default_rng(1000 + case).uniform(-1, 1, n_cols).astype(dt)


def case_csr(z, i):
    return z[f"c{i}_row_ptr"], z[f"c{i}_col_idx"], z[f"c{i}_values"]


def random_csr_arrays(rng, n, m, density, banded=False):
    """Random CSR (row_ptr, col_idx, values) with |v| in [0.01, 1] (reference conftest.py:9-29 family)."""
    if banded:
        lo = int(rng.integers(0, max(n // 4, 1)))
        hi = int(rng.integers(0, max(m // 4, 1)))
        i = np.arange(n)[:, None]
        j = np.arange(m)[None, :]
        mask = ((j >= i - lo) & (j <= i + hi)) & (rng.random((n, m)) < max(density, 0.5))
    else:
        mask = rng.random((n, m)) < density
    r, c = np.nonzero(mask)
    vals = rng.uniform(0.01, 1.0, len(r)) * rng.choice([-1.0, 1.0], len(r))
    rp = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=n))]).astype(np.int64)
    return rp, c.astype(np.int32), vals


@pytest.fixture
def rng():
    return np.random.default_rng(20260810)
