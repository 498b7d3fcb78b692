"""Shared test fixtures.

CPU tests (-m "not gpu"): oracle restatement vs golden vectors / the reference,
the product's host layer, and the C ABI surface.  GPU tests (-m gpu): parity of
the sm_100a path (through the C ABI) against the oracle restatement.
"""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def oc():
    import oracle

    return oracle.restatement()


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.reference_available():
        pytest.skip("oracle/_ref not built (needs /root/reference; build container only)")
    return oracle.reference()


@pytest.fixture(scope="session")
def gnp():
    import paper_2406_00809_b200 as g

    return g


@pytest.fixture(scope="session")
def capi():
    from paper_2406_00809_b200 import capi as c

    return c


@pytest.fixture(scope="session")
def cuda(capi):
    if capi.device_count() < 1:
        pytest.fail("gpu test on a machine without a CUDA device")
    return True


def rel_l2(y, ref_y):
    y = np.asarray(y, np.float64)
    ref_y = np.asarray(ref_y, np.float64)
    den = np.linalg.norm(ref_y)
    return np.linalg.norm(y - ref_y) / (den if den > 0 else 1.0)


def max_rel(y, ref_y):
    ref_y = np.asarray(ref_y, np.float64)
    m = np.max(np.abs(ref_y)) if ref_y.size else 0.0
    return np.max(np.abs(np.asarray(y) - ref_y)) / (m if m > 0 else 1.0)


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


def csr_of(prefix, d):
    from oracle import Csr

    return Csr(int(d[f"{prefix}_n"]), d[f"{prefix}_row_ptr"], d[f"{prefix}_col_idx"],
               d[f"{prefix}_values"])
