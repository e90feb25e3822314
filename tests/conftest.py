"""Shared fixtures.  ``-m gpu`` tests need a B200 (they call the CUDA path
through the C-ABI); everything else runs on CPU.  The oracle package is test
infrastructure: tests use it only as the checker."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# parity tolerance of the north star: |a-b| <= ABS + REL*max(|a|,|b|)
REL_TOL = 1e-5
ABS_TOL = 1e-6


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def orc():
    import oracle

    if not oracle.oracle_available():
        oracle.build(with_reference=False)
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.reference_available():
        if os.path.isdir("/root/reference/proj/src"):
            oracle.build(with_reference=True)
        else:
            pytest.skip("reference build (oracle/_ref) not available")
    return oracle.Reference()


@pytest.fixture(scope="session")
def gmi():
    import paper_2012_13257_b200 as gmi

    return gmi


@pytest.fixture(scope="session")
def ctx(gmi):
    return gmi.Context(0)


def assert_close(got, want, rel=REL_TOL, abs_=ABS_TOL, what=""):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert got.shape == want.shape, f"{what}: shape {got.shape} vs {want.shape}"
    diff = np.abs(got - want)
    bound = abs_ + rel * np.maximum(np.abs(got), np.abs(want))
    bad = diff > bound
    if bad.any():
        k = np.argmax(diff - bound)
        raise AssertionError(
            f"{what}: {int(bad.sum())}/{bad.size} entries out of tolerance; worst at flat "
            f"{k}: got {got.flat[k]!r} want {want.flat[k]!r} (|d|={diff.flat[k]:.3e})")
