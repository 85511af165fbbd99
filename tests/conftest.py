"""Shared fixtures.  `-m gpu` tests need a B200 (sm_100) and call the product
through the C ABI; everything else runs on the CPU container."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as R
    if not R.available():
        pytest.fail("oracle/_ref/libkrylov_ref.so missing: run `make -C oracle ref` (built by __graft_entry__.build())")
    return R


@pytest.fixture(scope="session")
def kb():
    import paper_2402_15033_b200 as K
    return K


@pytest.fixture(scope="session")
def ctx(kb):
    # A GPU test must run the CUDA path; no device is a hard failure, not a skip.
    c = kb.get_context()
    yield c


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
