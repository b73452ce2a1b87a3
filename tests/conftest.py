import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) — runs through librrsvd_b200.so")
    config.addinivalue_line("markers", "slow: longer parity cases")


@pytest.fixture(scope="session")
def ctx():
    """The library context.  On a GPU box a failure here is a hard error (no CPU fallback)."""
    from paper_1504_00992_b200 import Context
    return Context(0)


@pytest.fixture(scope="session")
def ref():
    """The reference implementation (oracle/_ref, built from /root/reference by oracle/Makefile)."""
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref not built (make -C oracle)")
    R.set_threads(min(8, os.cpu_count() or 1))
    return R


def cplx_randn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
