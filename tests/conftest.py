import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (runs through the C ABI)")
    config.addinivalue_line("markers", "slow: full-size configuration parity (GPU box)")


def rel_err(got, want):
    """reference tests/test_util.hpp:36-51 (relative L2)."""
    got = np.asarray(got)
    want = np.asarray(want)
    num = np.sqrt(np.sum(np.abs(got - want) ** 2))
    den = max(np.sqrt(np.sum(np.abs(want) ** 2)), 1e-300)
    return float(num / den)


def random_volume(dims, rng, lo=-1.0, hi=1.0):
    m, n, s = dims
    return rng.uniform(lo, hi, (s, n, m))


def random_spectrum(dims, rng):
    m, n, s = dims
    return rng.uniform(-1, 1, (s, n, m)) + 1j * rng.uniform(-1, 1, (s, n, m))


def random_psf(hr, ksz, rng):
    """reference tests/test_util.hpp:28-33 (explicit random ksz^3 kernel)."""
    import volsr_oracle as O
    w = rng.uniform(0.0, 1.0, ksz ** 3)
    return O.make_gaussian_psf((ksz, ksz, ksz), (0, 0, 0), hr, weights=w)


@pytest.fixture(scope="session")
def V():
    from paper_2010_15491_b200 import volsr
    return volsr


@pytest.fixture(scope="session")
def O():
    import volsr_oracle
    return volsr_oracle
