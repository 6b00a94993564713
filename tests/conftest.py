"""Shared fixtures.  Mirrors the reference suite's fixtures
(/root/reference/pkg/tests/conftest.py:13-66) so the parity tests read like
the reference's own tests; ``gpu`` marks tests that need a B200."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA sm_100 device (B200)")


@pytest.fixture
def rng():
    return np.random.default_rng(0)


@pytest.fixture
def cam32():
    from paper_2512_20943_b200.camera import look_at

    return look_at((0.0, 0.0, -2.5), (0.0, 0.0, 0.0), focal=40.0, resolution=(32, 32))


@pytest.fixture
def two_cams():
    from paper_2512_20943_b200.camera import look_at

    return [
        look_at((0.0, 0.0, -2.5), (0.0, 0.0, 0.0), focal=40.0, resolution=(32, 32)),
        look_at((2.5, 0.3, 0.0), (0.0, 0.0, 0.0), focal=40.0, resolution=(32, 32)),
    ]


def random_params(rng, n, sh_degree=0, spread=0.4):
    """The reference's random_frame recipe (conftest.py:31-43)."""
    width = 14 + 3 * (sh_degree + 1) ** 2
    p = np.zeros((n, width))
    p[:, 0:3] = rng.uniform(-spread, spread, (n, 3))
    p[:, 3:7] = rng.normal(size=(n, 4))
    p[:, 3:7] /= np.linalg.norm(p[:, 3:7], axis=1, keepdims=True)
    p[:, 7:10] = np.log(rng.uniform(0.05, 0.2, (n, 3)))
    p[:, 10] = rng.uniform(0.5, 3.0, n)
    p[:, 11:14] = rng.normal(0, 1.0, (n, 3))
    if sh_degree >= 1:
        p[:, 14:] = rng.normal(0, 0.1, (n, width - 14))
    return p


@pytest.fixture
def frame_factory():
    from paper_2512_20943_b200.model import GaussianFrame

    def make(rng, n, sh_degree=0, spread=0.4):
        return GaussianFrame(params=random_params(rng, n, sh_degree, spread), frame_index=0, group_key=0)

    return make


def load_golden(name):
    path = os.path.join(GOLDEN, name)
    with np.load(path, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}
