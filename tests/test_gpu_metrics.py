"""The trainer's image metrics on the GPU: SSIM,
SSIM gradient, L1, L1 gradient against the real reference's outputs
(tests/golden/metrics.npz, ss/metrics.py:77-121).  SSIM is a separable
11-tap stencil on device vs scipy's direct 2D sum in the reference, so values
agree to rounding (checked at 1e-12 relative), not bit for bit; L1 and its
gradient are exact up to the summation order of the mean."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cid", [0, 1, 2, 3])
def test_metrics_match_reference(cid):
    from paper_2512_20943_b200 import metrics

    g = load_golden("metrics.npz")
    a, b = g[f"c{cid}_a"], g[f"c{cid}_b"]
    assert abs(metrics.ssim(a, b) - float(g[f"c{cid}_ssim"])) <= 1e-12 * abs(float(g[f"c{cid}_ssim"]))
    assert metrics.ssim(a, a) == pytest.approx(float(g[f"c{cid}_ssim_self"]), rel=1e-14)
    ga = metrics.ssim_grad(a, b)
    ref = g[f"c{cid}_ssim_grad"]
    assert ga.shape == ref.shape
    assert np.max(np.abs(ga - ref)) <= 1e-12 * np.max(np.abs(ref))
    assert abs(metrics.l1(a, b) - float(g[f"c{cid}_l1"])) <= 1e-14
    np.testing.assert_array_equal(metrics.l1_grad(a, b), g[f"c{cid}_l1_grad"])


def test_ssim_errors():
    from paper_2512_20943_b200 import metrics
    from paper_2512_20943_b200.errors import StructuralError

    with pytest.raises(StructuralError):
        metrics.ssim(np.zeros((10, 12, 3)), np.zeros((10, 12, 3)))
    with pytest.raises(StructuralError):
        metrics.ssim(np.zeros((12, 12, 3)), np.zeros((12, 13, 3)))
    with pytest.raises(StructuralError):
        metrics.ssim_grad(np.zeros((12, 12, 2)), np.zeros((12, 12, 2)))


def test_ssim_full_size_properties():
    """1352x1014 colour pair: SSIM in (0, 1], identical images give 1, the
    gradient vanishes at the optimum and matches a finite difference."""
    from paper_2512_20943_b200 import metrics

    rng = np.random.default_rng(5)
    a = rng.uniform(0, 1, (1014, 1352, 3))
    b = np.clip(a + rng.normal(0, 0.05, a.shape), 0, 1)
    s = metrics.ssim(a, b)
    assert 0.0 < s < 1.0
    assert metrics.ssim(a, a) == pytest.approx(1.0, abs=1e-12)
    assert np.max(np.abs(metrics.ssim_grad(a, a))) <= 1e-12
    g = metrics.ssim_grad(a, b)
    y, x, c = 500, 700, 1
    e = 1e-3
    ap, am = a.copy(), a.copy()
    ap[y, x, c] += e
    am[y, x, c] -= e
    fd = (metrics.ssim(ap, b) - metrics.ssim(am, b)) / (2 * e)
    assert abs(fd - g[y, x, c]) <= 1e-3 * abs(g[y, x, c])
