"""Backward pass on the GPU against the real
reference's render_backward with its compiled _composite.backward
(tests/golden/backward.npz).  Every per-pixel recurrence replays the
reference's operations in the reference's order; only the summation over
pixels of each primitive's gradient is in a different (atomic) order, so
gradients agree to rounding: checked at 1e-9 relative to the largest
gradient of each parameter column (values are O(1e-3 .. 1e2))."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _cam(g, cid):
    from paper_2512_20943_b200.camera import Camera

    pose = g[f"c{cid}_cam_pose"][0]
    res = tuple(int(v) for v in g[f"c{cid}_cam_res"][0])
    return Camera(pose, float(g[f"c{cid}_cam_focal"][0]), res)


@pytest.mark.parametrize("cid", [0, 1, 2])
def test_render_backward_matches_reference(cid):
    from paper_2512_20943_b200 import rasterizer
    from paper_2512_20943_b200.model import GaussianFrame

    g = load_golden("backward.npz")
    frame = GaussianFrame(params=g[f"c{cid}_params"])
    cam = _cam(g, cid)
    image, state = rasterizer.render_forward(frame, cam)
    assert np.max(np.abs(image - g[f"c{cid}_image"])) <= 1e-12
    grads = rasterizer.render_backward(state, g[f"c{cid}_d_image"])
    ref = g[f"c{cid}_grads"]
    assert grads.shape == ref.shape
    scale = np.maximum(np.max(np.abs(ref), axis=0), 1e-300)
    err = np.max(np.abs(grads - ref), axis=0) / scale
    assert np.all(err <= 1e-9), err
    # primitives without a recorded contribution get exactly zero
    np.testing.assert_array_equal(grads[np.all(ref == 0, axis=1)], 0.0)


def test_render_backward_finite_difference():
    """Directional derivative of L = <d_image, render(params)> against a
    central difference on a small scene (same depth order at +-h)."""
    from paper_2512_20943_b200 import rasterizer
    from paper_2512_20943_b200.model import GaussianFrame

    g = load_golden("backward.npz")
    p = g["c0_params"].copy()
    cam = _cam(g, 0)
    rng = np.random.default_rng(9)
    d_image = rng.normal(0, 1, g["c0_image"].shape)
    _, st = rasterizer.render_forward(GaussianFrame(params=p), cam)
    grads = rasterizer.render_backward(st, d_image)
    direction = rng.normal(0, 1, p.shape) * 1e-3
    direction[:, 3:7] = 0.0  # keep quaternions away from the normalisation kink
    h = 1e-4

    def loss(q):
        im, _ = rasterizer.render_forward(GaussianFrame(params=q), cam)
        return float(np.sum(im * d_image))

    fd = (loss(p + h * direction) - loss(p - h * direction)) / (2 * h)
    an = float(np.sum(grads * direction))
    assert abs(fd - an) <= 1e-3 * abs(an) + 1e-9


@pytest.mark.parametrize("cid", [0, 1])
def test_seam_record_and_backward_match_reference(cid):
    """The kernel seam (ss/_composite.pyx:18-152): forward(record=True) image,
    T, usage and masks bit-identical to the reference's, backward(...) from the
    reference's masks and t_final to 1e-9 of each output's scale."""
    from paper_2512_20943_b200 import rasterizer

    g = load_golden("seam_backward.npz")
    a = [g[f"s{cid}_{k}"] for k in ("means2d", "conics", "alphas", "colors", "bboxes")]
    h, w = (int(v) for v in g[f"s{cid}_hw"])
    img, tr, us, masks = rasterizer.forward(*a, h, w, record=True)
    np.testing.assert_array_equal(us, g[f"s{cid}_usage"])
    np.testing.assert_array_equal(masks, g[f"s{cid}_masks"])
    # the compositing kernel is bit-identical to the reference's (its exp is glibc's)
    np.testing.assert_array_equal(img, g[f"s{cid}_image"])
    np.testing.assert_array_equal(tr, g[f"s{cid}_trans"])
    out = rasterizer.backward(*a, h, w, g[f"s{cid}_masks"], g[f"s{cid}_trans"], g[f"s{cid}_d_image"])
    for name, v in zip(("d_means2d", "d_conics", "d_alphas", "d_colors"), out):
        ref = g[f"s{cid}_{name}"]
        assert v.shape == ref.shape
        assert np.max(np.abs(v - ref)) <= 1e-9 * max(np.max(np.abs(ref)), 1e-300), name
