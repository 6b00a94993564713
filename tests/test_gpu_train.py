"""The trainer on the device path ("unlocks
training"): frozen compositing orders, a frozen-order forward/backward and
short fits of fit_group_frame / fit_keyframe against the real reference
(tests/golden/train.npz).  Host arithmetic is the reference's; device losses
and gradients agree to rounding, so the line-search decisions coincide and
the fitted parameters agree to ~1e-9."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _cams(g):
    from paper_2512_20943_b200.camera import Camera

    return [Camera(g["cam_pose"][k], float(g["cam_focal"][k]), tuple(int(v) for v in g["cam_res"][k]))
            for k in range(len(g["cam_focal"]))]


def test_compositing_orders_match_reference():
    from paper_2512_20943_b200 import rasterizer
    from paper_2512_20943_b200.model import GaussianFrame

    g = load_golden("train.npz")
    orders = rasterizer.compositing_orders(GaussianFrame(params=g["params"]), _cams(g))
    for k, o in enumerate(orders):
        np.testing.assert_array_equal(o, g[f"order{k}"])


def test_frozen_forward_backward_match_reference():
    from paper_2512_20943_b200 import rasterizer
    from paper_2512_20943_b200.model import GaussianFrame

    g = load_golden("train.npz")
    cam = _cams(g)[0]
    frame = GaussianFrame(params=g["frozen_q"])
    (fo,) = rasterizer.compositing_orders(frame, [cam], frozen_orders=[g["order0"]])
    np.testing.assert_array_equal(fo, g["frozen_order_used"])
    img, st = rasterizer.render_forward(frame, cam, frozen_order=g["order0"])
    assert np.max(np.abs(img - g["frozen_image"])) <= 1e-12
    grads = rasterizer.render_backward(st, g["frozen_d_image"])
    ref = g["frozen_grads"]
    scale = np.maximum(np.max(np.abs(ref), axis=0), 1e-300)
    assert np.all(np.max(np.abs(grads - ref), axis=0) / scale <= 1e-9)


def test_fit_group_frame_matches_reference():
    from paper_2512_20943_b200 import train
    from paper_2512_20943_b200.model import CanonicalSpace, DeltaTensor, GaussianFrame

    g = load_golden("train.npz")
    cams = _cams(g)
    target = train.GroundTruth(images=[g["target0"], g["target1"]])
    space = CanonicalSpace(GaussianFrame(params=g["params"], frame_index=0, group_key=0), capacity_U=250)
    d = train.fit_group_frame(space, DeltaTensor.empty(250, 17), target, cams, train.LossWeights(),
                              train.TrainConfig(iterations=3, step_size=0.05))
    ref = g["group_delta"]
    assert np.max(np.abs(d.dense() - ref)) <= 1e-9 * max(np.max(np.abs(ref)), 1e-12)


def test_fit_keyframe_matches_reference():
    from paper_2512_20943_b200 import train
    from paper_2512_20943_b200.model import GaussianFrame

    g = load_golden("train.npz")
    cams = _cams(g)
    target = train.GroundTruth(images=[g["target0"], g["target1"]])
    ks = train.fit_keyframe(GaussianFrame(params=g["params"], frame_index=0, group_key=0), target, cams,
                            train.LossWeights(),
                            train.TrainConfig(iterations=4, step_size=0.05, densify_interval=2,
                                              densify_grad_threshold=1e-5, capacity_U=260))
    ref = g["key_params"]
    assert ks.frame.params.shape == ref.shape
    assert ks.capacity_U == int(g["key_capacity"])
    assert np.max(np.abs(ks.frame.params - ref)) <= 1e-8 * max(np.max(np.abs(ref)), 1.0)


def test_build_groups_matches_reference():
    """The training-based grouping driver (ss/grouping.py:169-250) on a
    3-frame toy sequence: the same keyframe decisions (frame 1 a delta, frame
    2 a new group), qualities to 1e-6 dB, spaces and cumulative deltas 1e-8."""
    from paper_2512_20943_b200 import grouping, train

    g = load_golden("train.npz")
    cams = _cams(g)
    tgts = [train.GroundTruth(images=[g[f"bg_t{t}_c0"], g[f"bg_t{t}_c1"]]) for t in range(3)]
    stream = grouping.build_groups(tgts, cams, train.LossWeights(), train.TrainConfig(iterations=2, step_size=0.05),
                                   train.TrainConfig(iterations=3, step_size=0.05, densify_interval=2),
                                   (np.full(3, -0.5), np.full(3, 0.5)), 120, tau_db=18.9, seed=3)
    np.testing.assert_array_equal([r.is_keyframe for r in stream.records], g["bg_iskey"])
    assert np.max(np.abs(np.array([r.quality_db for r in stream.records]) - g["bg_quality"])) <= 1e-6
    for k, sp in stream.spaces.items():
        ref = g[f"bg_space{k}"]
        assert sp.frame.params.shape == ref.shape
        assert np.max(np.abs(sp.frame.params - ref)) <= 1e-8 * max(np.max(np.abs(ref)), 1.0)
    for r in stream.records:
        ref = g[f"bg_cum{r.frame_index}"]
        assert np.max(np.abs(r.cumulative_delta.dense() - ref)) <= 1e-8 * max(np.max(np.abs(ref)), 1e-12)
