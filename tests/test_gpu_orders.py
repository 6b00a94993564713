"""Training kernels on the device path: frozen
compositing orders and a frozen-order forward/backward against the real
reference (tests/golden/train.npz).  The trainer itself (ss/train.py) is out
of scope."""

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
