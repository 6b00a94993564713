"""Rasterizer parity on the GPU: the CUDA path against the CPU oracle
(which tests/test_oracle.py pins to the reference's golden vectors).

Gates (BASELINE.json north star): usage counts / cull set / decisions
bit-exact; pixels within 1e-3 -- asserted here much tighter (1e-12) because
the fp64 path replays the reference op-for-op and only transcendental ulps
(exp/tanh) can differ."""

import numpy as np
import pytest

from conftest import random_params
from oracle import airgs_oracle as orc

pytestmark = pytest.mark.gpu

PIX_TOL = 1e-12  # north star allows 1e-3


def _cams(count, res, focal=None):
    from paper_2512_20943_b200.camera import ring_rig

    f = focal if focal is not None else res[0] * 40.0 / 48.0
    return ring_rig(count, radius=3.0, height=0.3, focal=f, resolution=res)


@pytest.mark.parametrize("deg,n,res", [(0, 500, (32, 32)), (0, 4000, (200, 120)), (1, 2000, (96, 72)),
                                        (0, 20000, (256, 256))])
def test_render_with_usage_matches_oracle(deg, n, res):
    from paper_2512_20943_b200 import rasterizer
    from paper_2512_20943_b200.model import GaussianFrame

    rng = np.random.default_rng(n + deg)
    p = random_params(rng, n, deg, spread=0.6)
    cams = _cams(3, res)
    imgs, usage = rasterizer.render_with_usage(GaussianFrame(params=p), cams)
    ref_imgs, ref_usage = orc.render_with_usage(p, cams)
    np.testing.assert_array_equal(usage.counts, ref_usage)
    for a, b in zip(imgs, ref_imgs):
        assert np.max(np.abs(a.pixels - b)) <= PIX_TOL


@pytest.mark.parametrize("near", [-0.2, -1.0])
def test_negative_near_clip_matches_oracle(near):
    """Cameras inside the cloud with a negative near plane: primitives at
    near_clip < z <= 0 are kept and composited first, as the reference's
    stable depth argsort orders them (ss/rasterizer.py:126-127); their
    32-bit list keys sit between frozen positions and positive depths."""
    from paper_2512_20943_b200 import rasterizer
    from paper_2512_20943_b200.camera import Camera
    from paper_2512_20943_b200.model import GaussianFrame

    rng = np.random.default_rng(7)
    p = random_params(rng, 3000, 0, spread=0.6)
    base = _cams(3, (96, 72))
    from paper_2512_20943_b200.camera import ring_rig

    inner = ring_rig(3, radius=0.35, height=0.1, focal=80.0, resolution=(96, 72))
    cams = [Camera(c.pose, c.focal, c.resolution, near_clip=near) for c in inner + base[:1]]
    z = [(p[:, :3] @ np.asarray(c.pose)[:3, :3].T + np.asarray(c.pose)[:3, 3])[:, 2] for c in cams]
    assert any(np.count_nonzero((zz > near) & (zz < 0)) > 50 for zz in z)  # negative depths are present
    imgs, usage = rasterizer.render_with_usage(GaussianFrame(params=p), cams)
    ref_imgs, ref_usage = orc.render_with_usage(p, cams)
    np.testing.assert_array_equal(usage.counts, ref_usage)
    for a, b in zip(imgs, ref_imgs):
        assert np.max(np.abs(a.pixels - b)) <= PIX_TOL


def test_render_single_view(rng, frame_factory, cam32):
    from paper_2512_20943_b200 import rasterizer

    f = frame_factory(rng, 12)
    img = rasterizer.render(f, cam32)
    assert np.max(np.abs(img.pixels - orc.render(f.params, cam32))) <= PIX_TOL
    assert np.all(img.pixels >= 0.0) and np.all(img.pixels <= 1.0)


def test_deterministic(rng, frame_factory, cam32):
    from paper_2512_20943_b200 import rasterizer

    f = frame_factory(rng, 200)
    a = rasterizer.render(f, cam32)
    b = rasterizer.render(f, cam32)
    np.testing.assert_array_equal(a.pixels, b.pixels)


def test_empty_frame_rejected(cam32):
    from paper_2512_20943_b200 import rasterizer
    from paper_2512_20943_b200.errors import StructuralError
    from paper_2512_20943_b200.model import GaussianFrame

    with pytest.raises(StructuralError):
        rasterizer.render(GaussianFrame(params=np.zeros((0, 17))), cam32)


def test_invalid_parameters_rejected(rng, cam32):
    from paper_2512_20943_b200 import rasterizer
    from paper_2512_20943_b200.errors import ValidationError
    from paper_2512_20943_b200.model import GaussianFrame

    p = random_params(rng, 10)
    p[3, 3:7] = 0.0  # zero quaternion (ss/rasterizer.py:105-106)
    with pytest.raises(ValidationError):
        rasterizer.render(GaussianFrame(params=p), cam32)
    p = random_params(rng, 10)
    p[5, 12] = np.nan
    with pytest.raises(ValidationError):
        rasterizer.render(GaussianFrame(params=p), cam32)


def test_behind_camera_invisible(cam32):
    from paper_2512_20943_b200 import rasterizer
    from paper_2512_20943_b200.model import GaussianFrame

    params = np.zeros((1, 17))
    params[0, 0:3] = [0.0, 0.0, -10.0]
    params[0, 3] = 1.0
    params[0, 7:10] = np.log(0.2)
    params[0, 10] = 5.0
    params[0, 11:14] = 5.0
    img = rasterizer.render(GaussianFrame(params=params), cam32)
    assert np.all(img.pixels == 0.0)


def test_zero_usage_removal_is_bit_identical(rng, frame_factory, cam32):
    from paper_2512_20943_b200 import rasterizer

    f = frame_factory(rng, 15)
    params = f.params.copy()
    params[7, 0:3] = (50.0, 50.0, 0.0)
    f = f.with_params(params)
    _, usage = rasterizer.render_with_usage(f, [cam32])
    unused = np.nonzero(usage.counts == 0)[0]
    assert unused.size > 0
    keep = np.setdiff1d(np.arange(f.count), unused)
    ref = rasterizer.render(f, cam32)
    cut = rasterizer.render(f.with_params(f.params[keep]), cam32)
    np.testing.assert_array_equal(ref.pixels, cut.pixels)


def test_usage_merge(rng, frame_factory, two_cams):
    from paper_2512_20943_b200 import rasterizer

    f = frame_factory(rng, 10)
    _, u_all = rasterizer.render_with_usage(f, two_cams)
    _, u0 = rasterizer.render_with_usage(f, [two_cams[0]])
    _, u1 = rasterizer.render_with_usage(f, [two_cams[1]])
    np.testing.assert_array_equal(u_all.counts, u0.merged_with(u1).counts)


def _kernel_inputs(rng, n, side):
    means2d = rng.uniform(2, side - 2, (n, 2))
    conics = np.zeros((n, 3))
    conics[:, 0] = rng.uniform(0.05, 0.4, n)
    conics[:, 2] = rng.uniform(0.05, 0.4, n)
    alphas = rng.uniform(0.2, 0.95, n)
    colors = rng.uniform(0, 1, (n, 3))
    bboxes = np.zeros((n, 4), dtype=np.int64)
    bboxes[:, 1] = side
    bboxes[:, 3] = side
    return means2d, conics, alphas, colors, bboxes


def test_seam_forward_matches_oracle(rng):
    """The reference kernel seam (_composite.pyx:18): image, T and usage."""
    from paper_2512_20943_b200 import rasterizer

    args = _kernel_inputs(rng, 12, 28)
    img, tr, us, masks = rasterizer.forward(*args, 28, 28)
    ri, rt, ru = orc.composite(*args, 28, 28)
    assert masks is None
    assert np.max(np.abs(img - ri)) <= PIX_TOL
    assert np.max(np.abs(tr - rt)) <= PIX_TOL
    np.testing.assert_array_equal(us, ru)


def test_seam_conservation_unit_colors(rng):
    """rgb = 1 - T with unit colours (reference test_rasterizer.py:59-68)."""
    from paper_2512_20943_b200 import rasterizer

    m2, co, al, _, bb = _kernel_inputs(rng, 10, 24)
    img, tr, _, _ = rasterizer.forward(m2, co, al, np.ones((10, 3)), bb, 24, 24)
    np.testing.assert_allclose(img[:, :, 0], 1.0 - tr, atol=1e-12)
    np.testing.assert_array_equal(img[:, :, 0], img[:, :, 1])
    assert np.all(tr > 0.0) and np.all(tr <= 1.0)


def test_seam_prepared_scene(rng):
    """Seam on a projected scene at a non-multiple-of-16 resolution."""
    from paper_2512_20943_b200 import rasterizer

    p = random_params(rng, 3000, 0, spread=0.6)
    cam = _cams(1, (200, 120))[0]
    pr = orc.prepare(p, cam)
    img, tr, us, _ = rasterizer.forward(pr.means2d, pr.conics, pr.alphas, pr.colors, pr.bboxes, 120, 200)
    ri, rt, ru = orc.composite(pr.means2d, pr.conics, pr.alphas, pr.colors, pr.bboxes, 120, 200)
    np.testing.assert_array_equal(us, ru)
    assert np.max(np.abs(img - ri)) <= PIX_TOL
    assert np.max(np.abs(tr - rt)) <= PIX_TOL


def test_psnr_device(rng):
    from paper_2512_20943_b200 import metrics

    a = rng.uniform(0, 1, (16, 16, 3))
    assert metrics.psnr(a, a) == 100.0
    assert metrics.psnr(np.zeros((8, 8, 3)), np.full((8, 8, 3), 0.1)) == pytest.approx(20.0, abs=1e-12)
    b = rng.uniform(0, 1, (16, 16, 3))
    assert abs(metrics.psnr(a, b) - orc.psnr(a, b)) <= 1e-9
    from paper_2512_20943_b200.errors import StructuralError

    with pytest.raises(StructuralError):
        metrics.psnr(np.zeros((8, 8, 3)), np.zeros((9, 8, 3)))


def test_seam_oversized_tile_list_fallback(rng):
    """> 2048 primitives on one tile exercise the radix-sort fallback for
    lists too long for the shared-memory sort."""
    from paper_2512_20943_b200 import rasterizer

    n, side = 3000, 40
    means2d = rng.uniform(16, 32, (n, 2))
    conics = np.zeros((n, 3))
    conics[:, 0] = rng.uniform(0.2, 1.5, n)
    conics[:, 2] = rng.uniform(0.2, 1.5, n)
    alphas = rng.uniform(0.02, 0.3, n)
    colors = rng.uniform(0, 1, (n, 3))
    bboxes = np.zeros((n, 4), dtype=np.int64)
    bboxes[:, 0] = np.clip(np.floor(means2d[:, 0] - 6), 0, side)
    bboxes[:, 1] = np.clip(np.ceil(means2d[:, 0] + 6) + 1, 0, side)
    bboxes[:, 2] = np.clip(np.floor(means2d[:, 1] - 6), 0, side)
    bboxes[:, 3] = np.clip(np.ceil(means2d[:, 1] + 6) + 1, 0, side)
    img, tr, us, _ = rasterizer.forward(means2d, conics, alphas, colors, bboxes, side, side)
    ri, rt, ru = orc.composite(means2d, conics, alphas, colors, bboxes, side, side)
    np.testing.assert_array_equal(us, ru)
    assert np.max(np.abs(img - ri)) <= PIX_TOL
    assert np.max(np.abs(tr - rt)) <= PIX_TOL


@pytest.mark.parametrize("n,res", [(1500, (40, 32)), (6000, (48, 32))])
def test_render_bucket_overflow(n, res):
    """Dense views whose tiles overflow the fixed-capacity binning buckets
    (> 512 and > 2048 primitives per tile): the scanned-range fallback, the
    bucket capacity adaptation and the radix presort of oversized lists must
    give the oracle's result on every call."""
    from paper_2512_20943_b200 import rasterizer
    from paper_2512_20943_b200.model import GaussianFrame

    rng = np.random.default_rng(n)
    p = random_params(rng, n, 0, spread=0.25)
    cams = _cams(2, res)
    ref_imgs, ref_usage = orc.render_with_usage(p, cams)
    for _ in range(2):
        imgs, usage = rasterizer.render_with_usage(GaussianFrame(params=p), cams)
        np.testing.assert_array_equal(usage.counts, ref_usage)
        for a, b in zip(imgs, ref_imgs):
            assert np.max(np.abs(a.pixels - b)) <= PIX_TOL


def test_depth_ties_resolved_by_index(rng):
    """Primitives at identical depth composite in index order (stable
    argsort, ss/rasterizer.py:127)."""
    from paper_2512_20943_b200 import rasterizer
    from paper_2512_20943_b200.model import GaussianFrame

    p = random_params(rng, 400, 0, spread=0.5)
    p[:, 2] = 0.1  # every primitive at the same depth for a camera looking along z
    from paper_2512_20943_b200.camera import look_at

    cam = look_at((0.0, 0.0, -2.5), (0.0, 0.0, 0.0), focal=60.0, resolution=(64, 48))
    imgs, usage = rasterizer.render_with_usage(GaussianFrame(params=p), [cam])
    ri, ru = orc.render_with_usage(p, [cam])
    np.testing.assert_array_equal(usage.counts, ru)
    assert np.max(np.abs(imgs[0].pixels - ri[0])) <= PIX_TOL


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_eval_stats_match_reference_loop_counts(cfg):
    """The diagnostic counters behind bench.py's algorithmic-work roofline:
    bbox / live / contributing pair counts equal the reference loop's, per
    view, exactly (C1: 4 views; C2: one full view)."""
    from dataclasses import replace

    from paper_2512_20943_b200 import _lib, synth
    from paper_2512_20943_b200.model import GaussianFrame
    from paper_2512_20943_b200.rasterizer import render_views

    c = synth.CONFIGS[cfg]
    if cfg == "C2":
        c = replace(c, views=1)
    p = synth.Sequence(c, seed=7, event_every=0).frame(0)
    cams = synth.cameras(c)
    eng = _lib.engine()
    fr = GaussianFrame(params=p)
    eng.eval_stats(1)
    try:
        for v, cam in enumerate(cams):
            render_views([fr], cams, [(0, v)], want_images=True, usage_frames=[0])
            got = eng.eval_stats(1)  # read + reset
            assert (got["bbox"], got["live"], got["contrib"]) == orc.eval_counts(p, cam)
    finally:
        eng.eval_stats(0)


def test_decision_margins_match_reference_quantities(rng):
    """airgs_eval_margins against the same quantities computed from the
    oracle's projection and a direct replay of the reference loop: bbox
    floor/ceil, near-clip and opacity-cull margins exactly; the termination
    margin to 1e-9; the weight margin exactly where it is below the fp32
    guard band (every such pair is evaluated in fp64), else a lower bound;
    the tile-list depth gap is bounded below by the view's global one."""
    from paper_2512_20943_b200 import _lib, rasterizer
    from paper_2512_20943_b200.model import GaussianFrame

    p = random_params(rng, 300, 0, spread=0.5)
    cam = _cams(1, (40, 32))[0]
    eng = _lib.engine()
    eng.eval_stats(1)
    try:
        rasterizer.render_with_usage(GaussianFrame(params=p), [cam])
        m = eng.eval_margins()
    finally:
        eng.eval_stats(0)
    pr = orc.prepare(p, cam)
    eps = 1.0 / 255.0
    live = pr.alpha_all > eps
    mx, my, r = pr.means2d[:, 0], pr.means2d[:, 1], pr.radius
    dist = lambda x: np.abs(x - np.rint(x))  # noqa: E731
    bbm = min(dist(mx - r).min(), dist(mx + r).min(), dist(my - r).min(), dist(my + r).min())
    assert m["min_bbox_floor_margin_px"] == bbm
    assert m["min_near_clip_margin"] == np.abs(pr.z_all[live] - cam.near_clip).min()
    assert m["min_rel_alpha_cull_margin"] == (np.abs(pr.alpha_all - eps) / eps).min()
    z = np.sort(pr.depth)
    gaps = np.diff(z.view(np.int64))
    gaps = gaps[gaps > 0]
    if gaps.size:
        assert m["min_depth_gap_ulps"] >= gaps.min()
    # the reference loop, pixel-major, weight and termination margins
    H, W = cam.resolution[1], cam.resolution[0]
    wmin, wlive, tmin = np.inf, np.inf, np.inf
    a, b, c = pr.conics[:, 0], pr.conics[:, 1], pr.conics[:, 2]
    for y in range(H):
        for x in range(W):
            sel = np.nonzero((pr.bboxes[:, 0] <= x) & (x < pr.bboxes[:, 1]) & (pr.bboxes[:, 2] <= y)
                             & (y < pr.bboxes[:, 3]))[0]
            T = 1.0
            for k in sel:  # every pair, as the reference (no early exit)
                dx, dy = x + 0.5 - mx[k], y + 0.5 - my[k]
                e = 0.5 * (a[k] * dx * dx + c[k] * dy * dy) + b[k] * dx * dy
                ap = min(pr.alphas[k] * np.exp(-e), 0.999)
                w = ap * T
                if 0.999 * T > eps:
                    wlive = min(wlive, abs(w - eps) / eps)
                wmin = min(wmin, abs(w - eps) / eps)
                if w > eps:
                    T = T * (1.0 - ap)
                    tmin = min(tmin, abs(0.999 * T - eps) / eps)
    assert np.isfinite(tmin)
    assert abs(m["min_rel_termination_margin"] - tmin) <= 1e-9 * tmin
    # the device evaluates a subset of the weight tests in fp64 (the fp32 pass
    # rejects the rest with margin >= ~4e-5): never below the true minimum, and
    # equal to it when the minimum is a live test inside the guard band
    assert m["min_rel_weight_margin"] >= wmin * (1 - 1e-9)
    if wlive < 4e-5 and wlive < tmin:
        assert abs(m["min_rel_weight_margin"] - wlive) <= 1e-9 * wlive
