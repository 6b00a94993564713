"""GPU: the CUDA path against the reference's own outputs
(tests/golden/*.npz made by tests/golden/make_golden.py from the real
reference).  Integer/byte/index/decision outputs bit-exact; compositing
(the kernel seam) bit-exact; rendered pixels 1e-12;
PSNR-derived qualities 1e-6 dB (north star: 1e-3 px, 0.01 dB)."""

import numpy as np
import pytest

from conftest import load_golden
from test_oracle import cams_from

pytestmark = pytest.mark.gpu
PIX = 1e-12
DB = 1e-6


def test_render_and_usage_vs_reference():
    from paper_2512_20943_b200 import rasterizer
    from paper_2512_20943_b200.model import GaussianFrame

    g = load_golden("render.npz")
    for cid in range(4):
        cams = cams_from(g, f"c{cid}_")
        imgs, usage = rasterizer.render_with_usage(GaussianFrame(params=g[f"c{cid}_params"]), cams)
        np.testing.assert_array_equal(usage.counts, g[f"c{cid}_usage"])
        for v, im in enumerate(imgs):
            assert np.max(np.abs(im.pixels - g[f"c{cid}_v{v}_image"])) <= PIX


def test_seam_vs_reference_kernel():
    from paper_2512_20943_b200 import rasterizer

    g = load_golden("composite.npz")
    for cid in range(2):
        args = [g[f"k{cid}_{k}"] for k in ("means2d", "conics", "alphas", "colors", "bboxes")]
        h, w = (int(v) for v in g[f"k{cid}_hw"])
        img, tr, us, _ = rasterizer.forward(*args, h, w)
        np.testing.assert_array_equal(us, g[f"k{cid}_usage"])
        # compositing alone is bit-identical to the reference kernel (glibc's exp on the device)
        np.testing.assert_array_equal(img, g[f"k{cid}_image"])
        np.testing.assert_array_equal(tr, g[f"k{cid}_trans"])


def test_seam_on_reference_prepared_views():
    """The seam fed the reference's own _prepare outputs reproduces its
    images bit for bit and its usage counts per view (depth order given); the
    full render's pixels (next tests) differ only through the projection's
    NumPy SIMD exp/tanh (<= 1e-15)."""
    from paper_2512_20943_b200 import rasterizer

    g = load_golden("render.npz")
    for cid in range(4):
        cams = cams_from(g, f"c{cid}_")
        total = np.zeros(g[f"c{cid}_params"].shape[0], dtype=np.int64)
        for v, cam in enumerate(cams):
            W, H = cam.resolution
            img, _, us, _ = rasterizer.forward(*[g[f"c{cid}_v{v}_{k}"] for k in
                                                 ("means2d", "conics", "alphas", "colors", "bboxes")], H, W)
            total[g[f"c{cid}_v{v}_order"]] += us
            np.testing.assert_array_equal(np.clip(img, 0, 1), g[f"c{cid}_v{v}_image"])
        np.testing.assert_array_equal(total, g[f"c{cid}_usage"])


def test_codec_vs_reference():
    from paper_2512_20943_b200 import codec
    from paper_2512_20943_b200.model import DeltaTensor, GaussianFrame

    g = load_golden("codec.npz")
    for cid in range(3):
        blob = g[f"gsai{cid}_blob"].tobytes()
        enc = codec.encode_frame(GaussianFrame(params=g[f"gsai{cid}_params"], frame_index=3, group_key=3))
        assert enc.to_bytes() == blob
        dec = codec.decode_frame(codec.AttributeImageSet.from_bytes(blob))
        np.testing.assert_array_equal(dec.params, g[f"gsai{cid}_decoded"])
    for cid in range(4):
        n, step = int(g[f"gsdp{cid}_n"][0]), float(g[f"gsdp{cid}_step"][0])
        d = DeltaTensor(n, 17, {int(i): r for i, r in zip(g[f"gsdp{cid}_idx"], g[f"gsdp{cid}_rows"])})
        pay = codec.encode_delta(d, step, frame_index=7, base_key=2)
        assert pay.data == g[f"gsdp{cid}_blob"].tobytes()
        back = codec.decode_delta(pay, n, 17)
        np.testing.assert_array_equal(back.indices(), g[f"gsdp{cid}_dec_idx"])
        ent = back.entries
        for i, r in zip(g[f"gsdp{cid}_dec_idx"].tolist(), g[f"gsdp{cid}_dec_rows"]):
            np.testing.assert_array_equal(ent[i], r)


def test_delta_algebra_vs_reference():
    from paper_2512_20943_b200.model import CanonicalSpace, DeltaTensor, GaussianFrame, apply_delta, compose_deltas

    g = load_golden("delta.npz")
    n = g["canon"].shape[0]
    a = DeltaTensor(n, 17, {int(i): r for i, r in zip(g["a_idx"], g["a_rows"])})
    b = DeltaTensor(n, 17, {int(i): r for i, r in zip(g["b_idx"], g["b_rows"])})
    c = compose_deltas([a, b.negate(), a])
    np.testing.assert_array_equal(c.indices(), g["c_idx"])
    fr = apply_delta(CanonicalSpace(GaussianFrame(params=g["canon"]), n), c, frame_index=4)
    np.testing.assert_array_equal(fr.params, g["applied"])


@pytest.mark.parametrize("cid", [0, 1])
def test_level_space_vs_reference(cid):
    from paper_2512_20943_b200.model import CanonicalSpace, DeltaTensor, GaussianFrame
    from paper_2512_20943_b200.pruning import SelectionContext, build_level_space, ilp_optimal, select_pruning_level

    g = load_golden("pruning.npz")
    canon = g[f"p{cid}_canon"]
    n = canon.shape[0]
    space = CanonicalSpace(GaussianFrame(params=canon, frame_index=0, group_key=0), capacity_U=n)
    gap = DeltaTensor(n, 17, {int(i): r for i, r in zip(g[f"p{cid}_gap_idx"], g[f"p{cid}_gap_rows"])})
    base = None
    if g[f"p{cid}_base_idx"].size:
        base = DeltaTensor(n, 17, {int(i): r for i, r in zip(g[f"p{cid}_base_idx"], g[f"p{cid}_base_rows"])})
    ratios = [i / 10 for i in range(10)] + [1.0]
    lv = build_level_space(gap, space, cams_from(g, f"p{cid}_"), ratios, g[f"p{cid}_usage"], 1e-4, base=base,
                           frame_index=2)
    np.testing.assert_array_equal([x.ratio for x in lv.levels], g[f"p{cid}_ratios"])
    np.testing.assert_array_equal(lv.sizes(), g[f"p{cid}_sizes"])
    assert np.max(np.abs(np.array(lv.qualities()) - g[f"p{cid}_quality"])) <= DB
    flat = np.concatenate([np.array(x.pruned_indices, dtype=np.int64) for x in lv.levels])
    np.testing.assert_array_equal(flat, g[f"p{cid}_removed_flat"])
    for b, want, want_ilp in zip(g[f"p{cid}_budgets"], g[f"p{cid}_select"], g[f"p{cid}_ilp"]):
        ctx = SelectionContext(bandwidth_B=float(b) * 8.0, target_rate_R=1.0)
        assert select_pruning_level(lv, ctx) == want
        got = ilp_optimal([lv], [int(b)])[0]
        assert (-1 if got.level is None else got.level) == want_ilp


def test_frame_quality_vs_reference():
    from paper_2512_20943_b200 import grouping
    from paper_2512_20943_b200.model import CanonicalSpace, GaussianFrame, diff_frames

    g = load_golden("grouping.npz")
    cams = cams_from(g)
    target = grouping.GroundTruth(images=list(g["targets"]))
    q = grouping.frame_quality(GaussianFrame(params=g["a"]), cams, target)
    assert abs(q - float(g["q"][0])) <= DB
    space = CanonicalSpace(GaussianFrame(params=g["a"]), capacity_U=g["a"].shape[0])
    d = diff_frames(space.frame, GaussianFrame(params=g["b"]))
    assert abs(grouping.quality_probe(space, d, target, cams) - float(g["q_probe"][0])) <= DB


def test_session_vs_reference():
    """run_session through the device path: payload bytes, sizes, levels and
    ratios identical to the reference's own session; qualities 1e-6 dB."""
    from paper_2512_20943_b200 import grouping, streamsim
    from paper_2512_20943_b200.model import CanonicalSpace, DeltaTensor, GaussianFrame, diff_frames

    g = load_golden("session.npz")
    frames = g["frames"]
    n = frames.shape[1]
    space = CanonicalSpace(GaussianFrame(params=frames[0], frame_index=0, group_key=0), capacity_U=n)
    recs = []
    for t in range(frames.shape[0]):
        cum = diff_frames(space.frame, GaussianFrame(params=frames[t]))
        recs.append(grouping.FrameRecord(t, 0, t == 0, DeltaTensor.empty(n, 17), cum, 40.0))
    plan = grouping.GroupPlan(30.0, (grouping.GroupSpan(0, 0, frames.shape[0] - 1),))
    stream = grouping.TrainedStream(plan=plan, spaces={0: space}, records=recs)
    trace = streamsim.BandwidthTrace(g["trace_t"], g["trace_b"])
    cfg = streamsim.SimConfig(target_rate_R=1.0, quant_step=1e-4, ratios=(0.0, 0.3, 0.6, 0.9), cliff_beta=2.0)
    report, state, log = streamsim.run_session(stream, cams_from(g), trace, cfg)
    np.testing.assert_array_equal([f.sent_bytes for f in report.frames], g["sent"])
    np.testing.assert_array_equal([f.level for f in report.frames], g["level"])
    np.testing.assert_array_equal([f.prune_ratio for f in report.frames], g["ratio"])
    assert np.max(np.abs(np.array([f.client_quality_db for f in report.frames]) - g["quality"])) <= DB
    for t, pl in enumerate(log.payloads):
        data = pl if isinstance(pl, bytes) else pl.data
        assert data == g[f"payload{t}"].tobytes()
    np.testing.assert_array_equal(state.applied.dense(), g["applied_dense"])
    # pure client reconstruction from the received bytes matches the session state
    rec = streamsim.client_reconstruct(log.payloads[0], [p.data for p in log.payloads[1:]], frame_index=4)
    np.testing.assert_array_equal(rec.params, state.client_frame(4).params)
