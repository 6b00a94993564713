"""Generate tests/golden/*.npz by running the REAL reference implementation.

Requires /root/reference (read-only) and the reference's compiled kernel
built by `make -C oracle ref` (oracle/_ref/_composite*.so, compiled from the
reference's own Cython-generated C where it lies).  The reference package is
imported in place from /root/reference/pkg/src with that kernel injected as
`splatstream._composite`; nothing is copied into this repository.

    python tests/golden/make_golden.py

Every fixture stores the inputs and the reference outputs; tests/test_oracle.py
pins the CPU oracle to them and the GPU tests check the CUDA path against them.
"""

import glob
import importlib.util
import os
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"


def import_reference():
    sys.dont_write_bytecode = True
    hits = glob.glob(os.path.join(ROOT, "oracle", "_ref", "_composite*.so"))
    if not hits:
        raise SystemExit("build the reference kernel first: make -C oracle ref")
    spec = importlib.util.spec_from_file_location("splatstream._composite", hits[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    sys.modules["splatstream._composite"] = mod
    sys.path.insert(0, REF_SRC)
    import splatstream  # noqa: F401
    from splatstream import rasterizer

    assert rasterizer.KERNEL_BACKEND == "compiled", rasterizer.KERNEL_BACKEND
    return splatstream


def random_params(rng, n, sh_degree=0, spread=0.4):
    """The reference suite's random_frame recipe (tests/conftest.py:31-43)."""
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


def cam_arrays(cams):
    return {
        "cam_pose": np.stack([c.pose for c in cams]),
        "cam_focal": np.array([c.focal for c in cams], dtype=np.float64),
        "cam_res": np.array([c.resolution for c in cams], dtype=np.int64),
    }


def gen_render(ss):
    from splatstream import camera, model, rasterizer

    out = {}
    cases = [(0, 400, 0, (48, 40), 0.4, 3), (1, 300, 1, (33, 29), 0.4, 2), (2, 2000, 0, (96, 72), 0.6, 3),
             (3, 1500, 1, (64, 64), 0.6, 2)]
    for cid, n, deg, res, spread, ncam in cases:
        rng = np.random.default_rng(100 + cid)
        p = random_params(rng, n, deg, spread)
        cams = camera.ring_rig(ncam, radius=3.0, height=0.3, focal=res[0] * 40.0 / 48.0, resolution=res)
        f = model.GaussianFrame(params=p)
        imgs, usage = rasterizer.render_with_usage(f, cams)
        out[f"c{cid}_params"] = p
        for k, v in cam_arrays(cams).items():
            out[f"c{cid}_{k}"] = v
        out[f"c{cid}_usage"] = usage.counts
        for v, (cam, im) in enumerate(zip(cams, imgs)):
            pr = rasterizer._prepare(f, cam)
            out[f"c{cid}_v{v}_image"] = im.pixels
            out[f"c{cid}_v{v}_order"] = pr.order
            out[f"c{cid}_v{v}_means2d"] = pr.means2d
            out[f"c{cid}_v{v}_conics"] = pr.conics
            out[f"c{cid}_v{v}_alphas"] = pr.alphas
            out[f"c{cid}_v{v}_colors"] = pr.colors
            out[f"c{cid}_v{v}_bboxes"] = pr.bboxes
    np.savez_compressed(os.path.join(HERE, "render.npz"), **out)


def gen_composite(ss):
    from splatstream import _composite

    out = {}
    rng = np.random.default_rng(7)
    for cid, (n, side) in enumerate([(12, 28), (40, 37)]):
        means2d = rng.uniform(2, side - 2, (n, 2))
        conics = np.zeros((n, 3))
        conics[:, 0] = rng.uniform(0.05, 0.4, n)
        conics[:, 1] = rng.uniform(-0.02, 0.02, n)
        conics[:, 2] = rng.uniform(0.05, 0.4, n)
        alphas = rng.uniform(0.2, 0.95, n)
        colors = rng.uniform(0, 1, (n, 3))
        bboxes = np.zeros((n, 4), dtype=np.int64)
        bboxes[:, 1] = side
        bboxes[:, 3] = side
        img, tr, us, _ = _composite.forward(means2d, conics, alphas, colors, bboxes, side, side)
        for k, v in dict(means2d=means2d, conics=conics, alphas=alphas, colors=colors, bboxes=bboxes,
                         image=np.asarray(img), trans=np.asarray(tr), usage=np.asarray(us),
                         hw=np.array([side, side])).items():
            out[f"k{cid}_{k}"] = v
    np.savez_compressed(os.path.join(HERE, "composite.npz"), **out)


def gen_codec(ss):
    from splatstream import codec, model

    out = {}
    for cid, (n, deg) in enumerate([(5, 0), (37, 1), (1000, 0)]):
        rng = np.random.default_rng(200 + cid)
        p = random_params(rng, n, deg)
        blob = codec.encode_frame(model.GaussianFrame(params=p, frame_index=3, group_key=3)).to_bytes()
        back = codec.decode_frame(codec.AttributeImageSet.from_bytes(blob))
        out[f"gsai{cid}_params"] = p
        out[f"gsai{cid}_blob"] = np.frombuffer(blob, dtype=np.uint8)
        out[f"gsai{cid}_decoded"] = back.params
    for cid, (n, k, step) in enumerate([(12, 3, 1e-4), (5000, 1000, 1e-4), (100000, 2, 1e-3), (300, 300, 1e-2)]):
        rng = np.random.default_rng(300 + cid)
        idx = np.sort(rng.choice(n, k, replace=False))
        rows = rng.normal(0, 0.05, (k, 17))
        rows[::5] *= 1e-3  # some entries quantise to all zeros at coarse steps
        d = model.DeltaTensor(n, 17, {int(i): r for i, r in zip(idx, rows)})
        pay = codec.encode_delta(d, step, frame_index=7, base_key=2)
        back = codec.decode_delta(pay, n, 17)
        bi = np.array(sorted(back.entries), dtype=np.int64)
        out[f"gsdp{cid}_n"] = np.array([n])
        out[f"gsdp{cid}_step"] = np.array([step])
        out[f"gsdp{cid}_idx"] = idx
        out[f"gsdp{cid}_rows"] = rows
        out[f"gsdp{cid}_blob"] = np.frombuffer(pay.data, dtype=np.uint8)
        out[f"gsdp{cid}_dec_idx"] = bi
        out[f"gsdp{cid}_dec_rows"] = np.stack([back.entries[i] for i in bi.tolist()]) if bi.size else np.zeros((0, 17))
    np.savez_compressed(os.path.join(HERE, "codec.npz"), **out)


def gen_delta(ss):
    from splatstream import model

    out = {}
    rng = np.random.default_rng(400)
    n = 3000
    canon = random_params(rng, n)
    parts = []
    for k in (600, 900):
        idx = np.sort(rng.choice(n, k, replace=False))
        rows = rng.normal(0, 0.05, (k, 17))
        parts.append((idx, rows))
    a = model.DeltaTensor(n, 17, {int(i): r for i, r in zip(*parts[0])})
    b = model.DeltaTensor(n, 17, {int(i): r for i, r in zip(*parts[1])})
    c = model.compose_deltas([a, b.negate(), a])
    space = model.CanonicalSpace(model.GaussianFrame(params=canon), capacity_U=n)
    fr = model.apply_delta(space, c, frame_index=4)
    ci = np.array(sorted(c.entries), dtype=np.int64)
    out.update(canon=canon, a_idx=parts[0][0], a_rows=parts[0][1], b_idx=parts[1][0], b_rows=parts[1][1],
               c_idx=ci, c_rows=np.stack([c.entries[i] for i in ci.tolist()]), applied=fr.params)
    np.savez_compressed(os.path.join(HERE, "delta.npz"), **out)


def gen_pruning(ss):
    from splatstream import model, pruning, rasterizer, scene_gen

    out = {}
    # the reference suite's real level space (tests/test_pruning.py:130-138)
    spec = scene_gen.SceneSpec(num_blobs=5, num_frames=3, mover_fraction=0.6, motion_amplitude=0.12,
                               min_separation=0.4, blob_scale=0.18, seed=5)
    frames = scene_gen.gen_scene(spec)
    cams = scene_gen.default_rig(count=2, resolution=(32, 32))
    ratios = [i / 10 for i in range(10)] + [1.0]
    for cid, (fr0, fr1, base_scale) in enumerate([(frames[0], frames[2], 0.0), (frames[0], frames[2], 0.01)]):
        space = model.CanonicalSpace(frame=fr0, capacity_U=fr0.live_count())
        delta = model.diff_frames(fr0, fr1)
        _, usage = rasterizer.render_with_usage(fr1, cams)
        base = None
        bi = np.zeros(0, dtype=np.int64)
        br = np.zeros((0, 17))
        if base_scale:
            rng = np.random.default_rng(9)
            bi = np.arange(fr0.count, dtype=np.int64)[::2]
            br = rng.normal(0, base_scale, (bi.size, 17))
            base = model.DeltaTensor(fr0.count, 17, {int(i): r for i, r in zip(bi, br)})
        lv = pruning.build_level_space(delta, space, cams, ratios, usage, 1e-4, base=base, frame_index=2)
        di = np.array(sorted(delta.entries), dtype=np.int64)
        out[f"p{cid}_canon"] = fr0.params
        out[f"p{cid}_target"] = fr1.params
        out[f"p{cid}_gap_idx"] = di
        out[f"p{cid}_gap_rows"] = np.stack([delta.entries[i] for i in di.tolist()])
        out[f"p{cid}_base_idx"] = bi
        out[f"p{cid}_base_rows"] = br
        out[f"p{cid}_usage"] = usage.counts
        out[f"p{cid}_ratios"] = np.array([x.ratio for x in lv.levels])
        out[f"p{cid}_quality"] = np.array([x.quality_db for x in lv.levels])
        out[f"p{cid}_sizes"] = np.array([x.size_bytes for x in lv.levels], dtype=np.int64)
        rm = [np.array(x.pruned_indices, dtype=np.int64) for x in lv.levels]
        out[f"p{cid}_removed_flat"] = np.concatenate(rm) if rm else np.zeros(0, np.int64)
        out[f"p{cid}_removed_len"] = np.array([len(r) for r in rm], dtype=np.int64)
        budgets = sorted({24, 100, int(lv.levels[0].size_bytes), int(lv.levels[len(lv.levels) // 2].size_bytes), 10**7})
        sel = [pruning.select_pruning_level(lv, pruning.SelectionContext(bandwidth_B=b * 8.0, target_rate_R=1.0))
               for b in budgets]
        out[f"p{cid}_budgets"] = np.array(budgets, dtype=np.int64)
        out[f"p{cid}_select"] = np.array(sel, dtype=np.int64)
        ilp = pruning.ilp_optimal([lv] * len(budgets), budgets)
        out[f"p{cid}_ilp"] = np.array([-1 if s.level is None else s.level for s in ilp], dtype=np.int64)
        for k, v in cam_arrays(cams).items():
            out[f"p{cid}_{k}"] = v
    # hand-traced Algorithm 1 spaces (tests/test_pruning.py:90-101)
    np.savez_compressed(os.path.join(HERE, "pruning.npz"), **out)


def gen_grouping(ss):
    from splatstream import camera, grouping, model, rasterizer, train

    rng = np.random.default_rng(500)
    n = 1500
    a = random_params(rng, n, 0, 0.6)
    b = a.copy()
    m = rng.choice(n, 400, replace=False)
    b[m, 0:3] += rng.normal(0, 0.02, (m.size, 3))
    cams = camera.ring_rig(3, radius=3.0, height=0.3, focal=80 * 40.0 / 48.0, resolution=(80, 64))
    target = train.GroundTruth(images=tuple(rasterizer.render(model.GaussianFrame(params=b), c).pixels for c in cams))
    q = grouping.frame_quality(model.GaussianFrame(params=a), cams, target)
    space = model.CanonicalSpace(model.GaussianFrame(params=a), capacity_U=n)
    d = model.diff_frames(space.frame, model.GaussianFrame(params=b))
    qp = grouping.quality_probe(space, d, target, cams)
    out = dict(a=a, b=b, targets=np.stack(target.images), q=np.array([q]), q_probe=np.array([qp]), **cam_arrays(cams))
    np.savez_compressed(os.path.join(HERE, "grouping.npz"), **out)


def gen_session(ss):
    """A 5-frame streaming session over a training-free stream (records built
    from ground-truth deltas) through the reference's own
    run_session."""
    from splatstream import camera, grouping, model, streamsim

    rng = np.random.default_rng(600)
    n = 1200
    base = random_params(rng, n, 0, 0.6)
    movers = rng.choice(n, 240, replace=False)
    frames = [base]
    for t in range(1, 5):
        p = frames[-1].copy()
        p[movers, 0:3] += rng.normal(0, 0.004, (movers.size, 3))
        frames.append(p)
    space = model.CanonicalSpace(model.GaussianFrame(params=base, frame_index=0, group_key=0), capacity_U=n)
    recs = []
    for t, p in enumerate(frames):
        cum = model.diff_frames(space.frame, model.GaussianFrame(params=p))
        recs.append(grouping.FrameRecord(t, 0, t == 0, model.DeltaTensor.empty(n, 17), cum, 40.0))
    plan = grouping.GroupPlan(30.0, (grouping.GroupSpan(0, 0, 4),))
    stream = grouping.TrainedStream(plan=plan, spaces={0: space}, records=tuple(recs))
    cams = camera.ring_rig(2, radius=3.0, height=0.3, focal=64 * 40.0 / 48.0, resolution=(64, 48))
    trace = streamsim.BandwidthTrace(np.array([0.0, 2.0, 10.0]), np.array([2.0e6, 0.4e6, 0.4e6]))
    cfg = streamsim.SimConfig(target_rate_R=1.0, quant_step=1e-4, ratios=(0.0, 0.3, 0.6, 0.9), cliff_beta=2.0)
    report, state, log = streamsim.run_session(stream, cams, trace, cfg)
    out = dict(frames=np.stack(frames), **cam_arrays(cams),
               sent=np.array([f.sent_bytes for f in report.frames], dtype=np.int64),
               level=np.array([f.level for f in report.frames], dtype=np.int64),
               ratio=np.array([f.prune_ratio for f in report.frames]),
               quality=np.array([f.client_quality_db for f in report.frames]),
               is_key=np.array([f.is_keyframe for f in report.frames]),
               applied_dense=state.applied.dense(),
               trace_t=trace.times_s, trace_b=trace.bandwidth_bps)
    for t, pl in enumerate(log.payloads):
        data = pl if isinstance(pl, bytes) else pl.data
        out[f"payload{t}"] = np.frombuffer(data, dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "session.npz"), **out)


def gen_metrics(ss):
    """SSIM / SSIM gradient / L1 / L1 gradient (ss/metrics.py:77-121) on
    colour and grey image pairs."""
    from splatstream import metrics

    out = {}
    cases = [(0, (24, 31, 3)), (1, (16, 16)), (2, (40, 57, 3)), (3, (11, 11, 3))]
    for cid, shape in cases:
        rng = np.random.default_rng(700 + cid)
        a = rng.uniform(0, 1, shape)
        b = np.clip(a + rng.normal(0, 0.1, shape), 0, 1)
        out[f"c{cid}_a"], out[f"c{cid}_b"] = a, b
        out[f"c{cid}_ssim"] = np.array(metrics.ssim(a, b))
        out[f"c{cid}_ssim_grad"] = metrics.ssim_grad(a, b)
        out[f"c{cid}_l1"] = np.array(metrics.l1(a, b))
        out[f"c{cid}_l1_grad"] = metrics.l1_grad(a, b)
        out[f"c{cid}_ssim_self"] = np.array(metrics.ssim(a, a))
    np.savez_compressed(os.path.join(HERE, "metrics.npz"), **out)


def gen_backward(ss):
    """render_forward / render_backward (ss/rasterizer.py:248-369, the
    compiled _composite.backward): per-parameter gradients of a random
    image-space loss gradient, SH degrees 0 and 1."""
    from splatstream import camera, model, rasterizer

    out = {}
    cases = [(0, 300, 0, (40, 32), 0.4), (1, 250, 1, (33, 29), 0.4), (2, 1200, 0, (72, 56), 0.6)]
    for cid, n, deg, res, spread in cases:
        rng = np.random.default_rng(800 + cid)
        p = random_params(rng, n, deg, spread)
        cam = camera.ring_rig(2, radius=3.0, height=0.3, focal=res[0] * 40.0 / 48.0, resolution=res)[1]
        f = model.GaussianFrame(params=p)
        image, state = rasterizer.render_forward(f, cam)
        d_image = rng.normal(0, 1.0, image.shape)
        grads = rasterizer.render_backward(state, d_image)
        out[f"c{cid}_params"] = p
        for k, v in cam_arrays([cam]).items():
            out[f"c{cid}_{k}"] = v
        out[f"c{cid}_image"] = image
        out[f"c{cid}_d_image"] = d_image
        out[f"c{cid}_grads"] = grads
        prep, t_final, masks = state
        out[f"c{cid}_t_final"] = t_final
        d2 = rasterizer._kernels.backward(prep.means2d, prep.conics, prep.alphas, prep.colors, prep.bboxes,
                                          res[1], res[0], masks, t_final, np.ascontiguousarray(d_image))
        for name, v in zip(("d_means2d", "d_conics", "d_alphas", "d_colors"), d2):
            out[f"c{cid}_{name}"] = v
        out[f"c{cid}_order"] = prep.order
    np.savez_compressed(os.path.join(HERE, "backward.npz"), **out)


def gen_io(ss):
    """A GSSC scene (2 frames, SH degree 1) and a trained-stream .npz written
    by the reference's own save_scene / save_stream (ss/model.py:318-329,
    ss/grouping.py:108-122), plus the values they hold."""
    from splatstream import grouping, model

    rng = np.random.default_rng(900)
    frames = [model.GaussianFrame(params=random_params(rng, n, 1, 0.5), frame_index=t)
              for t, n in enumerate((37, 41))]
    model.save_scene(os.path.join(HERE, "io_scene.gssc"), frames)
    base = random_params(rng, 30, 0, 0.5)
    space = model.CanonicalSpace(model.GaussianFrame(params=base, frame_index=0, group_key=0), capacity_U=32)
    recs = []
    cum = model.DeltaTensor.empty(30, 17)
    for t in range(3):
        step = model.DeltaTensor.from_dense(np.where(rng.uniform(0, 1, (30, 17)) < 0.2,
                                                     rng.normal(0, 1e-3, (30, 17)), 0.0))
        cum = model.compose_deltas([cum, step])
        recs.append(grouping.FrameRecord(t, 0, t == 0, step, cum, 40.0 - t))
    plan = grouping.GroupPlan(30.0, (grouping.GroupSpan(0, 0, 2),))
    grouping.save_stream(os.path.join(HERE, "io_stream.npz"),
                         grouping.TrainedStream(plan=plan, spaces={0: space}, records=recs))
    np.savez_compressed(os.path.join(HERE, "io_values.npz"), f0=frames[0].params, f1=frames[1].params, base=base,
                        **{f"cum{t}": r.cumulative_delta.dense() for t, r in enumerate(recs)},
                        **{f"step{t}": r.step_delta.dense() for t, r in enumerate(recs)})


def gen_train(ss):
    """Frozen compositing orders and short fits of the reference trainer
    (ss/train.py:262-292, 370-486): compositing_orders, a frozen-order
    forward/backward, fit_group_frame and fit_keyframe (with one
    densification event) on a small scene."""
    from splatstream import camera, model, rasterizer, train

    out = {}
    rng = np.random.default_rng(1000)
    p = random_params(rng, 250, 0, 0.45)
    cams = camera.ring_rig(2, radius=3.0, height=0.3, focal=40.0, resolution=(48, 40))
    for k, v in cam_arrays(cams).items():
        out[k] = v
    out["params"] = p
    moved = p.copy()
    sel = rng.uniform(0, 1, p.shape[0]) < 0.3
    moved[sel, 0:3] += rng.normal(0, 0.02, (int(sel.sum()), 3))
    out["moved"] = moved
    # targets = renders of the moved scene plus noise: an exact render would sit
    # on L1's kink (sign(0)) wherever the fit's render equals it bit for bit,
    # where a 1-ulp exp difference flips the subgradient
    target = train.GroundTruth(images=tuple(
        np.clip(rasterizer.render(model.GaussianFrame(params=moved), c).pixels + rng.normal(0, 0.01, (40, 48, 3)),
                0, 1) for c in cams))
    for k, im in enumerate(target.images):
        out[f"target{k}"] = im
    orders = rasterizer.compositing_orders(model.GaussianFrame(params=p), cams)
    for k, o in enumerate(orders):
        out[f"order{k}"] = o
    # frozen forward / backward at the moved parameters (depths crossed, some primitives culled)
    q = moved.copy()
    q[:5, 10] = -8.0  # below the contribution quantum: absent from the frozen order's kept set
    img, st = rasterizer.render_forward(model.GaussianFrame(params=q), cams[0], frozen_order=orders[0])
    d_image = rng.normal(0, 1, img.shape)
    out["frozen_q"] = q
    out["frozen_image"] = img
    out["frozen_d_image"] = d_image
    out["frozen_grads"] = rasterizer.render_backward(st, d_image)
    out["frozen_order_used"] = st[0].order
    space = model.CanonicalSpace(model.GaussianFrame(params=p, frame_index=0, group_key=0), capacity_U=250)
    weights = train.LossWeights()
    d = train.fit_group_frame(space, model.DeltaTensor.empty(250, 17), target, cams, weights,
                              train.TrainConfig(iterations=3, step_size=0.05))
    out["group_delta"] = d.dense()
    ks = train.fit_keyframe(model.GaussianFrame(params=p, frame_index=0, group_key=0), target, cams, weights,
                            train.TrainConfig(iterations=4, step_size=0.05, densify_interval=2,
                                              densify_grad_threshold=1e-5, capacity_U=260))
    out["key_params"] = ks.frame.params
    out["key_capacity"] = np.array(ks.capacity_U)
    # the whole training-based grouping driver on a 3-frame toy sequence
    from splatstream import grouping

    seq = [moved.copy() for _ in range(3)]
    seq[2][:, 0:3] += 0.05  # a jump the motion fit cannot follow
    tgts = [train.GroundTruth(images=tuple(np.clip(rasterizer.render(model.GaussianFrame(params=f), c).pixels
                                                   + rng.normal(0, 0.01, (40, 48, 3)), 0, 1) for c in cams))
            for f in seq]
    for t, tg in enumerate(tgts):
        for k, im in enumerate(tg.images):
            out[f"bg_t{t}_c{k}"] = im
    stream = grouping.build_groups(tgts, cams, weights, train.TrainConfig(iterations=2, step_size=0.05),
                                   train.TrainConfig(iterations=3, step_size=0.05, densify_interval=2),
                                   (np.full(3, -0.5), np.full(3, 0.5)), 120, tau_db=18.9, seed=3)
    out["bg_iskey"] = np.array([r.is_keyframe for r in stream.records])
    out["bg_quality"] = np.array([r.quality_db for r in stream.records])
    for k, sp in stream.spaces.items():
        out[f"bg_space{k}"] = sp.frame.params
    for r in stream.records:
        out[f"bg_cum{r.frame_index}"] = r.cumulative_delta.dense()
    np.savez_compressed(os.path.join(HERE, "train.npz"), **out)


def gen_seam_backward(ss):
    """The kernel seam's forward(record=True) masks and backward
    (ss/_composite.pyx:18-152) on random primitives (with clipped and empty
    bboxes) and on a prepared scene."""
    from splatstream import _composite, camera, model, rasterizer

    out = {}
    rng = np.random.default_rng(1100)
    cases = []
    n, hh, ww = 60, 30, 37
    means2d = rng.uniform(-3, ww + 3, (n, 2))
    conics = np.zeros((n, 3))
    conics[:, 0] = rng.uniform(0.05, 0.5, n)
    conics[:, 1] = rng.uniform(-0.03, 0.03, n)
    conics[:, 2] = rng.uniform(0.05, 0.5, n)
    alphas = rng.uniform(0.2, 0.99, n)
    colors = rng.uniform(0, 1, (n, 3))
    r = rng.uniform(1, 9, n)
    bb = np.stack([np.clip(np.floor(means2d[:, 0] - r), 0, ww), np.clip(np.ceil(means2d[:, 0] + r) + 1, 0, ww),
                   np.clip(np.floor(means2d[:, 1] - r), 0, hh), np.clip(np.ceil(means2d[:, 1] + r) + 1, 0, hh)],
                  axis=1).astype(np.int64)
    bb[3] = [5, 5, 2, 9]  # empty bbox
    cases.append((means2d, conics, alphas, colors, bb, hh, ww))
    p = random_params(rng, 400, 0, 0.5)
    cam = camera.ring_rig(1, radius=3.0, height=0.3, focal=40.0, resolution=(48, 40))[0]
    pr = rasterizer._prepare(model.GaussianFrame(params=p), cam)
    cases.append((pr.means2d, pr.conics, pr.alphas, pr.colors, pr.bboxes, 40, 48))
    for cid, (m2, co, al, cl, bbx, h, w) in enumerate(cases):
        img, tr, us, masks = _composite.forward(m2, co, al, cl, bbx, h, w, record=True)
        d_image = rng.normal(0, 1, (h, w, 3))
        grads = _composite.backward(m2, co, al, cl, bbx, h, w, masks, np.asarray(tr), d_image)
        for k, v in dict(means2d=m2, conics=co, alphas=al, colors=cl, bboxes=bbx, hw=np.array([h, w]),
                         image=np.asarray(img), trans=np.asarray(tr), usage=np.asarray(us), masks=np.asarray(masks),
                         d_image=d_image).items():
            out[f"s{cid}_{k}"] = v
        for name, v in zip(("d_means2d", "d_conics", "d_alphas", "d_colors"), grads):
            out[f"s{cid}_{name}"] = np.asarray(v)
    np.savez_compressed(os.path.join(HERE, "seam_backward.npz"), **out)


GENERATORS = ("gen_render", "gen_composite", "gen_codec", "gen_delta", "gen_pruning", "gen_grouping", "gen_session",
              "gen_metrics", "gen_backward", "gen_io", "gen_train", "gen_seam_backward")


def main():
    ss = import_reference()
    only = sys.argv[1:] or GENERATORS  # e.g. `make_golden.py gen_metrics`
    for name in only:
        globals()[name](ss)
        print("ok", name)
    total = sum(os.path.getsize(p) for p in glob.glob(os.path.join(HERE, "*.npz")))
    print(f"fixtures: {total / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
