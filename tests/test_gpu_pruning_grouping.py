"""Pruning-level spaces, selection and keyframe probes on the GPU vs the
oracle: prune order, pruned index sets, level sizes and selected levels are
bit-exact; qualities within 1e-6 dB (north star: 0.01 dB)."""

import numpy as np
import pytest

from conftest import random_params
from oracle import airgs_oracle as orc

pytestmark = pytest.mark.gpu

DB_TOL = 1e-6


def _scene(seed, n=2000, movers=0.3, amp=0.02):
    rng = np.random.default_rng(seed)
    base = random_params(rng, n, 0, spread=0.6)
    moved = base.copy()
    m = rng.choice(n, int(movers * n), replace=False)
    moved[m, 0:3] += rng.normal(0, amp, (m.size, 3))
    moved[m[::3], 11:14] += rng.normal(0, 0.2, (m[::3].size, 3))
    return base, moved


def _cams(count=3, res=(64, 48)):
    from paper_2512_20943_b200.camera import ring_rig

    return ring_rig(count, radius=3.0, height=0.3, focal=res[0] * 40.0 / 48.0, resolution=res)


def test_prune_order_rules():
    from paper_2512_20943_b200.model import DeltaTensor
    from paper_2512_20943_b200.pruning import prune_delta, prune_order

    delta = DeltaTensor(4, 17, {i: np.ones(17) for i in range(4)})
    assert prune_order(delta, np.array([5, 1, 1, 7])) == [2, 1, 0, 3]
    delta = DeltaTensor(6, 17, {1: np.ones(17), 4: np.ones(17)})
    assert prune_order(delta, np.array([0, 9, 0, 0, 2, 0])) == [4, 1]
    five = DeltaTensor(5, 17, {i: np.ones(17) for i in range(5)})
    kept, removed = prune_delta(five, np.arange(5), 0.5)
    assert len(removed) == 3 and kept.entry_count == 2
    kept, removed = prune_delta(five, np.arange(5), 0.0)
    assert removed == () and kept.entry_count == 5
    kept, removed = prune_delta(five, np.arange(5), 1.0)
    assert kept.is_empty() and len(removed) == 5


def test_prune_order_matches_oracle_large(rng):
    from paper_2512_20943_b200.model import DeltaTensor
    from paper_2512_20943_b200.pruning import prune_order

    n = 50000
    idx = np.sort(rng.choice(n, 9000, replace=False))
    usage = rng.integers(0, 40, n)  # many ties
    d = DeltaTensor(n, 17, {int(i): np.ones(17) for i in idx})
    assert prune_order(d, usage) == orc.prune_order(idx, usage).tolist()


@pytest.mark.parametrize("with_base", [False, True])
def test_level_space_matches_oracle(with_base):
    from paper_2512_20943_b200 import rasterizer
    from paper_2512_20943_b200.model import CanonicalSpace, DeltaTensor, GaussianFrame, diff_frames
    from paper_2512_20943_b200.pruning import build_level_space

    base_p, moved = _scene(1 + with_base)
    cams = _cams()
    space = CanonicalSpace(GaussianFrame(params=base_p, frame_index=0, group_key=0), capacity_U=base_p.shape[0])
    gap = diff_frames(space.frame, GaussianFrame(params=moved))
    _, usage = rasterizer.render_with_usage(GaussianFrame(params=moved), cams)
    _, ref_usage = orc.render_with_usage(moved, cams)
    np.testing.assert_array_equal(usage.counts, ref_usage)
    ratios = [i / 10 for i in range(10)] + [1.0]
    bi = br = None
    base = None
    if with_base:
        rng = np.random.default_rng(9)
        bi = np.sort(rng.choice(base_p.shape[0], 300, replace=False))
        br = rng.normal(0, 0.003, (300, 17))
        base = DeltaTensor(base_p.shape[0], 17, {int(i): r for i, r in zip(bi, br)})
    got = build_level_space(gap, space, cams, ratios, usage, 1e-4, base=base, frame_index=2)
    gi, gr = gap.indices(), np.stack([gap.entries[i] for i in gap.indices().tolist()])
    ref = orc.level_space((gi, gr), base_p, cams, ratios, ref_usage, 1e-4, base=(bi, br) if with_base else None)
    assert len(got.levels) == len(ref)
    for lv, (r, q, s, rm) in zip(got.levels, ref):
        assert lv.ratio == r
        assert lv.size_bytes == s
        assert lv.pruned_indices == tuple(rm.tolist())
        assert abs(lv.quality_db - q) <= DB_TOL
    assert got.levels[0].quality_db == 100.0
    assert got.levels[-1].size_bytes == 24
    sizes = got.sizes()
    assert all(b < a for a, b in zip(sizes, sizes[1:]))


def test_selection_matches_oracle_on_real_space():
    from paper_2512_20943_b200 import rasterizer
    from paper_2512_20943_b200.model import CanonicalSpace, GaussianFrame, diff_frames
    from paper_2512_20943_b200.pruning import SelectionContext, build_level_space, ilp_optimal, select_pruning_level

    base_p, moved = _scene(5)
    cams = _cams(2)
    space = CanonicalSpace(GaussianFrame(params=base_p), capacity_U=base_p.shape[0])
    gap = diff_frames(space.frame, GaussianFrame(params=moved))
    _, usage = rasterizer.render_with_usage(GaussianFrame(params=moved), cams)
    sp = build_level_space(gap, space, cams, [i / 10 for i in range(10)], usage, 1e-4)
    q, s = sp.qualities(), sp.sizes()
    for budget in (24, 100, s[len(s) // 2], s[0], 10 * s[0]):
        ctx = SelectionContext(bandwidth_B=budget * 8.0, target_rate_R=1.0)
        assert select_pruning_level(sp, ctx) == orc.select_level(q, s, budget * 8.0, 1.0)
    sel = ilp_optimal([sp], [s[1]])
    assert sel[0].level == orc.ilp([(q, s)], [s[1]])[0]


def test_frame_quality_and_probe_match_oracle():
    from paper_2512_20943_b200 import grouping
    from paper_2512_20943_b200.model import CanonicalSpace, GaussianFrame, diff_frames

    base_p, moved = _scene(7)
    cams = _cams(3, (80, 64))
    targets = grouping.GroundTruth(images=orc.render_with_usage(moved, cams)[0])
    f = GaussianFrame(params=moved)
    assert grouping.frame_quality(f, cams, targets) == 100.0
    q = grouping.frame_quality(GaussianFrame(params=base_p), cams, targets)
    assert abs(q - orc.frame_quality(base_p, cams, targets.images)) <= DB_TOL
    space = CanonicalSpace(GaussianFrame(params=base_p), capacity_U=base_p.shape[0])
    d = diff_frames(space.frame, f)
    assert grouping.quality_probe(space, d, targets, cams) == 100.0
    assert grouping.is_keyframe(q, 200.0) and not grouping.is_keyframe(100.0, 30.0)


def test_probe_frames_batched_matches_oracle():
    from paper_2512_20943_b200 import grouping
    from paper_2512_20943_b200.model import GaussianFrame

    cams = _cams(4, (64, 64))
    frames, targets, ref = [], [], []
    for s in range(3):
        b, m = _scene(20 + s, n=1500)
        frames.append(GaussianFrame(params=b))
        imgs = orc.render_with_usage(m, cams)[0]
        targets.append(grouping.GroundTruth(images=imgs))
        ref.append(orc.frame_quality(b, cams, imgs))
    got = grouping.probe_frames(frames, cams, targets)
    assert np.max(np.abs(np.array(got) - np.array(ref))) <= DB_TOL


def test_sharded_drivers_world1_equal_unsharded():
    from paper_2512_20943_b200 import grouping, rasterizer, sharding
    from paper_2512_20943_b200.model import CanonicalSpace, GaussianFrame, diff_frames
    from paper_2512_20943_b200.pruning import build_level_space

    base_p, moved = _scene(31)
    cams = _cams(3)
    space = CanonicalSpace(GaussianFrame(params=base_p), capacity_U=base_p.shape[0])
    gap = diff_frames(space.frame, GaussianFrame(params=moved))
    _, usage = rasterizer.render_with_usage(GaussianFrame(params=moved), cams)
    u2 = sharding.usage_sharded(GaussianFrame(params=moved), cams)
    np.testing.assert_array_equal(u2.cpu().numpy(), usage.counts)
    a = build_level_space(gap, space, cams, [0, 0.25, 0.5, 0.75], usage, 1e-4)
    b = sharding.build_level_space_sharded(gap, space, cams, [0, 0.25, 0.5, 0.75], usage, 1e-4)
    assert a.sizes() == b.sizes() and a.qualities() == b.qualities()
    tg = grouping.GroundTruth(images=orc.render_with_usage(moved, cams)[0])
    assert sharding.probe_frames_sharded([GaussianFrame(params=base_p)], cams, [tg]) == \
        grouping.probe_frames([GaussianFrame(params=base_p)], cams, [tg])


def test_probe_sequence_streams_from_host():
    import torch

    from paper_2512_20943_b200 import codec, grouping
    from paper_2512_20943_b200.model import CanonicalSpace, GaussianFrame, diff_frames

    base_p, _ = _scene(41, n=1500)
    cams = _cams(3, (64, 48))
    space = CanonicalSpace(GaussianFrame(params=base_p), capacity_U=base_p.shape[0])
    payloads, targets, ref = [], [], []
    for s in range(4):
        _, moved = _scene(50 + s, n=1500)
        moved = base_p.copy()
        rng = np.random.default_rng(s)
        moved[::4, 0:3] += rng.normal(0, 0.01 * (s + 1), (moved[::4].shape[0], 3))
        d = diff_frames(space.frame, GaussianFrame(params=moved))
        pay = codec.encode_delta(d, 1e-4)
        payloads.append(pay)
        imgs = orc.render_with_usage(moved, cams)[0]
        targets.append([torch.from_numpy(im).pin_memory() for im in imgs])
        dec = codec.decode_delta(pay, base_p.shape[0], 17)
        ref.append(grouping.quality_probe(space, dec, grouping.GroundTruth(images=imgs), cams))
    got = grouping.probe_sequence(space, cams, payloads, targets, tau_db=60.0)
    assert [q for q, _ in got] == ref
    assert [k for _, k in got] == [not q >= 60.0 for q in ref]
    # the double buffers outlive a call: back-to-back calls (reversed frame
    # order, odd frame counts so buffer parity shifts) must not see each other's data
    got2 = grouping.probe_sequence(space, cams, payloads[::-1][:3], targets[::-1][:3], tau_db=60.0)
    got3 = grouping.probe_sequence(space, cams, payloads, targets, tau_db=60.0)
    assert [q for q, _ in got2] == ref[::-1][:3]
    assert [q for q, _ in got3] == ref


def test_probe_payloads_device_pipelined_and_checked_rerun():
    """The pipelined batch probe (deferred checking) gives the per-frame
    probe's qualities bit for bit; a malformed payload in the batch is caught
    by the deferred word and re-raised exactly by the checked re-run."""
    import torch

    from paper_2512_20943_b200 import codec, grouping
    from paper_2512_20943_b200.errors import DecodeError
    from paper_2512_20943_b200.model import CanonicalSpace, GaussianFrame, diff_frames

    base_p, _ = _scene(61, n=1500)
    cams = _cams(3, (64, 48))
    space = CanonicalSpace(GaussianFrame(params=base_p), capacity_U=base_p.shape[0])
    payloads, pdevs, targets, ref = [], [], [], []
    for s in range(4):
        moved = base_p.copy()
        rng = np.random.default_rng(s)
        moved[::3, 0:3] += rng.normal(0, 0.01 * (s + 1), (moved[::3].shape[0], 3))
        pay = codec.encode_delta(diff_frames(space.frame, GaussianFrame(params=moved)), 1e-4)
        imgs = orc.render_with_usage(moved, cams)[0]
        payloads.append(pay)
        pdevs.append(torch.frombuffer(bytearray(pay.data), dtype=torch.uint8).cuda())
        targets.append([torch.from_numpy(im).cuda() for im in imgs])
        dec = codec.decode_delta(pay, base_p.shape[0], 17)
        ref.append(grouping.quality_probe(space, dec, grouping.GroundTruth(images=imgs), cams))
    got = grouping.probe_payloads_device(space, cams, payloads, pdevs, targets, tau_db=60.0)
    assert [q for q, _ in got] == ref
    # corrupt frame 2's varint section: the batch must raise the checked-mode error
    bad = bytearray(payloads[2].data)
    bad[24 + 3] |= 0x80
    bad_dev = torch.frombuffer(bytearray(bad), dtype=torch.uint8).cuda()
    with pytest.raises(DecodeError):
        grouping.probe_payloads_device(space, cams, payloads[:2] + [bytes(bad)] + payloads[3:],
                                       pdevs[:2] + [bad_dev] + pdevs[3:], targets)
    # and the context is back in checked mode afterwards
    got2 = grouping.probe_payloads_device(space, cams, payloads, pdevs, targets, tau_db=60.0)
    assert [q for q, _ in got2] == ref


@pytest.mark.parametrize("lanes", [1, 2, 3])
def test_probe_lanes_equal(monkeypatch, lanes):
    """Frames of the pipelined probe alternate over engine lanes (own stream,
    own scratch, own decode-ahead slots); the qualities do not depend on the
    lane count, including an out-of-order, repeated frame sequence."""
    import torch

    from paper_2512_20943_b200 import codec, grouping
    from paper_2512_20943_b200.model import CanonicalSpace, GaussianFrame, diff_frames

    monkeypatch.setenv("AIRGS_PROBE_LANES", str(lanes))
    base_p, _ = _scene(62, n=1500)
    cams = _cams(3, (64, 48))
    space = CanonicalSpace(GaussianFrame(params=base_p), capacity_U=base_p.shape[0])
    payloads, pdevs, targets, ref = [], [], [], []
    for s in range(5):
        moved = base_p.copy()
        rng = np.random.default_rng(s + 10)
        moved[::3, 0:3] += rng.normal(0, 0.01 * (s + 1), (moved[::3].shape[0], 3))
        pay = codec.encode_delta(diff_frames(space.frame, GaussianFrame(params=moved)), 1e-4)
        imgs = orc.render_with_usage(moved, cams)[0]
        payloads.append(pay)
        pdevs.append(torch.frombuffer(bytearray(pay.data), dtype=torch.uint8).cuda())
        targets.append([torch.from_numpy(im).cuda() for im in imgs])
        dec = codec.decode_delta(pay, base_p.shape[0], 17)
        ref.append(grouping.quality_probe(space, dec, grouping.GroundTruth(images=imgs), cams))
    seq = [0, 1, 2, 4, 3, 3, 0, 1]
    got = grouping.probe_payloads_device(space, cams, [payloads[i] for i in seq], [pdevs[i] for i in seq],
                                         [targets[i] for i in seq], tau_db=60.0)
    assert [q for q, _ in got] == [ref[i] for i in seq]


def test_level_space_chunked_render_calls_equal_single_call(monkeypatch):
    """build_level_space splits its (level, view) renders into calls of bounded
    working set (RENDER_PAIRS_PER_CALL); the qualities do not depend on it."""
    from paper_2512_20943_b200 import pruning, rasterizer
    from paper_2512_20943_b200.model import CanonicalSpace, GaussianFrame, diff_frames

    base_p, moved = _scene(7)
    cams = _cams()
    space = CanonicalSpace(GaussianFrame(params=base_p, frame_index=0, group_key=0), capacity_U=base_p.shape[0])
    gap = diff_frames(space.frame, GaussianFrame(params=moved))
    _, usage = rasterizer.render_with_usage(GaussianFrame(params=moved), cams)
    ratios = [i / 10 for i in range(8)]
    one = pruning.build_level_space(gap, space, cams, ratios, usage, 1e-4)
    monkeypatch.setattr(pruning, "RENDER_PAIRS_PER_CALL", base_p.shape[0] * 3)  # 3 items per call
    many = pruning.build_level_space(gap, space, cams, ratios, usage, 1e-4)
    assert [lv.quality_db for lv in one.levels] == [lv.quality_db for lv in many.levels]
    assert [lv.size_bytes for lv in one.levels] == [lv.size_bytes for lv in many.levels]
