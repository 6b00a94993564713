"""The binning + sort stage read back directly (airgs_debug_tile_lists):
per-tile primitive lists against the oracle's tile keys (SURVEY.md s8(c):
key = tile_id << 32 | position in the reference's stable depth order,
ss/rasterizer.py:126-127) restricted by the binning's weight-threshold
narrowing (orc.threshold_tile_ranges; soundness of that narrowing is
tests/test_oracle.py::test_threshold_tile_narrowing_keeps_every_passing_pixel).
Bit-exact: same tiles, same members, same within-tile order."""

import numpy as np
import pytest

from oracle import airgs_oracle as orc

pytestmark = pytest.mark.gpu


def _compare(params, cam):
    from paper_2512_20943_b200 import rasterizer
    from paper_2512_20943_b200.model import GaussianFrame

    counts, lists = rasterizer.tile_lists(GaussianFrame(params=params), cam, max_per_tile=8192)
    want = orc.tile_lists_threshold(params, cam)
    got = {g: lst for g, lst in enumerate(lists) if lst.size}
    assert sorted(got) == sorted(want)
    for g, lst in want.items():
        np.testing.assert_array_equal(got[g], lst)
    return int(counts.sum()), int(counts.max())


def test_c2_view_tile_lists_bit_exact():
    """300k Gaussians, 1352x1014 (BASELINE configs[1])."""
    from paper_2512_20943_b200 import synth

    cfg = synth.CONFIGS["C2"]
    p = synth.Sequence(cfg, seed=0, event_every=0).frame(1)
    pairs, longest = _compare(p, synth.cameras(cfg)[5])
    assert pairs > 500_000 and longest > 32


def test_depth_ties_ordered_by_index():
    """Every primitive at exactly the same camera depth: the reference's
    stable argsort keeps index order, and so must every tile list (the
    sort's depth buckets all clash: each tile is one run, re-sorted in place
    on the exact (64-bit depth key, index))."""
    from paper_2512_20943_b200.camera import look_at

    rng = np.random.default_rng(11)
    n = 3000
    p = np.zeros((n, 17))
    p[:, 0:2] = rng.uniform(-0.8, 0.8, (n, 2))
    p[:, 2] = 0.25  # camera at z = -2.5 looking along +z: depth exactly 2.75 for all
    p[:, 3] = 1.0
    p[:, 7:10] = np.log(0.03)
    p[:, 10] = rng.uniform(0.5, 3.0, n)
    p[:, 11:14] = rng.normal(size=(n, 3))
    cam = look_at((0.0, 0.0, -2.5), (0.0, 0.0, 0.0), focal=120.0, resolution=(160, 128))
    pr = orc.prepare(p, cam)
    assert np.all(pr.depth == pr.depth[0])
    _compare(p, cam)


@pytest.mark.parametrize("count", [800, 1500, 6000])
def test_crowded_tiles_through_overflow_paths(count):
    """Lists longer than the warp sort (512: the 32-keys-per-lane warp sort
    up to 1024, the block sort up to 2048), the bucket capacity (512) and the
    in-shared-memory sort (2048: the call is redone through scanned ranges
    and a segmented radix presort); with exact depth ties inside the crowd,
    the lists are still the reference order."""
    from paper_2512_20943_b200.camera import look_at

    rng = np.random.default_rng(count)
    p = np.zeros((count, 17))
    p[:, 0:2] = rng.normal(0.0, 0.02, (count, 2))
    p[:, 2] = rng.uniform(-0.5, 0.5, count)
    q = rng.normal(size=(count, 4))
    p[:, 3:7] = q / np.linalg.norm(q, axis=1, keepdims=True)
    p[:, 7:10] = np.log(0.02)
    p[:, 10] = rng.uniform(-1.0, 3.0, count)
    p[:, 11:14] = rng.normal(size=(count, 3))
    p[::7, 2] = 0.1  # some exact depth ties among the crowd
    cam = look_at((0.0, 0.0, -2.5), (0.0, 0.0, 0.0), focal=80.0, resolution=(64, 64))
    _, longest = _compare(p, cam)
    assert longest > 512
