"""Clean-tile skip of the pruning-level sweep (pruning.tile_footprint,
airgs_view_item.tile_minrank): the reference re-renders every level in full
(ss/pruning.py:122-131); a tile that no primitive changed by the level
reaches, before or after pruning, composites exactly as the reference render,
so it is given SSE 0 without rendering.  Checked here: (1) soundness of the
footprint against the binning read back directly (every tile listing a
primitive the level changes, in the unpruned or the pruned frame, is marked
below the level's rank cut); (2) the qualities of the whole level space are
bit-identical with the skip on and off, at C3's full size; (3) the skip is
refused for items that need pixels or usage."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _c3_gap(views, count=None, seed=3):
    from dataclasses import replace

    from paper_2512_20943_b200 import rasterizer, synth
    from paper_2512_20943_b200.model import CanonicalSpace, GaussianFrame, diff_frames

    cfg = replace(synth.CONFIGS["C3"], views=views)
    if count is not None:
        cfg = replace(cfg, count=count)
    seq = synth.Sequence(cfg, seed=seed, event_every=0)
    base, moved = seq.frame(0), seq.frame(4)
    cams = synth.cameras(cfg)
    space = CanonicalSpace(GaussianFrame(params=base, frame_index=0, group_key=0), capacity_U=base.shape[0])
    gap = diff_frames(space.frame, GaussianFrame(params=moved))
    _, usage = rasterizer.render_with_usage(GaussianFrame(params=moved), cams)
    return gap, space, cams, usage


def test_footprint_covers_every_binned_tile_of_changed_primitives():
    from paper_2512_20943_b200 import rasterizer
    from paper_2512_20943_b200.model import GaussianFrame
    from paper_2512_20943_b200.pruning import level_frame_planes, level_table, tile_footprint

    gap, space, cams, usage = _c3_gap(views=3, count=60_000)
    t = level_table(gap, space, [i / 10 for i in range(8)], usage, 1e-4)
    p = t.plan
    kmax = max(t.kmins)
    minrank, _ = tile_footprint(p, cams, kmax)
    rank = p.rank[: p.n].cpu().numpy().astype(np.int64)
    nz = p.nz[: p.n].cpu().numpy().astype(bool)
    checked = clean = 0
    for k in sorted(set(t.kmins) - {0}):
        changed = nz & (rank < k)
        for planes in (level_frame_planes(p, None), level_frame_planes(p, k)):
            fr = GaussianFrame(device_params=planes, count=p.n)
            for v, cam in enumerate(cams):
                mr = minrank[v].cpu().numpy()
                counts, lists = rasterizer.tile_lists(fr, cam)
                for g, ids in enumerate(lists):
                    if len(ids) and changed[np.asarray(ids, dtype=np.int64)].any():
                        assert mr[g] < k, (k, v, g)
                        checked += 1
                clean += int((mr >= k).sum())
    assert checked > 0 and clean > 0  # both branches exercised


def test_c3_level_space_identical_with_and_without_tile_skip(monkeypatch):
    """C3 at full size (300k, 1080p, 8 levels; 6 views): every level's
    quality, size and pruned set bit-identical with the skip on and off."""
    from paper_2512_20943_b200.pruning import build_level_space

    gap, space, cams, usage = _c3_gap(views=6)
    ratios = [i / 10 for i in range(8)]
    monkeypatch.setenv("AIRGS_LEVEL_TILE_SKIP", "0")
    off = build_level_space(gap, space, cams, ratios, usage, 1e-4, frame_index=4)
    monkeypatch.setenv("AIRGS_LEVEL_TILE_SKIP", "1")
    on = build_level_space(gap, space, cams, ratios, usage, 1e-4, frame_index=4)
    assert len(on.levels) == len(off.levels) > 2
    for a, b in zip(on.levels, off.levels):
        assert a.ratio == b.ratio and a.size_bytes == b.size_bytes and a.pruned_indices == b.pruned_indices
        assert a.quality_db == b.quality_db  # bit for bit


@pytest.mark.parametrize("views,count", [(4, 20_000), (2, 60_000)])
def test_small_level_space_identical_with_and_without_tile_skip(monkeypatch, views, count):
    """Reduced C3 scenes (fast enough for compute-sanitizer): the skip path
    (k_tile_footprint, k_bin<true>, k_zero_clean) against full renders."""
    from paper_2512_20943_b200.pruning import build_level_space

    gap, space, cams, usage = _c3_gap(views=views, count=count, seed=5)
    ratios = [0.0, 0.05, 0.2, 0.5, 0.9]
    monkeypatch.setenv("AIRGS_LEVEL_TILE_SKIP", "0")
    off = build_level_space(gap, space, cams, ratios, usage, 1e-4)
    monkeypatch.setenv("AIRGS_LEVEL_TILE_SKIP", "1")
    on = build_level_space(gap, space, cams, ratios, usage, 1e-4)
    assert [x.quality_db for x in on.levels] == [x.quality_db for x in off.levels]
    assert [x.size_bytes for x in on.levels] == [x.size_bytes for x in off.levels]


def test_tile_skip_refused_for_items_with_pixels_or_usage():
    import torch

    from paper_2512_20943_b200 import synth
    from paper_2512_20943_b200.errors import StructuralError
    from paper_2512_20943_b200.model import GaussianFrame
    from paper_2512_20943_b200.rasterizer import render_views

    cfg = synth.CONFIGS["C1"]
    fr = GaussianFrame(params=synth.Sequence(cfg, seed=1).frame(0))
    cam = synth.cameras(cfg)[0]
    w, h = cam.resolution
    mr = torch.zeros((((w + 15) // 16) * ((h + 15) // 16),), dtype=torch.int32, device="cuda")
    tgt = torch.zeros((h, w, 3), dtype=torch.float64, device="cuda")
    with pytest.raises(StructuralError):
        render_views([fr], [cam], [(0, 0)], targets=[tgt], want_images=True, tile_skip=[(mr, 1)])
    with pytest.raises(StructuralError):
        render_views([fr], [cam], [(0, 0)], targets=[tgt], usage_frames=[0], tile_skip=[(mr, 1)])
    # keep_min 0: every tile clean -> SSE exactly 0 whatever the target
    out = render_views([fr], [cam], [(0, 0)], targets=[tgt], tile_skip=[(mr, 0)])
    assert float(out.sse[0]) == 0.0
