"""Break down build_level_space wall time (C3/C4 level sweep) by stage."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_20943_b200 import pruning, rasterizer, synth  # noqa: E402
from paper_2512_20943_b200.model import CanonicalSpace, GaussianFrame, diff_frames  # noqa: E402
from paper_2512_20943_b200.rasterizer import render_views  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
dev = torch.device("cuda", 0)
seq = synth.Sequence(cfg, seed=3, event_every=0)
base, moved = seq.frame(0), seq.frame(4)
cams = synth.cameras(cfg)
space = CanonicalSpace(GaussianFrame(params=base, frame_index=0, group_key=0), capacity_U=base.shape[0])
gap = diff_frames(space.frame, GaussianFrame(params=moved))
mv = GaussianFrame(params=moved)
ratios = [i / 10 for i in range(8)]


def t(label, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print(f"{label:28s} {1e3 * (time.perf_counter() - t0):9.2f} ms", flush=True)
    return r


for rep in range(3):
    print("rep", rep)
    from paper_2512_20943_b200.streamsim import _usage_only
    usage = t("usage pass (counts only)", lambda: _usage_only(mv, cams))
    p = t("plan_levels", lambda: pruning.plan_levels(gap, space, usage, 1e-4))
    kmins = [pruning._k_of(r, p.entries) for r in ratios]
    sizes = t("level_sizes", lambda: pruning.level_sizes(p.nz, p.rank, p.n, p.width, kmins, p.canon.device))
    t("removed sets", lambda: pruning._removed_sets(p, gap.overlay(), kmins))
    ref = GaussianFrame(device_params=pruning.level_frame_planes(p, None), count=p.n)
    rv = t("reference render", lambda: render_views([ref], cams, [(0, v) for v in range(len(cams))], want_images=True))
    frames = t("level planes", lambda: [GaussianFrame(device_params=pruning.level_frame_planes(p, k), count=p.n)
                                         for k in kmins])
    items = [(li, v) for li in range(len(frames)) for v in range(len(cams))]
    targets = [rv.images[v] for li in range(len(frames)) for v in range(len(cams))]
    lv = t("level renders (batched)", lambda: render_views(frames, cams, items, targets=targets))
    t("sse readback", lambda: lv.sse.cpu().numpy())
    t("build_level_space total", lambda: pruning.build_level_space(gap, space, cams, ratios, usage, 1e-4))
    os.environ["AIRGS_LEVEL_TILE_SKIP"] = "0"
    t("build_level_space (no skip)", lambda: pruning.build_level_space(gap, space, cams, ratios, usage, 1e-4))
    os.environ["AIRGS_LEVEL_TILE_SKIP"] = "1"
    mr, _ = pruning.tile_footprint(p, cams, max(kmins))
    tot = sum(int(m.numel()) for m in mr)
    print("clean tile share per level:",
          " ".join("%.3f" % (sum(int((m >= k).sum()) for m in mr) / tot) for k in kmins[1:]), flush=True)
