import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2512_20943_b200 import synth, rasterizer
from paper_2512_20943_b200.model import GaussianFrame
cfg = synth.CONFIGS["C5"]
p = synth.Sequence(cfg, seed=0, event_every=0).frame(1)
cams = synth.cameras(cfg)
tot = np.zeros(5)
for v in (0, 9, 20):
    counts, lists = rasterizer.tile_lists(GaussianFrame(params=p), cams[v], max_per_tile=8192)
    c = np.asarray(counts)
    h = [np.sum(c == 0), np.sum((c > 0) & (c <= 512)), np.sum((c > 512) & (c <= 1024)), np.sum((c > 1024) & (c <= 2048)), np.sum(c > 2048)]
    e = [0, c[(c > 0) & (c <= 512)].sum(), c[(c > 512) & (c <= 1024)].sum(), c[(c > 1024) & (c <= 2048)].sum(), c[c > 2048].sum()]
    print(v, "tiles by class", h, "entries by class", e, "mean", c.mean(), "max", c.max(), flush=True)
