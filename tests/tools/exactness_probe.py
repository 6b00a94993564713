"""How many output values of the CUDA path differ from the reference's own
outputs (tests/golden fixtures), split by stage: the compositing seam fed the
reference's prepared arrays (compositing alone) and the full render (projection
+ compositing).  Prints one JSON line.

  python tools/exactness_probe.py
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from conftest import load_golden  # noqa: E402
from test_oracle import cams_from  # noqa: E402


def diff(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    d = a != b
    ulps = np.abs(a.view(np.int64) - b.view(np.int64))
    return {"values": int(a.size), "differing": int(d.sum()), "max_abs": float(np.max(np.abs(a - b))) if a.size else 0.0,
            "max_ulps": int(ulps.max()) if a.size else 0}


def add(acc, d):
    acc["values"] += d["values"]
    acc["differing"] += d["differing"]
    acc["max_abs"] = max(acc["max_abs"], d["max_abs"])
    acc["max_ulps"] = max(acc["max_ulps"], d["max_ulps"])


def main():
    from paper_2512_20943_b200 import rasterizer
    from paper_2512_20943_b200.model import GaussianFrame

    out = {}
    seam = {"values": 0, "differing": 0, "max_abs": 0.0, "max_ulps": 0}
    g = load_golden("composite.npz")
    for cid in range(2):
        args = [g[f"k{cid}_{k}"] for k in ("means2d", "conics", "alphas", "colors", "bboxes")]
        h, w = (int(v) for v in g[f"k{cid}_hw"])
        img, tr, us, _ = rasterizer.forward(*args, h, w)
        add(seam, diff(img, g[f"k{cid}_image"]))
        add(seam, diff(tr, g[f"k{cid}_trans"]))
    g = load_golden("render.npz")
    seam_prep = {"values": 0, "differing": 0, "max_abs": 0.0, "max_ulps": 0}
    full = {"values": 0, "differing": 0, "max_abs": 0.0, "max_ulps": 0}
    for cid in range(4):
        cams = cams_from(g, f"c{cid}_")
        imgs, _ = rasterizer.render_with_usage(GaussianFrame(params=g[f"c{cid}_params"]), cams)
        for v, cam in enumerate(cams):
            W, H = cam.resolution
            img, _, _, _ = rasterizer.forward(*[g[f"c{cid}_v{v}_{k}"] for k in
                                                ("means2d", "conics", "alphas", "colors", "bboxes")], H, W)
            add(seam_prep, diff(np.clip(img, 0, 1), g[f"c{cid}_v{v}_image"]))
            add(full, diff(imgs[v].pixels, g[f"c{cid}_v{v}_image"]))
    out["seam_vs_reference_kernel (image+T)"] = seam
    out["seam_on_reference_prepared_views (image)"] = seam_prep
    out["render (projection+compositing, image)"] = full
    print(json.dumps(out))


if __name__ == "__main__":
    main()
