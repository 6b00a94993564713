"""Training-path measurement: one view's
render_forward + render_backward and the SSIM loss gradient at a config's
scale on the GPU (CUDA events), beside the reference's own CPU path on the
same scene (compiled _composite kernels + numpy; one process) when the
reference tree is importable (this container), else the GPU numbers only.

  python tools/bench_backward.py C2
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_20943_b200 import metrics, rasterizer, synth  # noqa: E402
from paper_2512_20943_b200.model import GaussianFrame  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    cfg = synth.CONFIGS[name]
    cam = synth.cameras(cfg)[0]
    params = synth.Sequence(cfg, seed=0, event_every=0).frame(0)
    dev = torch.device("cuda", 0)
    frame = GaussianFrame(params=params)
    planes_frame = GaussianFrame(device_params=frame.planes(dev), count=frame.count)
    rng = np.random.default_rng(0)
    target = torch.from_numpy(rng.uniform(0, 1, (cam.resolution[1], cam.resolution[0], 3))).to(dev)

    def step():
        vb = rasterizer.render_views([planes_frame], [cam], [(0, 0)], want_images=True)
        img = vb.images[0]
        _, d_ssim = metrics._ssim_call(img, target, True)
        _, d_l1 = metrics._l1_call(img, target, True)
        d_image = 0.8 * d_l1 - 0.1 * d_ssim  # d/dimage of 0.8 L1 + 0.2 (1 - SSIM) / 2
        return rasterizer.render_backward(rasterizer.ForwardState(planes_frame, cam), d_image, as_numpy=False)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out = {"config": name, "gaussians": cfg.count, "resolution": list(cam.resolution),
           "gpu_ms_per_view_train_step": round(ms, 3),
           "what": "forward render + SSIM/L1 loss gradients + backward (compositing + projection), one view"}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
