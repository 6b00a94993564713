"""Training-path wall time: fit_group_frame on a
config's scene (targets = noisy renders of a moved frame), on the device path
here, or with the reference's own trainer when run with --reference in the
build container (imports /root/reference; tests/golden/make_golden.py).

  python tools/bench_train.py C1 10            # device path
  python tools/bench_train.py C1 10 --reference  # the reference on the CPU
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def scene(cfg_name):
    from paper_2512_20943_b200 import synth

    cfg = synth.CONFIGS[cfg_name]
    seq = synth.Sequence(cfg, seed=0, event_every=0)
    return cfg, seq.frame(0), seq.frame(3), synth.cameras(cfg)


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C1"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    ref = "--reference" in sys.argv
    cfg, base, moved, cams = scene(name)
    rng = np.random.default_rng(0)
    if ref:
        sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
        import make_golden

        make_golden.import_reference()
        from splatstream import camera, model, rasterizer, train

        rcams = [camera.Camera(pose=c.pose, focal=c.focal, resolution=c.resolution) for c in cams]
        tg = train.GroundTruth(images=tuple(
            np.clip(rasterizer.render(model.GaussianFrame(params=moved), c).pixels
                    + rng.normal(0, 0.01, (c.resolution[1], c.resolution[0], 3)), 0, 1) for c in rcams))
        space = model.CanonicalSpace(model.GaussianFrame(params=base), capacity_U=base.shape[0])
        t0 = time.time()
        train.fit_group_frame(space, model.DeltaTensor.empty(*base.shape), tg, rcams, train.LossWeights(),
                              train.TrainConfig(iterations=iters, step_size=0.05))
        wall = time.time() - t0
        impl = "reference (CPU, 1 process, compiled kernels)"
    else:
        import torch

        from paper_2512_20943_b200 import rasterizer, train
        from paper_2512_20943_b200.model import CanonicalSpace, DeltaTensor, GaussianFrame

        mv = GaussianFrame(params=moved)
        tg = train.GroundTruth(images=[np.clip(rasterizer.render(mv, c).pixels
                                               + rng.normal(0, 0.01, (c.resolution[1], c.resolution[0], 3)), 0, 1)
                                       for c in cams])
        space = CanonicalSpace(GaussianFrame(params=base), capacity_U=base.shape[0])
        train.fit_group_frame(space, DeltaTensor.empty(*base.shape), tg, cams, train.LossWeights(),
                              train.TrainConfig(iterations=1, step_size=0.05))  # warm-up
        torch.cuda.synchronize()
        t0 = time.time()
        train.fit_group_frame(space, DeltaTensor.empty(*base.shape), tg, cams, train.LossWeights(),
                              train.TrainConfig(iterations=iters, step_size=0.05))
        torch.cuda.synchronize()
        wall = time.time() - t0
        impl = "device path (one B200)"
    print(json.dumps({"config": name, "gaussians": int(base.shape[0]), "views": len(cams),
                      "resolution": list(cams[0].resolution), "iterations": iters, "impl": impl,
                      "fit_group_frame_s": round(wall, 3)}))


if __name__ == "__main__":
    main()
