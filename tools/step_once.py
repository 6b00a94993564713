"""Profiling helper: build a small C2 workload, then run `--reps` timed
keyframe-probe steps between cudaProfilerStart/Stop so that
`ncu --profile-from-start off` captures exactly the hot path."""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_20943_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--frames", type=int, default=2)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = synth.CONFIGS[args.config]
    space, cams, payloads, targets = bench.build_workload(cfg, args.frames, 0, dev)
    pdev = [torch.frombuffer(bytearray(p.data), dtype=torch.uint8).to(dev) for p in payloads]
    bench.evaluate_frame(space, cams, pdev[0], payloads[0].data, targets[0], dev)  # warm
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for r in range(args.reps):
        i = r % len(payloads)
        q, _ = bench.evaluate_frame(space, cams, pdev[i], payloads[i].data, targets[i], dev)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("q =", q)


if __name__ == "__main__":
    main()
