"""Per-configuration measurements beside the headline bench line (one B200).

For every BASELINE.json config (C1..C5) on synthetic scenes:
  probe  : keyframe-probe step (decode GSDP delta + apply + render all views
           with fused SSE + PSNR + tau) -- views/s, device-resident inputs;
  sweep  : (C3, C4) pruning-level space of one delta frame: usage pass on the
           server frame + build_level_space over 8 ratios x all views --
           (level, view) evaluations/s and ms per frame;
  cpu    : the reference arm of bench.py (the vendored reference package:
           decode_delta + apply_delta + render + psnr, persistent fork pool of
           the host's cores) on one frame state x all views -- views/s.
Timing: CUDA events on the current stream around `--steps` repetitions after
`--warmup`; inputs larger than L2 for C2..C5 (targets).  Prints one JSON line
per config and writes them to --out.

  python tools/bench_configs.py --out profiles/r1_configs.jsonl
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_20943_b200 import synth  # noqa: E402
from paper_2512_20943_b200.model import CanonicalSpace, GaussianFrame, diff_frames  # noqa: E402
from paper_2512_20943_b200.pruning import (SelectionContext, build_level_space, select_pruning_level,  # noqa: E402
                                           selection_margins)


def cuda_time(fn, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def probe(cfg, dev, steps, warmup):
    space, cams, payloads, targets = bench.build_workload(cfg, 2, 0, dev)
    pdev = [torch.frombuffer(bytearray(p.data), dtype=torch.uint8).to(dev) for p in payloads]
    i = [0]

    def step():
        k = i[0] % len(payloads)
        i[0] += 1
        bench.evaluate_frame(space, cams, pdev[k], payloads[k].data, targets[k], dev)

    ms = cuda_time(step, steps, warmup)
    del targets
    torch.cuda.empty_cache()
    return {"views": len(cams), "ms_per_frame": round(ms, 3), "views_per_s": round(len(cams) / ms * 1e3, 1)}


def sweep(cfg, dev, steps, warmup, ratios=tuple(i / 10 for i in range(8))):
    seq = synth.Sequence(cfg, seed=3, event_every=0)
    base, moved = seq.frame(0), seq.frame(4)
    cams = synth.cameras(cfg)
    space = CanonicalSpace(GaussianFrame(params=base, frame_index=0, group_key=0), capacity_U=base.shape[0])
    gap = diff_frames(space.frame, GaussianFrame(params=moved))
    mv = GaussianFrame(params=moved)

    from paper_2512_20943_b200.streamsim import _usage_only

    out = {}

    def step():
        usage = _usage_only(mv, cams)  # the session's usage pass (counts only, ss/streamsim.py:223-225)
        out["space"] = build_level_space(gap, space, cams, list(ratios), usage, 1e-4, frame_index=4)

    ms = cuda_time(step, steps, warmup)
    evals = len(cams) * (len(ratios) + 1)  # usage pass + one render per (level, view)
    lv = out["space"]
    # selection at a budget between the middle levels' sizes (beta = 2, R = 1 frame/s)
    mid = len(lv.levels) // 2
    budget = 0.5 * (lv.levels[mid - 1].size_bytes + lv.levels[mid].size_bytes)
    ctx = SelectionContext(bandwidth_B=budget * 8.0, target_rate_R=1.0, cliff_beta=2.0)
    return {"levels": len(ratios), "views": len(cams), "ms_per_frame": round(ms, 2),
            "level_view_evals_per_s": round(evals / ms * 1e3, 1),
            "quality_table_db": [round(x.quality_db, 4) for x in lv.levels],
            "sizes_bytes": [x.size_bytes for x in lv.levels],
            "selected_level": select_pruning_level(lv, ctx),
            "decision_margins": selection_margins(lv, ctx, entries=len(gap.indices()))}


def cpu(cfg, steps=1):
    """The reference arm (bench.CpuArm: the vendored reference package on a
    persistent fork pool of the host's cores) on `steps` frame states."""
    arm = bench.CpuArm(cfg)
    try:
        arm.run(1)  # warm
        dt = arm.run(steps)
        return {"views_per_s": round(arm.V * steps / dt, 4), "cores": arm.cores, "kind": arm.kind,
                "sample": arm.describe(steps), "cpu_model": bench.cpu_model()}
    finally:
        arm.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--cpu-steps", type=int, default=1, help="frame states (x all views) in the CPU sample")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    lines = []
    for name in args.configs.split(","):
        cfg = synth.CONFIGS[name]
        rec = {"config": name, "gaussians": cfg.count, "views": cfg.views, "resolution": list(cfg.resolution),
               "data": "synthetic (seeded SURVEY s8(d) generator)", "gpu": torch.cuda.get_device_name(dev)}
        t0 = time.time()
        rec["probe"] = probe(cfg, dev, args.steps, args.warmup)
        if name in ("C3", "C4", "C5"):
            rec["sweep"] = sweep(cfg, dev, max(1, args.steps // 2), 1)
        if not args.no_cpu:
            rec["cpu_reference"] = cpu(cfg, args.cpu_steps)
            rec["gpu_over_cpu_probe"] = round(rec["probe"]["views_per_s"] / rec["cpu_reference"]["views_per_s"], 1)
        rec["wall_s"] = round(time.time() - t0, 1)
        print(json.dumps(rec), flush=True)
        lines.append(rec)
    if args.out:
        with open(args.out, "w") as fh:
            for r in lines:
                fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
