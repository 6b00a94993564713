"""Per-frame cost of the streaming session driver (SURVEY.md s8(a) a15,
ss/streamsim.py:189-301) at a BASELINE.json config scale: keyframe + delta
frames through streamsim.run_session on one GPU, with a per-stage breakdown of
one delta frame (usage pass, level space, selection, encode/decode, client
quality).  Synthetic stream: frame t's cumulative delta = GT_t - GT_0
(SURVEY.md s8(d) training-free stand-in).

  python tools/profile_session.py C4 6
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_20943_b200 import grouping, streamsim, synth  # noqa: E402
from paper_2512_20943_b200.model import CanonicalSpace, DeltaTensor, GaussianFrame, diff_frames  # noqa: E402


def build_stream(cfg, frames, seed=0):
    seq = synth.Sequence(cfg, seed=seed, event_every=0)
    gt0 = seq.frame(0)
    n = gt0.shape[0]
    space = CanonicalSpace(GaussianFrame(params=gt0, frame_index=0, group_key=0), capacity_U=n)
    recs = []
    for t in range(frames):
        cum = diff_frames(space.frame, GaussianFrame(params=seq.frame(t)[:n]))
        recs.append(grouping.FrameRecord(t, 0, t == 0, DeltaTensor.empty(n, gt0.shape[1]), cum, 40.0))
    plan = grouping.GroupPlan(30.0, (grouping.GroupSpan(0, 0, frames - 1),))
    return grouping.TrainedStream(plan=plan, spaces={0: space}, records=recs)


STAGES = {}


def instrument():
    """Wrap the session's stages with synchronising wall-clock timers."""
    from paper_2512_20943_b200 import codec, pruning

    def wrap(mod, name, label):
        fn = getattr(mod, name)

        def timed(*a, **k):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = fn(*a, **k)
            torch.cuda.synchronize()
            STAGES[label] = STAGES.get(label, 0.0) + time.perf_counter() - t0
            return r

        setattr(mod, name, timed)

    wrap(streamsim, "_server_pass", "server pass (usage + images)")
    wrap(pruning, "build_level_space", "level space")
    wrap(pruning, "prune_delta", "prune_delta")
    wrap(codec, "encode_delta", "encode_delta")
    wrap(codec, "decode_delta", "decode_delta")
    wrap(streamsim, "compose_deltas", "compose_deltas")
    wrap(streamsim, "_mean_psnr_vs", "client quality")
    wrap(grouping.TrainedStream, "reconstruct", "server reconstruct")
    wrap(codec, "encode_frame", "encode_frame (keyframe)")
    wrap(codec, "decode_frame", "decode_frame (keyframe)")


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    frames = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    cfg = synth.CONFIGS[name]
    cams = synth.cameras(cfg)
    stream = build_stream(cfg, frames)
    trace = streamsim.BandwidthTrace(np.array([0.0, 1e9]), np.array([2e7, 2e7]))
    scfg = streamsim.SimConfig(target_rate_R=1.0, quant_step=1e-4, ratios=tuple(i / 10 for i in range(8)),
                               cliff_beta=2.0)
    # warm-up (context, scratch growth)
    streamsim.run_session(build_stream(cfg, 2, seed=1), cams, trace, scfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    report, state, log = streamsim.run_session(stream, cams, trace, scfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    instrument()
    streamsim.run_session(stream, cams, trace, scfg)  # instrumented pass (synchronising timers)
    out = {"config": name, "frames": frames, "views": len(cams), "gaussians": cfg.count,
           "session_wall_s": round(wall, 3), "ms_per_frame": round(1e3 * wall / frames, 1),
           "levels": [f.level for f in report.frames], "sent_bytes": [f.sent_bytes for f in report.frames],
           "client_quality_db": [round(f.client_quality_db, 4) for f in report.frames],
           "stage_ms_per_frame (instrumented pass)": {k: round(1e3 * v / frames, 2) for k, v in
                                                      sorted(STAGES.items(), key=lambda kv: -kv[1])}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
