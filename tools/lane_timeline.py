"""GPU timeline of the pipelined probe, repeated: per frame, an event on its
lane's stream after the render; prints each repetition's device time and
its largest gap between consecutive frame completions, to locate the
occasional slow timed region (profiles/r2_composite_experiments.md,
"Bench timing hygiene").   python tools/lane_timeline.py [reps] [frames]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_20943_b200 import rasterizer, synth  # noqa: E402
from paper_2512_20943_b200.sharding import probe_payloads_sharded  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
space, cams, payloads, targets = bench.build_workload(synth.CONFIGS["C2"], 8, seed=0, device=dev)
pdev = [torch.frombuffer(bytearray(p.data), dtype=torch.uint8).to(dev) for p in payloads]
nf = len(payloads)
marks = []
orig = rasterizer.render_views


def render_marked(*a, **k):
    r = orig(*a, **k)
    e = torch.cuda.Event(enable_timing=True)
    e.record(torch.cuda.current_stream(dev))
    marks.append((e, time.perf_counter()))
    return r


rasterizer.render_views = render_marked


def frames(lo, hi):
    idx = [i % nf for i in range(lo, hi)]
    return [payloads[i] for i in idx], [pdev[i] for i in idx], [targets[i] for i in idx]


probe_payloads_sharded(space, cams, *frames(0, 3), tau_db=30.0, device=dev)
torch.cuda.synchronize()
stream = torch.cuda.current_stream(dev)
for r in range(reps):
    marks.clear()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    ev0.record(stream)
    probe_payloads_sharded(space, cams, *frames(3, 3 + K), tau_db=30.0, device=dev)
    ev1.record(stream)
    torch.cuda.synchronize()
    tot = ev0.elapsed_time(ev1)
    ends = [ev0.elapsed_time(e) for e, _ in marks]
    hosts = [1e3 * (h - h0) for _, h in marks]
    gaps = [ends[0]] + [ends[i] - ends[i - 1] for i in range(1, len(ends))]
    print(f"rep {r:2d}: {tot:7.2f} ms  frame ends " + " ".join(f"{x:6.1f}" for x in ends)
          + "  | host " + " ".join(f"{x:5.1f}" for x in hosts), flush=True)
