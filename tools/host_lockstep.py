"""Where does the host wait inside the pipelined probe?  Times each
per-frame host call (decode/apply enqueue, render enqueue) of one probe
batch; a call that lasts about a frame's GPU time is a blocking point.
   python tools/host_lockstep.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_20943_b200 import codec, grouping, rasterizer, synth  # noqa: E402

dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
cfg = synth.CONFIGS["C2"]
space, cams, payloads, targets = bench.build_workload(cfg, 8, seed=0, device=dev)
pdev = [torch.frombuffer(bytearray(p.data), dtype=torch.uint8).to(dev) for p in payloads]
log = []


def wrap(mod, name):
    fn = getattr(mod, name)

    def w(*a, **k):
        t0 = time.perf_counter()
        r = fn(*a, **k)
        log.append((name, 1e3 * (time.perf_counter() - t0)))
        return r
    setattr(mod, name, w)


wrap(codec, "decode_apply_device")
wrap(rasterizer, "render_views")
K = int(sys.argv[1]) if len(sys.argv) > 1 else 10
nf = len(payloads)


def window(lo, hi):
    idx = [i % nf for i in range(lo, hi)]
    return [payloads[i] for i in idx], [pdev[i] for i in idx], [targets[i] for i in idx]


# the bench's order: a 3-frame warm-up batch, then the K-frame batches
grouping.probe_payloads_device(space, cams, *window(0, 3))
torch.cuda.synchronize()
for rep in range(3):
    log.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    grouping.probe_payloads_device(space, cams, *window(3, 3 + K))
    print(f"rep {rep}: {1e3 * (time.perf_counter() - t0):.2f} ms total;",
          " ".join(f"{n[:6]} {ms:.2f}" for n, ms in log))
