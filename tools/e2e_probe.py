"""Diagnose the streamed e2e path: per-frame host timings of probe_sequence."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_20943_b200 import grouping, synth  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
cfg = synth.CONFIGS["C2"]
space, cams, payloads, targets = bench.build_workload(cfg, 2, 0, dev)
host_t = [[im.cpu().pin_memory() for im in targets[i]] for i in range(2)]
for sync_after in (False,):
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = grouping.probe_sequence(space, cams, [payloads[i % 2] for i in range(10)], [host_t[i % 2] for i in range(10)],
                                      device=dev)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"sync_after={sync_after} rep={rep}: {dt * 1e3 / 10:.2f} ms/frame -> {18 * 10 / dt:.1f} views/s")
