"""H2D pattern of the e2e step without compute: per frame 18 float64 C2
targets (33 MB each, pinned) + a 4.1 MB payload, on one copy stream,
against the streamed probe (tools/e2e_probe.py) -- where does the e2e
number leave the PCIe bound?"""
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
space, cams, payloads, targets = bench.build_workload(cfg, 4, 0, dev)
host_t = [[im.cpu().pin_memory() for im in targets[i]] for i in range(4)]
dtg = [[torch.empty_like(im, device=dev) for im in targets[0]] for _ in range(2)]
copy = torch.cuda.Stream(dev)
K = 20
for rep in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(copy)
    with torch.cuda.stream(copy):
        for k in range(K):
            for v, im in enumerate(host_t[k % 4]):
                dtg[k % 2][v].copy_(im, non_blocking=True)
    e1.record(copy)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    gb = K * sum(t.numel() * 8 for t in host_t[0]) / 1e9
    print(f"copies only: {ms / K:.2f} ms/frame, {gb / (ms / 1e3):.1f} GB/s -> {18 * K / (ms / 1e3):.0f} views/s bound")
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    grouping.probe_sequence(space, cams, [payloads[i % 4] for i in range(K)], [host_t[i % 4] for i in range(K)],
                            device=dev)
    e1.record()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"probe_sequence: {e0.elapsed_time(e1) / K:.2f} ms/frame (events), wall {dt * 1e3 / K:.2f} ms/frame "
          f"-> {18 * K / dt:.0f} views/s")

# copies concurrent with compositing on the compute stream: does the render slow the DMA?
from paper_2512_20943_b200.model import GaussianFrame  # noqa: E402
from paper_2512_20943_b200.rasterizer import render_views  # noqa: E402

fr = GaussianFrame(device_params=space.frame.planes(dev), count=space.frame.count)
for rep in range(2):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(copy)
    with torch.cuda.stream(copy):
        for k in range(K):
            for v, im in enumerate(host_t[k % 4]):
                dtg[k % 2][v].copy_(im, non_blocking=True)
    e1.record(copy)
    for k in range(3 * K):
        render_views([fr], cams, [(0, v) for v in range(len(cams))], targets=[targets[0][v] for v in range(len(cams))],
                     device=dev)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"copies under rendering: {ms / K:.2f} ms/frame")
