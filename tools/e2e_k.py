import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import bench
from paper_2512_20943_b200 import grouping, synth
from paper_2512_20943_b200.sharding import probe_sequence_sharded
dev = torch.device("cuda", 0); torch.cuda.set_device(dev)
cfg = synth.CONFIGS["C2"]
space, cams, payloads, targets = bench.build_workload(cfg, 4, 0, dev)
host_t = [[im.cpu().pin_memory() for im in targets[i]] for i in range(4)]
for K in (20, 60, 20, 60, 120):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    probe_sequence_sharded(space, cams, [payloads[i % 4] for i in range(K)], [host_t[i % 4] for i in range(K)], device=dev)
    e1.record(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"K={K}: {e0.elapsed_time(e1)/K:.3f} ms/frame events, wall {dt*1e3/K:.3f} -> {18*K/dt:.0f} views/s", flush=True)
