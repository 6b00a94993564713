"""Work counters of the evaluation compositing kernel (experiment builds with
-DC2_COUNT, tools/build_variant.sh): for one C2 step, candidate (pixel,
entry) evaluations, phase-B loop iterations per lane, warp-level iterations
(the max over lanes, i.e. what the warp actually executes), contributions,
phase-A entries per warp and staged entries per CTA.
    AIRGS_B200_LIB=paper_2512_20943_b200/lib/variants/count.so python tools/c2_counts.py"""

import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_20943_b200 import _lib, synth  # noqa: E402


def main():
    cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = synth.CONFIGS[cfgname]
    space, cams, payloads, targets = bench.build_workload(cfg, 2, 0, dev)
    pdev = [torch.frombuffer(bytearray(p.data), dtype=torch.uint8).to(dev) for p in payloads]
    lib = _lib.load_library()
    fn = lib.airgs_c2_counts
    out = (ctypes.c_ulonglong * 10)()
    bench.evaluate_frame(space, cams, pdev[0], payloads[0].data, targets[0], dev)
    fn(out, 1)
    bench.evaluate_frame(space, cams, pdev[1], payloads[1].data, targets[1], dev)
    fn(out, 1)
    V = len(cams)
    names = ["candidate_evals", "lane_iterations", "warp_iterations", "contributions", "phaseA_entries_per_warp",
             "staged_entries", "evals_after_termination", "evals_alive_failing", "subtile_pairs_aabb",
             "subtile_pairs_after_cull"]
    d = {k: out[i] / V for i, k in enumerate(names)}
    d["candidates_per_contribution"] = d["candidate_evals"] / max(d["contributions"], 1)
    d["lane_efficiency"] = d["lane_iterations"] / max(32 * d["warp_iterations"], 1)
    d["pixel_evals_per_union_iteration"] = d["candidate_evals"] / max(d["lane_iterations"], 1)
    print(json.dumps({"config": cfgname, "per_view": d}))


if __name__ == "__main__":
    main()
