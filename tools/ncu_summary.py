"""Summarise an ncu report: key metrics + top source lines by instructions.

  python tools/ncu_summary.py REPORT [TOP] [--traffic-json OUT]

--traffic-json writes the dominant kernel's measured DRAM bytes and SM-side
figures in the form bench.py reads (profiles/composite_traffic.json)."""
import csv
import json
import subprocess
import sys

args = [a for a in sys.argv[1:] if not a.startswith("--")]
rep = args[0]
top = int(args[1]) if len(args) > 1 else 20
tjson = sys.argv[sys.argv.index("--traffic-json") + 1] if "--traffic-json" in sys.argv else None
if tjson in args:
    args.remove(tjson)
    top = int(args[1]) if len(args) > 1 else 20
RAW = {}


def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout


rows = list(csv.reader(run(["--page", "details", "--csv"]).splitlines()))
h = rows[0]
want = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy", "Registers Per Thread",
        "Avg. Active Threads Per Warp", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "Executed Instructions",
        "L1/TEX Hit Rate", "L2 Hit Rate"]
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:<38} {d['Metric Value']} {d['Metric Unit']}")
raw = list(csv.reader(run(["--page", "raw", "--csv"]).splitlines()))
if len(raw) >= 3:
    stalls = []
    for name, unit, val in zip(raw[0], raw[1], raw[2]):
        if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
            try:
                stalls.append((float(val.replace(",", "")), name[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
        if name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
                    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
                    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "derived__memory_l1_wavefronts_shared_excessive",
                    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                    "sm__inst_executed.avg.per_cycle_active", "gpu__time_duration.sum"):
            print(f"{name:<60} {val} {unit}")
            try:
                scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit.strip(), 1.0)
                RAW[name] = float(val.replace(",", "")) * scale
            except ValueError:
                pass
    tot = sum(v for v, _ in stalls) or 1
    STALLS = ", ".join(f"{n} {100 * v / tot:.1f}%" for v, n in sorted(stalls, reverse=True)[:5])
    print("stalls:", ", ".join(f"{n} {100 * v / tot:.1f}%" for v, n in sorted(stalls, reverse=True)[:8]))
    if tjson:
        out = {"source": f"{rep} (ncu --set full --clock-control none, k_composite, one C2 step = 18 views "
                         "1352x1014, 300k Gaussians)",
               "dram_bytes_per_launch": int(RAW.get("dram__bytes_read.sum", 0) + RAW.get("dram__bytes_write.sum", 0)),
               "sm": {"fp64_pipe_active_pct": round(RAW.get(
                          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0), 1),
                      "issue_slots_busy_pct": round(RAW.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0), 1),
                      "ipc": round(RAW.get("sm__inst_executed.avg.per_cycle_active", 0), 2),
                      "achieved_occupancy_pct": round(RAW.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0), 1),
                      "lsu_data_pipe_wavefronts_pct": round(RAW.get(
                          "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", 0), 1),
                      "top_stalls": STALLS}}
        with open(tjson, "w") as fh:
            json.dump(out, fh, indent=1)
src = list(csv.reader(run(["--page", "source", "--csv", "--print-source=cuda,sass"]).splitlines()))
lines = []
for r in src[3:]:
    if r and r[0]:
        try:
            lines.append((int(r[0]), r[1][:90], int(r[7]), int(r[4])))
        except (ValueError, IndexError):
            pass
tot = sum(l[2] for l in lines) or 1
st = sum(l[3] for l in lines) or 1
print(f"source lines (instructions total {tot}):")
for l in sorted(lines, key=lambda x: -x[2])[:top]:
    print(f"{l[0]:5d} inst {100 * l[2] / tot:5.1f}% stall {100 * l[3] / st:5.1f}%  {l[1]}")
