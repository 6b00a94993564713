"""Summarise an ncu report: key metrics + top source lines by instructions."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20


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
                    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"):
            print(f"{name:<60} {val} {unit}")
    tot = sum(v for v, _ in stalls) or 1
    print("stalls:", ", ".join(f"{n} {100 * v / tot:.1f}%" for v, n in sorted(stalls, reverse=True)[:8]))
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
