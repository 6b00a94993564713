"""Key ncu details-page metrics for every kernel in a report, one line each.

  python tools/ncu_details.py REPORT
"""
import csv
import subprocess
import sys

WANT = ["Duration", "Memory Throughput", "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Achieved Occupancy", "Registers Per Thread", "Compute (SM) Throughput", "L2 Hit Rate"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in WANT:
        name = d.get("Kernel Name", "?").split("(")[0].replace("void airgs::", "")
        print(f"{name:<40} {d['Metric Name']:<28} {d['Metric Value']} {d['Metric Unit']}")
