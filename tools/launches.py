"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
tot = collections.OrderedDict()
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0][:70]
    v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
    tot.setdefault(k, [0.0, 0])
    tot[k][0] += v
    tot[k][1] += 1
s = sum(v[0] for v in tot.values())
print(f"{'us':>10} {'share':>6} {'n':>4}  kernel")
for k, (v, c) in sorted(tot.items(), key=lambda x: -x[1][0]):
    print(f"{v:10.1f} {100 * v / s:5.1f}% {c:4d}  {k}")
print(f"{s:10.1f} total us")
