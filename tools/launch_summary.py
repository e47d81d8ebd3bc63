"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
seq = []
tot = 0.0
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0][:60]
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
    agg.setdefault(k, [0.0, 0])
    agg[k][0] += v
    agg[k][1] += 1
    tot += v
    seq.append((k, v, d.get("Grid Size", ""), d.get("Block Size", "")))
print(f"total {tot/1e3:.3f} ms over {len(seq)} launches")
for k, (v, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{v/1e3:9.3f} ms {n:4d} {100*v/tot:5.1f}%  {k}")
if "-v" in sys.argv:
    for k, v, g, b in seq:
        print(f"{v:10.1f} us  {k} {g} {b}")
