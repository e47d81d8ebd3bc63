"""Achieved HBM bandwidth of the bandwidth-bound kernels (noise, analytic Phi,
blend, Laplacian / features / conditioning) from an ncu CSV captured with
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      -k regex:'noise|blend|phi_analytic|laplac|blur|signed|patch|condition|procedural|corrupt' \
      --csv --log-file hbm.csv python bench.py --phi analytic --steps 1 --warmup 3

python tools/hbm_kernels.py hbm.csv [out.json]
Prints per kernel: launches, mean DRAM bytes and time per launch, achieved GB/s
and the fraction of the measured HBM copy peak (MEASURED_PEAKS.json).
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6,
         "GB": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3}


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, per, names = None, collections.defaultdict(dict), {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            names[d["ID"]] = d["Kernel Name"].split("(")[0].replace("void ", "")
            per[d["ID"]][d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * \
                UNITS.get(d["Metric Unit"], 1.0)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    agg = collections.OrderedDict()
    for k, m in per.items():
        a = agg.setdefault(names[k], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        a[2] += m.get("gpu__time_duration.sum", 0)
    out = {}
    print(f"{'kernel':44s} {'n':>4s} {'MB/launch':>10s} {'us/launch':>10s} {'GB/s':>8s} {'frac':>6s}")
    for k, (n, b, t) in agg.items():
        gbs = b / t / 1e9 if t else 0.0
        out[k] = {"launches": n, "bytes_per_launch": b / n, "us_per_launch": t / n * 1e6,
                  "achieved_gbs": gbs, "frac_of_measured_hbm_peak": gbs / peak}
        print(f"{k[:44]:44s} {n:4d} {b / n / 1e6:10.2f} {t / n * 1e6:10.1f} {gbs:8.0f} {gbs / peak:6.2f}")
    if len(sys.argv) > 2:
        json.dump({"peak_gbs": peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)",
                   "note": "ncu replay: cold cache, serialised launches", "kernels": out},
                  open(sys.argv[2], "w"), indent=1)


if __name__ == "__main__":
    main()
