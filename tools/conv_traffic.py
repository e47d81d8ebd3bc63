"""DRAM traffic of the conv launches (bench.py's roofline "traffic").

Parses an ncu CSV captured with
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      -k regex:conv_ --csv --log-file conv_dram.csv python bench.py --steps 1 --warmup 3
and writes profiles/conv_traffic.json: mean DRAM bytes per conv launch (the
same averaging bench.py uses for "achieved": total over all ig_conv_tc
launches / launch count), plus the per-kernel breakdown.

python tools/conv_traffic.py conv_dram.csv [profiles/conv_traffic.json]
"""
import collections
import csv
import json
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def main():
    src = sys.argv[1]
    dst = sys.argv[2] if len(sys.argv) > 2 else "profiles/conv_traffic.json"
    rows = list(csv.reader(open(src)))
    hdr = None
    per = collections.defaultdict(dict)
    names = {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = d["ID"]
        names[k] = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", "")) * UNITS.get(d["Metric Unit"], 1.0)
        per[k][d["Metric Name"]] = v
    agg = collections.OrderedDict()
    tot_b = tot_t = 0.0
    n = 0
    for k, m in per.items():
        if "conv" not in names[k]:
            continue
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        t = m.get("gpu__time_duration.sum", 0.0)
        a = agg.setdefault(names[k], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += b
        a[2] += t
        tot_b += b
        tot_t += t
        n += 1
    out = {
        "bytes_per_launch": tot_b / n if n else None,
        "launches": n,
        "dram_gbs_under_ncu": tot_b / tot_t / 1e9 if tot_t else None,
        "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over every conv "
                  "launch of `bench.py --steps 1 --warmup 3` (cold-cache, serialised replay)",
        "per_kernel": {k: {"launches": v[0], "bytes_per_launch": v[1] / v[0],
                           "us_per_launch": v[2] / v[0] * 1e6} for k, v in agg.items()},
    }
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps({k: out[k] for k in ("bytes_per_launch", "launches", "dram_gbs_under_ncu")}))


if __name__ == "__main__":
    main()
