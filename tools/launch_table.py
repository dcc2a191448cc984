"""Markdown table of an ncu launch list (--metrics gpu__time_duration.sum --csv).
usage: python tools/launch_table.py gpurun_out/launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    x = dict(zip(hdr, r))
    if x.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = x["Kernel Name"]
    name = name.split("(")[0] if "(" in name else name
    u = x.get("Metric Unit", "")
    v = float(x["Metric Value"].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v for _, v in agg.values())
print("| launches | total us | share | kernel |")
print("|---|---|---|---|")
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| {c} | {v:.1f} | {100 * v / tot:.1f}% | `{k}` |")
