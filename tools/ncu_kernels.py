"""Summarise an ncu --csv launch list (gpu__time_duration.sum): mean time
and count per kernel.  python tools/ncu_kernels.py file.csv [filter]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
flt = sys.argv[2] if len(sys.argv) > 2 else ""
hdr = None
agg = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum" and flt in d["Kernel Name"]:
            agg[d["Kernel Name"][:70]].append(float(d["Metric Value"].replace(",", "")))
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{sum(v) / len(v) / 1e3:9.1f} us x{len(v):3d}  {k}")
