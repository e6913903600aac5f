"""Summarise ncu outputs into profiles/ (run in the build container).

  python tools/ncu_summary.py launches <launches.csv> <out.md>
  python tools/ncu_summary.py full <report.ncu-rep> <out.md>
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path, out):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[i]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[i + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("svdrec::<unnamed>::", "")
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        v = v / 1e3 if unit == "ns" else (v if unit == "us" else v * 1e3)
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    lines = ["| kernel | launches | total us | share |", "|---|---:|---:|---:|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| {k} | {cnt[k]} | {v:.1f} | {v / s:.3f} |")
    lines.append(f"| **all** | {sum(cnt.values())} | {s:.1f} | 1.000 |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


KEYS = ["Duration", "Elapsed Cycles", "SM Active Cycles", "DRAM Throughput", "Memory Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Issued Warp Per Scheduler", "Eligible Warps Per Scheduler",
        "Achieved Occupancy", "Registers Per Thread", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block"]


def full(path, out):
    txt = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    per = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        names[d["ID"]] = d["Kernel Name"].split("(")[0].replace("svdrec::<unnamed>::", "")
        if d["Metric Name"] in KEYS:
            per[d["ID"]][d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    rr = list(csv.reader(io.StringIO(raw)))
    traffic = {}
    pipes = {}
    if rr:
        h = rr[0]
        # FP64 tensor-core (DMMA) and FP64 pipe activity, where the report has them
        pk = [c for c in h if ("pipe_tensor" in c or "pipe_fp64" in c or "pipe_fmaheavy" in c)
              and "pct_of_peak_sustained_active" in c]
        for r in rr[2:]:
            d = dict(zip(h, r))
            pipes[d["ID"]] = [(c, d[c]) for c in pk if d.get(c) not in (None, "", "n/a")]
            try:
                rd = float(d.get("dram__bytes_read.sum", "0").replace(",", ""))
                wr = float(d.get("dram__bytes_write.sum", "0").replace(",", ""))
                traffic[d["ID"]] = (rd, wr, rr[1][h.index("dram__bytes_read.sum")])
            except (ValueError, KeyError):
                pass
    lines = []
    for i in sorted(per, key=int):
        lines.append(f"### launch {i}: {names[i]}")
        for k in KEYS:
            if k in per[i]:
                lines.append(f"- {k}: {per[i][k]}")
        if i in traffic:
            rd, wr, unit = traffic[i]
            lines.append(f"- dram__bytes_read.sum + dram__bytes_write.sum: {rd:.4g} + {wr:.4g} {unit}")
        for c, v in pipes.get(i, []):
            lines.append(f"- {c}: {v} %")
        lines.append("")
    open(out, "w").write("\n".join(lines))
    print("\n".join(lines))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
