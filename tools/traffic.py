"""DRAM traffic per launch of the two roofline kernels, from ncu --set full
captures, into profiles/traffic.json (read by bench.py for the roofline's
`traffic` field).

    python tools/traffic.py gpurun_out/traffic_cf.ncu-rep gpurun_out/traffic_spmm.ncu-rep

Each capture holds consecutive launches of one kernel from one bench step
(`-k regex:k_predict -c 13`: every CF scoring launch of a step, k = 20..260;
`-k regex:k_spmm_pipe -c 8`); the per-launch figure is the mean of
dram__bytes_read.sum + dram__bytes_write.sum over the captured launches.
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = {"k_predict": "cf_predict", "k_spmm_pipe": "spmm"}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    col = {c: h.index(c) for c in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                  "gpu__time_duration.sum")}
    scale = {c: UNIT.get(units[col[c]], 1) for c in ("dram__bytes_read.sum", "dram__bytes_write.sum")}
    for r in rows[2:]:
        rd = float(r[col["dram__bytes_read.sum"]].replace(",", "")) * scale["dram__bytes_read.sum"]
        wr = float(r[col["dram__bytes_write.sum"]].replace(",", "")) * scale["dram__bytes_write.sum"]
        yield r[col["Kernel Name"]], rd, wr


def main(reps):
    out = {}
    for rep in reps:
        per = {}
        for name, rd, wr in launches(rep):
            key = next((v for k, v in KEYS.items() if k in name), None)
            if key:
                per.setdefault(key, []).append((rd, wr))
        for key, v in per.items():
            n = len(v)
            out[key] = {"dram_bytes_per_launch": round(sum(a + b for a, b in v) / n),
                        "dram_read_bytes_per_launch": round(sum(a for a, _ in v) / n),
                        "dram_write_bytes_per_launch": round(sum(b for _, b in v) / n),
                        "launches": n, "capture": Path(rep).name}
    p = ROOT / "profiles" / "traffic.json"
    p.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
