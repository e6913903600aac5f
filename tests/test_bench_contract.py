"""bench.py's CPU reference arm (the oracle port timed on the host cores)
and its JSON contract, on config 0 (seconds of CPU work)."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path


ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_measures_full_runs():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "c0_100k",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                         check=True).stdout
    line = json.loads(out.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["unit"] == "s" and line["higher_is_better"] is False
    assert 1 <= line["steps"] <= 2 and len(line["runs_s"]) == line["steps"]
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and "not extrapolated" in cb["sample"]
    assert line["result"]["blocks"] >= 1 and line["result"]["k"] % 20 == 0
