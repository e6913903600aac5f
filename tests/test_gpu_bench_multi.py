"""bench.py --gpus N launches N ranks itself (torch.distributed.run) and
reports the whole job: two ranks sharing cuda:0 over gloo
(BENCH_SHARE_GPU: a flow check, not a timing -- gpurun grants one GPU)
must pick the same k and test errors as the one-GPU run, with n_gpus = 2."""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _bench(gpus, extra_env=None):
    env = dict(os.environ, BENCH_NO_CLOCKS="1", **(extra_env or {}))
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(gpus), "--config", "c0_100k",
                          "--steps", "2", "--warmup", "1", "--no-cpu-baseline", "--no-variants"],
                         capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # rank 0 alone prints
    return json.loads(lines[0])


def test_bench_spawns_ranks(gpu):
    one = _bench(1)
    two = _bench(2, {"BENCH_SHARE_GPU": "1"})
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["k"] == one["k"] and two["blocks"] == one["blocks"]
    assert abs(two["test_rmse"] - one["test_rmse"]) <= 1e-9 * one["test_rmse"]
    assert two["value"] > 0 and two["e2e"]["value"] > 0
