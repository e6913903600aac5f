"""Do clock samplers perturb the timed steps?  nvidia-smi -lms N vs NVML thread vs none."""
import subprocess
import sys
import threading
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2009_02251_b200 as P  # noqa: E402
from paper_2009_02251_b200.cf import _Samples  # noqa: E402

cfg, M, tr, va, te, _ = bench._workload()
lo, hi = cfg.bounds
A = P.SparseRatings(tr, lo, hi)
dev = torch.device("cuda")
vs, ts = _Samples(va, dev), _Samples(te, dev)


def step():
    f, trace = P.auto_latent_factors(A, vs, block_size=bench.BLOCK, passes=bench.PASSES, patience=bench.PATIENCE,
                                     min_improvement=bench.MIN_IMPROVEMENT, seed=bench.SEED, max_rank=bench.K_CAP)
    return P.evaluate_errors(A, f, ts)


def run(tag):
    ts_ = []
    for _ in range(15):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        torch.cuda.synchronize()
        ts_.append(e0.elapsed_time(e1))
    print(f"{tag:12s} max {max(ts_):6.1f} median {sorted(ts_)[7]:6.1f}  " + " ".join(f"{t:.0f}" for t in ts_), flush=True)


for _ in range(3):
    step()
run("none")
for lms in (50, 200):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", str(lms)],
                         stdout=subprocess.DEVNULL)
    time.sleep(2.0)
    run(f"smi {lms}ms")
    p.terminate()
    p.wait()
import pynvml  # noqa: E402
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
stop = False


def poll():
    while not stop:
        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        time.sleep(0.05)


th = threading.Thread(target=poll)
th.start()
time.sleep(0.5)
run("nvml 50ms")
stop = True
th.join()
