"""Where the end-to-end (host arrays in, MAE out) time goes.

python tools/probe_e2e.py   (GPU box)
"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2009_02251_b200 as P  # noqa: E402
from paper_2009_02251_b200.cf import _Samples  # noqa: E402

cfg, M, tr, va, te, _ = bench._workload()
lo, hi = cfg.bounds
dev = torch.device("cuda")


def run(verbose):
    T = {}
    torch.cuda.synchronize()
    t = time.perf_counter()

    def mark(name):
        torch.cuda.synchronize()
        nonlocal t
        now = time.perf_counter()
        T[name] = (now - t) * 1e3
        t = now

    A = P.SparseRatings(tr, lo, hi)
    mark("SparseRatings")
    d = A.device(dev)
    mark("device upload + A.T + plans")
    vs = _Samples(va, dev)
    ts = _Samples(te, dev)
    mark("samples (val+test)")
    f, trace = P.auto_latent_factors(A, vs, block_size=bench.BLOCK, passes=bench.PASSES, patience=bench.PATIENCE,
                                     min_improvement=bench.MIN_IMPROVEMENT, seed=bench.SEED, max_rank=bench.K_CAP)
    mark("auto_latent_factors")
    P.evaluate_errors(A, f, ts)
    mark("evaluate_errors")
    if verbose:
        print(" | ".join(f"{k} {v:.1f} ms" for k, v in T.items()), f"total {sum(T.values()):.1f} ms")


for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    run(i >= 1)
