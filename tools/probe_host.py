"""Host-side cost of one bench step: cProfile of the Python/ctypes layer.

python tools/probe_host.py   (GPU box)
"""
import cProfile
import pstats
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
A = P.SparseRatings(tr, lo, hi)
dev = torch.device("cuda")
A.device(dev)
vs, ts = _Samples(va, dev), _Samples(te, dev)


def step():
    f, trace = P.auto_latent_factors(A, vs, block_size=bench.BLOCK, passes=bench.PASSES, patience=bench.PATIENCE,
                                     min_improvement=bench.MIN_IMPROVEMENT, seed=bench.SEED, max_rank=bench.K_CAP)
    return P.evaluate_errors(A, f, ts)


for _ in range(3):
    step()
torch.cuda.synchronize()
t = time.perf_counter()
step()
torch.cuda.synchronize()
print(f"wall {1e3 * (time.perf_counter() - t):.2f} ms")
pr = cProfile.Profile()
pr.enable()
step()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
