"""Per-step GPU times over many steps (outlier hunt), with / without GC."""
import gc
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
vs, ts = _Samples(va, dev), _Samples(te, dev)


def step():
    f, trace = P.auto_latent_factors(A, vs, block_size=bench.BLOCK, passes=bench.PASSES, patience=bench.PATIENCE,
                                     min_improvement=bench.MIN_IMPROVEMENT, seed=bench.SEED, max_rank=bench.K_CAP)
    return P.evaluate_errors(A, f, ts)


for _ in range(3):
    step()
for mode in ("gc on", "gc off"):
    if mode == "gc off":
        gc.disable()
    ts_ = []
    for _ in range(12):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        e0.record()
        step()
        e1.record()
        torch.cuda.synchronize()
        ts_.append((e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t)))
    print(mode, " ".join(f"{a:.1f}/{b:.1f}" for a, b in ts_), flush=True)
    print("  mem allocated", torch.cuda.memory_allocated() >> 20, "MB reserved", torch.cuda.memory_reserved() >> 20, "MB")
