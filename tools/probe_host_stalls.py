"""Where do the occasional slow steps lose time on the host? (GPU box)"""
import gc
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2009_02251_b200 as P  # noqa: E402
from paper_2009_02251_b200 import cf  # noqa: E402
from paper_2009_02251_b200.cf import _Samples  # noqa: E402

cfg, M, tr, va, te, _ = bench._workload()
A = P.SparseRatings(tr, *cfg.bounds)
dev = torch.device("cuda")
vs, ts = _Samples(va, dev), _Samples(te, dev)


def step():
    f, trace = P.auto_latent_factors(A, vs, block_size=20, passes=4, patience=2, min_improvement=1e-4, seed=0,
                                     max_rank=400)
    return P.evaluate_errors(A, f, ts)


for _ in range(3):
    step()
gc.collect()
gc.freeze()
gc.disable()
for i in range(30):
    cf._HOST_TRACE = []
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record()
    step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    tr_ = cf._HOST_TRACE
    worst = max(tr_, key=lambda x: x[1] + x[2] + x[3])
    print(f"step {i}: {ms:.1f} ms; worst block k={worst[0]} submit {worst[1]*1e3:.1f} next {worst[2]*1e3:.1f} "
          f"collect {worst[3]*1e3:.1f} ms", flush=True)
