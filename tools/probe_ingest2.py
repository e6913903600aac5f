"""Breakdown of the end-to-end path's ingest (host CSR in -> device
image, plans, ranked CSR, sample grouping): every stage below is wrapped
with synchronize + wall clock (nested stages are included in their
parents).  python tools/probe_ingest2.py [pinned]   (GPU box)"""
import collections
import functools
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2009_02251_b200 as P  # noqa: E402
from paper_2009_02251_b200 import cf, hostio, sparse  # noqa: E402

T = collections.defaultdict(float)


def timed(owner, name, label=None):
    fn = getattr(owner, name)

    @functools.wraps(fn)
    def w(*a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        T[label or name] += (time.perf_counter() - t) * 1e3
        return r
    setattr(owner, name, w)


for owner, name in [(hostio, "to_device"), (sparse.DeviceCSR, "transposed"), (sparse.DeviceCSR, "ranked"),
                    (sparse, "segment_plan_t"), (sparse, "warp_plan_t"), (sparse.DeviceRatings, "check"),
                    (sparse.DeviceRatings, "_init_from"), (cf._Samples, "__init__"), (cf._Samples, "plan_for"),
                    (sparse.SparseRatings, "__init__")]:
    timed(owner, name, f"{getattr(owner, '__name__', owner)}.{name}")
sparse.to_device = hostio.to_device
cf.to_device = hostio.to_device

cfg, M, tr, va, te, _ = bench._workload()
lo, hi = cfg.bounds
dev = torch.device("cuda")
if len(sys.argv) > 1 and sys.argv[1] == "pinned":
    def pin(a):
        t = torch.empty(a.shape, dtype=torch.from_numpy(a[:1]).dtype, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()
    from scipy import sparse as sp
    tr = sp.csr_matrix((pin(tr.data), pin(tr.indices), pin(tr.indptr.astype(np.int64))), shape=tr.shape)
    va = tuple(pin(np.asarray(x)) for x in va)
    te = tuple(pin(np.asarray(x)) for x in te)
for it in range(4):
    T.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    A = P.SparseRatings(tr, lo, hi)
    f, trace = P.auto_latent_factors(A, va, block_size=bench.BLOCK, passes=bench.PASSES, patience=bench.PATIENCE,
                                     min_improvement=bench.MIN_IMPROVEMENT, seed=bench.SEED, max_rank=bench.K_CAP)
    mae, rmse = P.evaluate_errors(A, f, te)
    torch.cuda.synchronize()
    tot = (time.perf_counter() - t0) * 1e3
    if it:
        print(f"total {tot:.1f} ms | " + " | ".join(f"{k} {v:.1f}" for k, v in sorted(T.items(), key=lambda x: -x[1])),
              flush=True)
    del A, f, trace
