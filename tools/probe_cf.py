"""Per-call CF scoring times vs k on the headline workload, with the hot
(shared-memory) fraction of the streamed ratings and the L2 floor of the
cold part (GPU box)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2009_02251_b200 as P  # noqa: E402
from paper_2009_02251_b200 import kernels as K  # noqa: E402
from paper_2009_02251_b200.cf import _Samples  # noqa: E402

cfg, M, tr, va, te, _ = bench._workload()
lo, hi = cfg.bounds
A = P.SparseRatings(tr, lo, hi)
dev = torch.device("cuda")
vs = _Samples(va, dev)
kw = dict(block_size=20, passes=4, patience=2, min_improvement=1e-4, seed=0, max_rank=400)
prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
from paper_2009_02251_b200 import cf as _cf  # noqa: E402
_cf.PIPELINE = False
P.auto_latent_factors(A, vs, precision=prec, **kw)
torch.cuda.synchronize()
K.PROFILE = []
P.auto_latent_factors(A, vs, precision=prec, **kw)
torch.cuda.synchronize()
rec = [(n, e0.elapsed_time(e1), nb) for n, e0, e1, nb, _g in K.PROFILE if n == "cf_predict"]
K.PROFILE = None
d = A.device()
rk = d.A.ranked()[0].cpu().numpy()
deg_rated = int(d.A.nnz)
ks = [20 * (i + 1) for i in range(len(rec))]
tot = 0.0
for (n, ms, nb), k in zip(rec, ks):  # noqa: B007
    nhot = min(208 * 1024 // ((4 if prec == 'fp32' else 8) * k), A.n)
    hot = float(np.mean(rk < nhot))
    cold_gb = (1 - hot) * deg_rated * (4 if prec == 'fp32' else 8) * k / 1e9
    floor = cold_gb / 18.9  # ms at the measured 1920-B L2 gather ceiling
    tot += ms
    print(f"k={k:4d} ms={ms:6.3f} nhot={nhot:5d} hot={hot:.3f} cold={cold_gb:6.2f} GB floor={floor:.3f} ms "
          f"eff={floor / ms:.2f}", flush=True)
print("total", round(tot, 3))
