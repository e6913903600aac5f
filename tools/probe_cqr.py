"""Timing probe of the CholeskyQR pieces on a 138493 x b block (bench shape):
svdrec_orth (CholeskyQR2 + gated TSQR), svdrec_gram (Gram + two-level
reduction, no Cholesky) and svdrec_chol_apply (one-CTA Cholesky + apply),
back to back with CUDA events (the block stays in L2, as in the pipeline)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2009_02251_b200 import kernels as K  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 138493
for b in (20, 32):
    Y = torch.randn(r, b, dtype=torch.float64, device="cuda")
    Q = torch.empty_like(Y)
    G = torch.empty(b, b, dtype=torch.float64, device="cuda")
    K.gram(Y, G)
    res = {}
    for name, fn in (("orth", lambda: K.orth(Y, Q)), ("gram", lambda: K.gram(Y, G)),
                     ("chol_apply", lambda: K.chol_apply(G, Y, Q))):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 200
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name] = round(e0.elapsed_time(e1) / n * 1e3, 2)
    print(f"r={r} b={b} us/call", res, flush=True)
