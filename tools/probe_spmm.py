"""SpMM per-call times on the headline workload (A @ X and A.T @ Y, b = 20),
with and without the shared-memory hot set (GPU box)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2009_02251_b200 as P  # noqa: E402
from paper_2009_02251_b200 import kernels as K  # noqa: E402

cfg, M, tr, va, te, _ = bench._workload()
A = P.SparseRatings(tr, *cfg.bounds)
d = A.device()
dev = torch.device("cuda")
X = torch.randn(A.n, 20, dtype=torch.float64, device=dev)
Yu = torch.randn(A.m, 20, dtype=torch.float64, device=dev)
out_m = torch.empty(A.m, 20, dtype=torch.float64, device=dev)
out_n = torch.empty(A.n, 20, dtype=torch.float64, device=dev)


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for hot in (False, True):
    K.SPMM_HOT = hot
    ref = K.spmm(d.A, X, out_m).clone()
    print(f"hot={hot}: A@X {t(lambda: K.spmm(d.A, X, out_m)):.1f} us   A.T@Y {t(lambda: K.spmm(d.AT, Yu, out_n)):.1f} us",
          flush=True)
K.SPMM_HOT = False
a = K.spmm(d.A, X, out_m).clone()
K.SPMM_HOT = True
b = K.spmm(d.A, X, out_m).clone()
print("hot vs plain max rel diff", float(((a - b).abs().max() / a.abs().max())))

# one 40-column product vs two 20-column ones (the lookahead engine's fusion)
X40 = torch.randn(A.n, 40, dtype=torch.float64, device=dev)
Y40 = torch.randn(A.m, 40, dtype=torch.float64, device=dev)
o40m = torch.empty(A.m, 40, dtype=torch.float64, device=dev)
o40n = torch.empty(A.n, 40, dtype=torch.float64, device=dev)
K.SPMM_HOT = False
print(f"b=40: A@X {t(lambda: K.spmm(d.A, X40, o40m)):.1f} us   A.T@Y {t(lambda: K.spmm(d.AT, Y40, o40n)):.1f} us",
      flush=True)
ref = torch.cat([K.spmm(d.A, X40[:, :20].contiguous(), out_m).clone(), K.spmm(d.A, X40[:, 20:].contiguous(), out_m).clone()], 1)
got = K.spmm(d.A, X40, o40m)
print("b=40 vs 2 x b=20 max rel diff", float((got - ref).abs().max() / ref.abs().max()))
X64 = torch.randn(A.n, 64, dtype=torch.float64, device=dev)
o64 = torch.empty(A.m, 64, dtype=torch.float64, device=dev)
print(f"b=64: A@X {t(lambda: K.spmm(d.A, X64, o64)):.1f} us")

# fp32 variant: float copy of X (the conversion is part of the call)
for name, plan, src, dst in (("A@X", d.A, X, out_m), ("A.T@Y", d.AT, Yu, out_n)):
    print(f"fp32 {name} {t(lambda: K.spmm(plan, src, dst, 'fp32')):.1f} us", flush=True)
X32 = X.float()
Y32 = torch.empty(A.m, 20, dtype=torch.float64, device=dev)

# hot/cold split through sparse_dense_mul (dense hot block on the tensor cores)
from paper_2009_02251_b200 import linalg as L  # noqa: E402
for h in (0, 128, 256, 512):
    L.DENSE_HOT = h
    ax = t(lambda: P.sparse_dense_mul(A, X, False, out=out_m))
    aty = t(lambda: P.sparse_dense_mul(A, Yu, True, out=out_n))
    a1 = P.sparse_dense_mul(A, X, False, out=out_m).clone()
    a2 = P.sparse_dense_mul(A, Yu, True, out=out_n).clone()
    if h == 0:
        r1, r2 = a1, a2
    print(f"dense-hot h={h}: A@X {ax:.1f} us  A.T@Y {aty:.1f} us  rel diff {float((a1 - r1).abs().max() / r1.abs().max()):.1e} "
          f"{float((a2 - r2).abs().max() / r2.abs().max()):.1e}", flush=True)

L.DENSE_HOT = 256
sp = d.hybrid(256)
print("hot share of nnz", sp.hot_nnz / A.nnz)
xh = X.index_select(0, sp.hot_items)
print(f"parts: cold A@X {t(lambda: K.spmm(sp.A, X, out_m)):.1f} us, dense A_hot@X {t(lambda: K.gemm_nn(sp.dense, xh, out_m, alpha=1.0, beta=1.0)):.1f} us, "
      f"cold A.T@Y {t(lambda: K.spmm(sp.AT, Yu, out_n)):.1f} us, dense A_hot.T@Y {t(lambda: K.gemm_tn(sp.dense, Yu)):.1f} us", flush=True)
