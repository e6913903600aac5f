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
