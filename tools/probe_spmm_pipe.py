"""Pipelined SpMM (csrc/spmm.cu k_spmm_pipe) on the headline workload: per-call
times of A @ X and A.T @ Y at several widths, checked against the plain
row-per-warp kernel (GPU box)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2009_02251_b200 as P  # noqa: E402
from paper_2009_02251_b200 import kernels as K  # noqa: E402
from paper_2009_02251_b200.kernels import call, ptr, stream_handle  # noqa: E402

cfg, M, tr, va, te, _ = bench._workload()
A = P.SparseRatings(tr, *cfg.bounds)
d = A.device()
dev = torch.device("cuda")
K.SPMM_HOT = False


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


def plain(plan, X, Y):
    b = X.shape[1]
    call("svdrec_spmm", plan.nseg, ptr(plan.seg_row), ptr(plan.seg_begin), ptr(plan.seg_end), ptr(plan.seg_slot),
         ptr(plan.indices), ptr(plan.values), ptr(X), b, plan.n, ptr(Y), b, b, plan.nlong, ptr(plan.long_row),
         ptr(plan.long_s0), ptr(plan.long_s1), 0, None, None, None, None, None, ptr(plan.partial(b)), stream_handle())
    return Y


widths = [int(x) for x in sys.argv[1:]] or [2, 8, 16, 20, 32, 40, 64]
for b in widths:
    X = torch.randn(A.n, b, dtype=torch.float64, device=dev)
    Yu = torch.randn(A.m, b, dtype=torch.float64, device=dev)
    om, on = torch.empty(A.m, b, dtype=torch.float64, device=dev), torch.empty(A.n, b, dtype=torch.float64, device=dev)
    rm, rn = torch.empty_like(om), torch.empty_like(on)
    plain(d.A, X, rm)
    plain(d.AT, Yu, rn)
    K.spmm(d.A, X, om)
    K.spmm(d.AT, Yu, on)
    e1 = float((om - rm).abs().max() / rm.abs().max())
    e2 = float((on - rn).abs().max() / rn.abs().max())
    line = f"b={b}: A@X {t(lambda: K.spmm(d.A, X, om)):.1f} us  A.T@Y {t(lambda: K.spmm(d.AT, Yu, on)):.1f} us  err {e1:.1e} {e2:.1e}"
    if b % 4 == 0:
        K.spmm(d.A, X, om, "fp32")
        e3 = float((om - rm).abs().max() / rm.abs().max())
        line += f"  fp32-X: A@X {t(lambda: K.spmm(d.A, X, om, 'fp32')):.1f} us (err {e3:.1e})"
    print(line, flush=True)
