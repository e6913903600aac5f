"""A @ X on the headline workload: hot / cold chunk kernel (k_spmm_hc) vs the
TMA pipeline (k_spmm_pipe), per-call times and the difference of their
results (GPU box)."""
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


K.HC_WIDTHS = frozenset(range(2, 33, 2))  # measure every supported width
print("hc warps/SM", K.query("svdrec_spmm_hc_warps_per_sm"))
for b in [int(x) for x in sys.argv[1:]] or [2, 8, 16, 20, 32]:
    X = torch.randn(A.n, b, dtype=torch.float64, device=dev)
    o1, o2 = (torch.empty(A.m, b, dtype=torch.float64, device=dev) for _ in range(2))
    K.SPMM_HOT = True
    nh = K._hc_rows(d.A, b, b, b)
    K.spmm(d.A, X, o1)
    th = t(lambda: K.spmm(d.A, X, o1))
    K.SPMM_HOT = False
    K.spmm(d.A, X, o2)
    tp = t(lambda: K.spmm(d.A, X, o2))
    err = float((o1 - o2).abs().max() / o2.abs().max())
    print(f"b={b}: hot/cold ({nh} hot rows) {th:.1f} us   pipeline {tp:.1f} us   max rel diff {err:.1e}", flush=True)
