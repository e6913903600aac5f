"""The hot / cold chunk kernel with NO hot rows (every chunk gathered into
registers by LDG.128) against the TMA pipeline, A @ X and A.T @ Y on the
headline workload: is the register gather on chunk records competitive
without the shared-memory table? (GPU box)"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2009_02251_b200 as P  # noqa: E402
from paper_2009_02251_b200 import kernels as K  # noqa: E402
from paper_2009_02251_b200.kernels import call, ptr, query, stream_handle  # noqa: E402

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


def hc(plan, X, Y, nhot):
    b = X.shape[1]
    if getattr(plan, "item_rank", None) is None:
        plan.item_rank = torch.zeros(plan.n, dtype=torch.int32, device=dev)
        plan.hot_items = torch.zeros(1, dtype=torch.int32, device=dev)
    nwarp, wchunk, recs, ents, _ = plan.hot_packed(nhot, query("svdrec_spmm_hc_warps_per_sm"))
    call("svdrec_spmm_hc", plan.nseg, ptr(ents), ptr(X), b, plan.n, ptr(plan.hot_items), nhot, ptr(Y), b, b,
         plan.nlong, ptr(plan.long_row), ptr(plan.long_s0), ptr(plan.long_s1), nwarp, ptr(wchunk), ptr(recs),
         ptr(plan.partial(b)), stream_handle())


for b in [int(x) for x in sys.argv[1:]] or [8, 16, 20, 32]:
    for name, plan, rows in (("A@X", d.A, A.m), ("A.T@Y", d.AT, A.n)):
        X = torch.randn(plan.n, b, dtype=torch.float64, device=dev)
        o1, o2 = (torch.empty(rows, b, dtype=torch.float64, device=dev) for _ in range(2))
        hc(plan, X, o1, 0)
        K.spmm(plan, X, o2)
        err = float((o1 - o2).abs().max() / o2.abs().max())
        print(f"b={b} {name}: all-cold register gather {t(lambda: hc(plan, X, o1, 0)):.1f} us   "
              f"TMA pipeline {t(lambda: K.spmm(plan, X, o2)):.1f} us   max rel diff {err:.1e}", flush=True)
