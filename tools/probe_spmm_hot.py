"""A @ X on the headline matrix: the hot-set kernel (shared-memory hot rows
+ L2 gathers for the rest) against the TMA-gather kernel -- agreement and
CUDA-event time per call for several b.  python tools/probe_spmm_hot.py"""
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
K.HOT_WIDTHS = frozenset(range(2, 65, 2))  # measure every supported width
args = [a for a in sys.argv[1:] if a != "c4"]
if "c4" in sys.argv[1:]:  # the scale-out matrix (device-generated, 2e9 ratings)
    from paper_2009_02251_b200 import synth
    del A, d, M, tr, va, te
    A = synth.generate_device(synth.CONFIGS["c4_2b"], torch.device("cuda"))
    d = A.device()
for b in [int(x) for x in (args or ["20", "8", "32"])]:
    X = torch.randn(d.n, b, dtype=torch.float64, device=dev)
    out = {}
    reps = 20 if d.nnz < 1e9 else 3
    for mode in (False, True):
        K.SPMM_HOT = mode
        Y = torch.empty(d.m, b, dtype=torch.float64, device=dev)
        for _ in range(3):
            K.spmm(d.A, X, Y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            K.spmm(d.A, X, Y)
        e1.record()
        torch.cuda.synchronize()
        out[mode] = (Y.clone(), e0.elapsed_time(e1) / reps * 1e3)
    err = float((out[True][0] - out[False][0]).abs().max() / out[False][0].abs().max())
    print(f"b={b:3d} tma {out[False][1]:7.1f} us  hot {out[True][1]:7.1f} us  rel.diff {err:.2e}  "
          f"nhot={K._hot_rows(d.A, b, b, b) if K.SPMM_HOT else 0}", flush=True)
