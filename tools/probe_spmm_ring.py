"""TMA SpMM ring geometry (stages x warps per CTA, two CTAs per SM) on
config 3, b = 20: A @ X and A.T @ Y per call for library builds with
-DSVDREC_SPMM_S2=S -DSVDREC_SPMM_W2=W.  python tools/probe_spmm_ring.py lib1.so [lib2.so ...]"""
import subprocess
import sys
from pathlib import Path

if len(sys.argv) > 2 or (len(sys.argv) == 2 and not sys.argv[1].startswith("--one=")):
    for lib in sys.argv[1:]:
        subprocess.run([sys.executable, __file__, f"--one={lib}"], check=False)
    sys.exit(0)

import torch  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2009_02251_b200 import _lib  # noqa: E402

lib = sys.argv[1][len("--one="):] if len(sys.argv) > 1 else None
if lib:
    _lib.LIB_PATH = Path(lib).resolve()
import bench  # noqa: E402
import paper_2009_02251_b200 as P  # noqa: E402
from paper_2009_02251_b200 import kernels as K  # noqa: E402

cfg, M, tr, va, te, _ = bench._workload()
A = P.SparseRatings(tr, *cfg.bounds)
d = A.device()
b = 20
K.SPMM_HOT = False
res = []
for name, c in (("A @ X", d.A), ("A.T @ Y", d.AT)):
    X = torch.randn(c.n, b, dtype=torch.float64, device="cuda")
    Y = torch.empty(c.m, b, dtype=torch.float64, device="cuda")
    for _ in range(3):
        K.spmm(c, X, Y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        K.spmm(c, X, Y)
    e1.record()
    torch.cuda.synchronize()
    res.append(f"{name} {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
print(Path(lib).name if lib else "default", "|", " | ".join(res), flush=True)
