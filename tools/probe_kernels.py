"""Per-call device times of the main kernels at headline shapes (GPU box)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2009_02251_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda")
rng = np.random.default_rng(0)
m, n, b = 138493, 26744, 20


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


Y = torch.randn(m, b, dtype=torch.float64, device=dev)
Yc = Y.clone()
print(f"orth {m}x{b}: {t(lambda: K.orth(Yc.copy_(Y), Yc)):.1f} us (incl. copy)")
print(f"copy only: {t(lambda: Yc.copy_(Y)):.1f} us")
print(f"tsqr {m}x{b}: {t(lambda: K.tsqr(Y)):.1f} us")
for kk in (60, 140, 240):
    Q = torch.randn(m, 256, dtype=torch.float64, device=dev)[:, :kk]
    C = torch.randn(kk, b, dtype=torch.float64, device=dev)
    us_nn = t(lambda: K.gemm_nn(Q, C, Yc, -1.0, 1.0))
    us_tn = t(lambda: K.gemm_tn(Q, Y))
    gb = m * 256 * 8 / 1e9 * kk / 256
    print(f"K={kk}: gemm_nn {us_nn:.1f} us ({gb / us_nn * 1e6:.0f} GB/s of Q), gemm_tn {us_tn:.1f} us "
          f"({gb / us_tn * 1e6:.0f} GB/s)")
    G = torch.randn(kk + 50, kk, dtype=torch.float64, device=dev)
    G = G.T @ G
    st = K.new_status(dev)
    print(f"K={kk}: inv_sqrt {t(lambda: K.inv_sqrt(G, st)):.1f} us")
