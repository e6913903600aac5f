"""Tall-skinny Y += Q @ C and Bt @ Z at headline shapes (GPU box)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2009_02251_b200 import kernels as K  # noqa: E402

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


for Kd in (60, 140, 240):
    Q = torch.randn(138493, 256, dtype=torch.float64, device=dev)[:, :Kd]
    C = torch.randn(Kd, 20, dtype=torch.float64, device=dev)
    Y = torch.randn(138493, 20, dtype=torch.float64, device=dev)
    Bt = torch.randn(26744, 256, dtype=torch.float64, device=dev)[:, :Kd]
    Z = torch.randn(Kd, Kd, dtype=torch.float64, device=dev)
    a = t(lambda: K.gemm_nn(Q, C, Y, alpha=-1.0, beta=1.0))
    b = t(lambda: K.gemm_nn(Bt, Z))
    print(f"K={Kd}: Q@C {a:.1f} us ({138493 * Kd * 8 / a / 1e3:.0f} GB/s)   Bt@Z {b:.1f} us", flush=True)
