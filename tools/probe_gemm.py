"""Time the tall-skinny fp64 products of the QB/CF path: ours vs cuBLAS (torch)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2009_02251_b200 import kernels as K  # noqa: E402


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


d = torch.device("cuda")
for (r, p, q) in [(138493, 240, 20), (138493, 120, 20), (26744, 240, 20), (26744, 240, 240), (138493, 20, 20)]:
    X = torch.randn(r, p, dtype=torch.float64, device=d)
    C = torch.randn(p, q, dtype=torch.float64, device=d)
    Y = torch.randn(r, q, dtype=torch.float64, device=d)
    nn_ours = t(lambda: K.gemm_nn(X, C))
    nn_cub = t(lambda: torch.mm(X, C))
    tn_ours = t(lambda: K.gemm_tn(X, Y))
    tn_cub = t(lambda: torch.mm(X.T, Y))
    gb = (r * p + r * q) * 8 / 1e9
    print(f"r={r} p={p} q={q}: nn ours {nn_ours:.1f} us cublas {nn_cub:.1f} us | tn ours {tn_ours:.1f} us "
          f"cublas {tn_cub:.1f} us | bytes {gb*1e3:.0f} MB -> {gb/6.5e3*1e6:.1f} us at 6.5 TB/s", flush=True)
