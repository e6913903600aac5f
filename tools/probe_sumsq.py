import sys, torch
sys.path.insert(0, '.')
from paper_2009_02251_b200 import kernels as K
dev = torch.device('cuda')
for r, q, ld in ((26744, 20, 256), (138493, 20, 20), (18000000, 1, 1)):
    X = torch.randn(r, ld, dtype=torch.float64, device=dev)[:, :q]
    colsq = torch.empty(q, dtype=torch.float64, device=dev); tot = torch.empty(1, dtype=torch.float64, device=dev)
    K.sumsq(X, colsq, tot); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): K.sumsq(X, colsq, tot)
    e1.record(); torch.cuda.synchronize()
    ref = (X * X).sum(0)
    print(r, q, f"{e0.elapsed_time(e1) / 20 * 1e3:.1f} us", float((colsq - ref).abs().max() / ref.abs().max()))
