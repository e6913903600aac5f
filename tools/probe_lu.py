"""Time lu_lower on the bench shape (138493 x 20) with CUDA events."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2009_02251_b200 import kernels as K  # noqa: E402
Y0 = torch.randn(138493, 20, dtype=torch.float64, device="cuda")
st = K.new_status(Y0.device)
Y = Y0.clone()
K.lu_lower(Y, st)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    Y = Y0.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    K.lu_lower(Y, st)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(f"lu_lower 138493 x 20: {min(ts):.1f} us (min of 10)")
