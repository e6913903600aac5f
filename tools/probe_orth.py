"""Launch-list probe: svdrec_orth (CholeskyQR2 + gated TSQR) on r x b
(default 138493 x 20, the bench block).  Run under ncu for kernel times."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2009_02251_b200 import kernels as K  # noqa: E402
r = int(sys.argv[1]) if len(sys.argv) > 1 else 138493
b = int(sys.argv[2]) if len(sys.argv) > 2 else 20
Y = torch.randn(r, b, dtype=torch.float64, device="cuda")
for _ in range(3):
    K.orth(Y.clone())
torch.cuda.synchronize()
