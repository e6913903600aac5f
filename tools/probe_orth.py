"""Launch-list probe: svdrec_orth (CholeskyQR2 + gated TSQR) on 138493 x 20."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2009_02251_b200 import kernels as K  # noqa: E402
Y = torch.randn(138493, 20, dtype=torch.float64, device="cuda")
for _ in range(3):
    K.orth(Y.clone())
torch.cuda.synchronize()
