"""Launch-list probe: the Gaussian sketch stream for one 26744 x 20 block."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2009_02251_b200.linalg import GaussianStream  # noqa: E402
g = GaussianStream(0)
for _ in range(3):
    g.normal_device(26744, 20)
torch.cuda.synchronize()
