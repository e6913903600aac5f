import sys, torch
sys.path.insert(0, '.')
from paper_2009_02251_b200 import kernels as K
r = int(sys.argv[1])
Y = torch.randn(r, 20, dtype=torch.float64, device="cuda")
G = torch.empty(20, 20, dtype=torch.float64, device="cuda")
for _ in range(3):
    K.gram(Y, G)
torch.cuda.synchronize()
