"""Config 4 (8M x 1M, 2e9 ratings, b = 64): A @ X with X's rows in
popularity order (columns relabelled by rank -- entry order unchanged, so
the sums are bitwise equal) and a persisting L2 window over the hottest
rows, against the plain call.  python tools/probe_c4_l2.py   (GPU box)"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2009_02251_b200 import kernels as K, synth  # noqa: E402
from paper_2009_02251_b200._lib import load, ptr, stream_handle  # noqa: E402
from paper_2009_02251_b200.sparse import DeviceCSR  # noqa: E402

dev = torch.device("cuda")
A = synth.generate_device(synth.CONFIGS["c4_2b"], dev)
d = A.device()
c = d.A
lib = load()
b = int(sys.argv[1]) if len(sys.argv) > 1 else 64
X = torch.randn(c.n, b, dtype=torch.float64, device=dev)
Y = torch.empty(c.m, b, dtype=torch.float64, device=dev)
order = c.hot_items.to(torch.int64)
rank = c.item_rank
# relabelled copy of the CSR (same plans: the segment arrays are shared)
rc = object.__new__(DeviceCSR)
rc.__dict__.update(c.__dict__)
rc.indices = rank[c.indices.to(torch.int64)].to(torch.int32)
rc.item_rank = None  # keep the hot-set kernel out of it
Xr = X[order].contiguous()


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


K.SPMM_HOT = False
t0 = timeit(lambda: K.spmm(c, X, Y))
Y0 = Y.clone()
t1 = timeit(lambda: K.spmm(rc, Xr, Y))
same = bool(torch.equal(Y, Y0))
print(f"b={b}: plain {t0:.2f} ms | rank-ordered X {t1:.2f} ms (bitwise equal: {same})", flush=True)
for mb in (16, 32, 48, 64, 96):
    nbytes = min(mb << 20, Xr.numel() * 8)
    got = lib.svdrec_l2_window(stream_handle(), ptr(Xr), nbytes)
    t2 = timeit(lambda: K.spmm(rc, Xr, Y))
    lib.svdrec_l2_window(stream_handle(), None, 0)
    print(f"  + persisting window over the hottest {mb} MB (applied {got / 2**20:.0f} MB): {t2:.2f} ms "
          f"(equal: {bool(torch.equal(Y, Y0))})", flush=True)
