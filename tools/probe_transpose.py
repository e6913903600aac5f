"""Time the device ingest kernels on the headline matrix: the counting-sort
transpose (A -> A.T, and the ranked CSR) and the scoring work plan.
python tools/probe_transpose.py   (GPU box; run under ncu for per-kernel times)"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2009_02251_b200 import kernels as K  # noqa: E402
from paper_2009_02251_b200.sparse import DeviceCSR  # noqa: E402

cfg, M, tr, va, te, _ = bench._workload()
dev = torch.device("cuda")
ip = torch.as_tensor(tr.indptr.astype("int64"), device=dev)
ix = torch.as_tensor(tr.indices, device=dev)
dv = torch.as_tensor(tr.data, device=dev)
m, n = tr.shape
for it in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    tp, ti, tv = K.csr_transpose(ip, ix, dv, n)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    deg = tp[1:] - tp[:-1]
    order = torch.sort(-deg, stable=True).indices
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    rank = torch.empty(n, dtype=torch.int32, device=dev)
    rank[order] = torch.arange(n, dtype=torch.int32, device=dev)
    rk, rv = K.rank_rows(ip, ix, dv, n, rank)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    c = DeviceCSR(tp, ti, tv, (n, m))
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"transpose {1e3 * (t1 - t):.2f} ms | popularity sort {1e3 * (t2 - t1):.2f} | ranked {1e3 * (t3 - t2):.2f} "
          f"| DeviceCSR plans {1e3 * (t4 - t3):.2f}", flush=True)
