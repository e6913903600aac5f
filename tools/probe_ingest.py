"""Where the CSR ingest time goes (GPU box): upload, plans, transpose, checks."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2009_02251_b200 as P  # noqa: E402
from paper_2009_02251_b200 import sparse as S  # noqa: E402
from paper_2009_02251_b200.hostio import to_device  # noqa: E402

cfg, M, tr, va, te, _ = bench._workload()
dev = torch.device("cuda")
for rep in range(3):
    T = {}
    torch.cuda.synchronize()
    t = time.perf_counter()

    def mark(k):
        global t
        torch.cuda.synchronize()
        now = time.perf_counter()
        T[k] = round((now - t) * 1e3, 2)
        t = now

    ip = to_device(tr.indptr, np.int64, dev)
    ind = to_device(tr.indices, np.int32, dev)
    val = to_device(tr.data, np.float64, dev)
    mark("upload")
    A = S.DeviceCSR(ip, ind, val, tr.shape)
    mark("plans")
    AT = A.transposed()
    mark("transpose")
    P.SparseRatings(tr, *cfg.bounds)
    mark("full SparseRatings")
    print(T, flush=True)
