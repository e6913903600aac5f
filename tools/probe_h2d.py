"""Host->device upload of the headline CSR: pageable vs page-locked in place (GPU box)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

cfg, M, tr, va, te, _ = bench._workload()
arrs = [np.ascontiguousarray(tr.indptr.astype(np.int64)), np.ascontiguousarray(tr.indices.astype(np.int32)),
        np.ascontiguousarray(tr.data)]
nb = sum(a.nbytes for a in arrs)
cudart = torch.cuda.cudart()


def t_pageable():
    torch.cuda.synchronize()
    t = time.perf_counter()
    outs = [torch.from_numpy(a).to("cuda", non_blocking=False) for a in arrs]
    torch.cuda.synchronize()
    return time.perf_counter() - t


def t_registered():
    torch.cuda.synchronize()
    t = time.perf_counter()
    outs = []
    for a in arrs:
        cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter()
    s = torch.cuda.current_stream()
    for a in arrs:
        outs.append(torch.from_numpy(a).to("cuda", non_blocking=True))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    for a in arrs:
        cudart.cudaHostUnregister(a.ctypes.data)
    t3 = time.perf_counter()
    return t3 - t, t1 - t, t2 - t1, t3 - t2


for _ in range(3):
    p = t_pageable()
    r = t_registered()
    print(f"{nb / 1e6:.0f} MB: pageable {p * 1e3:.1f} ms ({nb / p / 1e9:.1f} GB/s) | registered total {r[0] * 1e3:.1f} ms "
          f"(register {r[1] * 1e3:.1f}, copy {r[2] * 1e3:.1f} = {nb / r[2] / 1e9:.1f} GB/s, unregister {r[3] * 1e3:.1f})",
          flush=True)
