"""Probe the eigensolver on a realistic Gram: time per call, sweeps, accuracy.

python tools/probe_syev.py   (GPU box)
"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2009_02251_b200 import kernels as K, _lib  # noqa: E402


def flags_sweeps(k):
    al = lambda x: (x + 255) // 256 * 256  # noqa: E731
    off = 2 * al(k * k * 8) + al(k * 8)
    buf = _lib.scratch().buf
    return int(buf[off + 12: off + 16].view(torch.int32).item())


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1))
    return min(t), out


rng = np.random.default_rng(0)
for k in (40, 120, 240, 400):
    n = 26744
    s = np.geomspace(1e4, 30, k)
    Bt = rng.standard_normal((n, k)) * s / np.sqrt(n)
    Btd = torch.from_numpy(Bt).cuda()
    G = K.gemm_tn(Btd, Btd)
    st = K.new_status(G.device)
    ms, (w, V) = timed(lambda: K.syev(G, st))
    sw = flags_sweeps(k)
    ref = np.linalg.eigvalsh(G.cpu().numpy())
    err = np.max(np.abs(w.cpu().numpy() - ref)) / ref[-1]
    # warm start from the leading (k-20) block's eigenvectors
    k0 = k - 20
    G0 = G[:k0, :k0].contiguous()
    _, V0s = K.syev(G0, st)
    V0 = torch.eye(k, dtype=torch.float64, device=G.device)
    V0[:k0, :k0] = V0s
    msw, (w2, V2) = timed(lambda: K.syev(G, st, V0))
    sw2 = flags_sweeps(k)
    err2 = np.max(np.abs(w2.cpu().numpy() - ref)) / ref[-1]
    it = torch.zeros(1, dtype=torch.int32, device=G.device)
    msn, Z = timed(lambda: K.inv_sqrt(G, st, it))
    Zr = (V2 * w2.rsqrt()) @ V2.T
    errn = float((Z - Zr).norm() / Zr.norm())
    print(f"k={k}: cold {ms:.3f} ms sweeps={sw} relerr={err:.1e} | warm {msw:.3f} ms sweeps={sw2} relerr={err2:.1e} "
          f"| NS {msn:.3f} ms iters={int(it.item())} relerr={errn:.1e} status={int(st.item())}", flush=True)
