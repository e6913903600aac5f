"""Feasibility of an L2-tiled SpMM on config 4 (8M x 1M, 2e9 ratings, b =
64): the product split into column tiles whose slice of the dense operand
fits L2 -- A @ X over T item tiles, A.T @ Y over T user tiles -- each tile a
pass of the TMA kernel over the row segments holding that tile's columns
(timing only: the passes overwrite instead of accumulating).
python tools/probe_c4_tiles.py   (GPU box)"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2009_02251_b200 import kernels as K, synth  # noqa: E402
from paper_2009_02251_b200._lib import call, ptr, query, stream_handle  # noqa: E402
from paper_2009_02251_b200.sparse import SEG_MAX, warp_plan_t  # noqa: E402

dev = torch.device("cuda")
A = synth.generate_device(synth.CONFIGS["c4_2b"], dev)
d = A.device()
b = 64
sms = torch.cuda.get_device_properties(dev).multi_processor_count
wps = query("svdrec_spmm_warps_per_sm", b)
K.SPMM_HOT = False


def plans(c, ntiles):
    cols = torch.linspace(0, c.n, ntiles + 1, device=dev).round().to(torch.int32)
    bounds = torch.empty((ntiles + 1) * c.m, dtype=torch.int64, device=dev)
    call("svdrec_csr_tile_bounds", c.m, ptr(c.indptr), ptr(c.indices), ntiles, ptr(cols), ptr(bounds),
         stream_handle())
    bounds = bounds.view(ntiles + 1, c.m)
    out = []
    for t in range(ntiles):
        beg, end = bounds[t], bounds[t + 1]
        deg = end - beg
        nps = (deg + SEG_MAX - 1) // SEG_MAX  # empty rows: no segment
        seg_row = torch.repeat_interleave(torch.arange(c.m, device=dev), nps)
        first = torch.cumsum(nps, 0) - nps
        within = torch.arange(seg_row.numel(), device=dev) - first[seg_row]
        sb = beg[seg_row] + within * SEG_MAX
        se = torch.minimum(sb + SEG_MAX, end[seg_row])
        slot = torch.full_like(seg_row, -1).to(torch.int32)  # (split rows overwrite: timing only)
        nw = int(max(1, min(seg_row.numel(), sms * wps)))
        out.append((seg_row.to(torch.int32), sb, se, slot, nw, warp_plan_t(sb, se, nw), int(seg_row.numel())))
    return out


def run(c, X, Y, pl):
    for sr, sb, se, sl, nw, ws, ns in pl:
        call("svdrec_spmm", ns, ptr(sr), ptr(sb), ptr(se), ptr(sl), ptr(c.indices), ptr(c.values), ptr(X), b,
             c.n, ptr(Y), b, b, 0, None, None, None, nw, ptr(ws), None, stream_handle())


def timeit(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name, c in (("A @ X", d.A), ("A.T @ Y", d.AT)):
    X = torch.randn(c.n, b, dtype=torch.float64, device=dev)
    Y = torch.empty(c.m, b, dtype=torch.float64, device=dev)
    t0 = timeit(lambda: K.spmm(c, X, Y))
    print(f"{name}: one pass {t0:.1f} ms (X = {X.numel() * 8 / 2**20:.0f} MB)", flush=True)
    for nt in ((2, 4, 6, 8) if c.n < 2_000_000 else (16, 32, 48, 64)):
        pl = plans(c, nt)
        t1 = timeit(lambda: run(c, X, Y, pl))
        print(f"  {nt:3d} column tiles ({X.numel() * 8 / nt / 2**20:.0f} MB each): {t1:.1f} ms", flush=True)
        del pl
    del X, Y
