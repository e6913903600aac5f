"""Is the TMA-gather SpMM bound by the SM's TMA unit?  Runs A @ X (b = 20,
config 3) as the TMA kernel on the first fraction f of the row segments and
the register-gather kernel (no TMA: LDG gathers) on the rest, on two streams
at once, against the TMA kernel alone on everything (timing only; split rows'
fix-up skipped).  python tools/probe_spmm_dual.py"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2009_02251_b200 as P  # noqa: E402
from paper_2009_02251_b200 import kernels as K  # noqa: E402
from paper_2009_02251_b200._lib import call, ptr, query  # noqa: E402
from paper_2009_02251_b200.sparse import warp_plan_t  # noqa: E402

cfg, M, tr, va, te, _ = bench._workload()
A = P.SparseRatings(tr, *cfg.bounds)
d = A.device()
c = d.A
dev = torch.device("cuda")
b = 20
X = torch.randn(c.n, b, dtype=torch.float64, device=dev)
Y = torch.empty(c.m, b, dtype=torch.float64, device=dev)
part = c.partial(b)
sms = torch.cuda.get_device_properties(dev).multi_processor_count
wps = query("svdrec_spmm_warps_per_sm", b)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def tma(lo, hi, nw, stream):
    sb, se = c.seg_begin[lo:hi], c.seg_end[lo:hi]
    ws = warp_plan_t(sb, se, nw)
    def run():
        with torch.cuda.stream(stream):
            call("svdrec_spmm", hi - lo, ptr(c.seg_row[lo:hi]), ptr(sb), ptr(se), ptr(c.seg_slot[lo:hi]),
                 ptr(c.indices), ptr(c.values), ptr(X), b, c.n, ptr(Y), b, b, 0, None, None, None, nw, ptr(ws),
                 ptr(part), K.stream_handle(stream))
    return run


def plain(lo, hi, stream):
    def run():
        with torch.cuda.stream(stream):
            call("svdrec_spmm", hi - lo, ptr(c.seg_row[lo:hi]), ptr(c.seg_begin[lo:hi]), ptr(c.seg_end[lo:hi]),
                 ptr(c.seg_slot[lo:hi]), ptr(c.indices), ptr(c.values), ptr(X), b, c.n, ptr(Y), b, b, 0, None, None,
                 None, 0, None, ptr(part), K.stream_handle(stream))
    return run


def timeit(fns, reps=20):
    torch.cuda.synchronize()
    for f in fns:
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cur = torch.cuda.current_stream()
    for _ in range(reps):
        for s in (s1, s2):
            s.wait_stream(cur)
        for f in fns:
            f()
        for s in (s1, s2):
            cur.wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


nseg = c.nseg
print(f"tma alone {timeit([tma(0, nseg, sms * wps, s1)]):.1f} us; plain alone {timeit([plain(0, nseg, s2)]):.1f} us",
      flush=True)
for f in (0.9, 0.8, 0.7, 0.6):
    mid = int(torch.searchsorted(torch.cumsum(c.seg_end - c.seg_begin, 0).double(),
                                 torch.tensor([f * c.nnz], dtype=torch.float64, device=dev)).item())
    t = timeit([tma(0, mid, sms * wps, s1), plain(mid, nseg, s2)])
    print(f"split {f:.1f}: tma + plain concurrently {t:.1f} us", flush=True)
