"""Which entry order does the hot-set SpMM need?  A @ X on config 3 through
k_spmm_hot with three encodings of the same CSR: (a) rows in full
popularity-rank order (the default), (b) rows stably partitioned into the
hot items first and the cold ones after, each in item order, (c) rows in
item order (hot / cold interleaved, split per batch by the ballot).
python tools/probe_hot_order.py [b ...]   (GPU box)"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2009_02251_b200 as P  # noqa: E402
from paper_2009_02251_b200 import kernels as K  # noqa: E402
from paper_2009_02251_b200._lib import call, ptr, query, stream_handle  # noqa: E402

cfg, M, tr, va, te, _ = bench._workload()
A = P.SparseRatings(tr, *cfg.bounds)
d = A.device()
c = d.A
dev = torch.device("cuda")
rank = c.item_rank.to(torch.int64)
rows = torch.repeat_interleave(torch.arange(c.m, device=dev), c.indptr[1:] - c.indptr[:-1])


def enc(order_key, nhot):
    perm = torch.sort(order_key, stable=True).indices
    idx = c.indices[perm].to(torch.int64)
    rk = rank[idx]
    hidx = torch.where(rk < nhot, -(rk + 1), idx).to(torch.int32)
    return hidx, c.values[perm].contiguous()


for b in [int(x) for x in (sys.argv[1:] or ["16", "64"])]:
    nhot = min(int(query("svdrec_spmm_hot_rows", b)), c.n)
    X = torch.randn(c.n, b, dtype=torch.float64, device=dev)
    Y = torch.empty(c.m, b, dtype=torch.float64, device=dev)
    rk_all = rank[c.indices.to(torch.int64)]
    variants = {
        "ranked": enc(rows * c.n + rk_all, nhot),
        "hot-first": enc(rows * 2 + (rk_all >= nhot).to(torch.int64), nhot),
        "item order": enc(torch.arange(c.nnz, device=dev), nhot),
    }
    nw, ws = c.schedule(16)
    for name, (hidx, hval) in variants.items():
        def run():
            call("svdrec_spmm_hot", c.nseg, ptr(c.seg_row), ptr(c.seg_begin), ptr(c.seg_end), ptr(c.seg_slot),
                 ptr(hidx), ptr(hval), ptr(X), b, c.n, ptr(c.hot_items), nhot, ptr(Y), b, b, c.nlong,
                 ptr(c.long_row), ptr(c.long_s0), ptr(c.long_s1), nw, ptr(ws), ptr(c.partial(b)), stream_handle())
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            run()
        e1.record()
        torch.cuda.synchronize()
        print(f"b={b:3d} {name:10s} {e0.elapsed_time(e1) / 20 * 1e3:7.1f} us", flush=True)
