"""Device ingest: the stable counting-sort transpose (csrc/ingest.cu)
against scipy's transpose and against a sort-based restatement of the
ranked CSR, bit for bit (integer / index work)."""
from __future__ import annotations

import numpy as np
import pytest
from scipy import sparse as sp

pytestmark = pytest.mark.gpu


def _rand_csr(m, n, density, seed, empty_rows=(), empty_cols=()):
    rng = np.random.default_rng(seed)
    M = sp.random(m, n, density=density, format="csr", random_state=rng, dtype=np.float64)
    M.data[:] = rng.integers(1, 11, M.nnz) * 0.5
    M = M.tolil()
    for r in empty_rows:
        M[r, :] = 0
    for c in empty_cols:
        M[:, c] = 0
    M = M.tocsr()
    M.eliminate_zeros()
    M.sort_indices()
    return M


def _dev(M, dev):
    import torch
    return (torch.as_tensor(M.indptr.astype(np.int64), device=dev), torch.as_tensor(M.indices.astype(np.int32), device=dev),
            torch.as_tensor(M.data, device=dev))


@pytest.mark.parametrize("m,n,density,seed", [(300, 200, 0.05, 0), (2000, 57000, 0.002, 1), (1, 5, 1.0, 2),
                                              (5000, 300, 0.2, 3)])
def test_transpose_matches_scipy(gpu, m, n, density, seed):
    from paper_2009_02251_b200 import kernels as K
    M = _rand_csr(m, n, density, seed, empty_rows=(0,) if m > 1 else (), empty_cols=(1,))
    ip, ix, dv = _dev(M, gpu)
    tp, ti, tv = K.csr_transpose(ip, ix, dv, n)
    T = M.T.tocsr()
    T.sort_indices()
    assert np.array_equal(tp.cpu().numpy(), T.indptr)
    assert np.array_equal(ti.cpu().numpy(), T.indices)
    assert np.array_equal(tv.cpu().numpy(), T.data)


@pytest.mark.parametrize("m,n,seed", [(800, 300, 4), (60000, 900, 5)])
def test_ranked_csr_matches_sort(gpu, m, n, seed):
    """Transpose of A.T taken in popularity order == each row of A relabelled
    by rank and sorted by rank (the previous sort-based construction)."""
    import torch
    from paper_2009_02251_b200 import kernels as K
    M = _rand_csr(m, n, 0.02, seed)
    T = M.T.tocsr()
    deg = np.diff(T.indptr)
    order = np.argsort(-deg, kind="stable")
    rank = np.empty(n, dtype=np.int64)
    rank[order] = np.arange(n)
    ip, ix, dv = _dev(T, gpu)
    _, rk, rv = K.csr_transpose(ip, ix, dv, m, perm=torch.as_tensor(order, device=gpu), relabel=True)
    rows = np.repeat(np.arange(m), np.diff(M.indptr))
    key = rows * n + rank[M.indices]
    perm = np.argsort(key, kind="stable")
    assert np.array_equal(rk.cpu().numpy(), rank[M.indices][perm])
    assert np.array_equal(rv.cpu().numpy(), M.data[perm])


def test_empty_transpose(gpu):
    from paper_2009_02251_b200 import kernels as K
    M = sp.csr_matrix((4, 6))
    ip, ix, dv = _dev(M, gpu)
    tp, ti, tv = K.csr_transpose(ip, ix, dv, 6)
    assert tp.cpu().numpy().tolist() == [0] * 7 and ti.numel() == 0


def _plan_torch(gd, group_start, row_start, chunk):
    """The work plan as plain torch ops (the restatement the kernels replaced)."""
    import torch
    nch = torch.clamp((gd + chunk - 1) // chunk, min=1)
    split = nch > 1
    cs = torch.cumsum(torch.where(split, nch, torch.zeros_like(nch)), 0)
    slot0 = torch.where(split, cs - nch, torch.full_like(nch, -1))
    done = torch.where(split, torch.cumsum(split.to(torch.int64), 0) - 1, torch.full_like(nch, -1))
    order = torch.sort(-gd, stable=True).indices
    no = nch[order]
    wg = torch.repeat_interleave(order, no)
    first = torch.repeat_interleave(torch.cumsum(no, 0) - no, no)
    wc = torch.arange(wg.numel(), device=gd.device) - first
    sp_w = split[wg]
    deg_w = gd[wg]
    off = torch.where(sp_w, wc * chunk, torch.zeros_like(wc))
    start = row_start[wg] + off
    length = torch.where(sp_w, torch.clamp(deg_w - off, max=chunk), deg_w)
    meta = torch.stack([length, deg_w, group_start[wg], group_start[wg + 1], nch[wg],
                        torch.where(sp_w, slot0[wg] + wc, torch.full_like(wc, -1)), done[wg], wc], 1)
    stats = (int(wg.numel()), int(split.sum()), int(torch.where(split, nch, torch.zeros_like(nch)).sum()),
             int(gd.sum()))
    return start, meta.to(torch.int32).flatten(), stats


@pytest.mark.parametrize("ng,seed", [(1, 0), (37, 1), (5000, 2), (130000, 3)])
def test_work_plan_kernels_match_torch(gpu, ng, seed):
    import torch
    from paper_2009_02251_b200.cf import WorkPlan
    rng = np.random.default_rng(seed)
    deg = np.minimum(rng.lognormal(4, 1.5, ng).astype(np.int64), 40000)
    deg[: min(ng, 4)] = [0, 512, 513, 1024][: min(ng, 4)]
    gd = torch.as_tensor(deg, device=gpu)
    gs = torch.as_tensor(np.concatenate([[0], np.cumsum(rng.integers(1, 9, ng))]), device=gpu)
    rs = torch.cumsum(gd, 0) - gd + 7
    p = WorkPlan(gd, gpu, gs, rs)
    start, meta, stats = _plan_torch(gd, gs, rs, WorkPlan.CHUNK)
    assert (p.nwork, p.ndone, p.nslots, p.rated) == stats
    assert torch.equal(p.start[: p.nwork], start)
    assert torch.equal(p.meta[: 8 * p.nwork], meta)


@pytest.mark.parametrize("m,n,seed", [(700, 300, 6), (3000, 40000, 7)])
def test_rank_rows_matches_transpose(gpu, m, n, seed):
    """The per-row bitset ranking (n <= 65536) and the transpose-of-A.T
    construction give the same ranked CSR."""
    import torch
    from paper_2009_02251_b200 import kernels as K
    M = _rand_csr(m, n, 0.03 if n < 1000 else 0.002, seed, empty_rows=(2,))
    T = M.T.tocsr()
    order = np.argsort(-np.diff(T.indptr), kind="stable")
    rank = np.empty(n, dtype=np.int32)
    rank[order] = np.arange(n)
    ip, ix, dv = _dev(M, gpu)
    rk, rv = K.rank_rows(ip, ix, dv, n, torch.as_tensor(rank, device=gpu))
    tp, ti, tv = _dev(T, gpu)
    _, rk2, rv2 = K.csr_transpose(tp, ti, tv, m, perm=torch.as_tensor(order, device=gpu), relabel=True)
    assert torch.equal(rk, rk2) and torch.equal(rv, rv2)


@pytest.mark.parametrize("n", [0, 1, 5000, 8192, 8193, 300001])
def test_scan_i64(gpu, n):
    import torch
    from paper_2009_02251_b200 import kernels as K
    x = torch.randint(0, 1000, (n,), dtype=torch.int64, device=gpu)
    tot = torch.empty(1, dtype=torch.int64, device=gpu)
    y = K.scan_i64(x, total=tot)
    ref = torch.cumsum(x, 0) - x
    assert torch.equal(y, ref) and int(tot) == int(x.sum())


@pytest.mark.parametrize("nhot", [0, 7, 50, 1000])
def test_hot_partition_matches_numpy(gpu, nhot):
    """The hot-set SpMM's copy of a CSR: each row stably partitioned into
    the entries of the nhot most rated items (index -(rank + 1)) and the
    rest (item id), values moved along."""
    import paper_2009_02251_b200 as P
    M = _rand_csr(400, 300, 0.05, 11 + nhot, empty_rows=(0, 5))
    A = P.SparseRatings(M, 0.5, 5.0)
    c = A.device(gpu).A
    idx, val = c.hot_encoded(nhot)
    rank = c.item_rank.cpu().numpy()
    want_i, want_v = [], []
    for r in range(M.shape[0]):
        cols = M.indices[M.indptr[r]:M.indptr[r + 1]]
        vals = M.data[M.indptr[r]:M.indptr[r + 1]]
        hot = rank[cols] < nhot
        want_i += list(-(rank[cols[hot]] + 1)) + list(cols[~hot])
        want_v += list(vals[hot]) + list(vals[~hot])
    assert np.array_equal(idx.cpu().numpy(), np.array(want_i, dtype=np.int32))
    assert np.array_equal(val.cpu().numpy(), np.array(want_v))


@pytest.mark.parametrize("nhot", [None, 0, 40])
def test_chunk_plan_matches_numpy(gpu, nhot):
    """The pipelined SpMMs' chunk records (svdrec_chunk_plan): every segment
    in chunks of <= 32 entries with first / last flags, an empty row as one
    empty chunk, split rows pointing at their partial slots; with the packed
    hot-first copy (svdrec_spmm_hot_pack) no chunk straddles a row's hot /
    cold boundary and hot chunks are flagged; per-warp record ranges."""
    import paper_2009_02251_b200 as P
    from paper_2009_02251_b200 import sparse as S
    rng = np.random.default_rng(3)
    m, n = 700, 3000
    deg = np.minimum(rng.lognormal(3.0, 1.5, m).astype(np.int64), n)
    deg[:4] = 0
    deg[4] = n  # split into segments
    rows = np.repeat(np.arange(m), deg)
    cols = np.concatenate([np.sort(rng.choice(n, d, replace=False)) for d in deg if d])
    M = sp.csr_matrix((rng.integers(1, 11, cols.size) * 0.5, (rows, cols)), shape=(m, n))
    c = P.SparseRatings(M, 0.5, 5.0).device(gpu).A
    indptr = c.indptr.cpu().numpy()
    if nhot is None:
        nw, wc, recs = c.chunk_schedule(16)
        cnt = np.zeros(m, dtype=np.int64)
    else:
        nw, wc, recs, ents, cnt = c.hot_packed(nhot, 16)
        cnt = cnt.cpu().numpy().astype(np.int64)[:m]
        rank = c.item_rank.cpu().numpy()
        want_c = np.array([int((rank[M.indices[indptr[r]:indptr[r + 1]]] < nhot).sum()) for r in range(m)])
        assert np.array_equal(cnt, want_c)
        e = ents.cpu().numpy().view(np.int32).reshape(-1, 4)
        ids, vals = e[:, 0], ents.cpu().numpy()[:, 1]
        want_i, want_v = [], []
        for r in range(m):
            cols_r, vals_r = M.indices[indptr[r]:indptr[r + 1]], M.data[indptr[r]:indptr[r + 1]]
            hot = rank[cols_r] < nhot
            want_i += list(rank[cols_r[hot]]) + list(cols_r[~hot])
            want_v += list(vals_r[hot]) + list(vals_r[~hot])
        assert np.array_equal(ids, np.array(want_i, dtype=np.int32)) and np.array_equal(vals, np.array(want_v))
    sr, sb, se, sl = (t.cpu().numpy() for t in (c.seg_row, c.seg_begin, c.seg_end, c.seg_slot))
    assert (sl >= 0).any()
    want, first = [], []
    for j in range(sr.size):
        a, e = int(sb[j]), int(se[j])
        h = min(max(int(indptr[sr[j]] + cnt[sr[j]]), a), e) if nhot is not None else a
        dst = int(sr[j]) if sl[j] < 0 else ~int(sl[j])
        parts = [(o, min(32, h - o), 1024) for o in range(a, h, 32)] + [(o, min(32, e - o), 0) for o in range(h, e, 32)]
        first.append(len(want))
        if not parts:
            want.append((0, dst, 256 | 512, 0))
        for t, (o, nv, hot) in enumerate(parts):
            want.append((o, dst, nv | (256 if t == 0 else 0) | (512 if t == len(parts) - 1 else 0) | hot, 0))
    first.append(len(want))
    assert np.array_equal(recs.cpu().numpy()[: len(want)], np.array(want, dtype=np.int32))
    wseg = c.schedule(16, S.CHUNK_COST)[1].cpu().numpy()
    assert nw == wseg.size - 1 and np.array_equal(wc.cpu().numpy(), np.array(first, dtype=np.int32)[wseg])


@pytest.mark.parametrize("seed", [0, 1])
def test_segment_and_warp_plan_kernels_match_numpy(gpu, seed):
    """The SpMM plan built by the kernels equals sparse.segment_plan /
    warp_plan (the numpy definitions) -- empty rows, rows split into
    several segments."""
    import torch
    from paper_2009_02251_b200 import sparse as S
    rng = np.random.default_rng(seed)
    deg = rng.zipf(1.3, size=5000).clip(0, 9000)
    deg[rng.random(5000) < 0.1] = 0
    indptr = np.r_[0, np.cumsum(deg)].astype(np.int64)
    ref = S.segment_plan(indptr, seg_max=256)
    got = S.segment_plan_dev(torch.as_tensor(indptr, device=gpu), seg_max=256)
    for a, b in zip(ref[:7], got[:7]):
        np.testing.assert_array_equal(np.asarray(a, dtype=np.int64), b.cpu().numpy().astype(np.int64))
    assert ref[7] == got[7]
    for nw in (1, 7, 64, 5000, 100000):
        for cost in (16, S.CHUNK_COST):
            np.testing.assert_array_equal(S.warp_plan(ref[1], ref[2], nw, cost),
                                          S.warp_plan_dev(got[1], got[2], nw, cost).cpu().numpy())
