"""Planning logic: the plan builders that run next to the data on the
device must reproduce the numpy definitions exactly (torch-op builders on
CPU tensors; the kernel-built ones, marked gpu, on the device)."""
import numpy as np
import pytest
import torch

from paper_2009_02251_b200 import sparse as S


def _np_workplan(group_deg, chunk):
    """The scoring work plan, restated in numpy (the kernel's contract)."""
    ng = group_deg.size
    nch = np.maximum(1, -(-group_deg // chunk)).astype(np.int64)
    split = nch > 1
    slot0 = np.full(ng, -1, dtype=np.int64)
    slot0[split] = np.cumsum(nch[split]) - nch[split]
    done = np.full(ng, -1, dtype=np.int64)
    done[split] = np.arange(int(split.sum()))
    order = np.argsort(-group_deg, kind="stable")
    wg = np.repeat(order, nch[order])
    first = np.repeat(np.cumsum(nch[order]) - nch[order], nch[order])
    wc = np.arange(wg.size) - first
    return np.stack([wg, wc], 1).ravel(), np.stack([nch, slot0, done], 1).ravel(), int(split.sum()), \
        int(nch[split].sum())


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_segment_and_warp_plans_match_numpy(seed):
    rng = np.random.default_rng(seed)
    deg = rng.zipf(1.3, size=3000).clip(0, 9000)
    deg[rng.random(3000) < 0.1] = 0  # empty rows
    indptr = np.r_[0, np.cumsum(deg)].astype(np.int64)
    ref = S.segment_plan(indptr, seg_max=256)
    got = S.segment_plan_t(torch.from_numpy(indptr), seg_max=256)
    for a, b in zip(ref[:7], got[:7]):
        np.testing.assert_array_equal(np.asarray(a, dtype=np.int64), b.numpy().astype(np.int64))
    assert ref[7] == got[7]
    sb, se = ref[1], ref[2]
    for nw in (1, 7, 64, 5000):
        np.testing.assert_array_equal(S.warp_plan(sb, se, nw), S.warp_plan_t(got[1], got[2], nw).numpy())


@pytest.mark.gpu
def test_device_transpose_matches_scipy(gpu):
    """DeviceCSR.transposed runs the counting-sort kernel (csrc/ingest.cu)."""
    import scipy.sparse as sp
    rng = np.random.default_rng(5)
    M = sp.random(300, 170, density=0.05, random_state=rng, format="csr")
    M.data = np.round(M.data * 9) / 2 + 0.5
    d = S.DeviceCSR(torch.from_numpy(M.indptr.astype(np.int64)).to(gpu),
                    torch.from_numpy(M.indices.astype(np.int32)).to(gpu), torch.from_numpy(M.data).to(gpu), M.shape)
    t = d.transposed()
    ref = M.T.tocsr()
    ref.sort_indices()
    np.testing.assert_array_equal(t.indptr.cpu().numpy(), ref.indptr)
    np.testing.assert_array_equal(t.indices.cpu().numpy(), ref.indices)
    np.testing.assert_array_equal(t.values.cpu().numpy(), ref.data)


@pytest.mark.gpu
@pytest.mark.parametrize("chunk", [1, 3, 512])
def test_workplan_matches_numpy(gpu, chunk, monkeypatch):
    """WorkPlan runs the plan kernels (csrc/cf.cu k_plan_scan / k_plan_emit)."""
    from paper_2009_02251_b200.cf import WorkPlan
    rng = np.random.default_rng(chunk)
    gd = rng.zipf(1.5, size=400).astype(np.int64) - 1
    gs = np.r_[0, np.cumsum(rng.integers(1, 4, size=400))]  # samples per group
    rs = np.r_[0, np.cumsum(gd)][:-1] + 7  # CSR offset of each group's row
    monkeypatch.setattr(WorkPlan, "CHUNK", chunk)
    p = WorkPlan(torch.from_numpy(gd).to(gpu), gpu, torch.from_numpy(gs).to(gpu), torch.from_numpy(rs).to(gpu))
    work, ginfo, ndone, nslots = _np_workplan(gd, chunk)
    wg, wc = work[0::2], work[1::2]
    nch, slot0, done = ginfo[0::3], ginfo[1::3], ginfo[2::3]
    split = nch[wg] > 1
    start = rs[wg] + np.where(split, wc * chunk, 0)
    length = np.where(split, np.minimum(gd[wg] - wc * chunk, chunk), gd[wg])
    meta = np.stack([length, gd[wg], gs[wg], gs[wg + 1], nch[wg], np.where(split, slot0[wg] + wc, -1), done[wg],
                     wc], 1)
    np.testing.assert_array_equal(p.start[: p.nwork].cpu().numpy(), start)
    np.testing.assert_array_equal(p.meta[: 8 * p.nwork].cpu().numpy(), meta.ravel().astype(np.int32))
    assert (p.ndone, p.nslots, p.nwork) == (ndone, nslots, wg.size)
    # every rating of every user is covered exactly once by the items
    cover = np.zeros(int(rs[-1] + gd[-1] + 8), dtype=np.int64)
    for a, n in zip(start, length):
        cover[a:a + n] += 1
    for g in range(gd.size):
        assert np.all(cover[rs[g]:rs[g] + gd[g]] == 1)


def test_samples_grouping_on_host_device():
    from paper_2009_02251_b200.cf import _Samples
    rng = np.random.default_rng(3)
    u = rng.integers(0, 50, 1000)
    i = rng.integers(0, 80, 1000)
    r = rng.random(1000)
    s = _Samples((u, i, r), torch.device("cpu"))
    order = np.argsort(u, kind="stable")
    np.testing.assert_array_equal(s.order, order)
    us = u[order]
    starts = np.flatnonzero(np.r_[True, us[1:] != us[:-1]])
    np.testing.assert_array_equal(s.groups.numpy(), np.r_[starts, us.size])
    np.testing.assert_array_equal(s.items.numpy(), i[order])
    np.testing.assert_array_equal(s.truth.numpy(), r[order])
    np.testing.assert_array_equal(s.group_users_dev.numpy(), us[starts])
