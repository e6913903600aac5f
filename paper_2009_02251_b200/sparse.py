"""Rating matrix container: the reference's SparseRatings plus its HBM image.

``SparseRatings`` keeps the reference contract (pkg/src/svdrec/sparse.py:
canonical CSR, rating bounds, from_coo / from_dense / transposed ...).  Its
``device()`` method uploads the matrix once and caches a
:class:`DeviceRatings` -- the CSR of A and the CSR of A.T (so A.T @ X is a
gather-only row product, no atomics) plus the SpMM segment plans -- which
every GPU routine of this package works on.

HBM layout per CSR: int64 indptr (m+1), int32 indices (nnz), float64
values (nnz) -> 12 B per nonzero; the plan adds 24 B per row segment.
"""
from __future__ import annotations

import numpy as np
import torch
from scipy import sparse as sp

SEG_MAX = 2048  # nonzeros per SpMM row segment; longer rows are split


class SparseRatings:
    """Immutable CSR of observed ratings with the legal rating range.

    Same contract as the reference (sparse.py:11-59): canonical CSR
    (strictly increasing columns per row), float64 values inside
    [rating_min, rating_max], finite.
    """

    __slots__ = ("matrix", "rating_min", "rating_max", "_dev")

    def __init__(self, matrix: sp.csr_matrix, rating_min: float, rating_max: float) -> None:
        if not sp.issparse(matrix) or matrix.format != "csr":
            raise TypeError("matrix must be a scipy CSR matrix")
        mat = matrix.astype(np.float64, copy=False)
        object.__setattr__(self, "matrix", mat)
        object.__setattr__(self, "rating_min", float(rating_min))
        object.__setattr__(self, "rating_max", float(rating_max))
        object.__setattr__(self, "_dev", {})
        if self.rating_min > self.rating_max:
            raise ValueError("rating_min exceeds rating_max")
        if torch.cuda.is_available() and mat.nnz:
            # O(nnz) checks where the matrix is going anyway: upload once,
            # check on the device, keep the image (see DeviceRatings.check)
            d = self.device()
            unsorted, finite, lo, hi = d.check()
            if unsorted:  # order the columns on the host, then re-check
                self._dev.clear()
                self._check_host()
                self.device()
                return
            self._raise_values(finite, lo, hi)
        else:
            self._check_host()

    def _check_host(self) -> None:
        mat = self.matrix
        mat.sort_indices()
        ind, ptr = mat.indices, mat.indptr
        if ind.size > 1:
            d = np.diff(ind)
            inner = np.ones(ind.size - 1, dtype=bool)
            starts = ptr[1:-1]
            starts = starts[(starts > 0) & (starts < ind.size)]
            inner[starts - 1] = False
            if np.any(d[inner] <= 0):
                raise ValueError("duplicate or unsorted column indices in a row")
        if mat.data.size:
            self._raise_values(bool(np.all(np.isfinite(mat.data))), mat.data.min(), mat.data.max())

    def _raise_values(self, finite: bool, lo, hi) -> None:
        if not finite:
            raise ValueError("ratings must be finite")
        if lo < self.rating_min or hi > self.rating_max:
            raise ValueError(f"ratings outside [{self.rating_min}, {self.rating_max}]: observed [{lo}, {hi}]")

    def __setattr__(self, k, v):
        raise AttributeError("SparseRatings is immutable")

    shape = property(lambda self: self.matrix.shape)
    m = property(lambda self: self.matrix.shape[0])
    n = property(lambda self: self.matrix.shape[1])
    nnz = property(lambda self: self.matrix.nnz)
    data = property(lambda self: self.matrix.data)
    indices = property(lambda self: self.matrix.indices)
    indptr = property(lambda self: self.matrix.indptr)

    def row_slice(self, i: int):
        if not 0 <= i < self.m:
            raise IndexError(f"row {i} out of range for {self.m} rows")
        a, b = self.matrix.indptr[i], self.matrix.indptr[i + 1]
        return self.matrix.indices[a:b], self.matrix.data[a:b]

    def to_dense(self) -> np.ndarray:
        return self.matrix.toarray()

    def transposed(self) -> "SparseRatings":
        return SparseRatings(self.matrix.transpose().tocsr(), self.rating_min, self.rating_max)

    @classmethod
    def from_coo(cls, rows, cols, values, shape, bounds=None) -> "SparseRatings":
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        values = np.asarray(values, dtype=np.float64)
        if not rows.size == cols.size == values.size:
            raise ValueError("rows, cols, values must have equal length")
        csr = sp.coo_matrix((values, (rows, cols)), shape=shape).tocsr()
        if csr.nnz != values.size:
            raise ValueError("duplicate coordinates are not allowed")
        if bounds is None:
            bounds = (0.0, 0.0) if values.size == 0 else (float(values.min()), float(values.max()))
        return cls(csr, float(bounds[0]), float(bounds[1]))

    @classmethod
    def from_dense(cls, arr, bounds=None) -> "SparseRatings":
        arr = np.asarray(arr, dtype=np.float64)
        if arr.ndim != 2:
            raise ValueError("expected a 2-d array")
        csr = sp.csr_matrix(arr)
        if bounds is None:
            bounds = (0.0, 0.0) if csr.nnz == 0 else (float(csr.data.min()), float(csr.data.max()))
        return cls(csr, float(bounds[0]), float(bounds[1]))

    def device(self, device=None) -> "DeviceRatings":
        """Upload (once) and return the HBM image on ``device``."""
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        key = dev.index if dev.index is not None else torch.cuda.current_device()
        d = self._dev.get(key)
        if d is None:
            d = self._dev[key] = DeviceRatings(self, torch.device("cuda", key))
        return d


def segment_plan(indptr: np.ndarray, seg_max: int = SEG_MAX):
    """Row segments of <= seg_max nonzeros; split rows get partial slots."""
    m = indptr.size - 1
    deg = np.diff(indptr).astype(np.int64)
    nps = np.maximum(1, -(-deg // seg_max))
    seg_row = np.repeat(np.arange(m, dtype=np.int64), nps)
    first = np.repeat(np.cumsum(nps) - nps, nps)
    within = np.arange(seg_row.size, dtype=np.int64) - first
    seg_begin = indptr[seg_row].astype(np.int64) + within * seg_max
    seg_end = np.minimum(seg_begin + seg_max, indptr[seg_row + 1].astype(np.int64))
    split = nps > 1
    slot = np.full(seg_row.size, -1, dtype=np.int64)
    is_split_seg = split[seg_row]
    slot[is_split_seg] = np.arange(int(is_split_seg.sum()))
    long_row = np.nonzero(split)[0]
    s0 = first[np.searchsorted(seg_row, long_row)] if long_row.size else np.empty(0, np.int64)
    s0 = slot[s0] if long_row.size else s0
    s1 = s0 + nps[long_row]
    return seg_row, seg_begin, seg_end, slot, long_row, s0, s1, int(is_split_seg.sum())


WARPS_PER_SM = 16  # pipelined SpMM: resident warps per SM (2 CTAs x 8 warps)
# segment cost of the chunk kernels' schedules (svdrec_warp_plan, seg_cost < 0):
# whole 32-entry chunks plus 5 entries' worth for the segment's fold and store
CHUNK_COST = -5


def _seg_cost(d, seg_cost: int):
    """Cost of segments of ``d`` entries: d + seg_cost, or for seg_cost < 0 the
    chunk kernels' cost (whole 32-entry chunks, at least one) - seg_cost."""
    if seg_cost >= 0:
        return d + seg_cost
    chunks = (d + 31) // 32
    chunks = np.maximum(chunks, 1) if isinstance(d, np.ndarray) else torch.clamp(chunks, min=1)
    return chunks * 32 - seg_cost


def warp_plan(seg_begin: np.ndarray, seg_end: np.ndarray, nwarp: int, seg_cost: int = 16) -> np.ndarray:
    """Split the row-ordered segments into ``nwarp`` contiguous ranges of
    about equal cost (nonzeros + ``seg_cost`` per segment); returns the
    ``nwarp + 1`` range starts (int32) the pipelined SpMM kernel reads."""
    nseg = seg_begin.size
    cost = np.cumsum(_seg_cost(seg_end - seg_begin, seg_cost), dtype=np.int64)
    total = int(cost[-1]) if nseg else 0
    targets = (np.arange(1, nwarp, dtype=np.float64) * (total / max(nwarp, 1)))
    cuts = np.searchsorted(cost, targets, side="left") + 1 if nseg else np.zeros(nwarp - 1, np.int64)
    out = np.empty(nwarp + 1, dtype=np.int64)
    out[0], out[-1] = 0, nseg
    out[1:-1] = np.minimum(cuts, nseg)
    return np.maximum.accumulate(out).astype(np.int32)


def segment_plan_t(indptr: torch.Tensor, seg_max: int = SEG_MAX):
    """segment_plan on torch tensors (any device; same arrays as the numpy
    version): built where the CSR lives, so the upload path never walks the
    rows on the host."""
    dev = indptr.device
    m = indptr.numel() - 1
    deg = indptr[1:] - indptr[:-1]
    nps = torch.clamp((deg + seg_max - 1) // seg_max, min=1)
    seg_row = torch.repeat_interleave(torch.arange(m, device=dev), nps)
    cum = torch.cumsum(nps, 0)
    first_of_row = cum - nps
    within = torch.arange(seg_row.numel(), device=dev) - first_of_row[seg_row]
    seg_begin = indptr[seg_row] + within * seg_max
    seg_end = torch.minimum(seg_begin + seg_max, indptr[seg_row + 1])
    split = nps > 1
    is_split_seg = split[seg_row]
    slot = torch.where(is_split_seg, torch.cumsum(is_split_seg.to(torch.int64), 0) - 1,
                       torch.full_like(seg_row, -1))
    long_row = torch.nonzero(split).flatten()
    s0 = slot[first_of_row[long_row]]
    s1 = s0 + nps[long_row]
    nslots = int(is_split_seg.sum().item()) if seg_row.numel() else 0
    return seg_row, seg_begin, seg_end, slot, long_row, s0, s1, nslots


def segment_plan_dev(indptr: torch.Tensor, seg_max: int = SEG_MAX):
    """segment_plan by the plan kernels (csrc/ingest.cu) on a CUDA tensor:
    the same arrays, one small read for the sizes."""
    from . import kernels as K

    dev = indptr.device
    m = indptr.numel() - 1
    first = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
    sbase = torch.empty_like(first)
    lidx = torch.empty_like(first)
    tot = torch.empty(3, dtype=torch.int64, device=dev)
    K.call("svdrec_seg_plan_count", m, K.ptr(indptr), int(seg_max), K.ptr(first), K.ptr(sbase), K.ptr(lidx),
           K.ptr(tot), K.stream_handle())
    nseg, nslots, nlong = (int(x) for x in tot.cpu().numpy())
    seg_row = torch.empty(nseg, dtype=torch.int32, device=dev)
    seg_begin = torch.empty(nseg, dtype=torch.int64, device=dev)
    seg_end = torch.empty(nseg, dtype=torch.int64, device=dev)
    seg_slot = torch.empty(nseg, dtype=torch.int32, device=dev)
    long_row = torch.empty(nlong, dtype=torch.int32, device=dev)
    s0 = torch.empty(nlong, dtype=torch.int32, device=dev)
    s1 = torch.empty(nlong, dtype=torch.int32, device=dev)
    K.call("svdrec_seg_plan_emit", m, K.ptr(indptr), int(seg_max), K.ptr(first), K.ptr(sbase), K.ptr(lidx),
           K.ptr(seg_row), K.ptr(seg_begin), K.ptr(seg_end), K.ptr(seg_slot), K.ptr(long_row), K.ptr(s0), K.ptr(s1),
           K.stream_handle())
    return seg_row, seg_begin, seg_end, seg_slot, long_row, s0, s1, nslots


def warp_plan_dev(seg_begin: torch.Tensor, seg_end: torch.Tensor, nwarp: int, seg_cost: int = 16) -> torch.Tensor:
    """warp_plan by a kernel (csrc/ingest.cu) on CUDA tensors (same result)."""
    from . import kernels as K

    nseg = seg_begin.numel()
    scratch = torch.empty(nseg + 1, dtype=torch.int64, device=seg_begin.device)
    out = torch.empty(nwarp + 1, dtype=torch.int32, device=seg_begin.device)
    K.call("svdrec_warp_plan", nseg, K.ptr(seg_begin), K.ptr(seg_end), int(nwarp), int(seg_cost), K.ptr(scratch),
           K.ptr(out), K.stream_handle())
    return out


def warp_plan_t(seg_begin: torch.Tensor, seg_end: torch.Tensor, nwarp: int, seg_cost: int = 16) -> torch.Tensor:
    """warp_plan on torch tensors (same result as the numpy version)."""
    dev = seg_begin.device
    nseg = seg_begin.numel()
    out = torch.zeros(nwarp + 1, dtype=torch.int64, device=dev)
    out[-1] = nseg
    if nseg and nwarp > 1:
        cost = torch.cumsum(_seg_cost(seg_end - seg_begin, seg_cost), 0)
        total = cost[-1].to(torch.float64)
        targets = torch.arange(1, nwarp, dtype=torch.float64, device=dev) * (total / nwarp)
        cuts = torch.searchsorted(cost.to(torch.float64), targets, side="left") + 1
        out[1:-1] = torch.clamp(cuts, max=nseg)
    return torch.cummax(out, 0).values.to(torch.int32)


_COPY: dict = {}


def _copy_stream(dev: torch.device) -> torch.cuda.Stream:
    """One cached host-to-device copy stream per device."""
    s = _COPY.get(dev.index)
    if s is None:
        s = _COPY[dev.index] = torch.cuda.Stream(device=dev)
    return s


class DeviceCSR:
    """One CSR in HBM plus its SpMM plan (built on the device)."""

    def __init__(self, indptr: torch.Tensor, indices: torch.Tensor, values: torch.Tensor, shape, h2d_bytes: int = 0):
        self.m, self.n = int(shape[0]), int(shape[1])
        self.device = indptr.device
        self.indptr = indptr.to(torch.int64)
        self.indices = indices.to(torch.int32)
        self.values = values.to(torch.float64)
        self.nnz = int(self.indices.numel())
        cuda = self.device.type == "cuda"
        sr, sb, se, sl, lr, s0, s1, nslots = (segment_plan_dev if cuda else segment_plan_t)(self.indptr)
        self.nseg = int(sr.numel())
        self.seg_row = sr.to(torch.int32)
        self.seg_begin = sb
        self.seg_end = se
        self.seg_slot = sl.to(torch.int32)
        self.nlong = int(lr.numel())
        self.long_row = lr.to(torch.int32)
        self.long_s0 = s0.to(torch.int32)
        self.long_s1 = s1.to(torch.int32)
        self.nslots = nslots
        # in-kernel fix-up of the split rows (pipelined SpMM): slot -> split-row
        # index and one ticket per split row (the kernel leaves them at zero)
        if self.nlong:
            self.slot_long = torch.repeat_interleave(
                torch.arange(self.nlong, dtype=torch.int32, device=self.device),
                (self.long_s1 - self.long_s0).to(torch.int64), output_size=int(nslots))
            self.long_done = torch.zeros(self.nlong, dtype=torch.int32, device=self.device)
        else:
            self.slot_long = self.long_done = None
        sms = torch.cuda.get_device_properties(self.device).multi_processor_count if self.device.type == "cuda" else 148
        self.nwarp = int(max(1, min(self.nseg, sms * WARPS_PER_SM)))
        self.warp_seg = (warp_plan_dev if cuda else warp_plan_t)(sb, se, self.nwarp)
        self._partial = {}
        self._ranked = None
        self._transpose = None
        self._hot = {}
        self._sched = {}
        self._chunks = None
        self._wchunk = {}
        self._hotpack = {}
        self.h2d_bytes = h2d_bytes

    @classmethod
    def upload(cls, csr: sp.csr_matrix, device: torch.device) -> "DeviceCSR":
        """Upload a host CSR.  The row pointers go first and the SpMM plans
        (row pointers only) are built on the current stream while the
        column indices and values are still copying on a side stream; the
        current stream then waits for the copies."""
        from .hostio import to_device

        dev = torch.device(device)
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        cur = torch.cuda.current_stream(dev)
        side = _copy_stream(dev)  # host sources: no device work to wait for
        with torch.cuda.stream(side):
            indptr = to_device(csr.indptr, np.int64, dev)
            ev_ptr = torch.cuda.Event()
            ev_ptr.record(side)
            indices = to_device(csr.indices, np.int32, dev)
            values = to_device(csr.data, np.float64, dev)
            ev_all = torch.cuda.Event()
            ev_all.record(side)
        for t in (indptr, indices, values):
            t.record_stream(cur)  # allocated on the side stream, used on this one
        cur.wait_event(ev_ptr)
        self = cls(indptr, indices, values, csr.shape, h2d_bytes=(csr.shape[0] + 1) * 8 + csr.nnz * 12)
        cur.wait_event(ev_all)
        return self

    def transposed(self) -> "DeviceCSR":
        """CSR of the transpose, built on the device: a stable counting-sort
        transpose (csrc/ingest.cu, no sort; rows stay ascending within each
        column)."""
        from . import kernels as K

        indptr, rows, vals = K.csr_transpose(self.indptr, self.indices, self.values, self.n)
        t = DeviceCSR(indptr, rows, vals, (self.n, self.m))
        self._transpose = t
        return t

    def schedule(self, warps_per_sm: int, seg_cost: int = 16) -> tuple[int, torch.Tensor]:
        """(nwarp, warp_seg) for a kernel running ``warps_per_sm`` warps per
        SM: contiguous segment ranges of about equal cost (entries +
        ``seg_cost`` per segment; CHUNK_COST: whole 32-entry chunks)."""
        if warps_per_sm == WARPS_PER_SM and seg_cost == 16:
            return self.nwarp, self.warp_seg
        hit = self._sched.get((warps_per_sm, seg_cost))
        if hit is None:
            sms = torch.cuda.get_device_properties(self.device).multi_processor_count \
                if self.device.type == "cuda" else 148
            nw = int(max(1, min(self.nseg, sms * warps_per_sm)))
            plan = warp_plan_dev if self.device.type == "cuda" else warp_plan_t
            hit = self._sched[(warps_per_sm, seg_cost)] = (nw, plan(self.seg_begin, self.seg_end, nw, seg_cost))
        return hit

    def _chunk_plan(self, indptr=None, hot_cnt=None):
        from . import kernels as K

        cbase = torch.empty(self.nseg + 1, dtype=torch.int64, device=self.device)
        recs = torch.empty((self.nnz // 32 + 2 * self.nseg, 4), dtype=torch.int32, device=self.device)
        K.call("svdrec_chunk_plan", self.nseg, K.ptr(self.seg_row), K.ptr(self.seg_begin), K.ptr(self.seg_end),
               K.ptr(self.seg_slot), K.ptr(indptr), K.ptr(hot_cnt), K.ptr(cbase), K.ptr(recs), K.stream_handle())
        return cbase, recs

    def _warp_chunks(self, cbase, warps_per_sm: int):
        from . import kernels as K

        nw, wseg = self.schedule(warps_per_sm, CHUNK_COST)
        wc = torch.empty(nw + 1, dtype=torch.int32, device=self.device)
        K.call("svdrec_warp_chunks", nw, K.ptr(wseg), self.nseg, K.ptr(cbase), K.ptr(wc), K.stream_handle())
        return nw, wc

    def chunk_schedule(self, warps_per_sm: int):
        """(nwarp, warp_chunk, records): the pipelined SpMM's chunk plan
        (csrc/ingest.cu svdrec_chunk_plan: <= 32-entry chunks of the
        segments, one 16-B record each; built once, on the device, without a
        read-back) and this schedule's per-warp record ranges."""
        if self._chunks is None:
            self._chunks = self._chunk_plan()
        cbase, recs = self._chunks
        hit = self._wchunk.get(warps_per_sm)
        if hit is None:
            hit = self._wchunk[warps_per_sm] = self._warp_chunks(cbase, warps_per_sm)
        return hit[0], hit[1], recs

    def hot_packed(self, nhot: int, warps_per_sm: int):
        """(nwarp, warp_chunk, records, entries, hot counts) of the hot /
        cold chunk SpMM (csrc/spmm.cu k_spmm_hc): the packed hot-first copy
        for ``nhot`` hot items (16-B {rank or item, value} entries, each
        row's hot entries first) and the chunk plan cut at every row's hot /
        cold boundary.  Built once per (nhot, schedule) on the device
        (cached; one at a time: 16 B per rating)."""
        key = (nhot, warps_per_sm)
        hit = self._hotpack.get(key)
        if hit is None:
            from . import kernels as K

            self._hotpack = {}  # release the previous copy first
            ents = torch.empty((self.nnz, 2), dtype=torch.float64, device=self.device)
            cnt = torch.empty(max(self.m, 1), dtype=torch.int32, device=self.device)
            K.call("svdrec_spmm_hot_pack", self.m, K.ptr(self.indptr), K.ptr(self.indices), K.ptr(self.values),
                   K.ptr(self.item_rank), int(nhot), K.ptr(ents), K.ptr(cnt), K.stream_handle())
            cbase, recs = self._chunk_plan(self.indptr, cnt)
            nw, wc = self._warp_chunks(cbase, warps_per_sm)
            hit = self._hotpack[key] = (nw, wc, recs, ents, cnt)
        return hit

    def ranked(self):
        """(ranked indices, values, rank -> item order) for the CF scoring
        kernel: item ids replaced by popularity rank, each row ordered by
        rank.  Built once on the device (cached), without a sort: per row
        with a rank bitset (csrc/ingest.cu k_rank_rows) for up to 65536
        items, else as the transpose of A.T taken in rank order."""
        if self._ranked is None:
            from . import kernels as K

            if self.n <= 65536:
                rk, rv = K.rank_rows(self.indptr, self.indices, self.values, self.n, self.item_rank)
            else:
                AT = self._transpose_of_self()
                _, rk, rv = K.csr_transpose(AT.indptr, AT.indices, AT.values, self.m, perm=self.hot_items,
                                            relabel=True)
            self._ranked = (rk, rv, self.hot_items.to(torch.int64))
        return self._ranked

    def hot_encoded(self, nhot: int):
        """(index, values) of this CSR for the hot-set SpMM: every row
        partitioned hot-first (the nhot most rated items' entries, index
        -(rank + 1), then the others, index = item id), built once per nhot
        on the device (cached; one width at a time: 12 B per rating)."""
        hit = self._hot.get(nhot)
        if hit is None:
            from . import kernels as K

            self._hot = {}  # release the previous width's copy first
            idx = torch.empty_like(self.indices)
            val = torch.empty_like(self.values)
            K.call("svdrec_spmm_hot_partition", self.m, K.ptr(self.indptr), K.ptr(self.indices), K.ptr(self.values),
                   K.ptr(self.item_rank), int(nhot), K.ptr(idx), K.ptr(val), K.stream_handle())
            hit = self._hot[nhot] = (idx, val)
        return hit

    def _transpose_of_self(self) -> "DeviceCSR":
        return self._transpose if self._transpose is not None else self.transposed()

    def partial(self, b: int) -> torch.Tensor | None:
        if self.nslots == 0:
            return None
        p = self._partial.get(b)
        if p is None:
            p = self._partial[b] = torch.empty(max(self.nslots * b, 2), dtype=torch.float64, device=self.device)
        return p

    @property
    def hbm_bytes(self) -> int:
        return self.nnz * 12 + (self.m + 1) * 8


class DeviceRatings:
    """A and A.T in HBM (both row-major CSRs) + scalar summaries."""

    def __init__(self, ratings: SparseRatings, device: torch.device):
        A = DeviceCSR.upload(ratings.matrix, device)
        self._init_from(A, device, ratings.m, ratings.n, ratings.nnz, ratings.rating_min, ratings.rating_max)

    def _init_from(self, A: "DeviceCSR", device, m, n, nnz, rating_min, rating_max) -> None:
        self.device = device
        self.m, self.n = m, n
        self.nnz = nnz
        self.rating_min, self.rating_max = rating_min, rating_max
        self.A = A
        self.AT = self.A.transposed()
        # item popularity order (column degree, descending) for on-chip
        # staging of the hottest items' rows in the CF scoring kernel
        col_deg = self.AT.indptr[1:] - self.AT.indptr[:-1]
        order = torch.sort(-col_deg, stable=True).indices
        rank = torch.empty(self.n, dtype=torch.int32, device=device)
        rank[order] = torch.arange(self.n, dtype=torch.int32, device=device)
        self.A.hot_items = order.to(torch.int32)
        self.A.item_rank = rank
        self.h2d_bytes = self.A.h2d_bytes
        # ||A||_F^2 and the global mean (fro_norm_sq, linalg.py:161-168;
        # _global_mean, cf.py:102-105) reduced on the device, read once.
        from . import kernels as K

        stats = torch.zeros(2, dtype=torch.float64, device=device)
        if self.nnz:
            K.sumsq(self.A.values.view(-1, 1), None, stats[0:1])
            K.vec_sum(self.A.values, stats[1:2])
        s = stats.cpu().numpy()
        self.frob_sq = float(s[0])
        self.global_mean = float(s[1] / self.nnz) if self.nnz else float("nan")

    @classmethod
    def from_csr(cls, csr: DeviceCSR, rating_min: float, rating_max: float) -> "DeviceRatings":
        """Wrap a CSR already in HBM (no host copy): A.T, popularity order
        and the scalar summaries are built on the device."""
        self = object.__new__(cls)
        self._init_from(csr, csr.device, csr.m, csr.n, csr.nnz, rating_min, rating_max)
        return self

    def check(self):
        """(any row not strictly increasing, all values finite, min, max) of
        the uploaded CSR -- the reference's constructor checks
        (sparse.py:11-59), one device pass and one small read."""
        A = self.A
        dev = self.device
        bad = torch.zeros((), dtype=torch.bool, device=dev)
        if A.nnz > 1:
            dif = A.indices[1:] - A.indices[:-1]
            cross = torch.zeros(A.nnz - 1, dtype=torch.bool, device=dev)
            st = A.indptr[1:-1]
            st = st[(st > 0) & (st < A.nnz)]
            cross[st - 1] = True
            bad = ((dif <= 0) & ~cross).any()
        v = A.values
        out = torch.stack([bad.to(torch.float64), torch.isfinite(v).all().to(torch.float64),
                           torch.nan_to_num(v, nan=0.0).min(), torch.nan_to_num(v, nan=0.0).max()]).cpu().numpy()
        return bool(out[0]), bool(out[1]), float(out[2]), float(out[3])

    def swapped(self) -> "DeviceRatings":
        """View of A.T (rows <-> columns) sharing the same buffers."""
        v = object.__new__(DeviceRatings)
        v.__dict__.update(self.__dict__)
        v.m, v.n = self.n, self.m
        v.A, v.AT = self.AT, self.A
        return v


class TransposedRatings:
    """A.T of a matrix whose HBM image is (or will be) built: the image
    already holds the CSR of A.T (DeviceRatings.AT, built on the device), so
    the transpose is the two CSRs swapped -- no host transpose and no second
    upload.  What adaptive_pca works on when m > n (reference rsvd.py:359,
    ``A.transposed()``); the QB engines need only shape / nnz / bounds and
    ``device()``.  ``matrix`` (the host CSR of A.T) is built only if asked."""

    def __init__(self, base) -> None:
        self.base = base
        self.rating_min, self.rating_max = base.rating_min, base.rating_max
        self._views: dict = {}

    shape = property(lambda self: (self.base.n, self.base.m))
    m = property(lambda self: self.base.n)
    n = property(lambda self: self.base.m)
    nnz = property(lambda self: self.base.nnz)

    def device(self, device=None) -> "DeviceRatings":
        d = self.base.device(device)
        v = self._views.get(id(d))
        if v is None:
            v = self._views[id(d)] = (d, d.swapped())
        return v[1]

    @property
    def matrix(self) -> sp.csr_matrix:
        return self.base.matrix.transpose().tocsr()

    def transposed(self):
        return self.base


class DeviceSparseRatings:
    """A rating matrix that lives only in HBM (e.g. generated on the device).

    The subset of the SparseRatings interface the QB engines and the SpMM
    use: shape / m / n / nnz, the rating bounds and ``device()`` (the CSR of
    A, the CSR of A.T built on the device, ||A||_F^2).  ``to_host()``
    copies it to a SparseRatings (e.g. for an oracle check of a row range).
    """

    def __init__(self, csr: DeviceCSR, rating_min: float, rating_max: float):
        self.rating_min, self.rating_max = float(rating_min), float(rating_max)
        self._d = DeviceRatings.from_csr(csr, self.rating_min, self.rating_max)

    shape = property(lambda self: (self._d.m, self._d.n))
    m = property(lambda self: self._d.m)
    n = property(lambda self: self._d.n)
    nnz = property(lambda self: self._d.nnz)

    def device(self, device=None) -> "DeviceRatings":
        if device is not None and torch.device(device) != self._d.device:
            raise ValueError("a DeviceSparseRatings lives on one device")
        return self._d

    def to_host(self, row0: int = 0, row1: int | None = None) -> SparseRatings:
        """Rows [row0, row1) as a host SparseRatings."""
        A = self._d.A
        row1 = A.m if row1 is None else row1
        ip = A.indptr[row0: row1 + 1].cpu().numpy()
        a, b = int(ip[0]), int(ip[-1])
        csr = sp.csr_matrix((A.values[a:b].cpu().numpy(), A.indices[a:b].cpu().numpy(), ip - a),
                            shape=(row1 - row0, A.n))
        return SparseRatings(csr, self.rating_min, self.rating_max)

