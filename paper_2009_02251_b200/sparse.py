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
        mat.sort_indices()
        object.__setattr__(self, "matrix", mat)
        object.__setattr__(self, "rating_min", float(rating_min))
        object.__setattr__(self, "rating_max", float(rating_max))
        object.__setattr__(self, "_dev", {})
        if self.rating_min > self.rating_max:
            raise ValueError("rating_min exceeds rating_max")
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
            if not np.all(np.isfinite(mat.data)):
                raise ValueError("ratings must be finite")
            lo, hi = mat.data.min(), mat.data.max()
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


def warp_plan(seg_begin: np.ndarray, seg_end: np.ndarray, nwarp: int, seg_cost: int = 16) -> np.ndarray:
    """Split the row-ordered segments into ``nwarp`` contiguous ranges of
    about equal cost (nonzeros + ``seg_cost`` per segment); returns the
    ``nwarp + 1`` range starts (int32) the pipelined SpMM kernel reads."""
    nseg = seg_begin.size
    cost = np.cumsum((seg_end - seg_begin) + seg_cost, dtype=np.int64)
    total = int(cost[-1]) if nseg else 0
    targets = (np.arange(1, nwarp, dtype=np.float64) * (total / max(nwarp, 1)))
    cuts = np.searchsorted(cost, targets, side="left") + 1 if nseg else np.zeros(nwarp - 1, np.int64)
    out = np.empty(nwarp + 1, dtype=np.int64)
    out[0], out[-1] = 0, nseg
    out[1:-1] = np.minimum(cuts, nseg)
    return np.maximum.accumulate(out).astype(np.int32)


class DeviceCSR:
    """One CSR in HBM plus its SpMM plan."""

    def __init__(self, csr: sp.csr_matrix, device: torch.device):
        self.m, self.n = csr.shape
        self.nnz = csr.nnz
        self.device = device
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).astype(dt, copy=False)).to(device, non_blocking=True)  # noqa: E731
        self.indptr = t(csr.indptr, np.int64)
        self.indices = t(csr.indices, np.int32)
        self.values = t(csr.data, np.float64)
        sr, sb, se, sl, lr, s0, s1, nslots = segment_plan(csr.indptr.astype(np.int64))
        self.nseg = int(sr.size)
        self.seg_row = t(sr, np.int32)
        self.seg_begin = t(sb, np.int64)
        self.seg_end = t(se, np.int64)
        self.seg_slot = t(sl, np.int32)
        self.nlong = int(lr.size)
        self.long_row = t(lr, np.int32)
        self.long_s0 = t(s0, np.int32)
        self.long_s1 = t(s1, np.int32)
        self.nslots = nslots
        sms = torch.cuda.get_device_properties(device).multi_processor_count if device.type == "cuda" else 148
        self.nwarp = int(max(1, min(sr.size, sms * WARPS_PER_SM)))
        self.warp_seg = t(warp_plan(sb, se, self.nwarp), np.int32)
        self._partial = {}
        self.h2d_bytes = (self.m + 1) * 8 + self.nnz * 12 + self.nseg * 24 + self.nlong * 12 + (self.nwarp + 1) * 4

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
        self.device = device
        self.m, self.n = ratings.shape
        self.nnz = ratings.nnz
        self.rating_min, self.rating_max = ratings.rating_min, ratings.rating_max
        self.A = DeviceCSR(ratings.matrix, device)
        at = ratings.matrix.T.tocsr()
        self.AT = DeviceCSR(at, device)
        # item popularity order (column degree, descending) for on-chip
        # staging of the hottest items' rows in the CF scoring kernel
        order = np.argsort(-np.diff(at.indptr), kind="stable").astype(np.int32)
        rank = np.empty(self.n, dtype=np.int32)
        rank[order] = np.arange(self.n, dtype=np.int32)
        self.A.hot_items = torch.from_numpy(order).to(device)
        self.A.item_rank = torch.from_numpy(rank).to(device)
        self.h2d_bytes = self.A.h2d_bytes + self.AT.h2d_bytes + 8 * self.n
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

    def swapped(self) -> "DeviceRatings":
        """View of A.T (rows <-> columns) sharing the same buffers."""
        v = object.__new__(DeviceRatings)
        v.__dict__.update(self.__dict__)
        v.m, v.n = self.n, self.m
        v.A, v.AT = self.AT, self.A
        return v
