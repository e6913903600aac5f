"""Item-based collaborative filtering on latent factors (Algs. 4 and 5).

Mirrors ``svdrec.cf`` (reference pkg/src/svdrec/cf.py): LatentFactors,
latent_from_qb, predict_rating, mae, evaluate_mae, ValidationMae and
auto_latent_factors, same contracts and exceptions.  All scoring runs in
csrc/cf.cu; held-out samples are grouped by user once (one warp per user
builds the two k-vectors P_u, S_u and scores all of that user's samples).

Alg. 5 scores every block, but Alg. 4 only needs cosines between item
columns of T = S^(1/2) U.T, and T.T T = B.T (B B.T)^(-1/2) B.  So
ValidationMae scores each block in "metric mode" -- x_l = B[:, l],
y_l = G^(-1/2) x_l with G = B B.T from a Newton-Schulz kernel -- and only
the factors it returns pay for the eigendecomposition (lazily, on first
access to ``T``), exactly as latent_from_qb computes it.
"""
from __future__ import annotations

import os
import time
from typing import Iterable, NamedTuple, Sequence

import numpy as np
import torch

from . import kernels as K
from .hostio import to_device
from ._lib import STATUS_NEAR_SINGULAR, STATUS_NS_CHECK
from .linalg import EIG_FLOOR, GaussianStream, NearSingularError
from .parallel import ShardedRatings, local_samples
from .rsvd import QbState, RankExhaustedError, qb_pass_blocks
from .sparse import SparseRatings

WEIGHT_FLOOR = 1e-9  # cf.py:23
F64 = torch.float64
# Score block l on a side stream while block l+1 is factored (on by default:
# 47.5 vs 48.1 ms per bench step with the ranked CF kernel; SVDREC_PIPELINE=0
# scores on the caller's stream).
PIPELINE = os.environ.get("SVDREC_PIPELINE", "1") == "1"
_SIDE: dict = {}


def _side_stream(dev) -> torch.cuda.Stream:
    s = _SIDE.get(dev.index)
    if s is None:
        s = _SIDE[dev.index] = torch.cuda.Stream(device=dev)
    return s


class Prediction(NamedTuple):
    """A predicted rating: clamped value, raw pre-clamp value, fallback flag."""

    value: float
    raw: float
    fallback: bool


class BlockEval(NamedTuple):
    """Validation result after one factorization block."""

    k: int
    mae: float
    seconds: float


def _eig_T(Bt: torch.Tensor, G: torch.Tensor | None = None, status: torch.Tensor | None = None) -> torch.Tensor:
    """T.T = B.T V diag(s^-1/2), eig(B B.T) descending (cf.py:77-92)."""
    st = K.new_status(Bt.device) if status is None else status
    if G is None:
        G = K.gemm_tn(Bt, Bt)
    w, V = K.syev(G, st)
    if status is None and K.check_status(st) & STATUS_NEAR_SINGULAR:
        raise NearSingularError(f"Gram eigenvalue {float(w[0].item()):.3e} below floor "
                                f"{EIG_FLOOR * float(torch.trace(G)):.3e}")
    Wm = V.flip(1) * torch.rsqrt(torch.sqrt(torch.clamp(w.flip(0), min=0.0)))
    return K.gemm_nn(Bt, Wm.contiguous())


_DEBUG_NS = bool(os.environ.get("SVDREC_DEBUG_NS"))
_HOST_TRACE: list | None = None  # (rank, submit s, next block s, collect s) per block when a list


class LatentFactors:
    """Item embedding T (k x items) with cached column norms (cf.py:42-74).

    Device-resident.  Scoring uses unit item rows ``Xn``/``Yn`` (equal to
    T's normalized columns for explicit factors; B's columns in the metric
    (B B.T)^(-1/2) for factors taken straight from a QB block) and
    ``norm_device``.  ``T`` and ``col_norms`` materialise numpy copies; for
    QB-block factors T is computed on first access by the same eig route
    as the reference's latent_from_qb.
    """

    def __init__(self, Tt: torch.Tensor | None = None, *, Xn=None, Yn=None, norm=None, Bt=None, G=None):
        self._Tt = None
        self._Bt, self._G = Bt, G
        if Tt is not None:
            if Tt.dim() != 2:
                raise ValueError("T must be 2-d")
            self._Tt = Tt.contiguous()
            Tn, norm = K.cf_normalize(self._Tt)
            Xn = Yn = Tn
        self.Xn, self.Yn, self.norm_device = Xn, Yn, norm
        self._T = None
        self._norms = None

    @property
    def k(self) -> int:
        return int(self.Xn.shape[1])

    @property
    def n_items(self) -> int:
        return int(self.Xn.shape[0])

    @property
    def Tt(self) -> torch.Tensor:
        if self._Tt is None:
            self._Tt = _eig_T(self._Bt, self._G)
        return self._Tt

    @property
    def T(self) -> np.ndarray:
        if self._T is None:
            self._T = np.asfortranarray(self.Tt.cpu().numpy().T)
        return self._T

    @property
    def col_norms(self) -> np.ndarray:
        # metric mode: n_l = sqrt(x_l.G^(-1/2).x_l) = |T_l| identically
        if self._norms is None:
            self._norms = self.norm_device.cpu().numpy()
        return self._norms

    @classmethod
    def from_matrix(cls, T) -> "LatentFactors":
        if isinstance(T, torch.Tensor):
            Tt = T.to(F64).T.contiguous().cuda()
        else:
            T = np.asarray(T, dtype=np.float64)
            if T.ndim != 2:
                raise ValueError("T must be 2-d")
            Tt = torch.from_numpy(np.ascontiguousarray(T.T)).cuda()
        return cls(Tt)

    @classmethod
    def from_qb_metric(cls, Bt: torch.Tensor, G: torch.Tensor, Z: torch.Tensor) -> "LatentFactors":
        """Metric-mode factors of a QB block: x_l = B[:, l], y_l = Z x_l."""
        Yt = K.gemm_nn(Bt, Z)
        Xn, Yn, norm = K.cf_normalize_pair(Bt, Yt)
        return cls(Xn=Xn, Yn=Yn, norm=norm, Bt=Bt, G=G)


def latent_from_qb(state: QbState) -> LatentFactors:
    """Distill item factors from a QB snapshot: T = sqrt(S) U.T, rows by
    descending singular value (cf.py:77-92)."""
    if state.rank == 0:
        raise ValueError("empty factorization has no latent factors")
    return LatentFactors(_eig_T(state.Bt_device))


class WorkPlan:
    """Work items of the CF scoring kernel for one (samples, matrix) pair.

    Groups (one per user with samples) are cut into chunks of at most
    ``CHUNK`` training ratings; items are ordered heaviest user first so the
    dynamic scheduler never ends behind a long row.  Each item is described
    up front (built on the device): ``start`` (its first CSR entry) and
    ``meta`` = (length, user degree, first sample, end sample, chunks of the
    user, partial slot, completion counter, chunk index) as int32.
    """

    CHUNK = 512

    def __init__(self, group_deg: torch.Tensor, device, group_start: torch.Tensor | None = None,
                 row_start: torch.Tensor | None = None):
        """``group_deg``: training degree of each group's user; ``group_start``
        (ngroups + 1) sample offsets; ``row_start``: CSR offset of each
        group's user row (all int64 tensors on ``device``)."""
        gd = torch.as_tensor(group_deg, device=device).to(torch.int64).contiguous()
        ng = gd.numel()
        if group_start is None:
            group_start = torch.arange(ng + 1, device=device)
        if row_start is None:
            row_start = torch.cumsum(gd, 0) - gd
        gs = group_start.to(torch.int64).contiguous()
        rs = row_start.to(torch.int64).contiguous()
        # heaviest user first (ties: group order), then two kernels: chunk
        # counts / slot bases / first items (one CTA), then the records
        order = torch.sort(-gd, stable=True).indices if ng else torch.zeros(0, dtype=torch.int64, device=device)
        first = torch.empty(max(ng, 1), dtype=torch.int64, device=device)
        slot0 = torch.empty(max(ng, 1), dtype=torch.int32, device=device)
        done_idx = torch.empty(max(ng, 1), dtype=torch.int32, device=device)
        stats = torch.empty(4, dtype=torch.int64, device=device)
        K.cf_plan_scan(gd, order, self.CHUNK, first, slot0, done_idx, stats)
        st = stats.cpu().numpy()  # the plan's sizes (one small read)
        self.nwork, self.ndone, self.nslots, self.rated = int(st[0]), int(st[1]), int(st[2]), int(st[3])
        self.start = torch.zeros(max(self.nwork, 1), dtype=torch.int64, device=device)
        self.meta = torch.zeros(8 * max(self.nwork, 1), dtype=torch.int32, device=device)
        K.cf_plan_emit(gd, order, first, slot0, done_idx, gs, rs, self.CHUNK, self.start, self.meta)
        self.done = torch.zeros(max(self.ndone, 1), dtype=torch.int32, device=device)
        self.counter = torch.zeros(1, dtype=torch.int32, device=device)
        self.chunk = self.CHUNK
        self.device = device
        self._part = None

    def partial(self, k: int) -> torch.Tensor:
        need = max(self.nslots * (2 * k + 1), 1)
        if self._part is None or self._part.numel() < need:
            self._part = torch.empty(need, dtype=torch.float64, device=self.device)
        return self._part


class _Samples:
    """Held-out (user, item, rating) triples, user-grouped, on the device."""

    def __init__(self, samples, device):
        if hasattr(samples, "arrays") and not callable(samples.arrays):  # data.SampleList
            samples = samples.arrays
        if isinstance(samples, tuple) and len(samples) == 3 and hasattr(samples[0], "__len__") and \
                not isinstance(samples[0], (int, np.integer)):
            u = np.asarray(samples[0], dtype=np.int64)
            i = np.asarray(samples[1], dtype=np.int64)
            r = np.asarray(samples[2], dtype=np.float64)
        else:
            arr = list(samples)
            u = np.array([int(s[0]) for s in arr], dtype=np.int64)
            i = np.array([int(s[1]) for s in arr], dtype=np.int64)
            r = np.array([float(s[2]) for s in arr], dtype=np.float64)
        self.n = int(u.size)
        self.users_np, self.items_np, self.truth_np = u, i, r
        # grouped by user on the device: stable sort of the raw arrays.  The
        # uploads run on the copy stream, so they overlap whatever the
        # current stream is computing (e.g. the first QB block)
        from .sparse import _copy_stream

        dv = torch.device(device)
        if dv.type == "cuda":
            if dv.index is None:
                dv = torch.device("cuda", torch.cuda.current_device())
            cur, side = torch.cuda.current_stream(dv), _copy_stream(dv)
            with torch.cuda.stream(side):
                ud = to_device(u, np.int64, device)
                idev = to_device(i, np.int64, device)
                rd = to_device(r, np.float64, device)
                ev = torch.cuda.Event()
                ev.record(side)
            for t in (ud, idev, rd):
                t.record_stream(cur)
            cur.wait_event(ev)
        else:  # host-side planning tests
            ud, idev, rd = (to_device(x, dt, device) for x, dt in ((u, np.int64), (i, np.int64), (r, np.float64)))
        self.h2d_bytes = self.n * 24
        order = torch.sort(ud, stable=True).indices if self.n else torch.zeros(0, dtype=torch.int64, device=device)
        us = ud[order]
        starts = torch.nonzero(us[1:] != us[:-1]).flatten() + 1 if self.n > 1 else \
            torch.zeros(0, dtype=torch.int64, device=device)
        self.groups = torch.cat([torch.zeros(1 if self.n else 0, dtype=torch.int64, device=device), starts,
                                 torch.full((1,), self.n, dtype=torch.int64, device=device)])
        self.users = us.to(torch.int32)
        self.items = idev[order].to(torch.int32)
        self.truth = rd[order]
        self._order_dev = order
        self._order = None
        self.group_users_dev = us[self.groups[:-1]] if self.n else torch.zeros(0, dtype=torch.int64, device=device)
        self.device = device
        self._plans = {}
        self._checked: set = set()  # matrix shapes the samples were bounds-checked against
        self._overlap: dict = {}    # id(matrix) -> (matrix, samples also stored in it); the
        #                             reference keeps the id from being reused

    @property
    def order(self) -> np.ndarray:
        """Input position of each user-sorted sample (host copy, on demand)."""
        if self._order is None:
            self._order = self._order_dev.cpu().numpy()
        return self._order

    def plan_for(self, A: SparseRatings) -> "WorkPlan":
        """Scoring work plan against training matrix ``A`` (cached)."""
        hit = self._plans.get(id(A))  # (matrix, plan): the reference pins the id
        if hit is None:
            d = A.device(self.device)
            deg = d.A.indptr[1:] - d.A.indptr[:-1]
            gu = self.group_users_dev
            hit = self._plans[id(A)] = (A, WorkPlan(deg[gu], self.device, self.groups, d.A.indptr[gu]))
        return hit[1]

    def check_bounds(self, A: SparseRatings, exc: type = ValueError) -> None:
        if self.n == 0 or A.shape in self._checked:
            return
        u, i = self.users_np, self.items_np
        if u.min() >= 0 and u.max() < A.m and i.min() >= 0 and i.max() < A.n:
            self._checked.add(A.shape)
            return
        bad = (u < 0) | (u >= A.m) | (i < 0) | (i >= A.n)
        if bad.any():
            j = int(np.flatnonzero(bad)[0])
            raise exc(f"sample ({self.users_np[j]}, {self.items_np[j]}) outside matrix bounds")
        self._checked.add(A.shape)


def _predict_device(A: SparseRatings, factors: LatentFactors, s: _Samples, gmean: float, precision: str = "fp64"):
    d = A.device(factors.Xn.device)
    return K.cf_predict(s.groups, s.users, s.items, d.A, factors.Yn, factors.Xn, factors.norm_device, gmean,
                        A.rating_min, A.rating_max, s.plan_for(A), precision, group_users=s.group_users_dev)


def predict_rating(A: SparseRatings, factors: LatentFactors, user: int, item: int) -> Prediction:
    """Alg. 4: cosine-weighted average of the user's ratings, clamped;
    user/global mean fallback (cf.py:146-164)."""
    if not 0 <= user < A.m:
        raise IndexError(f"user {user} out of range")
    if not 0 <= item < A.n:
        raise IndexError(f"item {item} out of range")
    if factors.n_items != A.n:
        raise ValueError("factor matrix does not cover this item set")
    if A.nnz == 0:
        raise ValueError("cannot take the mean of a matrix with no ratings")
    d = A.device(factors.Xn.device)
    s = _Samples(([user], [item], [0.0]), factors.Xn.device)
    val, raw, fb = _predict_device(A, factors, s, d.global_mean)
    out = torch.stack([val, raw, fb.to(F64)]).cpu().numpy()
    return Prediction(value=float(out[0, 0]), raw=float(out[1, 0]), fallback=bool(out[2, 0]))


def predict_many(A: SparseRatings, factors: LatentFactors, samples) -> np.ndarray:
    """Batch Alg. 4: (n, 3) array of value, raw, fallback in input order."""
    s = _Samples(samples, factors.Xn.device)
    s.check_bounds(A)
    val, raw, fb = _predict_device(A, factors, s, A.device(factors.Xn.device).global_mean)
    out = np.empty((s.n, 3))
    out[s.order, 0] = val.cpu().numpy()
    out[s.order, 1] = raw.cpu().numpy()
    out[s.order, 2] = fb.cpu().numpy()
    return out


def mae(predictions: Sequence[float], truths: Sequence[float]) -> float:
    """Mean absolute error between two equally long nonempty sequences (Eq. 6)."""
    p = np.asarray(predictions, dtype=np.float64)
    t = np.asarray(truths, dtype=np.float64)
    if p.shape != t.shape or p.ndim != 1:
        raise ValueError("predictions and truths must be 1-d of equal length")
    if p.size == 0:
        raise ValueError("cannot average zero errors")
    return float(np.abs(p - t).mean())


def _errors(A, factors, s: _Samples, precision: str = "fp64"):
    if A.nnz == 0:
        raise ValueError("cannot take the mean of a matrix with no ratings")
    if isinstance(A, ShardedRatings):
        return _sharded_errors(A, factors, s, precision)
    if s.n == 0:
        raise ValueError("cannot average zero errors")
    # the reference's per-sample loop fails on an out-of-range user or item
    # with IndexError (sparse.py row_slice, numpy indexing); checked here so
    # no out-of-range index reaches the device
    s.check_bounds(A, IndexError)
    if factors.n_items != A.n:
        raise ValueError("factor matrix does not cover this item set")
    val, _, _ = _predict_device(A, factors, s, A.device(factors.Xn.device).global_mean, precision)
    e = K.err_sum(val, s.truth).cpu().numpy()
    return float(e[0] / s.n), float(np.sqrt(e[1] / s.n))


def _shard_samples(A: ShardedRatings, samples, device) -> _Samples:
    """This rank's held-out triples (users re-based to the shard), after
    the bounds check against the global shape; ``n_total`` counts all ranks."""
    u, i, r = local_samples(samples, 0, A.m)  # all of them, as arrays
    if u.size != _count(samples):
        raise ValueError("sample outside matrix bounds")
    bad = (i < 0) | (i >= A.n)
    if bad.any():
        j = int(np.flatnonzero(bad)[0])
        raise ValueError(f"sample ({u[j]}, {i[j]}) outside matrix bounds")
    keep = (u >= A.row0) & (u < A.row1)
    s = _Samples((u[keep] - A.row0, i[keep], r[keep]), device)
    s.n_total = int(u.size)
    s._checked.add(A.local.shape)
    return s


def _count(samples) -> int:
    if hasattr(samples, "arrays") and not callable(samples.arrays):
        samples = samples.arrays
    if isinstance(samples, tuple) and len(samples) == 3 and hasattr(samples[0], "__len__"):
        return len(samples[0])
    return len(list(samples))


def _local_err_sums(A: ShardedRatings, factors, s: _Samples, out: torch.Tensor, precision: str = "fp64") -> torch.Tensor:
    """(sum |e|, sum e^2) over this rank's samples, then all-reduced on the
    scoring communicator (A.score_comm: scoring may run on a side stream,
    apart from the QB chain's collectives on A.comm)."""
    if s.n:
        val, _, _ = _predict_device(A.local, factors, s, A.global_mean, precision)
        K.err_sum(val, s.truth, out=out)
    else:
        out.zero_()
    return A.score_comm.all_reduce_(out)


def _sharded_errors(A: ShardedRatings, factors, s, precision: str = "fp64"):
    dev = factors.Xn.device
    if not isinstance(s, _Samples) or not hasattr(s, "n_total"):
        s = _shard_samples(A, s, dev)
    if s.n_total == 0:
        raise ValueError("cannot average zero errors")
    e = _local_err_sums(A, factors, s, torch.zeros(2, dtype=F64, device=dev), precision).cpu().numpy()
    return float(e[0] / s.n_total), float(np.sqrt(e[1] / s.n_total))


def evaluate_mae(A: SparseRatings, factors: LatentFactors, samples: Iterable, precision: str = "fp64") -> float:
    """MAE of clamped predictions over held-out triples (cf.py:178-190).
    ``precision="fp32"`` (not in the reference) stores the gathered item
    rows as float, accumulating in double."""
    if isinstance(A, ShardedRatings):
        return _errors(A, factors, samples, precision)[0]
    s = samples if isinstance(samples, _Samples) else _Samples(samples, factors.Xn.device)
    return _errors(A, factors, s, precision)[0]


def evaluate_errors(A: SparseRatings, factors: LatentFactors, samples, precision: str = "fp64") -> tuple[float, float]:
    """(MAE, RMSE) of clamped Alg. 4 predictions (RMSE: BASELINE metric)."""
    if isinstance(A, ShardedRatings):
        return _errors(A, factors, samples, precision)
    s = samples if isinstance(samples, _Samples) else _Samples(samples, factors.Xn.device)
    return _errors(A, factors, s, precision)


class ValidationMae:
    """Termination criterion tracking held-out MAE (cf.py:193-240).

    After each block the factors are scored on the validation samples;
    ``patience`` consecutive blocks improving the best MAE by less than
    ``min_improvement`` stop the scan.  The best block's factors and the
    (k, MAE, seconds) trace stay on the instance.  The Gram B B.T is grown
    incrementally when successive states extend one another, and each
    block costs one small host read (error sums + status word).
    """

    def __init__(self, train: SparseRatings, validation, patience: int = 2, min_improvement: float = 1e-4,
                 precision: str = "fp64") -> None:
        if precision not in ("fp64", "fp32"):
            raise ValueError(f"precision must be 'fp64' or 'fp32', not {precision!r}")
        self.precision = precision
        if patience < 1:
            raise ValueError("patience must be at least 1")
        if min_improvement < 0.0:
            raise ValueError("min_improvement must be nonnegative")
        dev = torch.device("cuda", torch.cuda.current_device())
        self.shard = train if isinstance(train, ShardedRatings) else None
        if self.shard is not None:
            s = validation if isinstance(validation, _Samples) and hasattr(validation, "n_total") else \
                _shard_samples(train, validation, dev)
            if s.n_total == 0:
                raise ValueError("validation set is empty")
            train = train.local
        else:
            s = validation if isinstance(validation, _Samples) else _Samples(validation, dev)
            if s.n == 0:
                raise ValueError("validation set is empty")
            s.check_bounds(train)
        d = train.device(dev)
        hit = s._overlap.get(id(train))
        if hit is None:
            c = K.count_overlap(s.users, s.items, d.A).to(F64) if s.n else torch.zeros(1, dtype=F64, device=dev)
            if self.shard is not None:
                c = self.shard.comm.all_reduce_(c.reshape(1).clone())
            hit = s._overlap[id(train)] = (train, int(c.item()))
        cnt = hit[1]
        if cnt:
            raise ValueError(f"{cnt} validation samples are present in the training matrix")
        if (self.shard or train).nnz == 0:
            raise ValueError("cannot take the mean of a matrix with no ratings")
        self.train = train  # this rank's rows when sharded
        self.n_total = s.n_total if self.shard is not None else s.n
        self.samples = s
        self.patience = patience
        self.min_improvement = min_improvement
        self.trace: list[BlockEval] = []
        self.best_mae = np.inf
        self.best_factors: LatentFactors | None = None
        self.best_rmse = np.inf
        self._stale = 0
        self._start = time.perf_counter()
        self._G = None
        self._Gsrc = None
        self._mb = K.Mailbox(dev, sums=("f8", 2), status=("u4", 1), iters=("u4", 1))
        self._gmean = self.shard.global_mean if self.shard is not None else d.global_mean
        # scoring stream: the caller's unless pipelining; one cached side
        # stream per device (a fresh stream per call would defeat the caching
        # allocator, whose free blocks are tied to the stream they served)
        self._stream = _side_stream(dev) if PIPELINE else torch.cuda.current_stream(dev)

    @property
    def validation(self):
        s = self.samples
        return list(zip(s.users_np.tolist(), s.items_np.tolist(), s.truth_np.tolist()))

    def _gram(self, Bt: torch.Tensor) -> torch.Tensor:
        """B B.T, grown by the new block's rows when ``Bt`` extends the
        previous state's columns (same buffer); else recomputed."""
        k = Bt.shape[1]
        G0, src = self._G, self._Gsrc
        if G0 is not None and src is not None and src.data_ptr() == Bt.data_ptr() and src.shape[1] < k and \
                src.stride() == Bt.stride():
            k0 = G0.shape[0]
            G = torch.empty(k, k, dtype=F64, device=Bt.device)
            G[:k0, :k0] = G0
            K.gemm_tn(Bt, Bt[:, k0:k], G[:, k0:k])  # new columns
            G[k0:k, :k0] = G[:k0, k0:k].T
        else:
            G = K.gemm_tn(Bt, Bt)
        self._G, self._Gsrc = G, Bt
        return G

    def submit(self, state: QbState):
        """Queue the scoring of ``state`` on the criterion's own stream and
        return a handle; nothing waits.  The QB engine can meanwhile queue
        its next block on the current stream (see auto_latent_factors)."""
        if state.rank == 0:
            raise ValueError("empty factorization has no latent factors")
        cur = torch.cuda.current_stream()
        s2 = self._stream
        s2.wait_stream(cur)  # block l's columns of B are complete
        Bt = state.Bt_device
        Bt.record_stream(s2)
        mb = self._mb
        with torch.cuda.stream(s2):
            G = self._gram(Bt)
            Z = K.inv_sqrt(G, mb["status"], mb["iters"])
            factors = LatentFactors.from_qb_metric(Bt, G, Z)
            s = self.samples
            if self.shard is not None:
                _local_err_sums(self.shard, factors, s, mb["sums"], self.precision)
            else:
                val, _, _ = _predict_device(self.train, factors, s, self._gmean, self.precision)
                K.err_sum(val, s.truth, out=mb["sums"])
            mb.read_async()
        return state, factors

    def collect(self, pending) -> bool:
        """Wait for a submitted block's score, update the trace, and return
        the stop decision (cf.py:227-240)."""
        state, factors = pending
        state.check()  # the engine's deferred per-block errors, if any
        mb = self._mb
        got = mb.get()  # one host read per block: error sums + status
        flags = int(got["status"][0])
        if _DEBUG_NS:
            print(f"[svdrec] k={state.rank} NS iterations={int(got['iters'][0])} status={flags}", flush=True)
        s = self.samples
        if flags:
            with torch.cuda.stream(self._stream):
                mb["status"].zero_()
        if flags & STATUS_NS_CHECK:
            # Newton-Schulz could not certify the eigenvalue floor: decide it
            # exactly like the reference (eigh) and score with its T
            with torch.cuda.stream(self._stream):
                factors = LatentFactors(_eig_T(state.Bt_device, factors._G))
                if self.shard is not None:
                    sums = _local_err_sums(self.shard, factors, s, torch.zeros(2, dtype=F64, device=s.device),
                                           self.precision)
                else:
                    val, _, _ = _predict_device(self.train, factors, s, self._gmean, self.precision)
                    sums = K.err_sum(val, s.truth)
                got = {"sums": sums.cpu().numpy()}
        n = self.n_total
        score, rmse = float(got["sums"][0] / n), float(np.sqrt(got["sums"][1] / n))
        self.trace.append(BlockEval(k=state.rank, mae=score, seconds=time.perf_counter() - self._start))
        if score < self.best_mae - self.min_improvement:
            self._stale = 0
        else:
            self._stale += 1
        if score < self.best_mae:
            self.best_mae = score
            self.best_rmse = rmse
            self.best_factors = factors
        return self._stale >= self.patience

    def __call__(self, state: QbState) -> bool:
        return self.collect(self.submit(state))

    def may_stop(self) -> bool:
        """Whether the next collected score can end the scan (one more
        stale block reaches ``patience``)."""
        return self._stale + 1 >= self.patience

    def join(self) -> None:
        """Make the current stream wait for everything scored so far and
        keep the best factors alive across streams."""
        cur = torch.cuda.current_stream()
        cur.wait_stream(self._stream)
        f = self.best_factors
        if f is not None:
            for t in (f.Xn, f.Yn, f.norm_device, f._G):
                if t is not None:
                    t.record_stream(cur)


def auto_latent_factors(A: SparseRatings, validation, block_size: int = 20, passes: int = 10, patience: int = 2,
                        min_improvement: float = 1e-4, seed: int = 0,
                        max_rank: int | None = None, precision: str = "fp64") -> tuple[LatentFactors, list[BlockEval]]:
    """Alg. 5: grow item factors until validation MAE stops improving
    (cf.py:257-294).  ``max_rank`` (not in the reference) ends the scan once
    that many factors are held and keeps the best block so far.
    ``precision="fp32"`` (not in the reference) is the fp32 variant: the
    gathered operands of the SpMMs and of the CF scoring are stored as float
    (accumulation, the QB algebra and all returned values stay double)."""
    if passes <= 2:
        raise ValueError("passes must exceed 2")
    if block_size < 1:
        raise ValueError("block_size must be positive")
    if 2 * block_size > min(A.shape):
        raise ValueError(f"block_size {block_size} too large for min(m, n) = {min(A.shape)}")
    stream = GaussianStream(seed)
    gen = qb_pass_blocks(A, block_size, passes, stream, max_rank=max_rank, precision=precision)
    # block 1 is queued before the validation samples are ingested (upload,
    # grouping, bounds and disjointness checks -- host work with a few
    # small reads), so that ingest overlaps the block on the GPU; a
    # criterion error still surfaces before any result exists
    state = next(gen, None)
    criterion = ValidationMae(A, validation, patience=patience, min_improvement=min_improvement, precision=precision)
    # Same criterion sequence as the reference's ``for state in ...: if
    # criterion(state): break``, pipelined: block l is scored on the
    # criterion's stream while block l+1 is factored on this one (a block
    # computed past the stop is simply discarded).
    # the next block is enqueued before the host waits for this block's
    # score (same stream unless PIPELINE), so the GPU never idles on the
    # stop decision; a block computed past the stop is discarded
    pipeline = PIPELINE
    while state is not None:
        t0 = time.perf_counter() if _HOST_TRACE is not None else 0.0
        pending = criterion.submit(state)
        capped = max_rank is not None and state.rank >= max_rank
        # speculate on the next block only when this score cannot end the
        # scan (fewer than patience - 1 stale blocks so far): a block queued
        # past the stop would be computed for nothing, next to the scoring
        if pipeline and not criterion.may_stop():
            t1 = time.perf_counter() if _HOST_TRACE is not None else 0.0
            nxt = None if capped else next(gen, None)
            t2 = time.perf_counter() if _HOST_TRACE is not None else 0.0
            stop = criterion.collect(pending) or capped
            if _HOST_TRACE is not None:
                _HOST_TRACE.append((state.rank, t1 - t0, t2 - t1, time.perf_counter() - t2))
            if stop:
                break
        else:
            if criterion.collect(pending) or capped:
                break
            nxt = next(gen, None)
        state = nxt
    criterion.join()
    if criterion.best_factors is None:
        raise RankExhaustedError("rank cap reached before any block was scored")
    return criterion.best_factors, criterion.trace


__all__ = ["BlockEval", "LatentFactors", "Prediction", "ValidationMae", "auto_latent_factors", "evaluate_errors",
           "evaluate_mae", "latent_from_qb", "mae", "predict_many", "predict_rating"]
