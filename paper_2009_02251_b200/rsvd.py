"""Randomized QB factorizations on the B200: Algs. 1-3 of the paper.

Mirrors ``svdrec.rsvd`` (reference pkg/src/svdrec/rsvd.py): basic_rsvd,
fixed_precision_qb (randQB_EI, Alg. 2), adaptive_pca (Alg. 3) and the two
block generators, with the same signatures, stop rules, rank caps and
exceptions.

Device layout (all float64, HBM-resident for the whole factorization):
  Q  : m x cap row-major; block l occupies columns [l*b, (l+1)*b)
  Bt : n x cap row-major = B.T, so appending B's block is writing columns
  work buffers: two m x b, one n x b
Per block the host reads back exactly one small vector (||B_l||_F^2 and the
b row energies) to evaluate the termination criterion; everything else --
sketch generation, SpMM, deflation, LU, TSQR -- is queued on one stream.
"""
from __future__ import annotations

import os

from dataclasses import dataclass
from typing import Callable, Iterator

import numpy as np
import torch

from . import kernels as K
from ._lib import STATUS_NEAR_SINGULAR, STATUS_STREAM_SHORT, STATUS_ZERO_PIVOT
from .linalg import (EIG_FLOOR, GaussianStream, NearSingularError, RankDeficientError, SvdTriplet, _check_rank,
                     sparse_dense_mul)
from .parallel import ColumnShardedView, Comm, ShardedRatings, sharded_orth
from .sparse import SparseRatings, TransposedRatings

F64 = torch.float64


# basis of the power steps' lu_lower_basis: 'cqr' (one-pass shifted
# CholeskyQR, ~45 us at 138493 x 20) or 'lu' (partial pivoting on-chip,
# ~130 us); both are Y times an upper-triangular matrix, so the block's
# final Q is the same up to column signs (bench: 42.8 vs 43.8 ms per step,
# same k, MAE trace and test RMSE to every printed digit)
LU_BASIS = os.environ.get("SVDREC_LU_BASIS", "cqr")
# SVDREC_LOOKAHEAD=0: every sketch matrix is drawn in place on the QB stream (A/B measurements)
LOOKAHEAD = os.environ.get("SVDREC_LOOKAHEAD", "1") != "0"

class QbState:
    """Snapshot of a growing QB factorization after a completed block.

    Same fields as the reference's QbState (rsvd.py:40-59).  ``Q`` and
    ``B`` are numpy arrays materialised lazily from the device views
    ``Q_device`` (m x k) and ``Bt_device`` (n x k, = B.T).  ``err`` and
    ``row_energy`` of an engine snapshot are read back from the device only
    when first used, so a criterion that ignores them (ValidationMae) costs
    no host round trip per block.
    """

    def __init__(self, Q_device, Bt_device, err, blocks, block_size, frob_sq, row_energy=None, engine=None):
        self.Q_device = Q_device
        self.Bt_device = Bt_device
        self._err = None if err is None else float(err)
        self.blocks = int(blocks)
        self.block_size = int(block_size)
        self.frob_sq = float(frob_sq)
        self._row_energy = row_energy
        self._engine = engine
        self._Q = None
        self._B = None

    def _materialise(self) -> None:
        if self._err is None:
            self._engine.flush(self.blocks)
            self._err = self._engine.errs[self.blocks - 1]
            self._row_energy = np.asarray(self._engine.row_energy[: self.rank])

    @property
    def err(self) -> float:
        self._materialise()
        return self._err

    @property
    def row_energy(self) -> np.ndarray:
        self._materialise()
        return self._row_energy

    def check(self) -> None:
        """Raise the deferred device-side errors of this block (if any)."""
        if self._engine is not None:
            self._engine.flush(self.blocks)

    @property
    def rank(self) -> int:
        return int(self.Q_device.shape[1])

    @property
    def Q(self) -> np.ndarray:
        if self._Q is None:
            self._Q = self.Q_device.cpu().numpy()
        return self._Q

    @property
    def B(self) -> np.ndarray:
        if self._B is None:
            self._B = np.ascontiguousarray(self.Bt_device.cpu().numpy().T)
        return self._B


class RankExhaustedError(RuntimeError):
    """The factorization hit its rank cap before the stop condition held."""

    def __init__(self, message: str, state: QbState | None = None) -> None:
        super().__init__(message)
        self.state = state


@dataclass(frozen=True)
class FixedRank:
    """Stop once the factorization holds at least ``k`` columns."""

    k: int

    def __post_init__(self) -> None:
        if self.k < 1:
            raise ValueError("k must be positive")

    def __call__(self, state: QbState) -> bool:
        return state.rank >= self.k


@dataclass(frozen=True)
class FrobTolerance:
    """Stop once ``||A - QB||_F <= eps * ||A||_F`` by the running estimate."""

    eps: float

    def __post_init__(self) -> None:
        if not 0.0 < self.eps < 1.0:
            raise ValueError("eps must lie in (0, 1)")

    def __call__(self, state: QbState) -> bool:
        return state.err < self.eps * self.eps * state.frob_sq


TerminationCriterion = Callable[[QbState], bool]


_LOOKAHEAD: dict = {}


def _lookahead_stream(dev: torch.device) -> torch.cuda.Stream:
    """One cached stream per device for the sketch look-ahead draws."""
    s = _LOOKAHEAD.get(dev.index)
    if s is None:
        s = _LOOKAHEAD[dev.index] = torch.cuda.Stream(device=dev)
    return s


class _QbEngine:
    """Device state of one growing QB factorization."""

    @staticmethod
    def create(A, b: int, stream: GaussianStream, cap: int, precision: str = "fp64") -> "_QbEngine":
        if precision not in ("fp64", "fp32"):
            raise ValueError(f"precision must be 'fp64' or 'fp32', not {precision!r}")
        if isinstance(A, ShardedRatings) and A.world > 1:
            E = _ShardedQbEngine(A, b, stream, cap)
        elif isinstance(A, ColumnShardedView) and A.world > 1:
            E = _ColShardedQbEngine(A, b, stream, cap)
        else:
            E = _QbEngine(A.local if isinstance(A, (ShardedRatings, ColumnShardedView)) else A, b, stream, cap)
        E.precision = precision
        return E

    def __init__(self, A: SparseRatings, b: int, stream: GaussianStream, cap: int, global_m: int | None = None,
                 frob_sq: float | None = None, global_n: int | None = None):
        self.A = A
        self.dev = stream.device
        self.d = A.device(self.dev)
        self.m, self.n = A.shape  # rows held here (all of them unless sharded)
        self.gm = self.m if global_m is None else int(global_m)
        self.gn = self.n if global_n is None else int(global_n)
        self.b = b
        self.stream = stream
        cap = max(b, min(cap, min(self.gm, self.gn)))
        self.cap = cap
        self.Q = torch.empty(self.m, self._alloc_cols(0), dtype=F64, device=self.dev)
        self.Bt = torch.empty(self.n, self._alloc_cols(0), dtype=F64, device=self.dev)
        self.K = 0
        self.ym = torch.empty(self.m, b, dtype=F64, device=self.dev)
        self.ym2 = torch.empty(self.m, b, dtype=F64, device=self.dev)
        self.yn = torch.empty(self.n, b, dtype=F64, device=self.dev)
        # per block: a small mailbox (||B_l||_F^2, row energies, status
        # flags of the block's LU / sketch draws), copied back asynchronously
        # and parsed only when someone needs err / row energies / errors
        self._new_mailbox()
        self.frob = (self.d.frob_sq if A.nnz else 0.0) if frob_sq is None else float(frob_sq)
        self.err = self.frob
        self.errs: list[float] = []
        self.blocks = 0
        self.row_energy: list[float] = []
        self._pending: list = []

    def _new_mailbox(self) -> None:
        self.mb = K.Mailbox(self.dev, colsq=("f8", self.b), total=("f8", 1), status=("u4", 1))
        self.status = self.mb["status"]

    def flush(self, upto: int | None = None) -> None:
        """Parse the read-backs of blocks 1..upto (default: all), in order;
        waits only for those blocks, not for work queued after them."""
        upto = self.blocks if upto is None else upto
        while self._pending and len(self.errs) < upto:
            got = self._pending.pop(0).get()
            flags = int(got["status"][0])
            if flags & STATUS_STREAM_SHORT:
                raise RuntimeError("Gaussian stream window exhausted (internal sizing error)")
            if flags & STATUS_ZERO_PIVOT:
                raise RankDeficientError("exactly singular pivot in LU factorization")
            self.err = max(self.err - float(got["total"][0]), 0.0)
            self.errs.append(self.err)
            self.row_energy.extend(float(x) for x in got["colsq"])

    def _alloc_cols(self, need: int) -> int:
        c = max(need, 4 * self.b, 64)
        c = 1 << (c - 1).bit_length() if c < self.cap else self.cap
        return min(max(c, need), max(self.cap, need))

    def _ensure(self, need: int) -> None:
        if need <= self.Q.shape[1]:
            return
        c = self._alloc_cols(max(need, 2 * self.Q.shape[1]))
        Q = torch.empty(self.m, c, dtype=F64, device=self.dev)
        Bt = torch.empty(self.n, c, dtype=F64, device=self.dev)
        if self.K:
            Q[:, : self.K].copy_(self.Q[:, : self.K])
            Bt[:, : self.K].copy_(self.Bt[:, : self.K])
        self.Q, self.Bt = Q, Bt

    precision = "fp64"  # "fp32": the SpMMs gather float copies of their dense operand

    # -- products through the (monkeypatchable) sparse_dense_mul -----------
    def A_mul(self, X, out):
        if self.precision == "fp32":
            return K.spmm(self.d.A, X, out, "fp32")
        return sparse_dense_mul(self.A, X, False, out=out)

    def AT_mul(self, X, out):
        if self.precision == "fp32":
            return K.spmm(self.d.AT, X, out, "fp32")
        return sparse_dense_mul(self.A, X, True, out=out)

    # -- deflations ----------------------------------------------------------
    def minus_QBX(self, Y, X):
        """Y -= Q @ (B @ X)   (rsvd.py:135, 140, 179, 187)."""
        if self.K:
            C = K.gemm_tn(self.Bt[:, : self.K], X)
            K.gemm_nn(self.Q[:, : self.K], C, Y, alpha=-1.0, beta=1.0)

    def minus_BtQtX(self, Y, X):
        """Y -= B.T @ (Q.T @ X)   (rsvd.py:138)."""
        if self.K:
            C = K.gemm_tn(self.Q[:, : self.K], X)
            K.gemm_nn(self.Bt[:, : self.K], C, Y, alpha=-1.0, beta=1.0)

    def minus_QQtX(self, Y):
        """Y -= Q @ (Q.T @ Y)   (rsvd.py:142, 193)."""
        if self.K:
            C = K.gemm_tn(self.Q[:, : self.K], Y)
            K.gemm_nn(self.Q[:, : self.K], C, Y, alpha=-1.0, beta=1.0)

    def lu(self, Y):
        """lu_lower_basis of a power step (rsvd.py:183-190) as a one-pass
        shifted CholeskyQR basis (LU_BASIS = "cqr", the default; with "lu"
        the on-chip partial-pivoting LU where the rows fit it): both are Y
        times an upper-triangular matrix, so the block's final Q is the same
        up to column signs (parallel.py), and an all-zero Y still flags a
        zero pivot."""
        r, b = Y.shape
        if LU_BASIS == "lu" and K.query("svdrec_lu_fast_path", r, b):
            K.lu_lower(Y, self.status)
        else:
            sharded_orth(Y, Y, _LOCAL, r, passes=1, status=self.status)

    def orth_into(self, Y, dst):
        K.orth(Y, dst)

    def orth_final(self, Y, dst):
        """Orthonormalisation of the block that is appended to Q."""
        self.orth_into(Y, dst)

    def append(self, src):
        """Re-orthogonalise ``src`` against Q, append it and B_l = q.T A."""
        b, k0 = self.b, self.K
        self._ensure(k0 + b)
        self.minus_QQtX(src)
        qdst = self.Q[:, k0 : k0 + b]
        self.orth_final(src, qdst)
        bdst = self.Bt[:, k0 : k0 + b]
        self.AT_mul(qdst, bdst)
        K.sumsq(bdst, self.mb["colsq"], self.mb["total"])
        self._reduce_energy()
        self._pending.append(self.mb.read_async())  # parsed lazily by flush()
        self._new_mailbox()
        self.K = k0 + b
        self.blocks += 1

    def _reduce_energy(self) -> None:
        """B_l's row energies are complete on this rank (B.T replicated)."""

    def normal(self, rows: int, cols: int, out):
        return self.stream.normal_device(rows, cols, out=out, status=self.status)

    # -- sketch look-ahead ----------------------------------------------------
    # The sketch matrix Omega of block l + 1 (rsvd.py:178: one
    # standard_normal((n, b)) per block) does not depend on the factorization,
    # and its draw is a chain of small latency-bound kernels (csrc/gaussian.cu:
    # ~77 us at 26,744 x 20).  It is drawn one block ahead on a side stream,
    # into the other of two Omega buffers, with its status flags going to the
    # mailbox the next block will use.  The stream position lives on the
    # device and all draws stay in order; a drawn-ahead Omega that is never
    # used (the consumer stopped) is rolled back, so the stream ends exactly
    # where the reference's would.
    LOOKAHEAD_BYTES = 64 << 20  # larger sketches are throughput-bound: drawn in place

    def next_omega(self, n: int):
        """Omega of the block being started (n x b; ``n`` is the global
        column count: a sharded sketch side draws the full matrix and keeps
        its rows, and is not drawn ahead)."""
        la, self._la = getattr(self, "_la", None), None
        if la is not None:
            ev, buf, _, mb = la
            torch.cuda.current_stream(self.dev).wait_event(ev)
            self.mb, self.status = mb, mb["status"]  # the flags of this block's draw are in this mailbox
            return buf
        if not hasattr(self, "_om"):
            self._om = [torch.empty(self.n, self.b, dtype=F64, device=self.dev) for _ in range(2)]
            self._om_i = 0
        self._om_i ^= 1
        return self.normal(n, self.b, self._om[self._om_i])

    def prefetch_omega(self, n: int) -> None:
        """Queue the draw of the next block's Omega on the look-ahead stream
        (after everything queued so far on this stream: the buffer's last
        reader is behind us)."""
        if n != self.n or n * self.b * 8 > self.LOOKAHEAD_BYTES or not hasattr(self, "_om"):
            return
        cur = torch.cuda.current_stream(self.dev)
        side = _lookahead_stream(self.dev)
        ev0 = torch.cuda.Event()
        ev0.record(cur)
        side.wait_event(ev0)
        mb = K.Mailbox(self.dev, colsq=("f8", self.b), total=("f8", 1), status=("u4", 1))
        self._om_i ^= 1
        buf = self._om[self._om_i]
        with torch.cuda.stream(side):
            saved = self.stream.pos.clone()
            self.stream.normal_device(self.n, self.b, out=buf, status=mb["status"])
            ev = torch.cuda.Event()
            ev.record(side)
        self._la = (ev, buf, saved, mb)

    def release_lookahead(self) -> None:
        """Undo a drawn-ahead Omega nobody used: the reference never drew it."""
        la, self._la = getattr(self, "_la", None), None
        if la is not None:
            ev, _, saved, _ = la
            torch.cuda.current_stream(self.dev).wait_event(ev)
            self.stream.pos.copy_(saved)

    def state(self) -> QbState:
        return QbState(self.Q[:, : self.K], self.Bt[:, : self.K], None, self.blocks, self.b, self.frob,
                       None, engine=self)


_LOCAL = Comm.local()  # one-rank communicator: every all-reduce is a no-op


class _ShardedQbEngine(_QbEngine):
    """QB engine over a row-sharded matrix (parallel.py): this rank holds
    rows [row0, row1) of A and Q; the item side (sketches of n rows, B.T)
    is replicated.  Exchanges: all-reduce of A.T products (n x b), of
    Q.T Y (k x b) and of the b x b Grams of the sharded CholeskyQR."""

    def __init__(self, A: ShardedRatings, b: int, stream: GaussianStream, cap: int):
        super().__init__(A.local, b, stream, cap, global_m=A.m, frob_sq=A.frob_sq)
        self.shard = A
        self.comm = A.comm

    def AT_mul(self, X, out):
        if self.precision == "fp32":
            K.spmm(self.d.AT, X, out, "fp32")
        else:
            sparse_dense_mul(self.A, X, True, out=out)
        return self.comm.all_reduce_(out)

    def minus_BtQtX(self, Y, X):
        if self.K:
            C = self.comm.all_reduce_(K.gemm_tn(self.Q[:, : self.K], X))
            K.gemm_nn(self.Bt[:, : self.K], C, Y, alpha=-1.0, beta=1.0)

    def minus_QQtX(self, Y):
        if self.K:
            C = self.comm.all_reduce_(K.gemm_tn(self.Q[:, : self.K], Y))
            K.gemm_nn(self.Q[:, : self.K], C, Y, alpha=-1.0, beta=1.0)

    def lu(self, Y):
        # Y U^-1 with U upper triangular, like the reference's P.L: the
        # block's final Q is the same up to column signs (parallel.py)
        # one shifted pass: a well-conditioned basis is all the next
        # product needs
        sharded_orth(Y, Y, self.comm, self.gm, passes=1, status=self.status)

    def orth_into(self, Y, dst):
        # intermediate bases (fed to a product, re-orthogonalised later)
        sharded_orth(Y, dst, self.comm, self.gm, passes=2)

    def orth_final(self, Y, dst):
        sharded_orth(Y, dst, self.comm, self.gm, passes=3)  # shifted CholeskyQR3

    def normal(self, rows: int, cols: int, out):
        if out.shape[0] == rows:  # item-side draw: replicated
            return self.stream.normal_device(rows, cols, out=out, status=self.status)
        full = self.stream.normal_device(rows, cols, status=self.status)  # same stream on every rank
        out.copy_(full[self.shard.row0: self.shard.row1])
        return out


class _ColShardedQbEngine(_QbEngine):
    """QB engine over A.T of a row-sharded A (parallel.ColumnShardedView;
    adaptive_pca of a tall matrix, reference rsvd.py:359).  The n rows of
    A.T (items) are replicated -- Q, the sketches A.T Omega and their
    orthonormalisations are computed identically on every rank -- and its
    m columns (users) are sharded: B.T = A Q holds this rank's rows.
    Exchanges: all-reduce of A_r.T X_r (n x b) and of B.T X (k x b), the
    b x b Grams of m-side orthonormalisations (power steps of Alg. 2), and
    B_l's row energies."""

    def __init__(self, A: ColumnShardedView, b: int, stream: GaussianStream, cap: int):
        super().__init__(A.local, b, stream, cap, frob_sq=A.frob_sq, global_n=A.n)
        self.shard = A
        self.comm = A.comm

    def A_mul(self, X, out):
        super().A_mul(X, out)  # A_r.T X_r
        return self.comm.all_reduce_(out)

    def minus_QBX(self, Y, X):
        if self.K:
            C = self.comm.all_reduce_(K.gemm_tn(self.Bt[:, : self.K], X))
            K.gemm_nn(self.Q[:, : self.K], C, Y, alpha=-1.0, beta=1.0)

    def orth_into(self, Y, dst):
        if Y.shape[0] == self.m:  # replicated n-side block
            K.orth(Y, dst)
        else:  # sharded m-side block (Alg. 2 power steps)
            sharded_orth(Y, dst, self.comm, self.gn, passes=2)

    def _reduce_energy(self) -> None:
        self.comm.all_reduce_(self.mb["colsq"])
        self.comm.all_reduce_(self.mb["total"])

    def normal(self, rows: int, cols: int, out):
        if out.shape[0] == rows:  # n-side draw: replicated
            return self.stream.normal_device(rows, cols, out=out, status=self.status)
        full = self.stream.normal_device(rows, cols, status=self.status)  # same stream on every rank
        out.copy_(full[self.shard.row0: self.shard.row1])
        return out


def qb_power_blocks(A: SparseRatings, block_size: int, power: int, stream: GaussianStream,
                    max_rank: int | None = None, precision: str = "fp64") -> Iterator[QbState]:
    """Alg. 2 block generator with power iteration (rsvd.py:112-148)."""
    m, n = A.shape
    b = block_size
    cap = min(m, n) if max_rank is None else min(min(m, n), max_rank + b)
    E = _QbEngine.create(A, b, stream, cap, precision)
    while (E.blocks + 1) * b <= min(m, n):
        om = E.normal(n, b, E.yn)
        y = E.A_mul(om, E.ym)
        E.minus_QBX(y, om)
        E.orth_into(y, y)
        for _ in range(power):
            g = E.AT_mul(y, E.yn)
            E.minus_BtQtX(g, y)
            E.orth_into(g, g)
            y = E.A_mul(g, E.ym)
            E.minus_QBX(y, g)
            E.orth_into(y, y)
        E.append(y)
        yield E.state()


def qb_pass_blocks(A: SparseRatings, block_size: int, passes: int, stream: GaussianStream,
                   max_rank: int | None = None, precision: str = "fp64") -> Iterator[QbState]:
    """Alg. 3 pass-capped block generator (rsvd.py:151-199)."""
    m, n = A.shape
    b = block_size
    if passes < 2:
        raise ValueError("passes must be at least 2")
    cap = min(m, n) if max_rank is None else min(min(m, n), max_rank + b)
    E = _QbEngine.create(A, b, stream, cap, precision)
    nsteps = (passes - 1) // 2
    try:
        while (E.blocks + 1) * b <= min(m, n) - b:
            if passes % 2 == 0:
                om = E.next_omega(n)
                ql = E.A_mul(om, E.ym)
                E.minus_QBX(ql, om)
                if LOOKAHEAD and (E.blocks + 2) * b <= min(m, n) - b:
                    E.prefetch_omega(n)  # block l + 1's sketch matrix, drawn beside this block
                E.lu(ql)
            else:
                ql = E.normal(m, b, E.ym)
            for t in range(1, nsteps + 1):
                r = E.AT_mul(ql, E.yn)
                y = E.A_mul(r, E.ym2 if ql is E.ym else E.ym)
                if t == nsteps:
                    E.minus_QBX(y, r)
                    E.orth_into(y, y)
                else:
                    E.lu(y)
                ql = y
            E.append(ql)
            yield E.state()
    finally:
        E.release_lookahead()


def _refined_rank(row_energy: np.ndarray, frob_sq: float, eps: float) -> tuple[int, float]:
    """Smallest prefix of B's rows meeting eps (rsvd.py:202-214)."""
    cum = np.cumsum(row_energy)
    hits = np.nonzero(frob_sq - cum < eps * eps * frob_sq)[0]
    k = int(hits[0]) + 1 if hits.size else row_energy.size
    return k, max(float(frob_sq - cum[k - 1]), 0.0)


def basic_rsvd(A: SparseRatings, k: int, power: int = 0, oversample: int = 0, seed: int = 0) -> SvdTriplet:
    """Alg. 1: rank-k randomized SVD with a single sketch (rsvd.py:217-264)."""
    m, n = A.shape
    if k < 1:
        raise ValueError("k must be positive")
    if power < 0 or oversample < 0:
        raise ValueError("power and oversample must be nonnegative")
    ell = k + oversample
    if ell > min(m, n):
        raise ValueError(f"k + oversample = {ell} exceeds min(m, n) = {min(m, n)}")
    stream = GaussianStream(seed)
    dev = stream.device
    om = stream.normal_device(n, ell)
    y = sparse_dense_mul(A, om)
    q, R = K.tsqr(y)
    _check_rank(y, R)
    for _ in range(power):
        g = sparse_dense_mul(A, q, True)
        gq, R = K.tsqr(g)
        _check_rank(g, R)
        y = sparse_dense_mul(A, gq)
        q, R = K.tsqr(y)
        _check_rank(y, R)
    bt = sparse_dense_mul(A, q, True)  # b.T (n x ell)
    st = K.new_status(dev)
    s, Ub, Vb = K.gesvj(bt, st)  # b.T = Ub diag(s) Vb.T  ->  b = Vb diag(s) Ub.T
    u = K.gemm_nn(q, Vb[:, :k].contiguous())
    return SvdTriplet(u.cpu().numpy(), s[:k].cpu().numpy(), Ub[:, :k].cpu().numpy(), k)


def fixed_precision_qb(A: SparseRatings, tol: float, block_size: int = 20, power: int = 0, seed: int = 0,
                       max_rank: int | None = None) -> QbState:
    """Alg. 2 (randQB_EI): grow QB until ||A - QB||_F <= tol ||A||_F, then
    trim the last block to the smallest sufficient rank (rsvd.py:267-319).

    ``max_rank`` (not in the reference) caps the scan; hitting it raises
    RankExhaustedError with the state, like the reference's own cap.
    """
    if not 0.0 < tol < 1.0:
        raise ValueError("tol must lie in (0, 1)")
    if block_size < 1:
        raise ValueError("block_size must be positive")
    if power < 0:
        raise ValueError("power must be nonnegative")
    if block_size > min(A.shape):
        raise ValueError(f"block_size {block_size} exceeds min(m, n) = {min(A.shape)}")
    frob = A.frob_sq if isinstance(A, ShardedRatings) else (A.device().frob_sq if A.nnz else 0.0)
    if A.nnz == 0 or frob == 0.0:
        dev = torch.device("cuda", torch.cuda.current_device())
        rows = A.local.m if isinstance(A, ShardedRatings) else A.m
        return QbState(torch.empty(rows, 0, dtype=F64, device=dev), torch.empty(A.n, 0, dtype=F64, device=dev),
                       0.0, 0, block_size, 0.0, np.empty(0))
    stream = GaussianStream(seed)
    last = None
    for state in qb_power_blocks(A, block_size, power, stream, max_rank=max_rank):
        last = state
        if state.err < tol * tol * state.frob_sq:
            k, err = _refined_rank(state.row_energy, state.frob_sq, tol)
            return QbState(state.Q_device[:, :k], state.Bt_device[:, :k], err, state.blocks, block_size,
                           state.frob_sq, state.row_energy[:k])
        if max_rank is not None and state.rank >= max_rank:
            break
    raise RankExhaustedError(f"residual target {tol:.3e} unmet at rank cap", state=last)


def _svd_from_qb(Qm: torch.Tensor, Btm: torch.Tensor, k: int, comm: Comm | None = None):
    """Top-k singular triplets of Q B through eig_svd(B.T) (rsvd.py:384-389).
    ``comm``: B.T's rows are sharded over it (the Gram is all-reduced)."""
    st = K.new_status(Qm.device)
    G = K.gemm_tn(Btm, Btm)  # B B.T
    if comm is not None:
        comm.all_reduce_(G)
    w, V = K.syev(G, st)
    if K.check_status(st) & STATUS_NEAR_SINGULAR:
        raise NearSingularError(f"Gram eigenvalue {float(w[0].item()):.3e} below floor "
                                f"{EIG_FLOOR * float(torch.trace(G)):.3e}")
    r = G.shape[0]
    idx = torch.arange(r - 1, r - 1 - k, -1, device=Qm.device)
    Vk = V[:, idx].contiguous()
    s = torch.sqrt(torch.clamp(w[idx], min=0.0))
    u = K.gemm_nn(Qm, Vk)  # Q @ dec.v[:, idx]
    v = K.gemm_nn(Btm, Vk)  # dec.u[:, idx] = (B.T @ V) / s
    v.div_(s)
    return u, s, v


def adaptive_pca(A: SparseRatings, criterion: TerminationCriterion, block_size: int = 20, passes: int = 10,
                 seed: int = 0, max_rank: int | None = None, device_output: bool = False) -> SvdTriplet:
    """Alg. 3: blocked randomized SVD, fixed pass budget, pluggable stop
    (rsvd.py:322-392).  ``device_output`` keeps u, s, v as CUDA tensors."""
    if passes <= 2:
        raise ValueError("passes must exceed 2")
    if block_size < 1:
        raise ValueError("block_size must be positive")
    m, n = A.shape
    # the transpose is a view of the HBM image (its CSR of A.T), not a host
    # transpose and a second upload
    if m > n:
        work = A.transposed() if isinstance(A, ShardedRatings) else TransposedRatings(A)
    else:
        work = A
    b = block_size
    if isinstance(criterion, FixedRank):
        b = min(b, criterion.k)
    if 2 * b > min(m, n):
        raise ValueError(f"block_size {b} too large for min(m, n) = {min(m, n)}")
    stream = GaussianStream(seed)
    met = last = None
    for state in qb_pass_blocks(work, b, passes, stream, max_rank=max_rank):
        last = state
        if criterion(state):
            met = state
            break
        if max_rank is not None and state.rank >= max_rank:
            break
    if last is not None:
        last.check()  # deferred LU / stream errors surface like the reference's
    if met is None:
        raise RankExhaustedError("termination criterion never met", state=last)
    if isinstance(criterion, FixedRank):
        k = criterion.k
        Qm, Btm = met.Q_device, met.Bt_device
    elif isinstance(criterion, FrobTolerance):
        k, _ = _refined_rank(met.row_energy, met.frob_sq, criterion.eps)
        Qm, Btm = met.Q_device[:, :k], met.Bt_device[:, :k]
    else:
        k = met.rank
        Qm, Btm = met.Q_device, met.Bt_device
    col_sharded = isinstance(work, ColumnShardedView) and work.world > 1
    u, s, v = _svd_from_qb(Qm, Btm, k, work.comm if col_sharded else None)
    if m > n:  # u: this rank's rows when A is row-sharded (as for m <= n)
        u, v = v, u
    if device_output:
        return SvdTriplet(u, s, v, int(k))
    return SvdTriplet(u.cpu().numpy(), s.cpu().numpy(), v.cpu().numpy(), int(k))


__all__ = ["FixedRank", "FrobTolerance", "QbState", "RankExhaustedError", "TerminationCriterion", "adaptive_pca",
           "basic_rsvd", "fixed_precision_qb", "qb_pass_blocks", "qb_power_blocks"]
