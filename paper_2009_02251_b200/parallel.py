"""Multi-GPU plumbing and the row-sharded rating matrix (one process per GPU).

The north star shards the users (rows of A) over the GPUs: each rank keeps
rows [row0, row1) of A -- and the matching rows of Q -- and runs its local
SpMMs; the item side (the n x b sketches, B.T, the Gram B B.T and the CF
item factors) is replicated.  The only data-path exchanges are all-reduces
of small partials:

  * A.T @ X = sum_r A_r.T @ X_r                (n x b, every power step and B_l)
  * Q.T @ Y = sum_r Q_r.T @ Y_r                (k x b, the re-orthogonalisation)
  * Y.T @ Y = sum_r Y_r.T @ Y_r                (b x b, row-sharded CholeskyQR)
  * the CF error sums and sample counts        (a few scalars per block)

Row-sharded orthonormalisation is shifted CholeskyQR3 (Fukaya et al.,
"Shifted CholeskyQR for computing the QR factorization of ill-conditioned
matrices", SISC 2020): one Gram all-reduce per pass and no pivot search
across ranks.  Because Q = Y R^-1 with R upper triangular, and the
reference's LU basis P.L = Y U^-1 is also Y times an upper-triangular
matrix, replacing the LU of a power step by this orthonormalisation leaves
the block's final Q unchanged up to column signs (QR uniqueness), so B_l's
row energies, the error indicator and every CF score match the one-GPU run
to rounding.

NCCL is the backend on GPUs (``torch.distributed`` over NVLink/NVSwitch);
the same code runs under ``gloo`` (tests: two ranks, CPU-side plumbing).
"""
from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist

from . import kernels as K
from .sparse import SparseRatings

UNIT_ROUNDOFF = 2.0 ** -53


def env_ranks() -> tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def max_over_ranks(value: float, device: torch.device | None = None) -> float:
    """The maximum of ``value`` over all ranks (every rank gets it); the
    timing rule for multi-GPU numbers (slowest rank).  Identity when no
    process group is initialised."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or torch.device("cpu"))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    return float(t.item())


_SIBLINGS: dict = {}


class Comm:
    """The process group the shards of one matrix live on.

    ``all_reduce_`` sums a tensor in place, stream-ordered on the current
    CUDA stream (NCCL), or synchronously (gloo).  ``world == 1`` makes every
    call a no-op, so a one-rank ShardedRatings behaves like SparseRatings.
    """

    def __init__(self, group=None) -> None:
        self.group = group
        on = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if on else 1
        self.rank = dist.get_rank(group) if on else 0
        self.backend = dist.get_backend(group) if on else None

    @classmethod
    def local(cls) -> "Comm":
        """A one-rank communicator regardless of any process group."""
        c = object.__new__(cls)
        c.group, c.world, c.rank, c.backend = None, 1, 0, None
        return c

    def all_reduce_(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            if t.is_contiguous():
                dist.all_reduce(t, group=self.group)
            else:  # e.g. a column block of B.T: reduce a packed copy
                c = t.contiguous()
                dist.all_reduce(c, group=self.group)
                t.copy_(c)
        return t

    def sibling(self) -> "Comm":
        """A second communicator over the same ranks (its own process group,
        hence its own NCCL communicator), for collectives issued from
        another CUDA stream: the CF scoring's error sums run on the scoring
        side stream while the QB chain's all-reduces run on the main one,
        and two streams must not share one NCCL communicator.  Created
        collectively on first use (every rank constructs its shards in the
        same order) and cached per parent group."""
        if self.world == 1:
            return self
        key = id(self.group) if self.group is not None else 0
        hit = _SIBLINGS.get(key)
        if hit is None:
            ranks = dist.get_process_group_ranks(self.group) if self.group is not None else None
            hit = _SIBLINGS[key] = Comm(dist.new_group(ranks=ranks, backend=self.backend))
        return hit

    def all_gather(self, t: torch.Tensor) -> list[torch.Tensor]:
        if self.world == 1:
            return [t]
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t.contiguous(), group=self.group)
        return out

    def gather_rows(self, t: torch.Tensor, counts) -> torch.Tensor:
        """Concatenate every rank's rows (``counts[r]`` rows on rank r)."""
        if self.world == 1:
            return t
        width = t.shape[1:]
        top = max(int(c) for c in counts)
        pad = torch.zeros((top,) + tuple(width), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        parts = self.all_gather(pad)
        return torch.cat([p[: int(c)] for p, c in zip(parts, counts)])


def row_partition(indptr: np.ndarray, world: int, row_cost: float = 16.0) -> np.ndarray:
    """Contiguous row ranges balancing nonzeros (+ ``row_cost`` per row):
    ``world + 1`` offsets.  Every rank gets at least one row when m >= world."""
    indptr = np.asarray(indptr, dtype=np.int64)
    m = indptr.size - 1
    if world < 1:
        raise ValueError("world must be positive")
    if m < world:
        raise ValueError(f"cannot shard {m} rows over {world} ranks")
    cost = indptr[1:].astype(np.float64) + row_cost * np.arange(1, m + 1)
    total = cost[-1] if m else 0.0
    targets = total * np.arange(1, world) / world
    cuts = np.searchsorted(cost, targets, side="left") + 1
    off = np.concatenate([[0], cuts, [m]]).astype(np.int64)
    # at least one row each, monotone
    for r in range(1, world):
        off[r] = min(max(off[r], off[r - 1] + 1), m - (world - r))
    return off


class ShardedRatings:
    """Rows [row0, row1) of an m x n rating matrix on this rank.

    Behaves like :class:`SparseRatings` for the QB engines and the CF
    criterion: ``shape``/``m``/``n``/``nnz``/``frob_sq``/``global_mean`` are
    global (all-reduced once at construction); ``local`` is this rank's
    SparseRatings (its HBM image holds the CSR of A_r and of A_r.T).
    """

    def __init__(self, local: SparseRatings, row0: int, m: int, comm: Comm | None = None,
                 offsets: np.ndarray | None = None) -> None:
        self.comm = comm or Comm()
        self.score_comm = self.comm.sibling()  # CF scoring collectives (side stream)
        self.local = local
        self.row0 = int(row0)
        self.row1 = self.row0 + local.m
        self._m = int(m)
        self.rating_min, self.rating_max = local.rating_min, local.rating_max
        dev = torch.device("cuda", torch.cuda.current_device())
        stats = torch.zeros(4, dtype=torch.float64, device=dev)
        if local.nnz:
            d = local.device(dev)
            stats[0] = d.frob_sq
            stats[1] = d.global_mean * d.nnz
        stats[2] = float(local.nnz)
        stats[3] = float(local.m)
        self.comm.all_reduce_(stats)
        s = stats.cpu().numpy()
        self.frob_sq = float(s[0])
        self._nnz = int(round(s[2]))
        self.global_mean = float(s[1] / s[2]) if s[2] else float("nan")
        if int(round(s[3])) != self._m:
            raise ValueError(f"shards cover {int(round(s[3]))} rows, expected {self._m}")
        if offsets is None:
            cnt = torch.tensor([local.m], dtype=torch.int64, device=dev)
            counts = [int(c.item()) for c in self.comm.all_gather(cnt)]
            offsets = np.concatenate([[0], np.cumsum(counts)])
        self.offsets = np.asarray(offsets, dtype=np.int64)
        if self.offsets[self.comm.rank] != self.row0:
            raise ValueError("shard offsets disagree with this rank's row0")

    @classmethod
    def from_full(cls, A: SparseRatings, comm: Comm | None = None) -> "ShardedRatings":
        """Keep this rank's nonzero-balanced row range of a matrix every
        rank holds (e.g. loaded from the same file)."""
        comm = comm or Comm()
        off = row_partition(A.indptr, comm.world)
        r0, r1 = int(off[comm.rank]), int(off[comm.rank + 1])
        local = SparseRatings(A.matrix[r0:r1], A.rating_min, A.rating_max)
        return cls(local, r0, A.m, comm, off)

    @classmethod
    def from_csr(cls, csr, rating_min: float, rating_max: float, comm: Comm | None = None) -> "ShardedRatings":
        """Like from_full, from a host CSR: only this rank's rows are ever
        uploaded and checked."""
        comm = comm or Comm()
        off = row_partition(csr.indptr, comm.world)
        r0, r1 = int(off[comm.rank]), int(off[comm.rank + 1])
        return cls(SparseRatings(csr[r0:r1], rating_min, rating_max), r0, csr.shape[0], comm, off)

    shape = property(lambda self: (self._m, self.local.n))
    m = property(lambda self: self._m)
    n = property(lambda self: self.local.n)
    nnz = property(lambda self: self._nnz)
    world = property(lambda self: self.comm.world)

    @property
    def counts(self) -> np.ndarray:
        return np.diff(self.offsets)

    def device(self, device=None):
        """HBM image of the LOCAL rows (A_r and A_r.T)."""
        return self.local.device(device)

    def transposed(self) -> "ColumnShardedView":
        """A.T, column-sharded: the same shards seen through their device
        transposes (no data moves)."""
        return ColumnShardedView(self)


class ColumnShardedView:
    """A.T of a row-sharded A: n x m with the m columns sharded (this rank
    holds columns [row0, row1), i.e. A_r.T from the local HBM image).  The
    QB engine over it (rsvd._ColShardedQbEngine) keeps the n-side (Q, the
    sketches A.T Omega) replicated and the m-side (B.T = A Q) sharded; its
    exchanges are the all-reduces of A_r.T X_r (n x b), of B.T X (k x b),
    of the m-side Grams (b x b) and of B_l's row energies."""

    def __init__(self, base: ShardedRatings) -> None:
        from .sparse import TransposedRatings

        self.base = base
        self.local = TransposedRatings(base.local)  # n x m_r
        self.comm = base.comm
        self.frob_sq = base.frob_sq
        self.rating_min, self.rating_max = base.rating_min, base.rating_max

    shape = property(lambda self: (self.base.n, self.base.m))
    m = property(lambda self: self.base.n)
    n = property(lambda self: self.base.m)
    nnz = property(lambda self: self.base.nnz)
    world = property(lambda self: self.base.world)
    row0 = property(lambda self: self.base.row0)
    row1 = property(lambda self: self.base.row1)

    def device(self, device=None):
        return self.local.device(device)

    def transposed(self) -> ShardedRatings:
        return self.base


def sharded_orth(Y: torch.Tensor, dst: torch.Tensor, comm: Comm, m_global: int, passes: int = 3,
                 status: torch.Tensor | None = None) -> torch.Tensor:
    """Orthonormal basis of a row-sharded tall block: shifted CholeskyQR
    (first pass shifted by 11 (m b + b (b + 1)) u ||Y||_F^2, then plain
    passes), one b x b Gram all-reduce per pass.  ``dst`` may alias ``Y``;
    ``status`` receives SVDREC_STATUS_ZERO_PIVOT if the first (shifted)
    pass meets a non-positive pivot (Y == 0)."""
    b = Y.shape[1]
    shift = 11.0 * (m_global * b + b * (b + 1)) * UNIT_ROUNDOFF
    G = comm.all_reduce_(K.gram(Y))
    K.chol_apply(G, Y, dst, shift, status)
    for _ in range(passes - 1):
        G = comm.all_reduce_(K.gram(dst))
        K.chol_apply(G, dst, dst, 0.0)
    return dst


def local_samples(samples, row0: int, row1: int):
    """(users - row0, items, ratings) of the held-out triples whose user
    lives on this shard, as arrays (input order kept)."""
    if hasattr(samples, "arrays") and not callable(samples.arrays):
        samples = samples.arrays
    if isinstance(samples, tuple) and len(samples) == 3 and hasattr(samples[0], "__len__"):
        u, i, r = (np.asarray(samples[0], dtype=np.int64), np.asarray(samples[1], dtype=np.int64),
                   np.asarray(samples[2], dtype=np.float64))
    else:
        arr = list(samples)
        u = np.array([int(s[0]) for s in arr], dtype=np.int64)
        i = np.array([int(s[1]) for s in arr], dtype=np.int64)
        r = np.array([float(s[2]) for s in arr], dtype=np.float64)
    keep = (u >= row0) & (u < row1)
    return u[keep] - row0, i[keep], r[keep]


__all__ = ["ColumnShardedView", "Comm", "ShardedRatings", "env_ranks", "local_samples", "max_over_ranks", "row_partition",
           "sharded_orth"]
