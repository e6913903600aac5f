"""Dense/sparse building blocks -- reference API, B200 kernels underneath.

Mirrors ``svdrec.linalg`` (reference pkg/src/svdrec/linalg.py): same names,
argument meaning, return conventions and exceptions.  Inputs may be numpy
arrays (results come back as numpy, like the reference) or CUDA tensors
(results stay on the device).  Every computation runs in
libsvdrec_b200.so; without a CUDA device these raise
``ExtensionUnavailable`` -- there is no CPU path.
"""
from __future__ import annotations

from typing import NamedTuple

import numpy as np
import torch

from . import kernels as K
from ._lib import STATUS_NEAR_SINGULAR, STATUS_STREAM_SHORT, STATUS_ZERO_PIVOT, ExtensionUnavailable, load
from .sparse import SparseRatings

ORTH_RANK_FLOOR = 1e-12  # linalg.py:16
EIG_FLOOR = 1e-14  # linalg.py:17
MASK64 = (1 << 64) - 1


class RankDeficientError(ValueError):
    """A matrix that must have full column rank does not."""


class NearSingularError(ValueError):
    """A Gram matrix has eigenvalues at or below the numerical floor."""


def _device():
    load()
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(M) -> tuple[torch.Tensor, bool]:
    """(CUDA float64 row-major tensor, came_from_numpy)."""
    if isinstance(M, torch.Tensor):
        if not M.is_cuda:
            return M.to(_device(), torch.float64).contiguous(), True
        t = M if M.dtype == torch.float64 else M.double()
        if t.dim() == 2 and t.stride(1) != 1:
            t = t.contiguous()
        return t, False
    a = np.asarray(M, dtype=np.float64)
    return torch.from_numpy(np.ascontiguousarray(a)).to(_device()), True


def _out(t: torch.Tensor, host: bool):
    return t.cpu().numpy() if host else t


class GaussianStream:
    """Counter-based deterministic source of standard normal matrices.

    Bit-identical to the reference's ``np.random.Generator(Philox(key=seed))``
    stream (linalg.py:28-44): successive draws of the same shapes from the
    same seed give the same matrices as the reference, computed on the GPU
    (Philox4x64-10 + ziggurat transducer, csrc/gaussian.cu).  The stream
    position lives on the device, so consecutive draws never synchronise.
    """

    def __init__(self, seed: int, device=None) -> None:
        seed = int(seed)
        if seed < 0 or seed >= 1 << 128:
            raise ValueError("seed must lie in [0, 2**128)")
        self.seed = seed
        self.key = (seed & MASK64, (seed >> 64) & MASK64)
        self.device = torch.device(device) if device is not None else _device()
        self.pos = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.status = K.new_status(self.device)

    def normal_device(self, rows: int, cols: int, out: torch.Tensor | None = None,
                      row_perm: torch.Tensor | None = None, status: torch.Tensor | None = None) -> torch.Tensor:
        """Draw on the device; ``status`` (a uint32 word) overrides the
        stream's own status word so callers can batch their status reads."""
        if out is None:
            out = torch.empty(rows, cols, dtype=torch.float64, device=self.device)
        K.normal_fill(self.key, self.pos, rows, cols, out, self.status if status is None else status, row_perm)
        return out

    def check(self) -> None:
        if K.check_status(self.status) & STATUS_STREAM_SHORT:
            raise RuntimeError("Gaussian stream: raw window exhausted (internal sizing error)")

    def normal(self, rows: int, cols: int) -> np.ndarray:
        out = self.normal_device(rows, cols).cpu().numpy()
        self.check()
        return out


def gaussian_matrix(rows: int, cols: int, seed) -> np.ndarray:
    """Standard normal matrix, deterministic for a seed (linalg.py:40-51)."""
    if rows < 1 or cols < 1:
        raise ValueError("rows and cols must be positive")
    stream = seed if isinstance(seed, GaussianStream) else GaussianStream(seed)
    return stream.normal(rows, cols)


def orthonormal_basis(M, check_rank: bool = True):
    """Orthonormal basis of range(M) via Householder QR (linalg.py:54-81)."""
    t, host = _to_dev(M)
    if t.dim() != 2 or t.shape[0] < t.shape[1]:
        raise ValueError(f"expected rows >= cols, got shape {tuple(t.shape)}")
    if t.shape[1] == 0:
        return _out(t.clone(), host)
    Q, R = K.tsqr(t)
    if check_rank:
        _check_rank(t, R)
    return _out(Q, host)


def _check_rank(M: torch.Tensor, R: torch.Tensor) -> None:
    tot = torch.zeros(1, dtype=torch.float64, device=M.device)
    K.sumsq(M, None, tot)
    diag = torch.diagonal(R).abs().min()
    d, nrm = float(diag.item()), float(tot.item()) ** 0.5
    floor = ORTH_RANK_FLOOR * nrm
    if d < floor:
        raise RankDeficientError(f"column rank below {M.shape[1]}: min |R_ii| = {d:.3e}, floor {floor:.3e}")


def lu_lower_basis(M):
    """Permuted lower factor P.L of a partial-pivoting LU (linalg.py:84-97)."""
    t, host = _to_dev(M)
    if t.dim() != 2 or t.shape[0] < t.shape[1]:
        raise ValueError(f"expected rows >= cols, got shape {tuple(t.shape)}")
    out = t.clone() if not host else t
    st = K.new_status(out.device)
    K.lu_lower(out, st)
    if K.check_status(st) & STATUS_ZERO_PIVOT:
        raise RankDeficientError("exactly singular pivot in LU factorization")
    return _out(out, host)


class EigSvd(NamedTuple):
    """SVD factors with singular values in ascending order."""

    u: object
    s: object
    v: object


def eig_svd_device(M: torch.Tensor, status: torch.Tensor | None = None, check: bool = True):
    """Device eig_svd of a tall row-major block: (u, s, v) ascending."""
    st = status if status is not None else K.new_status(M.device)
    G = K.gemm_tn(M, M)
    w, V = K.syev(G, st)
    if check and K.check_status(st) & STATUS_NEAR_SINGULAR:
        w0 = float(w[0].item())
        raise NearSingularError(f"Gram eigenvalue {w0:.3e} below floor {EIG_FLOOR * float(torch.trace(G)):.3e}")
    s = torch.sqrt(torch.clamp(w, min=0.0))
    u = K.gemm_nn(M, V)
    u.div_(s)
    return u, s, V


def eig_svd(M) -> EigSvd:
    """SVD of a tall matrix through the eigendecomposition of its Gram
    matrix, ascending values (linalg.py:108-138)."""
    t, host = _to_dev(M)
    if t.dim() != 2 or t.shape[0] < t.shape[1]:
        raise ValueError(f"expected rows >= cols, got shape {tuple(t.shape)}")
    u, s, v = eig_svd_device(t)
    return EigSvd(_out(u, host), _out(s, host), _out(v, host))


def sparse_dense_mul(A: SparseRatings, X, transpose_a: bool = False, out: torch.Tensor | None = None):
    """A @ X or A.T @ X (linalg.py:141-158); the only route to A."""
    t, host = _to_dev(X)
    if t.dim() != 2:
        raise ValueError("X must be 2-d")
    inner = A.m if transpose_a else A.n
    if t.shape[0] != inner:
        side = "A.T" if transpose_a else "A"
        raise ValueError(f"dimension mismatch: {side} has {inner} columns, X has {t.shape[0]} rows")
    d = A.device(t.device)
    csr = d.AT if transpose_a else d.A
    if out is None:
        out = torch.empty(csr.m, t.shape[1], dtype=torch.float64, device=t.device)
    K.spmm(csr, t, out)
    return _out(out, host)


def fro_norm_sq(M) -> float:
    """Squared Frobenius norm; stored values only for sparse input."""
    if isinstance(M, SparseRatings):
        return M.device().frob_sq if M.nnz else 0.0
    t, _ = _to_dev(M)
    if t.dim() != 2:
        t = t.reshape(-1, 1).contiguous()
    tot = torch.zeros(1, dtype=torch.float64, device=t.device)
    if t.numel():
        K.sumsq(t, None, tot)
    return float(tot.item())


class SvdTriplet(NamedTuple):
    """Rank-k factorization ``u @ diag(s) @ v.T`` with s descending."""

    u: object
    s: object
    v: object
    k: int

    def reconstruct(self):
        if isinstance(self.u, torch.Tensor):
            return (self.u * self.s) @ self.v.T
        return (self.u * self.s) @ self.v.T


__all__ = [
    "EigSvd", "ExtensionUnavailable", "GaussianStream", "NearSingularError", "RankDeficientError", "SvdTriplet",
    "eig_svd", "fro_norm_sq", "gaussian_matrix", "lu_lower_basis", "orthonormal_basis", "sparse_dense_mul",
]
