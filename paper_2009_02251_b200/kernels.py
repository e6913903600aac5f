"""Typed wrappers: torch CUDA tensors in, C-ABI calls, torch tensors out.

Every function here is one (or two) calls into libsvdrec_b200.so on the
current CUDA stream.  Dense operands are 2-d float64 tensors whose rows are
contiguous (``stride(1) == 1``); their ``stride(0)`` is the leading
dimension, so column blocks such as ``Q[:, k0:k1]`` are passed without
copies.  Nothing here synchronises the device.
"""
from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, query, scratch, stream_handle

F64 = torch.float64

# Optional live instrumentation: when ``PROFILE`` is a list, every wrapper
# below appends (name, start_event, end_event, hbm_bytes, gathered_bytes)
# recorded on the launching stream.  ``hbm_bytes`` are the launch's
# compulsory HBM bytes (every input byte read once, every output byte
# written once); ``gathered_bytes`` (gather kernels only) count each
# gathered row every time it is fetched, whether L2, L1 or shared memory
# serves it.  bench.py uses them for the roofline numbers.
PROFILE: list | None = None


class _span:
    __slots__ = ("name", "nbytes", "gathered", "e0")

    def __init__(self, name: str, nbytes: int = 0, gathered: int = 0):
        self.name, self.nbytes, self.gathered, self.e0 = name, nbytes, gathered, None

    def __enter__(self):
        if PROFILE is not None:
            self.e0 = torch.cuda.Event(enable_timing=True)
            self.e0.record()
        return self

    def __exit__(self, *exc):
        if self.e0 is not None and exc[0] is None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            PROFILE.append((self.name, self.e0, e1, self.nbytes, self.gathered))
        return False


def profile_summary(records) -> dict:
    """{name: (calls, total_ms, total_hbm_bytes, total_gathered_bytes)} after a sync."""
    out: dict = {}
    for name, e0, e1, nb, ng in records:
        c, t, b, g = out.get(name, (0, 0.0, 0, 0))
        out[name] = (c + 1, t + e0.elapsed_time(e1), b + nb, g + ng)
    return out


def _mat(t: torch.Tensor, name: str) -> int:
    if t.dim() != 2 or t.dtype != F64 or not t.is_cuda:
        raise ValueError(f"{name}: expected a 2-d float64 CUDA tensor, got {tuple(t.shape)} {t.dtype} {t.device}")
    if t.stride(1) != 1 and t.shape[1] > 1:
        raise ValueError(f"{name}: rows must be contiguous (stride {t.stride()})")
    return max(t.stride(0), t.shape[1], 1)


def new_status(device) -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device=device)


class Mailbox:
    """Small device buffer holding several result fields (float64 vectors
    and uint32 status words) that the host reads back with ONE copy."""

    def __init__(self, device, **fields):
        self.off = {}
        o = 0
        for name, spec in fields.items():
            kind, n = spec
            size = 8 * n if kind == "f8" else 4 * n
            o = (o + 7) // 8 * 8
            self.off[name] = (kind, o, n)
            o += size
        self.buf = torch.zeros((o + 7) // 8 * 8, dtype=torch.uint8, device=device)

    def __getitem__(self, name) -> torch.Tensor:
        kind, o, n = self.off[name]
        view = self.buf[o: o + (8 if kind == "f8" else 4) * n]
        return view.view(F64) if kind == "f8" else view.view(torch.int32)

    def read_async(self) -> "Mailbox":
        """Queue the device->host copy (pinned) on the current stream; get()
        then waits for just that copy, not for later work on the stream."""
        self._host = torch.empty(self.buf.numel(), dtype=torch.uint8, pin_memory=True)
        self._host.copy_(self.buf, non_blocking=True)
        self._ev = torch.cuda.Event()
        self._ev.record()
        return self

    def get(self) -> dict:
        self._ev.synchronize()
        return self._parse(self._host.numpy(), reset=False)

    def read(self) -> dict:
        return self._parse(self.buf.cpu().numpy(), reset=True)

    def _parse(self, host, reset: bool) -> dict:
        out = {}
        dirty = False
        for name, (kind, o, n) in self.off.items():
            a = host[o: o + (8 if kind == "f8" else 4) * n].view(np.float64 if kind == "f8" else np.uint32)
            out[name] = a.copy()
            if kind == "u4" and a.any():
                dirty = True
        if dirty and reset:
            for name, (kind, o, n) in self.off.items():
                if kind == "u4":
                    self[name].zero_()
        return out


def normal_fill(key: tuple[int, int], pos: torch.Tensor, rows: int, cols: int, out: torch.Tensor,
                status: torch.Tensor, row_perm: torch.Tensor | None = None) -> torch.Tensor:
    ld = _mat(out, "normal.out")
    count = rows * cols
    ws, nb = scratch(out.device).get(query("svdrec_normal_workspace_bytes", count))
    with _span("normal", count * 8):
        call("svdrec_normal_fill", key[0], key[1], ptr(pos), count, cols, ptr(row_perm), ptr(out), ld, ws, nb,
             ptr(status), stream_handle())
    return out


def spmm(plan, X: torch.Tensor, Y: torch.Tensor, precision: str = "fp64") -> torch.Tensor:
    """Y = A @ X for the CSR described by ``plan`` (a sparse.DeviceCSR):
    the TMA-gather kernel of csrc/spmm.cu (``precision="fp32"``: its variant
    gathering a float copy of X)."""
    ldx, ldy = _mat(X, "spmm.X"), _mat(Y, "spmm.Y")
    b = X.shape[1]
    if Y.shape[1] != b or X.shape[0] != plan.n or Y.shape[0] != plan.m:
        raise ValueError(f"spmm: shape mismatch A{(plan.m, plan.n)} X{tuple(X.shape)} Y{tuple(Y.shape)}")
    part = plan.partial(b)
    # compulsory HBM bytes: the CSR once (12 B per nonzero + row pointers),
    # X once, Y written once; gathered: one X row (8b B) per nonzero
    nbytes = plan.nnz * 12 + (plan.m + 1) * 8 + plan.n * b * 8 + plan.m * b * 8
    gathered = plan.nnz * 8 * b
    if precision == "fp32" and b % 4 == 0 and b <= 64 and ldy % (2 if b <= 32 else 4) == 0 and plan.nnz:
        # fp32 variant: X stored as float (a rounded copy), fp64 values / accumulation / Y
        X32 = torch.empty(X.shape[0], b, dtype=torch.float32, device=X.device)
        X32.copy_(X)
        nw, wseg, wc, recs = _schedules(plan, query("svdrec_spmm_x32_warps_per_sm", b), b)
        with _span("spmm", plan.nnz * 12 + (plan.m + 1) * 8 + plan.n * b * 4 + plan.m * b * 8, plan.nnz * 4 * b):
            call("svdrec_spmm_x32", plan.nseg, ptr(plan.seg_row), ptr(plan.seg_begin), ptr(plan.seg_end),
                 ptr(plan.seg_slot), ptr(plan.indices), ptr(plan.values), ptr(X32), b, plan.n, ptr(Y), ldy, b,
                 plan.nlong, ptr(plan.long_row), ptr(plan.long_s0), ptr(plan.long_s1), nw, ptr(wseg), ptr(wc),
                 ptr(recs), ptr(plan.slot_long), ptr(plan.long_done), ptr(part), stream_handle())
        return Y
    hc = _hc_rows(plan, b, ldx, ldy)
    hot = 0 if hc else _hot_rows(plan, b, ldx, ldy)
    with _span("spmm", nbytes, gathered):
        if hc:
            _spmm_hc(plan, X, ldx, Y, ldy, b, hc)
        elif hot:
            _spmm_hot(plan, X, ldx, Y, ldy, b, hot)
        else:
            _spmm_tma(plan, X, ldx, Y, ldy, b)
    return Y


# SVDREC_SPMM_HOT=0 keeps A @ X on the TMA-gather kernels (A/B measurements)
SPMM_HOT = os.environ.get("SVDREC_SPMM_HOT", "1") != "0"
# A @ X of a rating matrix (a CSR with a popularity order), config 3, us per
# call, hot / cold chunk kernel (k_spmm_hc) vs TMA pipeline (k_spmm_pipe):
# b = 2 208 vs 245, 4 198 vs 228, 6 220 vs 333, 8 202 vs 230, 10 256 vs 334,
# 12 255 vs 254, 14 297 vs 331, 16 248 vs 255, 18 325 vs 313, 20 311 vs 288,
# 22 387 vs 394, 24 361 vs 326, 26 430 vs 525, 28 396 vs 499, 30 435 vs 527,
# 32 362 vs 494.  The pipeline keeps the widths where it ties or wins (it
# needs no second copy of A); b = 64 runs the register-gather hot-set kernel
# (k_spmm_hot: 554 vs 917 us for the wide TMA kernel; at b = 40, 668 vs 650,
# it is not used).
HC_WIDTHS = frozenset(range(2, 33, 2)) - {12, 18, 20, 24}
HOT_WIDTHS = frozenset({64})


def _hc_rows(plan, b: int, ldx: int, ldy: int) -> int:
    """Hot rows of X the hot / cold chunk kernel stages in shared memory, or
    0 when it does not apply (no popularity order on this CSR, b odd or
    > 32, unaligned rows)."""
    if not SPMM_HOT or getattr(plan, "item_rank", None) is None or ldx % 2 or ldy % 2 or b not in HC_WIDTHS:
        return 0
    return min(int(query("svdrec_spmm_hc_rows", b)), plan.n)


def _spmm_hc(plan, X, ldx, Y, ldy, b, nhot):
    """The hot / cold chunk kernel (csrc/spmm.cu k_spmm_hc) on the packed hot-first copy."""
    nwarp, wchunk, recs, ents, _ = plan.hot_packed(nhot, query("svdrec_spmm_hc_warps_per_sm"))
    call("svdrec_spmm_hc", plan.nseg, ptr(ents), ptr(X), ldx, plan.n, ptr(plan.hot_items), nhot, ptr(Y), ldy, b,
         plan.nlong, ptr(plan.long_row), ptr(plan.long_s0), ptr(plan.long_s1), nwarp, ptr(wchunk), ptr(recs),
         ptr(plan.partial(b)), stream_handle())


def _hot_rows(plan, b: int, ldx: int, ldy: int, widths=None) -> int:
    """Hot rows of X staged in shared memory by the hot-set kernel, or 0
    when it is not used (no popularity order on this CSR, a width where the
    TMA kernels are faster, unaligned rows)."""
    if not SPMM_HOT or getattr(plan, "item_rank", None) is None or ldx % 2 or ldy % 2:
        return 0
    if b not in (HOT_WIDTHS if widths is None else widths) or (b > 32 and (ldx % 4 or ldy % 4)):
        return 0
    if plan.n * (ldx // 2) >= 1 << 31:
        return 0
    return min(int(query("svdrec_spmm_hot_rows", b)), plan.n)


def _spmm_hot(plan, X, ldx, Y, ldy, b, nhot):
    """The hot-set kernel (csrc/spmm.cu k_spmm_hot) on the hot-first copy of this CSR."""
    hidx, hval = plan.hot_encoded(nhot)
    nwarp, wseg = plan.schedule(16)
    call("svdrec_spmm_hot", plan.nseg, ptr(plan.seg_row), ptr(plan.seg_begin), ptr(plan.seg_end), ptr(plan.seg_slot),
         ptr(hidx), ptr(hval), ptr(X), ldx, plan.n, ptr(plan.hot_items), nhot, ptr(Y), ldy, b, plan.nlong,
         ptr(plan.long_row), ptr(plan.long_s0), ptr(plan.long_s1), nwarp, ptr(wseg), ptr(plan.partial(b)),
         stream_handle())


def _schedules(plan, warps_per_sm: int, b: int):
    """(nwarp, warp_seg, warp_chunk, records) for width b: the chunk plan
    for the pipelined kernel (b <= 32), the segment ranges for the wide one."""
    if b <= 32:
        nwarp, wchunk, recs = plan.chunk_schedule(warps_per_sm)
        return nwarp, None, wchunk, recs
    nwarp, wseg = plan.schedule(warps_per_sm)
    return nwarp, wseg, None, None


def _spmm_tma(plan, X, ldx, Y, ldy, b):
    """The TMA-gather kernels (csrc/spmm.cu: k_spmm_pipe for even b <= 32,
    k_spmm_tma for the wide blocks) on one CSR."""
    nwarp, wseg, wchunk, recs = _schedules(plan, query("svdrec_spmm_warps_per_sm", b), b)
    call("svdrec_spmm", plan.nseg, ptr(plan.seg_row), ptr(plan.seg_begin), ptr(plan.seg_end), ptr(plan.seg_slot),
         ptr(plan.indices), ptr(plan.values), ptr(X), ldx, plan.n, ptr(Y), ldy, b, plan.nlong, ptr(plan.long_row),
         ptr(plan.long_s0), ptr(plan.long_s1), nwarp, ptr(wseg), ptr(wchunk), ptr(recs), ptr(plan.slot_long),
         ptr(plan.long_done), ptr(plan.partial(b)), stream_handle())


def gemm_tn(X: torch.Tensor, Y: torch.Tensor, C: torch.Tensor | None = None, alpha: float = 1.0,
            beta: float = 0.0) -> torch.Tensor:
    """C = alpha X.T @ Y + beta C (reduction over the tall dimension)."""
    ldx, ldy = _mat(X, "gemm_tn.X"), _mat(Y, "gemm_tn.Y")
    r, p = X.shape
    q = Y.shape[1]
    if Y.shape[0] != r:
        raise ValueError("gemm_tn: row mismatch")
    if C is None:
        C = torch.empty(p, q, dtype=F64, device=X.device)
    ldc = _mat(C, "gemm_tn.C")
    ws, nb = scratch(X.device).get(query("svdrec_gemm_tn_workspace_bytes", r, p, q))
    with _span("gemm_tn", (r * (p + q) + p * q) * 8):
        call("svdrec_gemm_tn", r, p, q, float(alpha), ptr(X), ldx, ptr(Y), ldy, float(beta), ptr(C), ldc, ws, nb,
             stream_handle())
    return C


def gemm_nn(X: torch.Tensor, Cm: torch.Tensor, Y: torch.Tensor | None = None, alpha: float = 1.0,
            beta: float = 0.0) -> torch.Tensor:
    """Y = alpha X @ Cm + beta Y."""
    ldx, ldc = _mat(X, "gemm_nn.X"), _mat(Cm, "gemm_nn.C")
    r, p = X.shape
    q = Cm.shape[1]
    if Cm.shape[0] != p:
        raise ValueError("gemm_nn: inner mismatch")
    if Y is None:
        Y = torch.empty(r, q, dtype=F64, device=X.device)
    ldy = _mat(Y, "gemm_nn.Y")
    with _span("gemm_nn", (r * (p + 2 * q) + p * q) * 8):
        call("svdrec_gemm_nn", r, p, q, float(alpha), ptr(X), ldx, ptr(Cm), ldc, float(beta), ptr(Y), ldy,
             stream_handle())
    return Y


def sumsq(X: torch.Tensor, colsq: torch.Tensor | None = None, total: torch.Tensor | None = None):
    ldx = _mat(X, "sumsq.X")
    r, q = X.shape
    ws, nb = scratch(X.device).get(query("svdrec_sumsq_workspace_bytes", r, q))
    with _span("sumsq", r * q * 8):
        call("svdrec_sumsq", r, q, ptr(X), ldx, ptr(colsq), ptr(total), ws, nb, stream_handle())
    return colsq, total


def vec_sum(x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    if out is None:
        out = torch.empty(1, dtype=F64, device=x.device)
    ws, nb = scratch(x.device).get(query("svdrec_vec_sum_workspace_bytes", x.numel()))
    call("svdrec_vec_sum", x.numel(), ptr(x), ptr(out), ws, nb, stream_handle())
    return out


def tsqr(A: torch.Tensor, Q: torch.Tensor | None = None, R: torch.Tensor | None = None):
    """Householder TSQR; Q may alias A."""
    lda = _mat(A, "tsqr.A")
    r, b = A.shape
    if Q is None:
        Q = torch.empty(r, b, dtype=F64, device=A.device)
    if R is None:
        R = torch.empty(b, b, dtype=F64, device=A.device)
    ldq = _mat(Q, "tsqr.Q")
    ws, nb = scratch(A.device).get(query("svdrec_tsqr_workspace_bytes", r, b))
    with _span("tsqr", 2 * r * b * 8):
        call("svdrec_tsqr", r, b, ptr(A), lda, ptr(Q), ldq, ptr(R), ws, nb, stream_handle())
    return Q, R


def orth(A: torch.Tensor, Q: torch.Tensor | None = None) -> torch.Tensor:
    """Orthonormal basis (CholeskyQR2 with in-device TSQR fallback); Q may alias A."""
    lda = _mat(A, "orth.A")
    r, b = A.shape
    if Q is None:
        Q = torch.empty(r, b, dtype=F64, device=A.device)
    ldq = _mat(Q, "orth.Q")
    ws, nb = scratch(A.device).get(query("svdrec_orth_workspace_bytes", r, b))
    with _span("orth", 2 * r * b * 8):
        call("svdrec_orth", r, b, ptr(A), lda, ptr(Q), ldq, ws, nb, stream_handle())
    return Q


def gram(Y: torch.Tensor, G: torch.Tensor | None = None) -> torch.Tensor:
    """Full symmetric b x b Gram Y.T Y of (this rank's rows of) Y."""
    r, b = Y.shape
    ldy = _mat(Y, "gram.Y") if r else b
    if G is None:
        G = torch.empty(b, b, dtype=F64, device=Y.device)
    ws, nb = scratch(Y.device).get(query("svdrec_gram_workspace_bytes", r, b))
    with _span("gram", r * b * 8):
        call("svdrec_gram", r, b, ptr(Y) if r else None, ldy, ptr(G), ws, nb, stream_handle())
    return G


def chol_apply(G: torch.Tensor, Y: torch.Tensor, Q: torch.Tensor | None = None, shift_rel: float = 0.0,
               status: torch.Tensor | None = None) -> torch.Tensor:
    """Q = Y R^-1 with R = chol(G + shift_rel trace(G) I); Q may alias Y."""
    r, b = Y.shape
    if Q is None:
        Q = torch.empty(r, b, dtype=F64, device=Y.device)
    ldy = _mat(Y, "chol_apply.Y") if r else b
    ldq = _mat(Q, "chol_apply.Q") if r else b
    ldg = _mat(G, "chol_apply.G")
    if status is None:
        status = _orth_status(Y.device)
    ws, nb = scratch(Y.device).get(query("svdrec_chol_apply_workspace_bytes", r, b))
    with _span("chol_apply", 2 * r * b * 8):
        call("svdrec_chol_apply", r, b, ptr(G), ldg, float(shift_rel), ptr(Y) if r else None, ldy,
             ptr(Q) if r else None, ldq, ptr(status), ws, nb, stream_handle())
    return Q


_ORTH_STATUS: dict = {}


def _orth_status(device) -> torch.Tensor:
    """Discarded status word for orthonormalisation calls (Householder QR
    in the reference never fails on rank deficiency)."""
    key = torch.device(device).index
    st = _ORTH_STATUS.get(key)
    if st is None:
        st = _ORTH_STATUS[key] = new_status(device)
    return st


def lu_lower(A: torch.Tensor, status: torch.Tensor, udiag: torch.Tensor | None = None) -> torch.Tensor:
    """In-place P.L of partial-pivoting LU; returns U's diagonal (device)."""
    lda = _mat(A, "lu.A")
    r, b = A.shape
    if udiag is None:
        udiag = torch.empty(b, dtype=F64, device=A.device)
    ws, nb = scratch(A.device).get(query("svdrec_lu_workspace_bytes", r, b))
    with _span("lu", 2 * r * b * 8):
        call("svdrec_lu_lower", r, b, ptr(A), lda, ptr(udiag), ws, nb, ptr(status), stream_handle())
    return udiag


def syev(G: torch.Tensor, status: torch.Tensor, V0: torch.Tensor | None = None):
    """Eigen-decomposition of a symmetric PSD k x k: (w ascending, V columns).

    ``V0`` (k x k orthonormal columns) warm-starts the Jacobi sweeps."""
    ldg = _mat(G, "syev.G")
    ldv0 = _mat(V0, "syev.V0") if V0 is not None else 0
    k = G.shape[0]
    w = torch.empty(k, dtype=F64, device=G.device)
    V = torch.empty(k, k, dtype=F64, device=G.device)
    ws, nb = scratch(G.device).get(query("svdrec_syev_workspace_bytes", k))
    with _span("syev", 2 * k * k * 8):
        call("svdrec_syev", k, ptr(G), ldg, ptr(V0), ldv0, ptr(w), ptr(V), k, ws, nb, ptr(status),
             stream_handle())
    return w, V


def gesvj(A: torch.Tensor, status: torch.Tensor):
    """One-sided Jacobi SVD of a tall block: (s descending, U, V)."""
    lda = _mat(A, "gesvj.A")
    rows, k = A.shape
    s = torch.empty(k, dtype=F64, device=A.device)
    U = torch.empty(rows, k, dtype=F64, device=A.device)
    V = torch.empty(k, k, dtype=F64, device=A.device)
    ws, nb = scratch(A.device).get(query("svdrec_gesvj_workspace_bytes", rows, k))
    call("svdrec_gesvj", rows, k, ptr(A), lda, ptr(s), ptr(U), k, ptr(V), k, ws, nb, ptr(status), stream_handle())
    return s, U, V


def cf_normalize(Tt: torch.Tensor):
    ldt = _mat(Tt, "cf.Tt")
    n, k = Tt.shape
    Tn = torch.empty(n, k, dtype=F64, device=Tt.device)
    norm = torch.empty(n, dtype=F64, device=Tt.device)
    with _span("cf_normalize", 2 * n * k * 8):
        call("svdrec_cf_normalize", n, k, ptr(Tt), ldt, ptr(Tn), k, ptr(norm), stream_handle())
    return Tn, norm


def cf_normalize_pair(X: torch.Tensor, Y: torch.Tensor):
    """(Xn, Yn, n) with n_l = sqrt(x_l . y_l) (metric-mode item factors)."""
    ldx, ldy = _mat(X, "cf.X"), _mat(Y, "cf.Y")
    n, k = X.shape
    Xn = torch.empty(n, k, dtype=F64, device=X.device)
    Yn = torch.empty(n, k, dtype=F64, device=X.device)
    norm = torch.empty(n, dtype=F64, device=X.device)
    with _span("cf_normalize", 4 * n * k * 8):
        call("svdrec_cf_normalize_pair", n, k, ptr(X), ldx, ptr(Y), ldy, ptr(Xn), ptr(Yn), k, ptr(norm),
             stream_handle())
    return Xn, Yn, norm


def inv_sqrt(G: torch.Tensor, status: torch.Tensor, iters: torch.Tensor | None = None) -> torch.Tensor:
    """G^(-1/2) by coupled Newton-Schulz (device); flags NS_CHECK if unsure."""
    ldg = _mat(G, "inv_sqrt.G")
    k = G.shape[0]
    Z = torch.empty(k, k, dtype=F64, device=G.device)
    ws, nb = scratch(G.device).get(query("svdrec_inv_sqrt_workspace_bytes", k))
    with _span("inv_sqrt", 2 * k * k * 8):
        call("svdrec_inv_sqrt", k, ptr(G), ldg, ptr(Z), k, ws, nb, ptr(status), ptr(iters), stream_handle())
    return Z


def cf_predict(groups: torch.Tensor, users: torch.Tensor, items: torch.Tensor, csr, Yn: torch.Tensor,
               Xn: torch.Tensor, norm: torch.Tensor, gmean: float, lo: float, hi: float, plan,
               precision: str = "fp64", group_users: torch.Tensor | None = None):
    """Alg. 4 over user-grouped samples.  ``csr`` is a sparse.DeviceCSR (its
    ranked copy is used); ``plan`` is a cf.WorkPlan (work items, per-group
    chunk info, completion counters, counter).  ``precision="fp32"`` stores
    the gathered item rows as float (fp64 accumulation)."""
    ldn = _mat(Xn, "cf.Xn")
    if Xn.shape != Yn.shape:
        raise ValueError("cf_predict: Xn and Yn must share their shape")
    if precision not in ("fp64", "fp32"):
        raise ValueError(f"precision must be 'fp64' or 'fp32', not {precision!r}")
    rind, rval, order = csr.ranked()
    n, k = Yn.shape
    f32 = precision == "fp32" and k <= 1024  # the wide kernel gathers fp64 rows
    # rank order + a zero row; rows zero-padded to a 16-B multiple (vector loads)
    ldy = (k + 3) // 4 * 4 if f32 else (k + 1) // 2 * 2
    Yr = torch.empty(n + 1, ldy, dtype=torch.float32 if f32 else F64, device=Yn.device)
    Yr[n].zero_()
    if ldy > k:
        Yr[:, k:].zero_()
    if not f32 and ldy == k and Yn.is_contiguous():
        torch.index_select(Yn, 0, order, out=Yr[:n])
    else:
        Yr[:n, :k].copy_(Yn.index_select(0, order))
    ns = users.shape[0]
    val = torch.empty(ns, dtype=F64, device=Yn.device)
    raw = torch.empty(ns, dtype=F64, device=Yn.device)
    fb = torch.empty(ns, dtype=torch.uint8, device=Yn.device)
    # compulsory HBM bytes: the scored users' ranked CSR rows once (12 B per
    # rating), the two n x k item tables once, per sample its item id, norm
    # and the three outputs; gathered: one item row per streamed rating and
    # one Xn row per sample
    es = 4 if f32 else 8
    rated = getattr(plan, "rated", 0)
    nbytes = rated * 12 + n * k * (es + 8) + ns * (4 + 8 + 17)
    gathered = rated * es * k + ns * 8 * k
    if k > 1024:  # wide factors: the k-tiled kernel (fp64 rows)
        with _span("cf_predict", nbytes, gathered):
            call("svdrec_cf_predict_wide", groups.numel() - 1, ptr(groups), ptr(group_users), ptr(csr.indptr),
                 ptr(items), ptr(rind), ptr(rval), k, ptr(Yr), ldy, ptr(Xn), ldn, ptr(norm), float(gmean), float(lo),
                 float(hi), ptr(val), ptr(raw), ptr(fb), stream_handle())
        return val, raw, fb
    common = (plan.nwork, ptr(plan.start), ptr(plan.meta), ptr(items), ptr(rind), ptr(rval), k)
    tail = (ptr(norm), float(gmean), float(lo), float(hi), n, ptr(plan.done), plan.ndone, ptr(plan.partial(k)),
            ptr(plan.counter), ptr(val), ptr(raw), ptr(fb), stream_handle())
    with _span("cf_predict", nbytes, gathered):
        if f32:
            call("svdrec_cf_predict_f32", *common, ptr(Yr), ldy, ptr(Xn), ldn, *tail)
        else:
            call("svdrec_cf_predict", *common, ptr(Yr), ldy, ptr(Xn), ldn, *tail)
    return val, raw, fb


def cf_plan_scan(gd, order, chunk, first, slot0, done_idx, stats):
    """Scoring work plan, step 1 (csrc/cf.cu k_plan_scan)."""
    call("svdrec_cf_plan_scan", gd.numel(), ptr(gd), ptr(order), int(chunk), ptr(first), ptr(slot0),
         ptr(done_idx), ptr(stats), stream_handle())


def cf_plan_emit(gd, order, first, slot0, done_idx, group_start, row_start, chunk, start, meta):
    """Scoring work plan, step 2 (csrc/cf.cu k_plan_emit): start / meta records."""
    call("svdrec_cf_plan_emit", gd.numel(), ptr(gd), ptr(order), ptr(first), ptr(slot0), ptr(done_idx),
         ptr(group_start), ptr(row_start), int(chunk), ptr(start), ptr(meta), stream_handle())


def rank_rows(indptr: torch.Tensor, indices: torch.Tensor, values: torch.Tensor, n: int, rank: torch.Tensor):
    """(ranked indices, values): columns relabelled by ``rank`` (int32, n
    entries) and every row ordered by rank (csrc/ingest.cu k_rank_rows)."""
    nnz = int(indices.numel())
    out_idx = torch.empty(nnz, dtype=torch.int32, device=indices.device)
    out_val = torch.empty(nnz, dtype=torch.float64, device=indices.device)
    if nnz:
        with _span("rank_rows", nnz * 24 + n * 4):
            call("svdrec_rank_rows", indptr.numel() - 1, n, ptr(indptr), ptr(indices), ptr(values),
                 ptr(rank.to(torch.int32).contiguous()), ptr(out_idx), ptr(out_val), stream_handle())
    return out_idx, out_val


def scan_i64(x: torch.Tensor, out: torch.Tensor | None = None, total: torch.Tensor | None = None) -> torch.Tensor:
    """Exclusive scan of an int64 vector (csrc/ingest.cu)."""
    x = x.to(torch.int64).contiguous()
    if out is None:
        out = torch.empty_like(x)
    call("svdrec_scan_i64", x.numel(), ptr(x), ptr(out), ptr(total), stream_handle())
    return out


def csr_transpose(indptr: torch.Tensor, indices: torch.Tensor, values: torch.Tensor, n_out: int,
                  perm: torch.Tensor | None = None, relabel: bool = False):
    """Stable counting-sort transpose (csrc/ingest.cu): returns (indptr,
    indices, values) of the n_out-row transpose, the input rows taken in
    the order ``perm`` (default: 0..m-1); entries carry the input row index,
    or its position in ``perm`` when ``relabel``."""
    dev = indptr.device
    m = indptr.numel() - 1
    if perm is None:
        pptr = indptr
    else:
        pptr = torch.zeros(m + 1, dtype=torch.int64, device=dev)
        if m:
            torch.cumsum((indptr[1:] - indptr[:-1])[perm], 0, out=pptr[1:])
        perm = perm.to(torch.int32).contiguous()
    nnz = int(indices.numel())
    out_ptr = torch.empty(n_out + 1, dtype=torch.int64, device=dev)
    out_idx = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    out_val = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    if nnz == 0 or n_out == 0:
        out_ptr.zero_()
        return out_ptr, out_idx[:nnz], out_val[:nnz]
    sb = int(query("svdrec_csr_transpose_scratch", n_out)) + 2 * ((nnz * 4 + 255) // 256 * 256)
    ws = torch.empty(sb, dtype=torch.uint8, device=dev)  # transient (allocator-cached)
    with _span("csr_transpose", nnz * (12 * 3 + 16)):
        call("svdrec_csr_transpose", m, n_out, nnz, ptr(indptr), ptr(indices), ptr(values),
             ptr(perm) if perm is not None else None, ptr(pptr), int(relabel), ptr(out_ptr), ptr(out_idx),
             ptr(out_val), ptr(ws), sb, stream_handle())
    return out_ptr, out_idx, out_val


def err_sum(pred: torch.Tensor, truth: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Device (sum |p - t|, sum (p - t)^2)."""
    if out is None:
        out = torch.empty(2, dtype=F64, device=pred.device)
    n = pred.shape[0]
    ws, nb = scratch(pred.device).get(query("svdrec_err_sum_workspace_bytes", n))
    call("svdrec_err_sum", n, ptr(pred), ptr(truth), ptr(out), ws, nb, stream_handle())
    return out


def count_overlap(users: torch.Tensor, items: torch.Tensor, csr) -> torch.Tensor:
    cnt = torch.empty(1, dtype=torch.int32, device=users.device)
    call("svdrec_count_overlap", users.shape[0], ptr(users), ptr(items), ptr(csr.indptr), ptr(csr.indices),
         ptr(cnt), stream_handle())
    return cnt


def check_status(status: torch.Tensor) -> int:
    """Synchronising read of a status word (then cleared)."""
    v = int(status.item())
    if v:
        status.zero_()
    return v


__all__ = [n for n in dir() if not n.startswith("_")] + ["_lib"]
