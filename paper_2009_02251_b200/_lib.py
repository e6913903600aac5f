"""ctypes binding of libsvdrec_b200.so (the C ABI in include/svdrec_b200.h).

This is the same binding a maintainer of the reference would add (see
INTEGRATION.md): plain pointers, sizes and a stream handle.  There is no
fallback: if the shared library or a CUDA device is missing, every call
raises :class:`ExtensionUnavailable`.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import torch

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libsvdrec_b200.so"

STATUS_ZERO_PIVOT = 1
STATUS_NEAR_SINGULAR = 2
STATUS_STREAM_SHORT = 4
STATUS_NO_CONVERGE = 8
STATUS_NS_CHECK = 16

_i64, _i32, _u64, _f64, _sz, _p = C.c_int64, C.c_int32, C.c_uint64, C.c_double, C.c_size_t, C.c_void_p

# name -> (restype, argtypes)
SIGNATURES = {
    "svdrec_abi_version": (C.c_int, []),
    "svdrec_last_error": (C.c_char_p, []),
    "svdrec_device_sm_count": (C.c_int, []),
    "svdrec_launch_count": (C.c_longlong, []),
    "svdrec_normal_workspace_bytes": (_sz, [_i64]),
    "svdrec_normal_fill": (C.c_int, [_u64, _u64, _p, _i64, _i64, _p, _p, _i64, _p, _sz, _p, _p]),
    "svdrec_spmm": (C.c_int, [_i64, _p, _p, _p, _p, _p, _p, _p, _i64, _i64, _p, _i64, _i32, _i64, _p, _p, _p, _i64, _p, _p, _p, _p,
                              _p, _p, _p]),
    "svdrec_chunk_plan": (C.c_int, [_i64, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "svdrec_spmm_hc_warps_per_sm": (C.c_int, []),
    "svdrec_spmm_hc_rows": (C.c_int, [_i32]),
    "svdrec_spmm_hot_pack": (C.c_int, [_i64, _p, _p, _p, _p, _i32, _p, _p, _p]),
    "svdrec_spmm_hc": (C.c_int, [_i64, _p, _p, _i64, _i64, _p, _i32, _p, _i64, _i32, _i64, _p, _p, _p, _i64, _p, _p, _p,
                                 _p]),
    "svdrec_warp_chunks": (C.c_int, [_i64, _p, _i64, _p, _p, _p]),
    "svdrec_spmm_warps_per_sm": (C.c_int, [_i32]),
    "svdrec_spmm_hot_rows": (C.c_int, [_i32]),
    "svdrec_spmm_hot_partition": (C.c_int, [_i64, _p, _p, _p, _p, _i32, _p, _p, _p]),
    "svdrec_spmm_hot": (C.c_int, [_i64, _p, _p, _p, _p, _p, _p, _p, _i64, _i64, _p, _i32, _p, _i64, _i32, _i64, _p, _p,
                                  _p, _i64, _p, _p, _p]),
    "svdrec_spmm_x32_warps_per_sm": (C.c_int, [_i32]),
    "svdrec_spmm_x32": (C.c_int, [_i64, _p, _p, _p, _p, _p, _p, _p, _i64, _i64, _p, _i64, _i32, _i64, _p, _p, _p, _i64, _p, _p,
                                  _p, _p, _p, _p, _p]),
    "svdrec_gemm_tn_workspace_bytes": (_sz, [_i64, _i64, _i64]),
    "svdrec_gemm_tn": (C.c_int, [_i64, _i64, _i64, _f64, _p, _i64, _p, _i64, _f64, _p, _i64, _p, _sz, _p]),
    "svdrec_gemm_nn": (C.c_int, [_i64, _i64, _i64, _f64, _p, _i64, _p, _i64, _f64, _p, _i64, _p]),
    "svdrec_sumsq_workspace_bytes": (_sz, [_i64, _i64]),
    "svdrec_sumsq": (C.c_int, [_i64, _i64, _p, _i64, _p, _p, _p, _sz, _p]),
    "svdrec_vec_sum_workspace_bytes": (_sz, [_i64]),
    "svdrec_vec_sum": (C.c_int, [_i64, _p, _p, _p, _sz, _p]),
    "svdrec_tsqr_workspace_bytes": (_sz, [_i64, _i32]),
    "svdrec_tsqr": (C.c_int, [_i64, _i32, _p, _i64, _p, _i64, _p, _p, _sz, _p]),
    "svdrec_orth_workspace_bytes": (_sz, [_i64, _i32]),
    "svdrec_orth": (C.c_int, [_i64, _i32, _p, _i64, _p, _i64, _p, _sz, _p]),
    "svdrec_gram_workspace_bytes": (_sz, [_i64, _i32]),
    "svdrec_gram": (C.c_int, [_i64, _i32, _p, _i64, _p, _p, _sz, _p]),
    "svdrec_chol_apply_workspace_bytes": (_sz, [_i64, _i32]),
    "svdrec_chol_apply": (C.c_int, [_i64, _i32, _p, _i64, _f64, _p, _i64, _p, _i64, _p, _p, _sz, _p]),
    "svdrec_lu_workspace_bytes": (_sz, [_i64, _i32]),
    "svdrec_lu_fast_path": (C.c_int, [_i64, _i32]),
    "svdrec_lu_lower": (C.c_int, [_i64, _i32, _p, _i64, _p, _p, _sz, _p, _p]),
    "svdrec_syev_workspace_bytes": (_sz, [_i32]),
    "svdrec_syev": (C.c_int, [_i32, _p, _i64, _p, _i64, _p, _p, _i64, _p, _sz, _p, _p]),
    "svdrec_gesvj_workspace_bytes": (_sz, [_i64, _i32]),
    "svdrec_gesvj": (C.c_int, [_i64, _i32, _p, _i64, _p, _p, _i64, _p, _i64, _p, _sz, _p, _p]),
    "svdrec_cf_normalize": (C.c_int, [_i64, _i32, _p, _i64, _p, _i64, _p, _p]),
    "svdrec_cf_normalize_pair": (C.c_int, [_i64, _i32, _p, _i64, _p, _i64, _p, _p, _i64, _p, _p]),
    "svdrec_cf_predict": (C.c_int, [_i64, _p, _p, _p, _p, _p, _i32, _p, _i64, _p, _i64, _p, _f64, _f64, _f64,
                                    _i32, _p, _i64, _p, _p, _p, _p, _p, _p]),
    "svdrec_cf_predict_f32": (C.c_int, [_i64, _p, _p, _p, _p, _p, _i32, _p, _i64, _p, _i64, _p, _f64, _f64, _f64,
                                        _i32, _p, _i64, _p, _p, _p, _p, _p, _p]),
    "svdrec_cf_predict_wide": (C.c_int, [_i64, _p, _p, _p, _p, _p, _p, _i32, _p, _i64, _p, _i64, _p, _f64, _f64,
                                         _f64, _p, _p, _p, _p]),
    "svdrec_cf_plan_scan": (C.c_int, [_i64, _p, _p, _i32, _p, _p, _p, _p, _p]),
    "svdrec_cf_plan_emit": (C.c_int, [_i64, _p, _p, _p, _p, _p, _p, _p, _i32, _p, _p, _p]),
    "svdrec_csr_transpose_scratch": (_i64, [_i64]),
    "svdrec_rank_rows": (C.c_int, [_i64, _i32, _p, _p, _p, _p, _p, _p, _p]),
    "svdrec_scan_i64": (C.c_int, [_i64, _p, _p, _p, _p]),
    "svdrec_seg_plan_count": (C.c_int, [_i64, _p, _i32, _p, _p, _p, _p, _p]),
    "svdrec_seg_plan_emit": (C.c_int, [_i64, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "svdrec_warp_plan": (C.c_int, [_i64, _p, _p, _i64, _i32, _p, _p, _p]),
    "svdrec_csr_transpose": (C.c_int, [_i64, _i64, _i64, _p, _p, _p, _p, _p, _i32, _p, _p, _p, _p, _i64, _p]),
    "svdrec_inv_sqrt_workspace_bytes": (_sz, [_i32]),
    "svdrec_inv_sqrt": (C.c_int, [_i32, _p, _i64, _p, _i64, _p, _sz, _p, _p, _p]),
    "svdrec_err_sum_workspace_bytes": (_sz, [_i64]),
    "svdrec_err_sum": (C.c_int, [_i64, _p, _p, _p, _p, _sz, _p]),
    "svdrec_count_overlap": (C.c_int, [_i64, _p, _p, _p, _p, _p, _p]),
}


class ExtensionUnavailable(RuntimeError):
    """The CUDA extension could not be used (no library or no device)."""


class KernelError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


_LIB = None


def load_library(path: Path | None = None) -> C.CDLL:
    """dlopen the library and declare every exported symbol (no GPU needed)."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path or os.environ.get("SVDREC_B200_LIB", LIB_PATH))
    if not p.is_file():
        raise ExtensionUnavailable(
            f"{p} not built; run `python -c 'import __graft_entry__ as g; g.build()'` (make -C {_HERE / 'csrc'})")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _LIB = lib
    return lib


def load() -> C.CDLL:
    """Library + a usable CUDA device, or ExtensionUnavailable."""
    lib = load_library()
    if not torch.cuda.is_available():
        raise ExtensionUnavailable("no CUDA device: the svdrec_b200 path has no CPU fallback")
    return lib


def call(name: str, *args) -> int:
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.svdrec_last_error().decode(errors="replace")
        raise KernelError(f"{name} failed ({rc}): {msg}")
    return rc


def query(name: str, *args) -> int:
    return int(getattr(load(), name)(*args))


def ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    return C.c_void_p(t.data_ptr())


def stream_handle(stream: torch.cuda.Stream | None = None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class Scratch:
    """Grow-only device scratch, reused by successive stream-ordered calls."""

    def __init__(self, device):
        self.device = torch.device(device)
        self.buf = torch.empty(0, dtype=torch.uint8, device=self.device)

    def get(self, nbytes: int) -> tuple[C.c_void_p, int]:
        nbytes = max(int(nbytes), 256)
        if self.buf.numel() < nbytes:
            self.buf = torch.empty(int(nbytes * 1.25) + 4096, dtype=torch.uint8, device=self.device)
        return C.c_void_p(self.buf.data_ptr()), self.buf.numel()


_SCRATCH: dict = {}


def scratch(device=None) -> Scratch:
    """Scratch for (device, current stream): calls on one stream are ordered,
    so they can share it; concurrent streams each get their own."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    key = (idx, torch.cuda.current_stream(idx).cuda_stream)
    s = _SCRATCH.get(key)
    if s is None:
        s = _SCRATCH[key] = Scratch(torch.device("cuda", idx))
    return s
