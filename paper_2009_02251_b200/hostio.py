"""Host -> device upload of large numpy arrays (the rating CSR, held-out
triples).

torch's copy from pageable memory stages through a single-threaded pinned
bounce buffer (~11 GB/s measured on the GPU box for the 217 MB headline
CSR); page-locking the numpy buffers in place costs more than it saves
(cudaHostRegister 21-55 ms for 217 MB).  Here the array is cut into chunks
that a thread pool copies (numpy releases the GIL) into page-locked
buffers from torch's caching host allocator, each chunk's DMA issued as
soon as its copy lands, so host copies and PCIe transfers overlap.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

CHUNK_BYTES = int(os.environ.get("SVDREC_H2D_CHUNK_MB", "8")) << 20
MIN_BYTES = 32 << 20  # smaller arrays: plain copy (a single chunk gains nothing)
_POOL: ThreadPoolExecutor | None = None


def _pool() -> ThreadPoolExecutor:
    global _POOL
    if _POOL is None:
        workers = int(os.environ.get("SVDREC_H2D_THREADS", "0")) or max(2, min(8, (os.cpu_count() or 4) // 2))
        _POOL = ThreadPoolExecutor(max_workers=workers,
                                   thread_name_prefix="svdrec-h2d")
    return _POOL


def to_device(a: np.ndarray, dtype, device) -> torch.Tensor:
    """``torch.from_numpy(a.astype(dtype)).to(device)``, overlapped."""
    a = np.ascontiguousarray(a)
    if a.dtype != dtype:
        a = a.astype(dtype)
    src = torch.from_numpy(a)
    if not torch.cuda.is_available():
        return src.to(device)
    if src.is_pinned():
        # already page-locked (e.g. a view of a pinned torch tensor): one
        # DMA straight from the caller's buffer, stream-ordered; the caller
        # keeps the buffer alive (SparseRatings holds its matrix)
        return src.to(device, non_blocking=True)
    if a.nbytes < MIN_BYTES:
        return src.to(device)
    flat = src.reshape(-1)
    out = torch.empty(flat.shape, dtype=flat.dtype, device=device)
    stage = torch.empty(flat.shape, dtype=flat.dtype, pin_memory=True)
    per = max(1, CHUNK_BYTES // flat.element_size())
    bounds = [(s, min(s + per, flat.numel())) for s in range(0, flat.numel(), per)]
    sv, fv = stage.numpy(), flat.numpy()
    futs = [_pool().submit(np.copyto, sv[s:e], fv[s:e]) for s, e in bounds]
    for (s, e), f in zip(bounds, futs):
        f.result()
        out[s:e].copy_(stage[s:e], non_blocking=True)
    # the stage returns to torch's pinned cache when it goes out of scope;
    # the allocator recorded the copies' stream and reuses the block only
    # after they complete
    return out.reshape(src.shape)
