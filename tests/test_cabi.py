"""The C-ABI library loads without a GPU and exports every declared symbol."""
from __future__ import annotations

import re

import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "svdrec_b200.h"


def declared():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(svdrec_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared()
    assert "svdrec_normal_fill" in names and "svdrec_spmm" in names and "svdrec_tsqr" in names
    assert len(names) >= 20


def test_library_exports_every_declared_symbol():
    from paper_2009_02251_b200 import _lib

    if not _lib.LIB_PATH.is_file():
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = _lib.load_library()
    for name in declared():
        assert hasattr(lib, name), name
    assert set(declared()) == set(_lib.SIGNATURES), "ctypes table out of sync with the header"
    assert lib.svdrec_abi_version() == 1


def test_workspace_queries_without_gpu():
    from paper_2009_02251_b200 import _lib

    if not _lib.LIB_PATH.is_file():
        pytest.skip("library not built")
    lib = _lib.load_library()
    assert lib.svdrec_normal_workspace_bytes(535_000) > 0
    assert lib.svdrec_tsqr_workspace_bytes(138_493, 20) > 138_493 * 20 * 8
    assert lib.svdrec_gemm_tn_workspace_bytes(138_493, 400, 20) > 0


def test_no_cpu_fallback():
    """Without a device the product path raises instead of computing."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_2009_02251_b200 as P

    with pytest.raises(P.ExtensionUnavailable):
        P.orthonormal_basis(np.eye(3))
    with pytest.raises(P.ExtensionUnavailable):
        P.GaussianStream(0)
