"""The power steps' basis (rsvd.LU_BASIS): the partial-pivoting LU of the
reference (lu_lower_basis, linalg.py:84-97) and the one-pass shifted
CholeskyQR used by default are both Y times an upper-triangular matrix, so
every block's final Q agrees up to column signs -- projector, B's row
energies, error indicator and the Alg. 5 trace match to rounding."""
from __future__ import annotations

import numpy as np
import pytest

import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(gpu):
    import paper_2009_02251_b200 as P
    return P


def _blocks(P, monkeypatch, basis, A, b, passes, seed, n):
    from paper_2009_02251_b200 import rsvd
    monkeypatch.setattr(rsvd, "LU_BASIS", basis)
    out = []
    for s in P.qb_pass_blocks(A, b, passes, P.GaussianStream(seed)):
        out.append((s.Q.copy(), (s.B * s.B).sum(1), s.err))
        if len(out) == n:
            break
    return out


@pytest.mark.parametrize("passes", [4, 6])
def test_same_blocks_both_bases(P, monkeypatch, passes):
    dense, csr = inputs.rand_sparse(900, 400, 0.05, 71)
    A = P.SparseRatings(csr, 0.5, 5.0)
    frob = float((dense * dense).sum())
    lu = _blocks(P, monkeypatch, "lu", A, 16, passes, 3, 5)
    cq = _blocks(P, monkeypatch, "cqr", A, 16, passes, 3, 5)
    for (q1, e1, r1), (q2, e2, r2) in zip(lu, cq):
        assert np.linalg.norm(q1 @ q1.T - q2 @ q2.T) <= 1e-9
        np.testing.assert_allclose(e1, e2, rtol=1e-9, atol=1e-9 * frob)
        assert abs(r1 - r2) <= 1e-10 * frob


def test_same_alg5_trace_both_bases(P, monkeypatch):
    from paper_2009_02251_b200 import rsvd
    train, (vu, vi, vr), _ = inputs.group_model(300, 240, 6, 0.6, seed=5)
    A = P.SparseRatings(train, 1.0, 5.0)
    val = (vu, vi, vr)
    traces = {}
    for basis in ("lu", "cqr"):
        monkeypatch.setattr(rsvd, "LU_BASIS", basis)
        f, tr = P.auto_latent_factors(A, val, block_size=3, passes=6, seed=2)
        traces[basis] = (f.k, [(e.k, e.mae) for e in tr])
    (k1, t1), (k2, t2) = traces["lu"], traces["cqr"]
    assert k1 == k2 and [k for k, _ in t1] == [k for k, _ in t2]
    np.testing.assert_allclose([m for _, m in t1], [m for _, m in t2], rtol=0, atol=1e-10)
