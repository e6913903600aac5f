"""Alg. 4 with wide factors (k > 1024: svdrec_cf_predict_wide) against the
oracle's per-sample loop (reference cf.py:108-143)."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k", [1025, 1500, 2100])
def test_wide_factors_match_oracle(gpu, k):
    import paper_2009_02251_b200 as P
    from paper_2009_02251_b200.cf import predict_many
    from oracle import svdrec_oracle as O
    from scipy import sparse as sp

    rng = np.random.default_rng(k)
    m, n = 300, 700
    dense = np.where(rng.random((m, n)) < 0.05, rng.integers(1, 11, (m, n)) * 0.5, 0.0)
    dense[7] = 0.0  # a user without ratings: global-mean fallback
    M = sp.csr_matrix(dense)
    A = P.SparseRatings(M, 0.5, 5.0)
    T = rng.standard_normal((k, n))
    T[:, 11] = 0.0  # an item with a zero column: fallback
    f = P.LatentFactors.from_matrix(T)
    users = rng.integers(0, m, 3000)
    items = rng.integers(0, n, 3000)
    users[:3] = 7
    items[3:6] = 11
    got = predict_many(A, f, (users, items, np.zeros(3000)))
    ref = O.predict_many(M, T, 0.5, 5.0, users, items)
    np.testing.assert_allclose(got[:, 0], ref[:, 0], rtol=0, atol=1e-10)
    np.testing.assert_allclose(got[:, 1], ref[:, 1], rtol=1e-9, atol=1e-10)
    assert np.array_equal(got[:, 2], ref[:, 2])
