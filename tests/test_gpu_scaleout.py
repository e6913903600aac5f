"""The scale-out config (BASELINE configs[4]) path: a rating matrix generated
and kept on the device (synth.generate_device -> DeviceSparseRatings), run
through the same QB engine.  Small instances here; tools/scaleout.py runs
the 2e9-rating configuration (or a stated fraction of it)."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cfg():
    from paper_2009_02251_b200.synth import SynthConfig
    return SynthConfig("t4", 3000, 5000, 240_000, 8, 1.2, True)


def test_device_generator_is_canonical_and_seeded(gpu):
    import torch
    from paper_2009_02251_b200 import synth
    A = synth.generate_device(_cfg())
    d = A.device()
    ip = d.A.indptr.cpu().numpy()
    ind = d.A.indices.cpu().numpy()
    val = d.A.values.cpu().numpy()
    assert A.shape == (3000, 5000) and A.nnz == 240_000 == ip[-1]
    deg = np.diff(ip)
    assert deg.min() >= 20
    for r in range(0, 3000, 7):  # distinct, increasing columns per row
        row = ind[ip[r]:ip[r + 1]]
        assert np.all(np.diff(row) > 0)
    assert val.min() >= 0.5 and val.max() <= 5.0 and np.all(val * 2 == np.round(val * 2))
    # popular items (Zipf): the top 1 % of items hold far more than 1 % of ratings
    cnt = np.sort(np.bincount(ind, minlength=5000))[::-1]
    assert cnt[:50].sum() > 0.1 * A.nnz
    B = synth.generate_device(_cfg())
    assert torch.equal(B.device().A.indices, d.A.indices) and torch.equal(B.device().A.values, d.A.values)
    # A.T built on the device matches the host transpose
    H = A.to_host()
    np.testing.assert_array_equal(H.matrix.toarray().T.nonzero()[1][:1000],
                                  d.AT.indices[:1000].cpu().numpy())


def test_device_matrix_qb_matches_oracle(gpu):
    import paper_2009_02251_b200 as P
    from paper_2009_02251_b200 import synth
    from oracle import svdrec_oracle as O
    A = synth.generate_device(_cfg())
    H = A.to_host()
    fro = A.device().frob_sq
    assert fro == pytest.approx(O.frob2(H.matrix), rel=1e-13)
    g = P.qb_pass_blocks(A, 16, 6, P.GaussianStream(2))  # b = 16, p = 2 (the config's pass budget)
    o = O.pass_blocks(H.matrix, 16, 6, O.Stream(2))
    for _ in range(3):
        s, so = next(g), next(o)
        assert abs(s.err - so.err) <= 1e-10 * fro
        sgn = np.where(np.sum(s.B * so.B, axis=1, keepdims=True) < 0, -1.0, 1.0)
        np.testing.assert_allclose(s.B * sgn, so.B, atol=1e-9 * np.sqrt(fro))
