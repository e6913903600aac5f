"""GPU QB engines / drivers / CF against the reference's golden outputs."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _R(csr, lo=None, hi=None):
    import paper_2009_02251_b200 as P
    if lo is None:
        lo, hi = float(csr.data.min()), float(csr.data.max())
    return P.SparseRatings(csr, lo, hi)


def _check_state(prefix, s, g):
    fro = s.frob_sq
    assert s.rank == int(g[f"{prefix}_rank"])
    assert abs(s.err - float(g[f"{prefix}_err"])) <= 1e-10 * fro
    np.testing.assert_allclose(s.Q @ s.B, g[f"{prefix}_QB"], atol=1e-9 * np.sqrt(fro))
    np.testing.assert_allclose(np.linalg.svd(s.B, compute_uv=False), g[f"{prefix}_svals"], rtol=1e-9, atol=1e-10)
    np.testing.assert_allclose(np.einsum("ij,ij->i", s.B, s.B), g[f"{prefix}_rowE"], rtol=1e-7, atol=1e-9 * fro)
    assert np.linalg.norm(s.Q.T @ s.Q - np.eye(s.rank)) <= 1e-10 * np.sqrt(s.rank)


@pytest.mark.parametrize("power", [0, 1, 2])
def test_power_engine_golden(gpu, power):
    import paper_2009_02251_b200 as P
    import inputs
    g = golden("engines")
    _, A = inputs.rand_sparse(120, 150, 0.08, seed=1)
    for blk, s in enumerate(P.qb_power_blocks(_R(A), 15, power, P.GaussianStream(3)), 1):
        _check_state(f"pow{power}_b{blk}", s, g)
        if blk == 3:
            break


@pytest.mark.parametrize("passes", [3, 4, 5, 10])
def test_pass_engine_golden(gpu, passes):
    import paper_2009_02251_b200 as P
    import inputs
    g = golden("engines")
    _, A = inputs.rand_sparse(120, 150, 0.08, seed=1)
    for blk, s in enumerate(P.qb_pass_blocks(_R(A), 15, passes, P.GaussianStream(4)), 1):
        _check_state(f"pass{passes}_b{blk}", s, g)
        if blk == 3:
            break


@pytest.mark.parametrize("passes", [4, 6])
def test_sketch_lookahead_leaves_the_stream_where_the_reference_would(gpu, passes):
    """Alg. 3's sketch matrix of block l + 1 is drawn one block ahead on a side
    stream (rsvd._QbEngine.prefetch_omega).  A consumer that stops after l
    blocks must find the Gaussian stream exactly where the reference leaves
    it -- l draws of (n, b) (reference rsvd.py:178) -- and the blocks must
    equal the ones computed without the look-ahead."""
    import paper_2009_02251_b200 as P
    from paper_2009_02251_b200 import rsvd
    import inputs
    _, A = inputs.rand_sparse(120, 150, 0.08, seed=1)
    R = _R(A)
    n, b = 150, 15
    st = P.GaussianStream(4)
    gen = P.qb_pass_blocks(R, b, passes, st)
    got = [next(gen) for _ in range(2)]
    Bs = [s.B.copy() for s in got]
    gen.close()
    after = st.normal(4, 3)
    ref = P.GaussianStream(4)
    for _ in range(2):
        ref.normal_device(n, b)
    np.testing.assert_array_equal(after, ref.normal(4, 3))
    old, rsvd.LOOKAHEAD = rsvd.LOOKAHEAD, False
    try:
        plain = [s.B.copy() for s, _ in zip(P.qb_pass_blocks(R, b, passes, P.GaussianStream(4)), range(2))]
    finally:
        rsvd.LOOKAHEAD = old
    for x, y in zip(Bs, plain):
        np.testing.assert_array_equal(x, y)


def test_drivers_golden(gpu):
    import paper_2009_02251_b200 as P
    import inputs
    g = golden("drivers")
    _, A = inputs.rand_sparse(100, 140, 0.07, seed=50)
    s = P.fixed_precision_qb(_R(A), 0.6, block_size=12, power=1, seed=5)
    _check_state("fpqb_rand", s, g)
    _, A = inputs.exact_rank(90, 70, 5, seed=51)
    assert P.fixed_precision_qb(_R(A), 1e-6, block_size=20, power=0, seed=0).rank == int(g["fpqb_exact_rank"])
    _, A = inputs.rand_sparse(110, 160, 0.07, seed=70)
    t = P.adaptive_pca(_R(A), P.FrobTolerance(0.6), block_size=12, passes=10, seed=0)
    assert t.k == int(g["apca_tol_k"])
    np.testing.assert_allclose(t.s, g["apca_tol_s"], rtol=1e-10)
    np.testing.assert_allclose(t.reconstruct(), g["apca_tol_recon"], atol=1e-9)
    _, A = inputs.decay(100, 120, 0.7, seed=71)
    t = P.adaptive_pca(_R(A), P.FixedRank(10), block_size=5, passes=10, seed=6)
    np.testing.assert_allclose(t.s, g["apca_rank_s"], rtol=1e-10)
    _, A = inputs.exact_rank(150, 40, 6, seed=72)
    t = P.adaptive_pca(_R(A), P.FrobTolerance(1e-7), block_size=6, passes=10, seed=7)
    assert t.k == int(g["apca_tall_k"])
    np.testing.assert_allclose(t.s, g["apca_tall_s"], rtol=1e-8)
    assert t.u.shape == (150, t.k) and t.v.shape == (40, t.k)
    _, A = inputs.rand_sparse(90, 130, 0.1, seed=73)
    t = P.adaptive_pca(_R(A), lambda st: st.blocks >= 3, block_size=7, passes=6, seed=8)
    assert t.k == int(g["apca_cb_k"])
    np.testing.assert_allclose(t.s, g["apca_cb_s"], rtol=1e-10)
    _, A = inputs.decay(100, 80, 0.7, seed=61)
    t = P.basic_rsvd(_R(A), k=10, power=6, oversample=10, seed=3)
    np.testing.assert_allclose(t.s, g["basic_s"], rtol=1e-10)


def test_config0_drivers_golden(gpu):
    import paper_2009_02251_b200 as P
    from paper_2009_02251_b200 import synth
    g = golden("drivers")
    A = _R(synth.generate(synth.CONFIGS["c0_100k"]), 1.0, 5.0)
    t = P.adaptive_pca(A, P.FrobTolerance(0.5), block_size=10, passes=4, seed=0)
    assert t.k == int(g["c0_apca_k"])
    np.testing.assert_allclose(t.s, g["c0_apca_s"], rtol=1e-9)
    st = P.fixed_precision_qb(A, 0.5, block_size=10, power=1, seed=0)
    assert st.rank == int(g["c0_fpqb_k"])
    np.testing.assert_allclose(np.linalg.svd(st.B, compute_uv=False), g["c0_fpqb_svals"], rtol=1e-9)


def test_cf_golden(gpu):
    import paper_2009_02251_b200 as P
    import inputs
    g = golden("cf")
    train, val, test = inputs.group_model(240, 200, 6, 0.7, seed=0)
    A = _R(train, 1.0, 5.0)
    f, trace = P.auto_latent_factors(A, val, block_size=2, passes=10, seed=0)
    assert f.k == int(g["auto_k"])
    assert [e.k for e in trace] == list(g["auto_trace_k"])
    np.testing.assert_allclose([e.mae for e in trace], g["auto_trace_mae"], rtol=1e-10)
    np.testing.assert_allclose(f.T.T @ f.T, g["auto_T"].T @ g["auto_T"], atol=1e-9)
    p = P.predict_many(A, f, (g["pred_users"], g["pred_items"], np.zeros(len(g["pred_users"]))))
    np.testing.assert_allclose(p[:, 0], g["pred_value"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(p[:, 1], g["pred_raw"], rtol=1e-10, atol=1e-12)
    assert np.array_equal(p[:, 2].astype(bool), g["pred_fallback"])
    one = P.predict_rating(A, f, int(g["pred_users"][0]), int(g["pred_items"][0]))
    assert one.value == pytest.approx(float(g["pred_value"][0]), rel=1e-10, abs=1e-12)
    assert abs(P.evaluate_mae(A, f, test) - float(g["auto_test_mae"])) <= 1e-10


def test_config0_cf_golden(gpu):
    import paper_2009_02251_b200 as P
    from paper_2009_02251_b200 import synth
    g = golden("cf")
    M = synth.generate(synth.CONFIGS["c0_100k"])
    tr, va, te = synth.split_holdout(M, (0.8, 0.1, 0.1), seed=0)
    A = _R(tr, 1.0, 5.0)
    f, trace = P.auto_latent_factors(A, va, block_size=10, passes=4, seed=0)
    assert f.k == int(g["c0_k"])
    np.testing.assert_allclose([e.mae for e in trace], g["c0_trace_mae"], rtol=1e-9)
    p = P.predict_many(A, f, te)
    np.testing.assert_allclose(p[:, 0], g["c0_test_pred"], rtol=1e-9, atol=1e-9)
    mae_, rmse = P.evaluate_errors(A, f, te)
    assert abs(mae_ - float(g["c0_test_mae"])) <= 1e-9
    assert abs(rmse - float(g["c0_test_rmse"])) <= 1e-9 * float(g["c0_test_rmse"])


@pytest.mark.slow
@pytest.mark.parametrize("power", [0, 1, 2])
def test_config1_fixed_precision_golden(gpu, power):
    """BASELINE config 1: 6040x3706 / 1M nnz, eps=0.1, b=20 -> same k, sigma."""
    import paper_2009_02251_b200 as P
    from paper_2009_02251_b200 import synth
    g = golden("c1_fpqb")
    A = _R(synth.generate(synth.CONFIGS["c1_1m"]), 1.0, 5.0)
    st = P.fixed_precision_qb(A, 0.1, block_size=20, power=power, seed=0)
    assert st.rank == int(g[f"p{power}_k"])
    assert st.blocks == int(g[f"p{power}_blocks"])
    sv = np.linalg.svd(st.B, compute_uv=False)
    np.testing.assert_allclose(sv, g[f"p{power}_svals"], rtol=1e-6)
