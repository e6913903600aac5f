"""Behavioural contract of the drop-in API on the GPU path.

The reference's own test suite (pkg/tests/test_cf.py, test_linalg.py,
test_rsvd.py) pins behaviours beyond numerics: fallbacks, clamping, error
types, validation, determinism, stopping rules.  These tests exercise the
same behaviours through this package (every numeric call goes through the
C ABI / CUDA kernels), with inputs built here and the CPU oracle
(oracle/svdrec_oracle.py) as the numeric checker.
"""
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(gpu):
    import paper_2009_02251_b200 as P
    return P


def _ratings(P, m, n, density, seed, lo=0.5, hi=5.0):
    import inputs
    dense, M = inputs.rand_sparse(m, n, density, seed)
    return dense, P.SparseRatings(M, lo, hi)


def _unit(*deg):
    r = np.deg2rad(np.asarray(deg, dtype=np.float64))
    return np.vstack([np.cos(r), np.sin(r)])


def _tiny(P):
    """2 users x 3 items; user 0 rated item 0 (5.0) and item 1 (1.0)."""
    return P.SparseRatings.from_coo([0, 0], [0, 1], [5.0, 1.0], shape=(2, 3), bounds=(1.0, 5.0))


# ---------------------------------------------------------------------------
# CF: latent factors and Alg. 4 predictions

def test_latent_factors_shape_and_descending_energy(P):
    _, A = _ratings(P, 80, 60, 0.15, 0)
    st = P.fixed_precision_qb(A, tol=0.7, block_size=8, power=1, seed=1)
    f = P.latent_from_qb(st)
    assert f.T.shape == (st.rank, 60) and f.k == st.rank
    e = np.sum(f.T ** 2, axis=1)
    assert np.all(np.diff(e) <= 1e-9 * e[0])


def test_unrated_items_have_zero_factor_columns(P):
    dense, _ = _ratings(P, 50, 40, 0.2, 2)
    dense[:, [7, 23]] = 0.0
    A = P.SparseRatings.from_dense(dense, bounds=(0.5, 5.0))
    f = P.latent_from_qb(P.fixed_precision_qb(A, tol=0.8, block_size=5, seed=3))
    assert f.col_norms[7] == 0.0 and f.col_norms[23] == 0.0 and np.any(f.col_norms > 0)


def test_empty_factorization_rejected(P):
    A = P.SparseRatings.from_dense(np.zeros((6, 5)))
    st = P.fixed_precision_qb(A, tol=0.5, block_size=2)
    assert st.rank == 0
    with pytest.raises(ValueError):
        P.latent_from_qb(st)


def test_factor_gram_spectrum_is_b_spectrum_squared(P):
    _, A = _ratings(P, 60, 45, 0.2, 4)
    st = P.fixed_precision_qb(A, tol=0.6, block_size=6, seed=5)
    f = P.latent_from_qb(st)
    wt = np.linalg.eigvalsh(f.T.T @ f.T)
    wb = np.linalg.eigvalsh(st.B.T @ st.B)
    keep = wb > 1e-9 * wb.max()
    np.testing.assert_allclose(np.sort(wt[keep]) ** 2, np.sort(wb[keep]), rtol=1e-8)


def test_predictions_match_bruteforce_oracle(P):
    from oracle import svdrec_oracle as O
    _, A = _ratings(P, 60, 50, 0.15, 6)
    f = P.latent_from_qb(P.fixed_precision_qb(A, tol=0.6, block_size=6, seed=7))
    T = f.T
    norms = np.linalg.norm(T, axis=0)
    g = float(A.matrix.data.mean())
    rng = np.random.default_rng(8)
    for _ in range(40):
        u, i = int(rng.integers(0, 60)), int(rng.integers(0, 50))
        got = P.predict_rating(A, f, u, i)
        val, raw, fb = O.predict(A.matrix, T, norms, 0.5, 5.0, u, i, g)
        assert got.fallback == fb
        assert got.raw == pytest.approx(raw, rel=1e-10, abs=1e-12)
        assert got.value == pytest.approx(val, rel=1e-10, abs=1e-12)


def test_prediction_is_clamped(P):
    pred = P.predict_rating(_tiny(P), P.LatentFactors.from_matrix(_unit(30, 120, 0)), 0, 2)
    assert pred.raw > 5.0 and pred.value == 5.0 and not pred.fallback


def test_cancelling_weights_fall_back_to_user_mean(P):
    pred = P.predict_rating(_tiny(P), P.LatentFactors.from_matrix(_unit(60, 120, 0)), 0, 2)
    assert pred.fallback and pred.value == pytest.approx(3.0)


def test_zero_norm_target_falls_back(P):
    T = _unit(30, 120, 0)
    T[:, 2] = 0.0
    pred = P.predict_rating(_tiny(P), P.LatentFactors.from_matrix(T), 0, 2)
    assert pred.fallback and pred.value == pytest.approx(3.0)


def test_user_without_ratings_gets_global_mean(P):
    pred = P.predict_rating(_tiny(P), P.LatentFactors.from_matrix(_unit(30, 120, 0)), 1, 2)
    assert pred.fallback and pred.value == pytest.approx(3.0)


def test_zero_norm_rated_items_are_skipped(P):
    T = _unit(30, 10, 0)
    T[:, 0] = 0.0
    pred = P.predict_rating(_tiny(P), P.LatentFactors.from_matrix(T), 0, 2)
    assert not pred.fallback and pred.value == pytest.approx(1.0)


def test_prediction_bounds_checking(P):
    A = _tiny(P)
    f = P.LatentFactors.from_matrix(_unit(30, 120, 0))
    with pytest.raises(IndexError):
        P.predict_rating(A, f, 2, 0)
    with pytest.raises(IndexError):
        P.predict_rating(A, f, 0, 3)
    with pytest.raises(ValueError):
        P.predict_rating(A, P.LatentFactors.from_matrix(_unit(30, 120)), 0, 1)


@pytest.mark.parametrize("scale", [1e-6, 3.7e-2, 1.0, 41.0, 1e6])
def test_prediction_invariant_under_positive_scaling(P, scale):
    A = _tiny(P)
    base = _unit(25, 110, 5)
    p0 = P.predict_rating(A, P.LatentFactors.from_matrix(base), 0, 2)
    p1 = P.predict_rating(A, P.LatentFactors.from_matrix(base * scale), 0, 2)
    assert p1.raw == pytest.approx(p0.raw, rel=1e-12, abs=1e-12) and p1.fallback == p0.fallback


def test_mae_values_and_validation(P):
    assert P.mae([1.0, 2.0, 3.0], [2.0, 2.0, 1.0]) == pytest.approx(1.0)
    assert P.mae([0.5, -3.0], [0.5, -3.0]) == 0.0
    with pytest.raises(ValueError):
        P.mae([], [])
    with pytest.raises(ValueError):
        P.mae([1.0], [1.0, 2.0])


def test_evaluate_mae_matches_per_sample_loop(P):
    _, A = _ratings(P, 40, 30, 0.2, 9)
    f = P.latent_from_qb(P.fixed_precision_qb(A, tol=0.7, block_size=5, seed=10))
    samples = [(3, 4, 2.5), (10, 7, 4.0), (0, 0, 1.0), (39, 29, 5.0)]
    want = np.mean([abs(P.predict_rating(A, f, u, i).value - r) for u, i, r in samples])
    assert P.evaluate_mae(A, f, samples) == pytest.approx(want, rel=1e-12)
    many = P.predict_many(A, f, samples)
    np.testing.assert_allclose(many[:, 0], [P.predict_rating(A, f, u, i).value for u, i, _ in samples], rtol=1e-12)


def test_evaluate_rejects_out_of_range_samples(P):
    """An out-of-range user or item raises IndexError (the reference's
    per-sample loop fails there: sparse.py row_slice / numpy indexing)
    before anything reaches the device; factors for another item set raise
    ValueError.  The process's CUDA context stays usable."""
    _, A = _ratings(P, 40, 30, 0.2, 9)
    f = P.latent_from_qb(P.fixed_precision_qb(A, tol=0.7, block_size=5, seed=10))
    for bad in ([(40, 3, 1.0)], [(3, 30, 1.0)], [(-1, 3, 1.0)]):
        with pytest.raises(IndexError):
            P.evaluate_mae(A, f, bad)
        with pytest.raises(IndexError):
            P.evaluate_errors(A, f, bad)
    _, A2 = _ratings(P, 40, 31, 0.2, 9)
    with pytest.raises(ValueError):
        P.evaluate_mae(A2, f, [(1, 2, 3.0)])
    assert np.isfinite(P.evaluate_mae(A, f, [(1, 2, 3.0)]))


# ---------------------------------------------------------------------------
# CF: the validation criterion and Alg. 5

def _model(P, m, n, r, seed):
    import inputs
    tr, va, te = inputs.group_model(m, n, r, 0.7, seed)
    lo = min(tr.data.min(), va[2].min(), te[2].min())
    hi = max(tr.data.max(), va[2].max(), te[2].max())
    train = P.SparseRatings(tr, lo, hi)
    val = list(zip(va[0].tolist(), va[1].tolist(), va[2].tolist()))
    return train, val


def test_validation_trace_and_best_snapshot(P):
    train, val = _model(P, 200, 160, 6, 12)
    crit = P.ValidationMae(train, val, patience=2, min_improvement=1e-4)
    stopped = False
    for st in P.qb_pass_blocks(train, 2, 10, P.GaussianStream(0)):
        if crit(st):
            stopped = True
            break
    assert stopped
    ks = [e.k for e in crit.trace]
    assert ks == sorted(ks)
    assert all(b.seconds >= a.seconds for a, b in zip(crit.trace, crit.trace[1:]))
    best = min(crit.trace, key=lambda e: e.mae)
    assert crit.best_mae == best.mae and crit.best_factors is not None and crit.best_factors.k == best.k


def test_validation_stops_after_patience_stale_blocks(P):
    train, val = _model(P, 200, 160, 6, 13)
    crit = P.ValidationMae(train, val, patience=2, min_improvement=0.5)
    blocks = 0
    for st in P.qb_pass_blocks(train, 2, 10, P.GaussianStream(0)):
        blocks += 1
        if crit(st):
            break
    assert blocks == 3  # block 1 beats +inf; blocks 2 and 3 cannot gain 0.5


def test_validation_rejects_bad_arguments_and_overlap(P):
    train, val = _model(P, 120, 100, 4, 14)
    with pytest.raises(ValueError):
        P.ValidationMae(train, val, patience=0)
    with pytest.raises(ValueError):
        P.ValidationMae(train, val, min_improvement=-1.0)
    with pytest.raises(ValueError):
        P.ValidationMae(train, [])
    cols, vals = train.row_slice(0)
    with pytest.raises(ValueError):
        P.ValidationMae(train, val + [(0, int(cols[0]), float(vals[0]))])


def test_auto_latent_factors_finds_the_model_rank(P):
    train, val = _model(P, 240, 200, 6, 0)
    f, trace = P.auto_latent_factors(train, val, block_size=2, passes=10, seed=0)
    assert 6 <= f.k <= 10
    assert min(e.mae for e in trace) <= trace[0].mae
    assert f.k == min(trace, key=lambda e: e.mae).k


def test_auto_latent_factors_deterministic_and_patience(P):
    train, val = _model(P, 200, 160, 5, 16)
    f1, t1 = P.auto_latent_factors(train, val, block_size=3, passes=8, seed=4)
    f2, t2 = P.auto_latent_factors(train, val, block_size=3, passes=8, seed=4)
    assert [(e.k, e.mae) for e in t1] == [(e.k, e.mae) for e in t2]
    assert np.array_equal(f1.T, f2.T)
    _, short = P.auto_latent_factors(train, val, block_size=3, passes=8, patience=1, seed=5)
    _, long = P.auto_latent_factors(train, val, block_size=3, passes=8, patience=3, seed=5)
    assert len(short) <= len(long)


def test_auto_latent_factors_parameter_validation(P):
    train, val = _model(P, 120, 100, 4, 18)
    with pytest.raises(ValueError):
        P.auto_latent_factors(train, val, passes=2)
    with pytest.raises(ValueError):
        P.auto_latent_factors(train, val, block_size=0)
    with pytest.raises(ValueError):
        P.auto_latent_factors(train, [])


# ---------------------------------------------------------------------------
# linalg

def test_gaussian_stream_determinism_and_sequential_draws(P):
    a = P.GaussianStream(11).normal(40, 3)
    b = P.GaussianStream(11).normal(40, 3)
    np.testing.assert_array_equal(a, b)
    s = P.GaussianStream(11)
    first, second = s.normal(20, 3), s.normal(20, 3)
    assert not np.array_equal(first, second)
    np.testing.assert_array_equal(np.vstack([first, second]), P.GaussianStream(11).normal(40, 3))
    big = P.GaussianStream(3).normal(20000, 5)
    assert abs(big.mean()) < 0.02 and abs(big.std() - 1.0) < 0.02
    with pytest.raises(ValueError):
        P.gaussian_matrix(0, 3, 1)


def test_orthonormal_basis_contract(P):
    rng = np.random.default_rng(20)
    M = rng.standard_normal((300, 12))
    Q = P.orthonormal_basis(M)
    np.testing.assert_allclose(Q.T @ Q, np.eye(12), atol=1e-13)
    np.testing.assert_allclose(Q @ (Q.T @ M), M, atol=1e-12 * np.abs(M).max())
    D = M.copy()
    D[:, 5] = D[:, 1] + 2 * D[:, 3]
    with pytest.raises(P.RankDeficientError):
        P.orthonormal_basis(D)
    Qd = P.orthonormal_basis(D, check_rank=False)
    np.testing.assert_allclose(Qd.T @ Qd, np.eye(12), atol=1e-10)
    with pytest.raises(ValueError):
        P.orthonormal_basis(rng.standard_normal((5, 8)))


def test_lu_lower_basis_contract(P):
    import scipy.linalg as sl
    M = np.array([[1e-8, 1.0], [1.0, 1.0], [2.0, 3.0]])
    L = P.lu_lower_basis(M)
    np.testing.assert_allclose(L, sl.lu(M, permute_l=True)[0], rtol=1e-13, atol=1e-15)
    rng = np.random.default_rng(21)
    R = rng.standard_normal((400, 9))
    Lr = P.lu_lower_basis(R)
    Q = np.linalg.qr(Lr)[0]
    np.testing.assert_allclose(Q @ (Q.T @ R), R, atol=1e-10 * np.abs(R).max())  # same range
    S = R.copy()
    S[:, 4] = 0.0
    with pytest.raises(P.RankDeficientError):
        P.lu_lower_basis(S)
    with pytest.raises(ValueError):
        P.lu_lower_basis(rng.standard_normal((3, 7)))


def test_eig_svd_contract(P):
    rng = np.random.default_rng(22)
    M = rng.standard_normal((200, 10)) @ np.diag(np.geomspace(10, 1, 10))
    u, s, v = P.eig_svd(M)
    assert np.all(np.diff(s) >= 0)  # ascending
    np.testing.assert_allclose((u * s) @ v.T, M, atol=1e-10 * np.abs(M).max())
    np.testing.assert_allclose(u.T @ u, np.eye(10), atol=1e-10)
    np.testing.assert_allclose(v.T @ v, np.eye(10), atol=1e-12)
    np.testing.assert_allclose(s, np.sort(np.linalg.svd(M, compute_uv=False)), rtol=1e-10)
    N = M.copy()
    N[:, 3] = N[:, 2]
    with pytest.raises(P.NearSingularError):
        P.eig_svd(N)
    with pytest.raises(ValueError):
        P.eig_svd(rng.standard_normal((4, 9)))


def test_sparse_dense_mul_and_norms(P):
    dense, A = _ratings(P, 70, 50, 0.2, 23)
    rng = np.random.default_rng(24)
    X = rng.standard_normal((50, 6))
    Z = rng.standard_normal((70, 4))
    np.testing.assert_allclose(P.sparse_dense_mul(A, X), dense @ X, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(P.sparse_dense_mul(A, Z, transpose_a=True), dense.T @ Z, rtol=1e-12, atol=1e-12)
    with pytest.raises(ValueError):
        P.sparse_dense_mul(A, rng.standard_normal((49, 2)))
    assert P.fro_norm_sq(A) == float(np.sum(dense * dense))  # exact on the half-point grid
    assert P.fro_norm_sq(P.SparseRatings.from_dense(np.zeros((4, 3)))) == 0.0


# ---------------------------------------------------------------------------
# rsvd engines and drivers

def test_fixed_precision_meets_tolerance_with_minimal_rank(P):
    dense, A = _ratings(P, 90, 70, 0.25, 30)
    tol = 0.5
    st = P.fixed_precision_qb(A, tol=tol, block_size=5, power=1, seed=2)
    fro2 = float(np.sum(dense ** 2))
    resid2 = float(np.sum((dense - st.Q @ st.B) ** 2))
    assert resid2 <= tol * tol * fro2 * (1 + 1e-9)
    assert st.err == pytest.approx(resid2, rel=1e-8, abs=1e-9 * fro2)
    # one row fewer would miss the target (rank is the smallest sufficient)
    Bm = st.B[:-1]
    assert float(np.sum((dense - st.Q[:, :-1] @ Bm) ** 2)) > tol * tol * fro2


def test_fixed_precision_zero_matrix_and_validation(P):
    A = P.SparseRatings.from_dense(np.zeros((10, 8)))
    st = P.fixed_precision_qb(A, tol=0.3, block_size=2)
    assert st.rank == 0
    _, B = _ratings(P, 20, 15, 0.3, 31)
    for kw in (dict(tol=0.0), dict(tol=1.0), dict(tol=0.5, block_size=0), dict(tol=0.5, power=-1),
               dict(tol=0.5, block_size=16)):
        with pytest.raises(ValueError):
            P.fixed_precision_qb(B, **kw)


def test_rank_exhaustion_carries_state(P):
    _, A = _ratings(P, 40, 30, 0.4, 32, lo=0.5, hi=5.0)
    with pytest.raises(P.RankExhaustedError) as ei:
        P.fixed_precision_qb(A, tol=1e-6, block_size=4, seed=1, max_rank=8)
    assert ei.value.state is not None and ei.value.state.rank >= 8


def test_exact_rank_recovery(P):
    import inputs
    dense, M = inputs.exact_rank(120, 90, 7, 33)
    A = P.SparseRatings(M, float(dense.min()), float(dense.max()))
    usv = P.basic_rsvd(A, k=7, power=1, oversample=0, seed=0)
    rec = (usv.u * usv.s) @ usv.v.T
    np.testing.assert_allclose(rec, dense, atol=1e-9 * np.abs(dense).max())
    np.testing.assert_allclose(usv.u.T @ usv.u, np.eye(7), atol=1e-10)
    np.testing.assert_allclose(usv.v.T @ usv.v, np.eye(7), atol=1e-10)
    with pytest.raises(P.RankDeficientError):  # a sketch wider than the rank is rank deficient
        P.basic_rsvd(A, k=7, oversample=3, seed=0)


def test_basic_rsvd_validation(P):
    _, A = _ratings(P, 30, 20, 0.3, 34)
    with pytest.raises(ValueError):
        P.basic_rsvd(A, k=15, oversample=6)  # sketch wider than min(m, n)
    with pytest.raises(ValueError):
        P.basic_rsvd(A, k=0)
    with pytest.raises(ValueError):
        P.basic_rsvd(A, k=3, power=-1)


def test_adaptive_pca_criteria_and_validation(P):
    dense, A = _ratings(P, 60, 90, 0.3, 35)  # wide: handled through A.T internally as in the reference
    usv = P.adaptive_pca(A, P.FrobTolerance(0.6), block_size=4, passes=6, seed=1)
    assert np.all(np.diff(usv.s) <= 1e-12 * usv.s[0])  # descending
    np.testing.assert_allclose(usv.u.T @ usv.u, np.eye(usv.u.shape[1]), atol=1e-9)
    fixed = P.adaptive_pca(A, P.FixedRank(6), block_size=4, passes=6, seed=1)
    assert fixed.s.size == 6
    custom = P.adaptive_pca(A, lambda st: st.rank >= 8, block_size=4, passes=6, seed=1)
    assert custom.s.size >= 8
    with pytest.raises(ValueError):
        P.adaptive_pca(A, P.FixedRank(4), passes=2)
    with pytest.raises(ValueError):
        P.FixedRank(0)
    with pytest.raises(ValueError):
        P.FrobTolerance(1.5)
    with pytest.raises(P.RankExhaustedError):
        P.adaptive_pca(A, P.FixedRank(500), block_size=4, passes=6, seed=1)


# ---------------------------------------------------------------------------
# acceptance-style properties (the reference's criteria 3, 4 and 8, on
# seeded synthetic matrices)

def test_pass_engine_matches_power_engine_at_matched_budget(P):
    import inputs
    dense, M = inputs.rand_sparse(200, 300, 0.05, 33, grid=False)
    A = P.SparseRatings(M, 0.5, 5.0)
    norm = np.linalg.norm(dense)
    for power in (0, 1, 2):
        s1 = next(P.qb_power_blocks(A, 20, power, P.GaussianStream(7)))
        s2 = next(P.qb_pass_blocks(A, 20, 2 * power + 2, P.GaussianStream(7)))
        assert np.linalg.norm(s1.Q @ s1.B - s2.Q @ s2.B) / norm <= 1e-6
        assert np.linalg.norm(s1.Q @ s1.Q.T - s2.Q @ s2.Q.T) <= 1e-6


def test_error_indicator_equals_explicit_residual(P):
    import inputs
    rng = np.random.default_rng(99)
    worst = 0.0
    for trial in range(8):
        m, n = int(rng.integers(60, 400)), int(rng.integers(60, 400))
        dense, M = inputs.rand_sparse(m, n, float(rng.uniform(0.02, 0.2)), 1000 + trial)
        A = P.SparseRatings(M, 0.5, 5.0)
        frob = float(np.sum(dense * dense))
        for st in P.qb_power_blocks(A, int(rng.integers(10, 31)), trial % 2, P.GaussianStream(trial)):
            explicit = np.linalg.norm(dense - st.Q @ st.B) ** 2
            worst = max(worst, abs(st.err - explicit) / frob)
            if st.blocks >= 4:
                break
    assert worst <= 1e-8


def test_exact_rank_matrices_reconstructed_by_all_drivers(P):
    import inputs
    worst = 0.0
    for r in (3, 7, 10):
        dense, M = inputs.exact_rank(100, 80, r, 200 + r)
        A = P.SparseRatings(M, float(dense.min()), float(dense.max()))
        norm = np.linalg.norm(dense)
        t = P.basic_rsvd(A, k=r, power=1, seed=r)
        worst = max(worst, np.linalg.norm(dense - t.reconstruct()) / norm)
        st = P.fixed_precision_qb(A, tol=1e-6, block_size=20, power=0, seed=r)
        worst = max(worst, np.linalg.norm(dense - st.Q @ st.B) / norm)
        tri = P.adaptive_pca(A, P.FrobTolerance(1e-6), block_size=20, passes=10, seed=r)
        worst = max(worst, np.linalg.norm(dense - tri.reconstruct()) / norm)
    assert worst <= 1e-8
