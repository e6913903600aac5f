"""The reference's acceptance gate (its tests/test_acceptance.py), criterion
by criterion, against this package on the GPU.  Criteria 3, 4, 7, 8 and 9
are data-free and run as stated.  Criteria 1 and 6 need MovieLens, which
is not on disk (no network); their data-independent guarantee -- leading
singular values within 1 % of an exact sparse SVD, the validation-chosen
block within 0.01 of the best test MAE -- is checked on the seeded
ML-100K-shaped synthetic matrix (BASELINE configs[0]).  Criteria 2 and 5
state dataset-specific bands (rank in [110, 128], MAE <= 0.70 on ML-100K)
and are skipped here, as the reference skips them without the dataset."""
from __future__ import annotations

import time

import numpy as np
import pytest
import scipy.sparse.linalg

import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(gpu):
    import paper_2009_02251_b200 as P
    return P


@pytest.fixture(scope="module")
def c0():
    from paper_2009_02251_b200 import synth
    return synth.generate(synth.CONFIGS["c0_100k"])


def test_criterion_1_singular_value_accuracy_synthetic(P, c0):
    """Synthetic stand-in: its noise floor is flat (no decaying tail as in
    ML-100K), so the 1 % bound holds for the leading 50 values; all 100 equal
    the reference algorithm's own output (the oracle) to 1e-9."""
    from oracle import svdrec_oracle as O
    A = P.SparseRatings(c0, 1.0, 5.0)
    t = P.adaptive_pca(A, P.FixedRank(118), block_size=20, passes=10, seed=0)
    v0 = np.random.default_rng(0).standard_normal(min(A.shape))
    ref = np.sort(scipy.sparse.linalg.svds(c0, k=100, v0=v0, return_singular_vectors=False))[::-1]
    assert np.max(np.abs(t.s[:50] - ref[:50]) / ref[:50]) <= 0.01
    _, s_oracle, _, _ = O.adaptive_pca(c0, ("rank", 118), block_size=20, passes=10, seed=0)
    np.testing.assert_allclose(t.s[:100], s_oracle[:100], rtol=1e-9)


@pytest.mark.skip(reason="ML-100K rank band [110, 128]: dataset-specific, MovieLens not on disk (no network)")
def test_criterion_2_ml100k_fixed_precision_rank_band():
    pass


def test_criterion_3_engine_equivalence(P):
    dense, csr = inputs.rand_sparse(200, 300, 0.05, 33, grid=False)
    A = P.SparseRatings(csr, 0.5, 5.0)
    norm = np.linalg.norm(dense)
    for power in (0, 1, 2):
        a = next(P.qb_power_blocks(A, 20, power, P.GaussianStream(7)))
        b = next(P.qb_pass_blocks(A, 20, 2 * power + 2, P.GaussianStream(7)))
        assert np.linalg.norm(a.Q @ a.B - b.Q @ b.B) / norm <= 1e-6
        assert np.linalg.norm(a.Q @ a.Q.T - b.Q @ b.Q.T) <= 1e-6


def test_criterion_4_error_indicator_identity(P):
    rng = np.random.default_rng(99)
    worst = 0.0
    for trial in range(20):
        m, n = int(rng.integers(60, 501)), int(rng.integers(60, 501))
        density = float(rng.uniform(0.02, 0.2))
        dense, csr = inputs.rand_sparse(m, n, density, 1000 + trial)
        A = P.SparseRatings(csr, 0.5, 5.0)
        frob = float((dense * dense).sum())
        block = int(rng.integers(10, 31))
        for s in P.qb_power_blocks(A, block, trial % 2, P.GaussianStream(trial)):
            gap = abs((frob - float((s.B * s.B).sum())) - np.linalg.norm(dense - s.Q @ s.B) ** 2)
            worst = max(worst, gap / frob)
            if s.blocks >= 5:
                break
    assert worst <= 1e-8


@pytest.mark.skip(reason="ML-100K MAE <= 0.70 at rank in [140, 320]: dataset-specific, MovieLens not on disk")
def test_criterion_5_ml100k_recommendation_quality():
    pass


def test_criterion_6_validation_tracks_test_synthetic(P, c0):
    from paper_2009_02251_b200 import synth
    worst = 0.0
    for seed in range(3):
        tr, va, te = synth.split_holdout(c0, (0.9, 0.05, 0.05), seed=seed)
        A = P.SparseRatings(tr, 1.0, 5.0)
        crit = P.ValidationMae(A, va, patience=2, min_improvement=1e-4)
        test_mae = []
        for s in P.qb_pass_blocks(A, 20, 10, P.GaussianStream(seed)):
            stop = crit(s)
            test_mae.append(P.evaluate_mae(A, P.latent_from_qb(s), te))
            if stop:
                break
        chosen = int(np.argmin([e.mae for e in crit.trace]))
        worst = max(worst, test_mae[chosen] - min(test_mae))
    assert worst <= 0.01


def test_criterion_7_prediction_matches_bruteforce_oracle(P):
    from test_gpu_reference_cf import _bruteforce
    train, _, _ = inputs.group_model(150, 120, 5, 0.3, seed=42)
    A = P.SparseRatings(train, 1.0, 5.0)
    f = P.latent_from_qb(P.fixed_precision_qb(A, tol=0.5, block_size=10, power=1, seed=0))
    T = f.T
    rng = np.random.default_rng(7)
    worst, mismatches = 0.0, 0
    users = rng.integers(0, A.m, 1000)
    items = rng.integers(0, A.n, 1000)
    got = P.predict_many(A, f, (users, items, np.zeros(1000)))
    for t, (u, i) in enumerate(zip(users.tolist(), items.tolist())):
        raw, val, fb = _bruteforce(A, T, u, i)
        if bool(got[t, 2]) != fb:
            mismatches += 1
            continue
        worst = max(worst, abs(got[t, 1] - raw) / max(1.0, abs(raw)), abs(got[t, 0] - val))
    assert mismatches == 0 and worst <= 1e-12


def test_criterion_8_exact_rank_recovery(P):
    worst = 0.0
    for r in (3, 7, 10):
        dense, csr = inputs.exact_rank(100, 80, r, 200 + r)
        A = P.SparseRatings(csr, float(dense.min()), float(dense.max()))
        norm = np.linalg.norm(dense)
        worst = max(worst, np.linalg.norm(dense - P.basic_rsvd(A, k=r, power=1, seed=r).reconstruct()) / norm)
        s = P.fixed_precision_qb(A, tol=1e-6, block_size=20, power=0, seed=r)
        worst = max(worst, np.linalg.norm(dense - s.Q @ s.B) / norm)
        t = P.adaptive_pca(A, P.FrobTolerance(1e-6), block_size=20, passes=10, seed=r)
        worst = max(worst, np.linalg.norm(dense - t.reconstruct()) / norm)
    assert worst <= 1e-8


def test_criterion_9_mae_evaluation_scales_linearly(P):
    import torch
    _, csr = inputs.rand_sparse(500, 1500, 0.07, 55)
    A = P.SparseRatings(csr, 0.5, 5.0)
    rng = np.random.default_rng(8)
    samples = (rng.integers(0, 500, 800), rng.integers(0, 1500, 800), rng.uniform(1, 5, 800))

    def timed(k):
        f = P.LatentFactors.from_matrix(np.random.default_rng(k).standard_normal((k, 1500)))
        P.evaluate_mae(A, f, samples)
        runs = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            P.evaluate_mae(A, f, samples)
            runs.append(time.perf_counter() - t0)
        return float(np.median(runs))

    assert timed(300) / timed(150) <= 2.2
