"""The reference's engine / driver behaviour suite (its tests/test_rsvd.py:
engine invariants, engine equivalence, fixed-precision QB, basic rSVD,
adaptive PCA, criteria), restated against this package on the GPU -- same
test names and inputs, so a reader of the reference's tests recognises each
case.  Tolerances are the reference's own."""
from __future__ import annotations

import itertools

import numpy as np
import pytest

import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(gpu):
    import paper_2009_02251_b200 as P
    return P


def _sparse(P, m, n, density, seed):
    dense, csr = inputs.rand_sparse(m, n, density, seed)
    return dense, P.SparseRatings(csr, 0.5, 5.0)


def _exact(P, m, n, r, seed):
    dense, csr = inputs.exact_rank(m, n, r, seed)
    return dense, P.SparseRatings(csr, float(dense.min()), float(dense.max()))


def _decay(P, m, n, base, seed):
    dense, csr = inputs.decay(m, n, base, seed)
    return dense, P.SparseRatings(csr, float(dense.min()), float(dense.max()))


def _nth(gen, n):
    return next(itertools.islice(gen, n - 1, None))


def _count_products(monkeypatch):
    """Count the engines' sparse products (the reference counts its
    sparse_dense_mul calls the same way)."""
    from paper_2009_02251_b200 import rsvd
    calls = []
    real = rsvd.sparse_dense_mul

    def counting(A, X, transpose_a=False, out=None):
        calls.append(transpose_a)
        return real(A, X, transpose_a, out=out)

    monkeypatch.setattr(rsvd, "sparse_dense_mul", counting)
    return calls


class TestEngineInvariants:
    @pytest.mark.parametrize("power", [0, 1, 2])
    def test_power_engine_state(self, P, power):
        dense, A = _sparse(P, 120, 150, 0.08, seed=power)
        frob = float((dense ** 2).sum())
        last = np.inf
        for s in P.qb_power_blocks(A, 15, power, P.GaussianStream(3)):
            k = s.rank
            assert k == 15 * s.blocks
            assert np.linalg.norm(s.Q.T @ s.Q - np.eye(k)) <= 1e-10 * np.sqrt(k)
            assert abs(s.err - (frob - float((s.B ** 2).sum()))) <= 1e-8 * frob
            assert abs(s.err - np.linalg.norm(dense - s.Q @ s.B) ** 2) <= 1e-8 * frob
            assert s.err <= last + 1e-8 * frob
            last = s.err
            if s.blocks == 5:
                break

    @pytest.mark.parametrize("passes", [4, 5, 10])
    def test_pass_engine_state(self, P, passes):
        dense, A = _sparse(P, 120, 150, 0.08, seed=passes)
        frob = float((dense ** 2).sum())
        for s in P.qb_pass_blocks(A, 15, passes, P.GaussianStream(4)):
            k = s.rank
            assert np.linalg.norm(s.Q.T @ s.Q - np.eye(k)) <= 1e-10 * np.sqrt(k)
            assert abs(s.err - np.linalg.norm(dense - s.Q @ s.B) ** 2) <= 1e-8 * frob
            if s.blocks == 4:
                break

    @pytest.mark.parametrize("passes", [2, 3, 4, 5, 10])
    def test_pass_budget_is_exact(self, P, passes, monkeypatch):
        _, A = _sparse(P, 80, 100, 0.1, seed=20)
        calls = _count_products(monkeypatch)
        gen = P.qb_pass_blocks(A, 10, passes, P.GaussianStream(0))
        next(gen)
        assert len(calls) == passes
        next(gen)
        assert len(calls) == 2 * passes

    @pytest.mark.parametrize("power", [0, 2])
    def test_power_engine_pass_count(self, P, power, monkeypatch):
        _, A = _sparse(P, 80, 100, 0.1, seed=21)
        calls = _count_products(monkeypatch)
        next(P.qb_power_blocks(A, 10, power, P.GaussianStream(0)))
        assert len(calls) == 2 * power + 2

    def test_rank_cap_power(self, P):
        _, A = _sparse(P, 30, 45, 0.3, seed=22)
        assert [s.rank for s in P.qb_power_blocks(A, 8, 0, P.GaussianStream(1))][-1] == 24

    def test_rank_cap_pass(self, P):
        _, A = _sparse(P, 30, 45, 0.3, seed=23)
        assert [s.rank for s in P.qb_pass_blocks(A, 8, 4, P.GaussianStream(1))][-1] == 16

    def test_invalid_passes(self, P):
        _, A = _sparse(P, 20, 20, 0.3, seed=24)
        with pytest.raises(ValueError):
            next(P.qb_pass_blocks(A, 4, 1, P.GaussianStream(0)))


class TestEngineEquivalence:
    @pytest.mark.parametrize("power,blocks", [(0, 1), (1, 1), (2, 1), (0, 3), (1, 3)])
    def test_products_and_projectors_match(self, P, power, blocks):
        dense, A = _sparse(P, 150, 200, 0.06, seed=31)
        a = _nth(P.qb_power_blocks(A, 20, power, P.GaussianStream(9)), blocks)
        b = _nth(P.qb_pass_blocks(A, 20, 2 * power + 2, P.GaussianStream(9)), blocks)
        assert np.linalg.norm(a.Q @ a.B - b.Q @ b.B) <= 1e-6 * np.linalg.norm(dense)
        assert np.linalg.norm(a.Q @ a.Q.T - b.Q @ b.Q.T) <= 1e-6


class TestFixedPrecisionQb:
    def test_meets_tolerance_explicitly(self, P):
        for seed in range(4):
            dense, A = _sparse(P, 100, 140, 0.07, seed=40 + seed)
            s = P.fixed_precision_qb(A, tol=0.6, block_size=12, power=1, seed=seed)
            assert np.linalg.norm(dense - s.Q @ s.B) <= 0.6 * np.linalg.norm(dense)

    def test_final_rank_is_minimal(self, P):
        dense, A = _sparse(P, 100, 140, 0.07, seed=50)
        s = P.fixed_precision_qb(A, tol=0.6, block_size=12, power=1, seed=5)
        total = float((dense ** 2).sum())
        assert total - float((s.B ** 2).sum()) < 0.36 * total
        if s.rank > 1:
            assert total - float((s.B[:-1] ** 2).sum()) >= 0.36 * total

    def test_exact_rank_recovery_with_oversized_block(self, P):
        dense, A = _exact(P, 90, 70, 5, seed=51)
        s = P.fixed_precision_qb(A, tol=1e-6, block_size=20, power=0, seed=0)
        assert s.rank == 5
        assert np.linalg.norm(dense - s.Q @ s.B) <= 1e-6 * np.linalg.norm(dense)

    def test_zero_matrix_gives_rank_zero(self, P):
        s = P.fixed_precision_qb(P.SparseRatings.from_dense(np.zeros((12, 9))), tol=0.5, block_size=3)
        assert (s.rank, s.err) == (0, 0.0)
        assert s.Q.shape == (12, 0) and s.B.shape == (0, 9)

    def test_parameter_validation(self, P):
        _, A = _sparse(P, 20, 25, 0.3, seed=52)
        for kw in (dict(tol=0.0), dict(tol=1.0), dict(tol=0.5, block_size=0), dict(tol=0.5, block_size=21),
                   dict(tol=0.5, power=-1)):
            with pytest.raises(ValueError):
                P.fixed_precision_qb(A, **kw)

    def test_rank_exhaustion_carries_state(self, P):
        _, A = _sparse(P, 30, 40, 0.5, seed=53)
        with pytest.raises(P.RankExhaustedError) as err:
            P.fixed_precision_qb(A, tol=1e-9, block_size=8, power=0, seed=1)
        assert err.value.state is not None and err.value.state.rank == 24


class TestBasicRsvd:
    def test_exact_rank_reconstruction(self, P):
        dense, A = _exact(P, 80, 60, 9, seed=60)
        t = P.basic_rsvd(A, k=9, power=1, seed=2)
        assert np.linalg.norm(dense - t.reconstruct()) <= 1e-8 * np.linalg.norm(dense)

    def test_singular_values_match_oracle_with_power(self, P):
        dense, A = _decay(P, 100, 80, 0.7, seed=61)
        sv = np.linalg.svd(dense, compute_uv=False)
        t = P.basic_rsvd(A, k=10, power=6, oversample=10, seed=3)
        assert np.max(np.abs(t.s[:5] - sv[:5]) / sv[:5]) <= 1e-6

    def test_factors_orthonormal(self, P):
        _, A = _sparse(P, 70, 90, 0.1, seed=62)
        t = P.basic_rsvd(A, k=8, power=2, oversample=4, seed=4)
        assert np.linalg.norm(t.u.T @ t.u - np.eye(8)) <= 1e-10
        assert np.linalg.norm(t.v.T @ t.v - np.eye(8)) <= 1e-10
        assert np.all(np.diff(t.s) <= 0)

    def test_sketch_wider_than_matrix_rejected(self, P):
        _, A = _sparse(P, 20, 30, 0.3, seed=63)
        with pytest.raises(ValueError):
            P.basic_rsvd(A, k=15, oversample=10)

    def test_rank_deficient_sketch_raises(self, P):
        _, A = _exact(P, 40, 30, 3, seed=64)
        with pytest.raises(P.RankDeficientError):
            P.basic_rsvd(A, k=8, seed=5)


class TestAdaptivePca:
    def test_frob_tolerance_met(self, P):
        for seed in range(3):
            dense, A = _sparse(P, 110, 160, 0.07, seed=70 + seed)
            t = P.adaptive_pca(A, P.FrobTolerance(0.6), block_size=12, passes=10, seed=seed)
            assert np.linalg.norm(dense - t.reconstruct()) <= 0.6 * np.linalg.norm(dense)

    def test_fixed_rank_values_match_oracle(self, P):
        dense, A = _decay(P, 100, 120, 0.7, seed=71)
        sv = np.linalg.svd(dense, compute_uv=False)
        t = P.adaptive_pca(A, P.FixedRank(10), block_size=5, passes=10, seed=6)
        assert t.k == 10
        assert np.max(np.abs(t.s[:5] - sv[:5]) / sv[:5]) <= 1e-6

    def test_tall_matrix_transposed_internally(self, P):
        dense, A = _exact(P, 150, 40, 6, seed=72)
        t = P.adaptive_pca(A, P.FrobTolerance(1e-7), block_size=6, passes=10, seed=7)
        assert t.u.shape == (150, t.k) and t.v.shape == (40, t.k)
        assert np.linalg.norm(dense - t.reconstruct()) <= 1e-7 * np.linalg.norm(dense)

    def test_custom_callable_criterion(self, P):
        _, A = _sparse(P, 90, 130, 0.1, seed=73)
        assert P.adaptive_pca(A, lambda s: s.blocks >= 3, block_size=7, passes=6, seed=8).k == 21

    def test_descending_order_and_orthonormal(self, P):
        _, A = _sparse(P, 90, 130, 0.1, seed=74)
        t = P.adaptive_pca(A, P.FixedRank(12), block_size=6, passes=8, seed=9)
        assert np.all(np.diff(t.s) <= 0)
        assert np.linalg.norm(t.u.T @ t.u - np.eye(12)) <= 1e-8
        assert np.linalg.norm(t.v.T @ t.v - np.eye(12)) <= 1e-8

    def test_pass_budget_validation(self, P):
        _, A = _sparse(P, 30, 30, 0.3, seed=75)
        with pytest.raises(ValueError):
            P.adaptive_pca(A, P.FixedRank(4), passes=2)
        with pytest.raises(ValueError):
            P.adaptive_pca(A, P.FixedRank(4), block_size=0)

    def test_unreachable_rank_exhausts(self, P):
        _, A = _sparse(P, 30, 40, 0.5, seed=76)
        with pytest.raises(P.RankExhaustedError):
            P.adaptive_pca(A, P.FixedRank(25), block_size=10, passes=4, seed=10)

    def test_unreachable_tolerance_exhausts(self, P):
        _, A = _sparse(P, 30, 40, 0.5, seed=77)
        with pytest.raises(P.RankExhaustedError):
            P.adaptive_pca(A, P.FrobTolerance(1e-9), block_size=8, passes=4, seed=11)

    def test_rank_beyond_numerical_rank_near_singular(self, P):
        _, A = _exact(P, 60, 50, 3, seed=78)
        with pytest.raises(P.NearSingularError):
            P.adaptive_pca(A, P.FixedRank(10), block_size=10, passes=6, seed=12)


class TestCriteria:
    def test_fixed_rank_fires_at_rank(self, P):
        crit = P.FixedRank(10)
        _, A = _sparse(P, 40, 50, 0.2, seed=80)
        gen = P.qb_power_blocks(A, 5, 0, P.GaussianStream(0))
        first, second = next(gen), next(gen)
        assert (first.rank, crit(first)) == (5, False)
        assert (second.rank, crit(second)) == (10, True)

    def test_frob_tolerance_uses_relative_error(self, P):
        crit = P.FrobTolerance(0.5)
        _, A = _sparse(P, 40, 50, 0.2, seed=81)
        fired = [crit(s) for s in P.qb_power_blocks(A, 10, 1, P.GaussianStream(0))]
        if True in fired:
            assert all(fired[fired.index(True):])

    def test_validation(self, P):
        for bad in (lambda: P.FixedRank(0), lambda: P.FrobTolerance(0.0), lambda: P.FrobTolerance(1.0)):
            with pytest.raises(ValueError):
                bad()
