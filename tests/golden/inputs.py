"""Seeded small test matrices shared by the golden generator and the tests.

Pure numpy, no reference imports: the same inputs are rebuilt on the GPU
box from these functions, so only the reference's *outputs* are stored in
the fixtures.
"""
from __future__ import annotations

import numpy as np
from scipy import sparse as sp


def rand_sparse(m, n, density, seed, grid=True):
    """Sparse ratings on the half-point grid (exact Frobenius sums)."""
    rng = np.random.default_rng(seed)
    keep = rng.random((m, n)) < density
    vals = rng.integers(1, 11, size=(m, n)) * 0.5 if grid else rng.uniform(0.5, 5.0, (m, n))
    dense = np.where(keep, vals, 0.0)
    return dense, sp.csr_matrix(dense)


def exact_rank(m, n, r, seed):
    rng = np.random.default_rng(seed)
    dense = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    return dense, sp.csr_matrix(dense)


def decay(m, n, base, seed):
    """Dense full-rank matrix with geometric spectrum base**i."""
    rng = np.random.default_rng(seed)
    r = min(m, n)
    u = np.linalg.qr(rng.standard_normal((m, r)))[0]
    v = np.linalg.qr(rng.standard_normal((n, r)))[0]
    dense = (u * base ** np.arange(r)) @ v.T
    return dense, sp.csr_matrix(dense)


def group_model(m, n, r, density, seed, holdout=0.1):
    """Exact rank-r rating model with r item groups; (train, val, test).

    val/test are (users, items, ratings) arrays of equal size holdout/2.
    """
    rng = np.random.default_rng(seed)
    levels = np.linspace(1.0, 5.0, r)
    prof = np.take_along_axis(np.tile(levels, (m, 1)), np.argsort(rng.random((m, r)), axis=1), axis=1)
    full = prof[:, rng.integers(0, r, size=n)]
    oi, oj = np.nonzero(rng.random((m, n)) < density)
    order = rng.permutation(oi.size)
    h = int(oi.size * holdout / 2)
    va, te, tr = order[:h], order[h:2 * h], order[2 * h:]
    train = sp.coo_matrix((full[oi[tr], oj[tr]], (oi[tr], oj[tr])), shape=(m, n)).tocsr()
    train.sort_indices()

    def part(idx):
        return oi[idx].astype(np.int64), oj[idx].astype(np.int64), full[oi[idx], oj[idx]].astype(np.float64)

    return train, part(va), part(te)
