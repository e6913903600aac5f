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


def ratings_csv_text(seed, nrows, nusers=60, nitems=40, delimiter=",", header=True, dup_frac=0.1):
    """A delimited ratings file as text: string identifiers with stray
    whitespace, half-star ratings, repeated (user, item) pairs."""
    rng = np.random.default_rng(seed)
    u = rng.integers(0, nusers, nrows)
    i = rng.integers(0, nitems, nrows)
    dup = rng.random(nrows) < dup_frac
    src = rng.integers(0, max(nrows, 1), nrows)
    u = np.where(dup, u[src], u)
    i = np.where(dup, i[src], i)
    r = rng.integers(1, 11, nrows) * 0.5
    lines = ["userId{0}movieId{0}rating{0}timestamp".format(delimiter)] if header else []
    for a, b, c in zip(u, i, r):
        pad = " " if (a + b) % 7 == 0 else ""
        lines.append(f"{pad}u{a}{delimiter}m{b}{pad}{delimiter}{c}{delimiter}1700000000")
        if (a * 31 + b) % 97 == 0:
            lines.append("")  # blank lines are skipped
    return "\n".join(lines) + "\n"


def matrix_market_text(seed, m, n, nnz, field="real"):
    rng = np.random.default_rng(seed)
    cells = rng.choice(m * n, size=nnz, replace=False)
    vals = rng.integers(1, 11, nnz) * (0.5 if field == "real" else 1)
    body = [f"{c // n + 1} {c % n + 1} {v if field == 'real' else int(v)}" for c, v in zip(cells, vals)]
    return "\n".join([f"%%MatrixMarket matrix coordinate {field} general", "% a comment", f"{m} {n} {nnz}"]
                     + body) + "\n"
