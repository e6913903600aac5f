"""Seeded synthetic rating matrices standing in for BASELINE.json's configs.

BASELINE.json names MovieLens-shaped workloads (943x1682/100k, 6040x3706/1M,
69878x10677/10M, 138493x26744/20M and an 8M x 1M scale-out).  No dataset is
fetched: every matrix here is drawn from a rank-r latent model with the
shape, nnz and value grid of its config:

* item popularity ~ Zipf(s) over a seeded permutation of the item ids;
* user activity ~ log-normal(mu, sigma), floored at ``min_per_user``
  ratings and rescaled so the total hits the requested nnz exactly;
* value = 3.5 + u_i . v_j + N(0, 0.5^2), with u, v ~ N(0, 1/sqrt(r)) per
  entry (variance 1/sqrt(r), so u.v has unit variance), rounded to the
  config's grid (integers 1..5 or half stars 0.5..5.0) and clipped.

Ratings are returned in canonical CSR order (row-major, columns increasing
per row); that order is the sample order used by :func:`split_holdout`,
which mirrors the reference's seeded 90/5/5 shuffle (reference
pkg/src/svdrec/data.py:200-232) without materialising Python objects.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy import sparse as sp


@dataclass(frozen=True)
class SynthConfig:
    name: str
    users: int
    items: int
    nnz: int
    rank: int
    zipf: float
    half_stars: bool
    lognorm_mu: float = 4.0
    lognorm_sigma: float = 1.2
    min_per_user: int = 20
    noise: float = 0.5
    seed: int = 0

    @property
    def bounds(self) -> tuple[float, float]:
        return (0.5, 5.0) if self.half_stars else (1.0, 5.0)


# BASELINE.json "configs", in order.
CONFIGS = {
    "c0_100k": SynthConfig("c0_100k", 943, 1682, 100_000, 10, 1.1, False),
    "c1_1m": SynthConfig("c1_1m", 6040, 3706, 1_000_209, 20, 1.0, False),
    "c2_10m": SynthConfig("c2_10m", 69_878, 10_677, 10_000_054, 30, 1.1, True),
    "c3_20m": SynthConfig("c3_20m", 138_493, 26_744, 20_000_263, 40, 1.2, True),
}


def _degrees(cfg: SynthConfig, rng: np.random.Generator) -> np.ndarray:
    m, n, nnz = cfg.users, cfg.items, cfg.nnz
    lo = min(cfg.min_per_user, n)
    if lo * m > nnz:
        lo = max(1, nnz // m)
    hi = max(lo, min(n, n // 2 if n >= 2 * lo else n))
    raw = rng.lognormal(cfg.lognorm_mu, cfg.lognorm_sigma, size=m)
    # find a scale c with sum(clip(round(c*raw), lo, hi)) ~= nnz by bisection
    a, b = 1e-9, 1.0
    while np.clip(np.rint(b * raw), lo, hi).sum() < nnz and b < 1e12:
        b *= 2.0
    for _ in range(200):
        c = 0.5 * (a + b)
        if np.clip(np.rint(c * raw), lo, hi).sum() < nnz:
            a = c
        else:
            b = c
    deg = np.clip(np.rint(b * raw), lo, hi).astype(np.int64)
    diff = int(deg.sum() - nnz)
    order = np.argsort(-raw, kind="stable")
    # remove (or add) the residual one rating at a time from the heaviest users
    i = 0
    while diff != 0:
        u = order[i % m]
        if diff > 0 and deg[u] > lo:
            deg[u] -= 1
            diff -= 1
        elif diff < 0 and deg[u] < hi:
            deg[u] += 1
            diff += 1
        i += 1
    return deg


def _pick_items(cfg: SynthConfig, deg: np.ndarray, rng: np.random.Generator) -> np.ndarray:
    """Per user, ``deg[u]`` distinct items drawn ~ Zipf popularity.

    Returns the flat sorted (user * n + item) keys.
    """
    m, n = cfg.users, cfg.items
    weights = 1.0 / np.arange(1, n + 1, dtype=np.float64) ** cfg.zipf
    perm = rng.permutation(n)  # popularity rank -> item id
    cdf = np.cumsum(weights)
    cdf /= cdf[-1]
    heavy_cut = max(64, n // 16)
    heavy = np.nonzero(deg > heavy_cut)[0]
    light = np.nonzero(deg <= heavy_cut)[0]
    keys = []
    # heavy users: Gumbel top-k == sampling without replacement ~ weights
    logw = np.log(weights)
    for u in heavy:
        g = logw + rng.gumbel(size=n)
        top = np.argpartition(-g, deg[u] - 1)[: deg[u]]
        keys.append(u * np.int64(n) + perm[top])
    # light users: draw with replacement (2x oversampled), drop keys already
    # held, keep a random subset of the fresh ones up to each user's deficit
    need = deg[light].copy()
    users = light
    got = np.empty(0, dtype=np.int64)
    for _ in range(64):
        if users.size == 0:
            break
        rows = np.repeat(users, 2 * need + 2)
        ranks = np.searchsorted(cdf, rng.random(rows.size), side="right")
        cand = rows * np.int64(n) + perm[np.minimum(ranks, n - 1)]
        cand.sort()
        cand = cand[np.concatenate(([True], cand[1:] != cand[:-1]))]
        if got.size:
            pos = np.minimum(np.searchsorted(got, cand), got.size - 1)
            cand = cand[got[pos] != cand]
        cu = cand // n
        order = np.lexsort((rng.random(cand.size), cu))
        cand, cu = cand[order], cu[order]
        first = np.searchsorted(cu, cu, side="left")
        quota = np.zeros(m, dtype=np.int64)
        quota[users] = need
        take = (np.arange(cand.size) - first) < quota[cu]
        got = np.sort(np.concatenate([got, cand[take]]))
        have = np.bincount((got // n).astype(np.int64), minlength=m)
        deficit = deg - have
        deficit[heavy] = 0
        users = np.nonzero(deficit > 0)[0]
        need = deficit[users]
    keys.append(got)
    return np.sort(np.concatenate(keys))


def generate(cfg: SynthConfig) -> sp.csr_matrix:
    """Seeded synthetic rating matrix (scipy CSR, float64, canonical)."""
    rng = np.random.default_rng(np.random.SeedSequence([cfg.seed, cfg.users, cfg.items, cfg.nnz]))
    deg = _degrees(cfg, rng)
    keys = _pick_items(cfg, deg, rng)
    rows = keys // cfg.items
    cols = keys - rows * cfg.items
    sd = (1.0 / np.sqrt(cfg.rank)) ** 0.5
    U = rng.normal(0.0, sd, size=(cfg.users, cfg.rank))
    V = rng.normal(0.0, sd, size=(cfg.items, cfg.rank))
    vals = np.empty(keys.size, dtype=np.float64)
    step = 1 << 21
    for s in range(0, keys.size, step):
        e = min(keys.size, s + step)
        vals[s:e] = np.einsum("ij,ij->i", U[rows[s:e]], V[cols[s:e]])
    vals += 3.5 + rng.normal(0.0, cfg.noise, size=keys.size)
    lo, hi = cfg.bounds
    if cfg.half_stars:
        vals = np.rint(vals * 2.0) / 2.0
    else:
        vals = np.rint(vals)
    np.clip(vals, lo, hi, out=vals)
    indptr = np.zeros(cfg.users + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=cfg.users), out=indptr[1:])
    return sp.csr_matrix((vals, cols.astype(np.int32), indptr), shape=(cfg.users, cfg.items))


def split_holdout(mat: sp.csr_matrix, fractions=(0.9, 0.05, 0.05), seed: int = 0):
    """Seeded train/validation/test split of a CSR matrix's stored ratings.

    Same rule as the reference (pkg/src/svdrec/data.py:212-225): validation
    and test sizes are the rounded fractions, ``rng.permutation(total)``
    with ``np.random.default_rng(seed)`` orders the samples (here: CSR
    order), train takes the head.  Returns ``(train_csr, val, test)`` where
    val/test are ``(users int64, items int64, ratings float64)`` arrays.
    """
    total = mat.nnz
    n_val = round(fractions[1] * total)
    n_test = round(fractions[2] * total)
    n_train = total - n_val - n_test
    if min(n_train, n_val, n_test) <= 0:
        raise ValueError("every part of the split must be nonempty")
    order = np.random.default_rng(seed).permutation(total)
    rows = np.repeat(np.arange(mat.shape[0], dtype=np.int64), np.diff(mat.indptr))
    cols = mat.indices.astype(np.int64)
    vals = mat.data
    tr = order[:n_train]
    va = order[n_train:n_train + n_val]
    te = order[n_train + n_val:]
    train = sp.coo_matrix((vals[tr], (rows[tr], cols[tr])), shape=mat.shape).tocsr()
    train.sort_indices()
    return train, (rows[va], cols[va], vals[va]), (rows[te], cols[te], vals[te])
