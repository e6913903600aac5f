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
    # scale-out: generated on the device (generate_device), fp32-range values
    "c4_2b": SynthConfig("c4_2b", 8_000_000, 1_000_000, 2_000_000_000, 64, 1.2, True),
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


def generate_device(cfg: SynthConfig, device=None, scale: float = 1.0, chunk_nnz: int = 1 << 27):
    """The same rating model drawn on the GPU (for the scale-out config,
    whose 2e9 ratings the host generator cannot build in reasonable time).

    ``scale`` shrinks the users and the rating count together (items stay:
    the dense item-side operands keep their size, so the SpMM gathers stay
    out of L2).  Degrees come from the host rule (_degrees); each user's
    items are drawn ~ Zipf over a seeded permutation, with replacement and
    re-drawn until ``deg`` distinct ones are held (heavy users by Gumbel
    top-k), values as in :func:`generate`.  A different random stream than
    :func:`generate` (torch's device Philox), so the matrix differs from a
    host-generated one of the same config.  Returns a
    :class:`sparse.DeviceSparseRatings` whose CSR never leaves the device.
    """
    import torch

    from .sparse import DeviceCSR, DeviceSparseRatings

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    m = max(1, int(round(cfg.users * scale)))
    nnz = max(m, int(round(cfg.nnz * scale)))
    n = cfg.items
    sub = SynthConfig(cfg.name, m, n, nnz, cfg.rank, cfg.zipf, cfg.half_stars, cfg.lognorm_mu, cfg.lognorm_sigma,
                      cfg.min_per_user, cfg.noise, cfg.seed)
    rng = np.random.default_rng(np.random.SeedSequence([cfg.seed, m, n, nnz, 4]))
    deg_h = _degrees(sub, rng)
    g = torch.Generator(device=dev)
    g.manual_seed(int(rng.integers(1 << 62)))
    deg = torch.from_numpy(deg_h).to(dev)
    ranks_w = torch.arange(1, n + 1, dtype=torch.float64, device=dev).pow_(-cfg.zipf)
    cdf = torch.cumsum(ranks_w, 0)
    cdf /= cdf[-1].clone()
    logw = torch.log(ranks_w)
    perm = torch.randperm(n, generator=g, device=dev)
    indptr = torch.zeros(m + 1, dtype=torch.int64, device=dev)
    torch.cumsum(deg, 0, out=indptr[1:])
    total = int(indptr[-1].item())
    indices = torch.empty(total, dtype=torch.int32, device=dev)
    heavy_cut = max(64, n // 16)
    # user chunks of ~chunk_nnz ratings
    bounds = np.searchsorted(np.cumsum(deg_h), np.arange(chunk_nnz, total + chunk_nnz, chunk_nnz), side="right")
    starts = np.concatenate([[0], np.minimum(bounds + 1, m)])
    starts = np.unique(np.minimum(starts, m))
    if starts[-1] != m:
        starts = np.append(starts, m)
    for u0, u1 in zip(starts[:-1], starts[1:]):
        u0, u1 = int(u0), int(u1)
        dchunk = deg[u0:u1]
        heavy = torch.nonzero(dchunk > heavy_cut).flatten()
        light_need = torch.where(dchunk > heavy_cut, torch.zeros_like(dchunk), dchunk)
        keys = torch.empty(0, dtype=torch.int64, device=dev)
        need = light_need.clone()
        for _ in range(64):
            users = torch.nonzero(need > 0).flatten()
            if users.numel() == 0:
                break
            cnt = 2 * need[users] + 2
            rows = torch.repeat_interleave(users, cnt)
            r = torch.searchsorted(cdf, torch.rand(rows.numel(), generator=g, device=dev, dtype=torch.float64),
                                   right=True).clamp_(max=n - 1)
            cand = rows * n + perm[r]
            keys = torch.unique(torch.cat([keys, cand]))  # sorted, distinct
            have = torch.bincount(keys // n, minlength=u1 - u0)
            need = torch.clamp(light_need - have, min=0)
        # keep a random subset of deg distinct items for over-full users
        ku = keys // n
        pri = torch.rand(keys.numel(), generator=g, device=dev)
        order = torch.argsort(ku * 2.0 + pri)  # by user, random within user (pri < 1)
        keys, ku = keys[order], ku[order]
        first = torch.searchsorted(ku, ku, right=False)
        keys = keys[(torch.arange(keys.numel(), device=dev) - first) < light_need[ku]]
        parts = [keys]
        for h in heavy.tolist():
            gum = logw - torch.log(-torch.log(torch.rand(n, generator=g, device=dev, dtype=torch.float64)))
            top = torch.topk(gum, int(dchunk[h].item())).indices
            parts.append(h * n + perm[top])
        keys = torch.sort(torch.cat(parts)).values
        a, b = int(indptr[u0].item()), int(indptr[u1].item())
        if keys.numel() != b - a:
            raise RuntimeError(f"generator: {keys.numel()} ratings for users [{u0}, {u1}), expected {b - a}")
        indices[a:b] = (keys % n).to(torch.int32)
        del keys
    sd = (1.0 / np.sqrt(cfg.rank)) ** 0.5
    U = torch.randn(m, cfg.rank, generator=g, device=dev, dtype=torch.float64).mul_(sd)
    V = torch.randn(n, cfg.rank, generator=g, device=dev, dtype=torch.float64).mul_(sd)
    values = torch.empty(total, dtype=torch.float64, device=dev)
    rows_all = None
    step = 1 << 22
    lo, hi = cfg.bounds
    for s0 in range(0, total, step):
        s1 = min(total, s0 + step)
        rows_all = torch.searchsorted(indptr, torch.arange(s0, s1, device=dev), right=True) - 1
        cols = indices[s0:s1].to(torch.int64)
        v = (U[rows_all] * V[cols]).sum(1)
        v += 3.5 + cfg.noise * torch.randn(s1 - s0, generator=g, device=dev, dtype=torch.float64)
        v = torch.round(v * 2.0) / 2.0 if cfg.half_stars else torch.round(v)
        values[s0:s1] = v.clamp_(lo, hi)
    del U, V, rows_all
    csr = DeviceCSR(indptr, indices, values, (m, n))
    return DeviceSparseRatings(csr, lo, hi)
