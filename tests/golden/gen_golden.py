"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/gen_golden.py [--big]

It imports ``svdrec`` from /root/reference/pkg/src, feeds it the seeded
inputs of ``tests/golden/inputs.py`` / ``paper_2009_02251_b200.synth`` and
stores only outputs as ``tests/golden/*.npz``.  The fixtures travel with the
repo; nothing at test time reads /root/reference.

``--big`` also regenerates the BASELINE config-1 (6040x3706, 1M nnz)
fixed-precision fixtures (about two minutes).
"""
from __future__ import annotations

import argparse
import itertools
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(HERE))

import svdrec  # noqa: E402  (the reference)
from svdrec import (  # noqa: E402
    FixedRank, FrobTolerance, GaussianStream, LatentFactors, RatingSample,
    RatingsDataset, SparseRatings, SplitSpec, adaptive_pca, auto_latent_factors,
    basic_rsvd, eig_svd, evaluate_mae, fixed_precision_qb, latent_from_qb,
    lu_lower_basis, orthonormal_basis, predict_rating, qb_pass_blocks,
    qb_power_blocks, split,
)

import inputs  # noqa: E402
from paper_2009_02251_b200 import synth  # noqa: E402


def R(csr, lo=None, hi=None):
    if lo is None:
        lo, hi = (float(csr.data.min()), float(csr.data.max())) if csr.nnz else (0.0, 0.0)
    return SparseRatings(csr.tocsr(), lo, hi)


def save(name, **arrays):
    np.savez_compressed(HERE / f"{name}.npz", **arrays)
    print("wrote", name, {k: np.shape(v) for k, v in arrays.items()})


def gen_gaussian():
    out = {}
    for seed in (0, 7, 2**33 + 5):
        st = GaussianStream(seed)
        draws = [st.normal(r, c) for r, c in ((5, 3), (4, 7), (1000, 20), (3, 1))]
        out[f"s{seed}"] = np.concatenate([d.ravel() for d in draws])
    save("gaussian", **out)


def _state_arrays(prefix, st, out):
    out[f"{prefix}_err"] = np.float64(st.err)
    out[f"{prefix}_rank"] = np.int64(st.rank)
    out[f"{prefix}_rowE"] = np.einsum("ij,ij->i", st.B, st.B)
    out[f"{prefix}_QB"] = st.Q @ st.B
    out[f"{prefix}_svals"] = np.linalg.svd(st.B, compute_uv=False)


def gen_engines():
    _, A = inputs.rand_sparse(120, 150, 0.08, seed=1)
    out = {}
    for power in (0, 1, 2):
        for blk, st in enumerate(qb_power_blocks(R(A), 15, power, GaussianStream(3)), 1):
            _state_arrays(f"pow{power}_b{blk}", st, out)
            if blk == 3:
                break
    for passes in (3, 4, 5, 10):
        for blk, st in enumerate(qb_pass_blocks(R(A), 15, passes, GaussianStream(4)), 1):
            _state_arrays(f"pass{passes}_b{blk}", st, out)
            if blk == 3:
                break
    save("engines", **out)


def gen_drivers():
    out = {}
    _, A = inputs.rand_sparse(100, 140, 0.07, seed=50)
    st = fixed_precision_qb(R(A), 0.6, block_size=12, power=1, seed=5)
    _state_arrays("fpqb_rand", st, out)
    _, A = inputs.exact_rank(90, 70, 5, seed=51)
    st = fixed_precision_qb(R(A), 1e-6, block_size=20, power=0, seed=0)
    out["fpqb_exact_rank"] = np.int64(st.rank)
    _, A = inputs.rand_sparse(110, 160, 0.07, seed=70)
    t = adaptive_pca(R(A), FrobTolerance(0.6), block_size=12, passes=10, seed=0)
    out["apca_tol_k"], out["apca_tol_s"] = np.int64(t.k), t.s
    out["apca_tol_recon"] = t.reconstruct()
    _, A = inputs.decay(100, 120, 0.7, seed=71)
    t = adaptive_pca(R(A), FixedRank(10), block_size=5, passes=10, seed=6)
    out["apca_rank_s"], out["apca_rank_recon"] = t.s, t.reconstruct()
    _, A = inputs.exact_rank(150, 40, 6, seed=72)
    t = adaptive_pca(R(A), FrobTolerance(1e-7), block_size=6, passes=10, seed=7)
    out["apca_tall_k"], out["apca_tall_s"] = np.int64(t.k), t.s
    _, A = inputs.rand_sparse(90, 130, 0.1, seed=73)
    t = adaptive_pca(R(A), lambda s: s.blocks >= 3, block_size=7, passes=6, seed=8)
    out["apca_cb_k"], out["apca_cb_s"] = np.int64(t.k), t.s
    _, A = inputs.decay(100, 80, 0.7, seed=61)
    t = basic_rsvd(R(A), k=10, power=6, oversample=10, seed=3)
    out["basic_s"] = t.s
    # config-0 workload (943x1682, 100k nnz): tolerance run of Alg. 3, q=4
    A = synth.generate(synth.CONFIGS["c0_100k"])
    t = adaptive_pca(R(A, 1.0, 5.0), FrobTolerance(0.5), block_size=10, passes=4, seed=0)
    out["c0_apca_k"], out["c0_apca_s"] = np.int64(t.k), t.s
    st = fixed_precision_qb(R(A, 1.0, 5.0), 0.5, block_size=10, power=1, seed=0)
    out["c0_fpqb_k"], out["c0_fpqb_svals"] = np.int64(st.rank), np.linalg.svd(st.B, compute_uv=False)
    save("drivers", **out)


def gen_linalg():
    rng = np.random.default_rng(5)
    out = {}
    m = rng.standard_normal((40, 6))
    out["qr_in"] = m
    out["qr_q"] = orthonormal_basis(m)
    out["lu_in"] = m
    out["lu_pl"] = lu_lower_basis(m)
    g = rng.standard_normal((30, 5))
    d = eig_svd(g)
    out["eig_in"], out["eig_u"], out["eig_s"], out["eig_v"] = g, d.u, d.s, d.v
    save("linalg", **out)


def gen_cf():
    out = {}
    train, val, test = inputs.group_model(240, 200, 6, 0.7, seed=0)
    A = R(train, 1.0, 5.0)
    vs = [RatingSample(int(u), int(i), float(r)) for u, i, r in zip(*val)]
    ts = [RatingSample(int(u), int(i), float(r)) for u, i, r in zip(*test)]
    f, trace = auto_latent_factors(A, vs, block_size=2, passes=10, seed=0)
    out["auto_k"] = np.int64(f.k)
    out["auto_T"] = f.T
    out["auto_trace_k"] = np.array([e.k for e in trace])
    out["auto_trace_mae"] = np.array([e.mae for e in trace])
    out["auto_test_mae"] = np.float64(evaluate_mae(A, f, ts))
    rng = np.random.default_rng(8)
    us = rng.integers(0, 240, 400)
    it = rng.integers(0, 200, 400)
    p = [predict_rating(A, f, int(u), int(i)) for u, i in zip(us, it)]
    out["pred_users"], out["pred_items"] = us, it
    out["pred_value"] = np.array([x.value for x in p])
    out["pred_raw"] = np.array([x.raw for x in p])
    out["pred_fallback"] = np.array([x.fallback for x in p])
    # config 0 CF pipeline: 80/10/10 split, block 10, q = 4 (p = 1)
    M = synth.generate(synth.CONFIGS["c0_100k"])
    tr, va, te = synth.split_holdout(M, (0.8, 0.1, 0.1), seed=0)
    A0 = R(tr, 1.0, 5.0)
    vs = [RatingSample(int(u), int(i), float(r)) for u, i, r in zip(*va)]
    ts = [RatingSample(int(u), int(i), float(r)) for u, i, r in zip(*te)]
    f, trace = auto_latent_factors(A0, vs, block_size=10, passes=4, seed=0)
    preds = np.array([predict_rating(A0, f, s.user, s.item).value for s in ts])
    out["c0_k"] = np.int64(f.k)
    out["c0_trace_mae"] = np.array([e.mae for e in trace])
    out["c0_test_pred"] = preds
    out["c0_test_mae"] = np.float64(np.abs(preds - te[2]).mean())
    out["c0_test_rmse"] = np.float64(np.sqrt(np.mean((preds - te[2]) ** 2)))
    # the reference's own split on the same samples (CSR order) pins synth.split_holdout
    coo = M.tocoo()
    ds = RatingsDataset(
        user_index={str(i): i for i in range(M.shape[0])},
        item_index={str(j): j for j in range(M.shape[1])},
        samples=[RatingSample(int(i), int(j), float(v)) for i, j, v in zip(coo.row, coo.col, coo.data)],
        rating_min=1.0, rating_max=5.0)
    rtr, rva, rte = split(ds, SplitSpec(0.8, 0.1, 0.1, seed=0))
    out["split_val"] = np.array([(s.user, s.item, s.rating) for s in rva])
    out["split_test"] = np.array([(s.user, s.item, s.rating) for s in rte])
    out["split_train_indptr"] = rtr.indptr
    save("cf", **out)


def gen_big():
    A = synth.generate(synth.CONFIGS["c1_1m"])
    out = {}
    for p in (0, 1, 2):
        st = fixed_precision_qb(R(A, 1.0, 5.0), 0.1, block_size=20, power=p, seed=0)
        out[f"p{p}_k"] = np.int64(st.rank)
        out[f"p{p}_blocks"] = np.int64(st.blocks)
        out[f"p{p}_err"] = np.float64(st.err)
        out[f"p{p}_svals"] = np.linalg.svd(st.B, compute_uv=False)
        print("c1 p", p, st.rank, flush=True)
    save("c1_fpqb", **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    a = ap.parse_args()
    gen_gaussian()
    gen_engines()
    gen_drivers()
    gen_linalg()
    gen_cf()
    if a.big:
        gen_big()


if __name__ == "__main__":
    main()
