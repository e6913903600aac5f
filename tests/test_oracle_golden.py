"""The CPU oracle against the reference's own outputs (tests/golden)."""
from __future__ import annotations

import sys

import numpy as np
import pytest

from conftest import ROOT, golden

sys.path.insert(0, str(ROOT))
from oracle import svdrec_oracle as O  # noqa: E402
from oracle import ziggurat_ref as Z  # noqa: E402
import inputs  # noqa: E402
from paper_2009_02251_b200 import synth  # noqa: E402


def test_gaussian_stream_matches_reference():
    g = golden("gaussian")
    for seed in (0, 7, 2**33 + 5):
        st = O.Stream(seed)
        got = np.concatenate([st.normal(r, c).ravel() for r, c in ((5, 3), (4, 7), (1000, 20), (3, 1))])
        assert np.array_equal(got, g[f"s{seed}"])


def test_transducer_restatement_is_bit_exact():
    """The 3-state parse the GPU kernel runs reproduces numpy bit for bit."""
    g = golden("gaussian")
    for seed in (0, 2**33 + 5):
        ref = g[f"s{seed}"]
        vals, _ = Z.normals(seed, 0, 3000)
        assert np.array_equal(np.array(vals), ref[:3000])


def test_transducer_consumption_matches_numpy():
    import numpy.random as npr

    bg = npr.Philox(key=11)
    gen = npr.Generator(bg)
    gen.standard_normal(777)
    st = bg.state
    consumed = (int(st["state"]["counter"][0]) - 1) * 4 + st["buffer_pos"]
    _, end = Z.normals(11, 0, 777)
    assert end == consumed


def _check_state(prefix, s, g, rtol=1e-9):
    assert s.rank == int(g[f"{prefix}_rank"])
    fro = s.frob_sq
    assert abs(s.err - float(g[f"{prefix}_err"])) <= 1e-10 * fro
    np.testing.assert_allclose(s.Q @ s.B, g[f"{prefix}_QB"], atol=1e-9 * np.sqrt(fro))
    np.testing.assert_allclose(np.linalg.svd(s.B, compute_uv=False), g[f"{prefix}_svals"], rtol=rtol, atol=1e-10)
    # row energies are only basis-sign invariant, which both QRs share
    np.testing.assert_allclose(np.einsum("ij,ij->i", s.B, s.B), g[f"{prefix}_rowE"], rtol=1e-7, atol=1e-9 * fro)


@pytest.mark.parametrize("power", [0, 1, 2])
def test_power_engine_golden(power):
    g = golden("engines")
    _, A = inputs.rand_sparse(120, 150, 0.08, seed=1)
    for blk, s in enumerate(O.power_blocks(A, 15, power, O.Stream(3)), 1):
        _check_state(f"pow{power}_b{blk}", s, g)
        if blk == 3:
            break


@pytest.mark.parametrize("passes", [3, 4, 5, 10])
def test_pass_engine_golden(passes):
    g = golden("engines")
    _, A = inputs.rand_sparse(120, 150, 0.08, seed=1)
    for blk, s in enumerate(O.pass_blocks(A, 15, passes, O.Stream(4)), 1):
        _check_state(f"pass{passes}_b{blk}", s, g)
        if blk == 3:
            break


def test_drivers_golden():
    g = golden("drivers")
    _, A = inputs.rand_sparse(100, 140, 0.07, seed=50)
    s = O.fixed_precision_qb(A, 0.6, block_size=12, power=1, seed=5)
    _check_state("fpqb_rand", s, g)
    _, A = inputs.exact_rank(90, 70, 5, seed=51)
    assert O.fixed_precision_qb(A, 1e-6, block_size=20, power=0, seed=0).rank == int(g["fpqb_exact_rank"])
    _, A = inputs.rand_sparse(110, 160, 0.07, seed=70)
    u, s, v, k = O.adaptive_pca(A, ("tol", 0.6), block_size=12, passes=10, seed=0)
    assert k == int(g["apca_tol_k"])
    np.testing.assert_allclose(s, g["apca_tol_s"], rtol=1e-10)
    np.testing.assert_allclose((u * s) @ v.T, g["apca_tol_recon"], atol=1e-9)
    _, A = inputs.decay(100, 120, 0.7, seed=71)
    u, s, v, k = O.adaptive_pca(A, ("rank", 10), block_size=5, passes=10, seed=6)
    np.testing.assert_allclose(s, g["apca_rank_s"], rtol=1e-10)
    _, A = inputs.exact_rank(150, 40, 6, seed=72)
    u, s, v, k = O.adaptive_pca(A, ("tol", 1e-7), block_size=6, passes=10, seed=7)
    assert k == int(g["apca_tall_k"])
    np.testing.assert_allclose(s, g["apca_tall_s"], rtol=1e-8)
    _, A = inputs.rand_sparse(90, 130, 0.1, seed=73)
    u, s, v, k = O.adaptive_pca(A, lambda st: st.blocks >= 3, block_size=7, passes=6, seed=8)
    assert k == int(g["apca_cb_k"])
    np.testing.assert_allclose(s, g["apca_cb_s"], rtol=1e-10)
    _, A = inputs.decay(100, 80, 0.7, seed=61)
    _, s, _ = O.basic_rsvd(A, 10, power=6, oversample=10, seed=3)
    np.testing.assert_allclose(s, g["basic_s"], rtol=1e-10)


def test_config0_drivers_golden():
    g = golden("drivers")
    A = synth.generate(synth.CONFIGS["c0_100k"])
    u, s, v, k = O.adaptive_pca(A, ("tol", 0.5), block_size=10, passes=4, seed=0)
    assert k == int(g["c0_apca_k"])
    np.testing.assert_allclose(s, g["c0_apca_s"], rtol=1e-9)
    st = O.fixed_precision_qb(A, 0.5, block_size=10, power=1, seed=0)
    assert st.rank == int(g["c0_fpqb_k"])
    np.testing.assert_allclose(np.linalg.svd(st.B, compute_uv=False), g["c0_fpqb_svals"], rtol=1e-9)


def test_linalg_golden():
    g = golden("linalg")
    q = O.orth(g["qr_in"])
    np.testing.assert_allclose(q @ q.T, g["qr_q"] @ g["qr_q"].T, atol=1e-12)
    np.testing.assert_allclose(O.lu_basis(g["lu_in"]), g["lu_pl"], atol=1e-13)
    u, s, v = O.eig_svd(g["eig_in"])
    np.testing.assert_allclose(s, g["eig_s"], rtol=1e-12)


def test_cf_golden():
    g = golden("cf")
    train, val, test = inputs.group_model(240, 200, 6, 0.7, seed=0)
    res = O.auto_latent_factors(train, val, 1.0, 5.0, block_size=2, passes=10, seed=0)
    assert res.k == int(g["auto_k"])
    assert [t[0] for t in res.trace] == list(g["auto_trace_k"])
    np.testing.assert_allclose([t[1] for t in res.trace], g["auto_trace_mae"], rtol=1e-10)
    np.testing.assert_allclose(res.T.T @ res.T, g["auto_T"].T @ g["auto_T"], atol=1e-9)
    p = O.predict_many(train, res.T, 1.0, 5.0, g["pred_users"], g["pred_items"])
    np.testing.assert_allclose(p[:, 0], g["pred_value"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(p[:, 1], g["pred_raw"], rtol=1e-10, atol=1e-12)
    assert np.array_equal(p[:, 2].astype(bool), g["pred_fallback"])
    tp = O.predict_many(train, res.T, 1.0, 5.0, test[0], test[1])
    assert abs(O.mae(tp[:, 0], test[2]) - float(g["auto_test_mae"])) <= 1e-10


def test_config0_cf_golden_and_split():
    g = golden("cf")
    M = synth.generate(synth.CONFIGS["c0_100k"])
    tr, va, te = synth.split_holdout(M, (0.8, 0.1, 0.1), seed=0)
    assert np.array_equal(np.stack(va, 1), g["split_val"])
    assert np.array_equal(np.stack(te, 1), g["split_test"])
    assert np.array_equal(tr.indptr, g["split_train_indptr"])
    res = O.auto_latent_factors(tr, va, 1.0, 5.0, block_size=10, passes=4, seed=0)
    assert res.k == int(g["c0_k"])
    np.testing.assert_allclose([t[1] for t in res.trace], g["c0_trace_mae"], rtol=1e-9)
    tp = O.predict_many(tr, res.T, 1.0, 5.0, te[0], te[1])
    np.testing.assert_allclose(tp[:, 0], g["c0_test_pred"], rtol=1e-9, atol=1e-9)


def test_oracle_full_c1_pipeline_matches_reference():
    """The oracle's Alg. 5 + Alg. 4 on BASELINE config 1 (6040 x 3706, 1M
    ratings; 90/5/5 split) against the reference's own full run
    (tests/golden/full_c1_1m.npz): same k and blocks, MAE trace 1e-9,
    test MAE/RMSE 1e-9."""
    from oracle import svdrec_oracle as O
    from paper_2009_02251_b200 import synth

    g = golden("full_c1_1m")
    cfg = synth.CONFIGS["c1_1m"]
    tr, va, te = synth.split_holdout(synth.generate(cfg), (0.9, 0.05, 0.05), seed=0)
    lo, hi = cfg.bounds
    res = O.auto_latent_factors(tr, va, lo, hi, block_size=20, passes=4, patience=2, min_improvement=1e-4, seed=0)
    assert res.k == int(g["k"]) and len(res.trace) == int(g["blocks"])
    np.testing.assert_allclose([t[1] for t in res.trace], g["trace_mae"], rtol=1e-9)
    pred = O.predict_many(tr, res.T, lo, hi, te[0], te[1])[:, 0]
    assert abs(np.abs(pred - te[2]).mean() - float(g["test_mae"])) <= 1e-9
    assert abs(np.sqrt(np.mean((pred - te[2]) ** 2)) - float(g["test_rmse"])) <= 1e-9
