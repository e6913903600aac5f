"""The fp32 variant (BASELINE configs 2 and 4 ask for one): the gathered dense
operands of the SpMMs and of the CF scoring are stored as float, while
accumulation, the QB algebra and the returned values stay double.  Stated
bounds against the fp64 path (itself pinned to the reference): SpMM and
predictions within 1e-6 relative, the selected k identical, MAE traces and
test RMSE within 1e-5 relative."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REL = 1e-6   # single products / predictions
REL_PIPE = 1e-5  # whole Alg. 5 traces (errors compound over blocks)


def test_spmm_fp32_operand(gpu):
    import torch
    import paper_2009_02251_b200 as P
    from paper_2009_02251_b200 import kernels as K, synth
    M = synth.generate(synth.CONFIGS["c0_100k"])
    A = P.SparseRatings(M, 1.0, 5.0)
    d = A.device()
    rng = np.random.default_rng(1)
    for b in (4, 20, 32, 40, 64):
        X = torch.from_numpy(rng.standard_normal((A.n, b))).cuda()
        Y = torch.empty(A.m, b, dtype=torch.float64, device="cuda")
        K.spmm(d.A, X, Y, "fp32")
        ref = M @ X.cpu().numpy()
        np.testing.assert_allclose(Y.cpu().numpy(), ref, rtol=0, atol=REL * np.abs(ref).max())
        Z = torch.from_numpy(rng.standard_normal((A.m, b))).cuda()
        W = torch.empty(A.n, b, dtype=torch.float64, device="cuda")
        K.spmm(d.AT, Z, W, "fp32")
        ref = M.T @ Z.cpu().numpy()
        np.testing.assert_allclose(W.cpu().numpy(), ref, rtol=0, atol=REL * np.abs(ref).max())
    # strided operand (a column block of a wider buffer)
    Xw = torch.from_numpy(rng.standard_normal((A.n, 40))).cuda()
    Y = torch.empty(A.m, 20, dtype=torch.float64, device="cuda")
    K.spmm(d.A, Xw[:, 8:28], Y, "fp32")
    ref = M @ Xw[:, 8:28].cpu().numpy()
    np.testing.assert_allclose(Y.cpu().numpy(), ref, rtol=0, atol=REL * np.abs(ref).max())


def test_cf_scores_fp32_rows(gpu):
    import paper_2009_02251_b200 as P
    import inputs
    train, val, test = inputs.group_model(400, 300, 8, 0.4, seed=3)
    A = P.SparseRatings(train, 1.0, 5.0)
    f, _ = P.auto_latent_factors(A, val, block_size=4, passes=4, seed=1)
    e64 = P.evaluate_errors(A, f, test)
    e32 = P.evaluate_errors(A, f, test, precision="fp32")
    np.testing.assert_allclose(e32, e64, rtol=REL)
    with pytest.raises(ValueError):
        P.evaluate_errors(A, f, test, precision="fp16")


@pytest.mark.parametrize("cfg,split,b", [("c0_100k", (0.8, 0.1, 0.1), 10), ("c1_1m", (0.9, 0.05, 0.05), 20)])
def test_pipeline_fp32_variant(gpu, cfg, split, b):
    import paper_2009_02251_b200 as P
    from paper_2009_02251_b200 import synth
    c = synth.CONFIGS[cfg]
    M = synth.generate(c)
    tr, va, te = synth.split_holdout(M, split, seed=0)
    A = P.SparseRatings(tr, *c.bounds)
    f64, t64 = P.auto_latent_factors(A, va, block_size=b, passes=4, seed=0, max_rank=400)
    f32, t32 = P.auto_latent_factors(A, va, block_size=b, passes=4, seed=0, max_rank=400, precision="fp32")
    assert f32.k == f64.k
    assert [e.k for e in t32] == [e.k for e in t64]
    np.testing.assert_allclose([e.mae for e in t32], [e.mae for e in t64], rtol=REL_PIPE)
    r64 = P.evaluate_errors(A, f64, te)
    r32 = P.evaluate_errors(A, f32, te, precision="fp32")
    np.testing.assert_allclose(r32, r64, rtol=REL_PIPE)
