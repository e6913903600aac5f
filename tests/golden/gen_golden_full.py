"""Full-size golden fixtures: the REFERENCE's own CF pipeline run to completion.

Run in the build container (where /root/reference exists), one config per
process (each takes minutes to tens of minutes of CPU, single-threaded
Python scoring loop in the reference):

    python tests/golden/gen_golden_full.py c3_20m      # headline, ~30 min
    python tests/golden/gen_golden_full.py c2_10m
    python tests/golden/gen_golden_full.py c1_1m       # + fixed-precision QB -> test RMSE

For each config it imports ``svdrec`` from /root/reference/pkg/src, rebuilds
the seeded synthetic matrix (``paper_2009_02251_b200.synth``, the bench's
workload generator) and split (0.9/0.05/0.05, seed 0), and runs the
reference's ``auto_latent_factors`` (cf.py:257-294) with the bench's
settings: block_size=20, passes=4, patience=2, min_improvement=1e-4,
seed=0.  The test set is then scored exactly as reference ``evaluate_mae``
does (cf.py:178-190: ``_predict`` with the global mean per sample), keeping
every prediction for the RMSE.

Stored (outputs only, ``tests/golden/full_<config>.npz``): chosen k, the MAE
trace (k, mae, seconds), the singular values of the chosen B (= squared row
norms of T = sqrt(S) U^T), T's column norms, test MAE / RMSE, 4096 test
predictions (value, raw, fallback) at seeded indices, and the wall time of
every phase with the host's CPU model and thread settings -- the measured
CPU baseline of the reference package itself (profiles/ cites it).
"""
from __future__ import annotations

import json
import os
import platform
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

import svdrec  # noqa: E402  (the reference)
from svdrec import (  # noqa: E402
    RatingSample, SparseRatings, auto_latent_factors, fixed_precision_qb, latent_from_qb,
)
from svdrec.cf import _predict  # noqa: E402  (what evaluate_mae calls per sample)

from paper_2009_02251_b200 import synth  # noqa: E402

BLOCK, PASSES, PATIENCE, MIN_IMP, SEED = 20, 4, 2, 1e-4, 0
SPLIT = (0.9, 0.05, 0.05)
N_KEEP = 4096


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def score_test(A, f, te):
    """Reference evaluate_mae (cf.py:178-190), keeping every prediction."""
    gmean = float(A.data.mean())
    vals = np.empty(len(te[0]))
    raws = np.empty(len(te[0]))
    fbs = np.empty(len(te[0]), dtype=bool)
    for t, (u, i) in enumerate(zip(te[0].tolist(), te[1].tolist())):
        p = _predict(A, f, u, i, gmean)
        vals[t], raws[t], fbs[t] = p.value, p.raw, p.fallback
    mae = svdrec.mae(vals, te[2])
    rmse = float(np.sqrt(np.mean((vals - te[2]) ** 2)))
    return vals, raws, fbs, mae, rmse


def run(name: str) -> None:
    cfg = synth.CONFIGS[name]
    lo, hi = cfg.bounds
    t0 = time.perf_counter()
    M = synth.generate(cfg)
    tr, va, te = synth.split_holdout(M, SPLIT, seed=0)
    gen_s = time.perf_counter() - t0
    A = SparseRatings(tr, lo, hi)
    vs = [RatingSample(int(u), int(i), float(r)) for u, i, r in zip(va[0].tolist(), va[1].tolist(), va[2].tolist())]
    print(name, "generated", gen_s, flush=True)

    t1 = time.perf_counter()
    f, trace = auto_latent_factors(A, vs, block_size=BLOCK, passes=PASSES, patience=PATIENCE,
                                   min_improvement=MIN_IMP, seed=SEED)
    auto_s = time.perf_counter() - t1
    print(name, "auto k", f.k, "blocks", len(trace), "s", auto_s, flush=True)
    t2 = time.perf_counter()
    vals, raws, fbs, mae, rmse = score_test(A, f, te)
    test_s = time.perf_counter() - t2
    print(name, "test mae", mae, "rmse", rmse, "s", test_s, flush=True)

    keep = np.sort(np.random.default_rng(1).choice(len(te[0]), size=min(N_KEEP, len(te[0])), replace=False))
    sigma = np.einsum("ij,ij->i", f.T, f.T)  # T = sqrt(S) U^T: row norms^2 = singular values of B
    out = dict(
        k=np.int64(f.k), blocks=np.int64(len(trace)),
        trace_k=np.array([e.k for e in trace], dtype=np.int64),
        trace_mae=np.array([e.mae for e in trace]),
        trace_seconds=np.array([e.seconds for e in trace]),
        sigma=sigma, col_norms=f.col_norms,
        test_mae=np.float64(mae), test_rmse=np.float64(rmse),
        keep_idx=keep.astype(np.int64), keep_value=vals[keep], keep_raw=raws[keep], keep_fallback=fbs[keep],
        n_val=np.int64(len(va[0])), n_test=np.int64(len(te[0])), train_nnz=np.int64(tr.nnz),
    )
    timing = {
        "config": name, "reference": "svdrec (/root/reference/pkg/src), unmodified",
        "call": f"auto_latent_factors(train, val, block_size={BLOCK}, passes={PASSES}, patience={PATIENCE}, "
                f"min_improvement={MIN_IMP}, seed={SEED}) + evaluate_mae-equivalent test scoring",
        "auto_latent_factors_s": auto_s, "test_scoring_s": test_s, "total_s": auto_s + test_s,
        "generate_split_s": gen_s, "k": int(f.k), "blocks": len(trace), "test_mae": mae, "test_rmse": rmse,
        "cpu_model": cpu_model(), "host_cpus": os.cpu_count(),
        "threads": {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")},
        "note": "the reference's per-sample scoring loop is single-threaded Python; BLAS calls may use the "
                "threads listed",
    }
    if name == "c1_1m":
        # config 1: fixed-precision QB (eps = 0.1) on the train split, its
        # factors -> test RMSE (cf.py:77-92 latent_from_qb, cf.py:178-190)
        for p in (0, 1, 2):
            t3 = time.perf_counter()
            st = fixed_precision_qb(A, 0.1, block_size=BLOCK, power=p, seed=SEED)
            try:
                fq = latent_from_qb(st)
            except Exception as exc:  # NearSingularError: record it
                out[f"fpqb_p{p}_error"] = np.array(type(exc).__name__)
                print(name, "fpqb", p, "latent failed", exc, flush=True)
                continue
            v2, r2, f2, mae2, rmse2 = score_test(A, fq, te)
            out[f"fpqb_p{p}_k"] = np.int64(st.rank)
            out[f"fpqb_p{p}_svals"] = np.linalg.svd(st.B, compute_uv=False)
            out[f"fpqb_p{p}_test_mae"] = np.float64(mae2)
            out[f"fpqb_p{p}_test_rmse"] = np.float64(rmse2)
            out[f"fpqb_p{p}_keep_value"] = v2[keep]
            timing[f"fpqb_p{p}_s"] = time.perf_counter() - t3
            print(name, "fpqb", p, st.rank, mae2, rmse2, flush=True)
    np.savez_compressed(HERE / f"full_{name}.npz", **out)
    (ROOT / "profiles").mkdir(exist_ok=True)
    (ROOT / "profiles" / f"r2_reference_{name}.json").write_text(json.dumps(timing, indent=1) + "\n")
    print("wrote", name, timing, flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:]:
        run(nm)
