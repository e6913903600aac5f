"""Row-sharded engine (parallel.py) through the product path: two ranks.

Both ranks run on cuda:0 with the ``gloo`` backend (gpurun grants one GPU;
the collectives are host-mediated, so no kernel waits on another rank's
kernel).  On an 8-GPU box the same code runs with NCCL, one GPU per rank.
Each rank also runs the unsharded single-GPU path (itself parity-pinned to
the reference goldens) and the results are compared: same selected k and
MAE traces, B equal up to the sign of each row (QR uniqueness), Q's
gathered rows equal up to column signs, replicated state bitwise equal on
both ranks.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

WORLD = 2


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _matrix(P, kind):
    import inputs
    if kind == "rand":
        _, A = inputs.rand_sparse(310, 190, 0.09, seed=11)
        return P.SparseRatings(A, 0.5, 5.0), None
    train, val, test = inputs.group_model(400, 300, 8, 0.4, seed=3)
    return P.SparseRatings(train, 1.0, 5.0), (val, test)


def _engine_case(P, rank, comm, gen_name, arg):
    from paper_2009_02251_b200.parallel import ShardedRatings
    A, _ = _matrix(P, "rand")
    S = ShardedRatings.from_full(A, comm)
    gen = getattr(P, gen_name)
    out = {}
    for blk, (s1, s2) in enumerate(zip(gen(A, 10, arg, P.GaussianStream(5)),
                                       gen(S, 10, arg, P.GaussianStream(5))), 1):
        out[f"err1_{blk}"] = s1.err
        out[f"err2_{blk}"] = s2.err
        out[f"rowE1_{blk}"] = s1.row_energy
        out[f"rowE2_{blk}"] = s2.row_energy
        out[f"B1_{blk}"] = s1.B
        out[f"B2_{blk}"] = s2.B
        out[f"Q1_{blk}"] = s1.Q
        out[f"Q2_{blk}"] = comm.gather_rows(s2.Q_device, S.counts).cpu().numpy()
        if blk == 4:
            break
    out["frob"] = S.frob_sq
    out["row0"], out["row1"] = S.row0, S.row1
    return out


def _cf_case(P, rank, comm):
    from paper_2009_02251_b200.parallel import ShardedRatings
    A, (val, test) = _matrix(P, "model")
    S = ShardedRatings.from_full(A, comm)
    f1, t1 = P.auto_latent_factors(A, val, block_size=3, passes=4, seed=2)
    f2, t2 = P.auto_latent_factors(S, val, block_size=3, passes=4, seed=2)
    e1 = P.evaluate_errors(A, f1, test)
    e2 = P.evaluate_errors(S, f2, test)
    return {"k1": f1.k, "k2": f2.k, "mae1": [t.mae for t in t1], "mae2": [t.mae for t in t2],
            "test1": e1, "test2": e2, "Xn2": f2.Xn.cpu().numpy(), "Yn2": f2.Yn.cpu().numpy(),
            "Xn1": f1.Xn.cpu().numpy()}


def _apca_case(P, rank, comm, passes):
    """adaptive_pca of a TALL matrix (m > n: the reference transposes,
    rsvd.py:359) on row shards -> the column-sharded engine over A.T."""
    import inputs
    from paper_2009_02251_b200.parallel import ShardedRatings
    from paper_2009_02251_b200.sparse import TransposedRatings
    _, M = inputs.rand_sparse(420, 150, 0.1, seed=17)
    A = P.SparseRatings(M, 0.5, 5.0)
    S = ShardedRatings.from_full(A, comm)
    out = {"row0": S.row0, "row1": S.row1}
    for name, crit in (("tol", P.FrobTolerance(0.5)), ("fixed", P.FixedRank(23))):
        r1 = P.adaptive_pca(A, crit, block_size=8, passes=passes, seed=4)
        r2 = P.adaptive_pca(S, crit, block_size=8, passes=passes, seed=4)
        out[f"{name}_k1"], out[f"{name}_k2"] = r1.k, r2.k
        out[f"{name}_s1"], out[f"{name}_s2"] = r1.s, r2.s
        out[f"{name}_u1"], out[f"{name}_u2"] = r1.u[S.row0:S.row1], r2.u
        out[f"{name}_v1"], out[f"{name}_v2"] = r1.v, r2.v
    # Alg. 2 power steps on the column-sharded view (sharded m-side orth)
    g1 = P.qb_power_blocks(TransposedRatings(A), 8, 1, P.GaussianStream(6))
    g2 = P.qb_power_blocks(S.transposed(), 8, 1, P.GaussianStream(6))
    for blk, (s1, s2) in enumerate(zip(g1, g2), 1):
        out[f"pw_err1_{blk}"], out[f"pw_err2_{blk}"] = s1.err, s2.err
        out[f"pw_Q1_{blk}"], out[f"pw_Q2_{blk}"] = s1.Q, s2.Q
        if blk == 3:
            break
    out["frob"] = S.frob_sq
    return out


def _worker(rank, world, port, outdir, case, arg):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests" / "golden"))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2009_02251_b200 as P
        from paper_2009_02251_b200.parallel import Comm
        comm = Comm()
        if case == "cf":
            res = _cf_case(P, rank, comm)
        elif case == "apca":
            res = _apca_case(P, rank, comm, arg)
        else:
            res = _engine_case(P, rank, comm, case, arg)
        torch.cuda.synchronize()
        np.savez(os.path.join(outdir, f"r{rank}.npz"), **{k: np.asarray(v) for k, v in res.items()})
    finally:
        dist.destroy_process_group()


def _run(tmp_path, case, arg=None, world=WORLD):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), case, arg), nprocs=world, join=True)
    return [dict(np.load(tmp_path / f"r{r}.npz")) for r in range(world)]


def _same_up_to_sign(a, b, axis, tol):
    """a, b equal after flipping each row (axis=1) / column (axis=0) of b."""
    dots = np.sum(a * b, axis=axis, keepdims=True)
    sgn = np.where(dots < 0, -1.0, 1.0)
    np.testing.assert_allclose(a, b * sgn, atol=tol)


@pytest.mark.parametrize("case,arg", [("qb_pass_blocks", 4), ("qb_pass_blocks", 3), ("qb_pass_blocks", 5),
                                      ("qb_power_blocks", 1)])
def test_sharded_engine_matches_single_gpu(gpu, tmp_path, case, arg):
    res = _run(tmp_path, case, arg)
    r0, r1 = res
    assert int(r0["row1"]) == int(r1["row0"])  # contiguous, covering shards
    fro = float(r0["frob"])
    for blk in range(1, 5):
        for r in res:
            assert abs(float(r[f"err2_{blk}"]) - float(r[f"err1_{blk}"])) <= 1e-10 * fro
            np.testing.assert_allclose(r[f"rowE2_{blk}"], r[f"rowE1_{blk}"], rtol=1e-8, atol=1e-10 * fro)
            _same_up_to_sign(r[f"B1_{blk}"], r[f"B2_{blk}"], axis=1, tol=1e-9 * np.sqrt(fro))
            _same_up_to_sign(r[f"Q1_{blk}"], r[f"Q2_{blk}"], axis=0, tol=1e-9)
            Q = r[f"Q2_{blk}"]
            assert np.linalg.norm(Q.T @ Q - np.eye(Q.shape[1])) <= 1e-12 * Q.shape[1]
        # replicated item side: bitwise identical on both ranks
        assert np.array_equal(r0[f"B2_{blk}"], r1[f"B2_{blk}"])


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_cf_pipeline_matches_single_gpu(gpu, tmp_path, world):
    res = _run(tmp_path, "cf", world=world)
    for r in res:
        assert int(r["k2"]) == int(r["k1"])
        np.testing.assert_allclose(r["mae2"], r["mae1"], rtol=1e-9)
        np.testing.assert_allclose(r["test2"], r["test1"], rtol=1e-9)
        # item factors equal up to sign per latent column (B rows up to sign)
        _same_up_to_sign(r["Xn1"], r["Xn2"], axis=0, tol=1e-9)
    for r in res[1:]:
        assert np.array_equal(res[0]["Yn2"], r["Yn2"])
        assert np.array_equal(res[0]["mae2"], r["mae2"])


@pytest.mark.parametrize("passes", [4, 5])
def test_sharded_adaptive_pca_tall_matrix(gpu, tmp_path, passes):
    res = _run(tmp_path, "apca", passes)
    fro = float(res[0]["frob"])
    for r in res:
        for name in ("tol", "fixed"):
            assert int(r[f"{name}_k2"]) == int(r[f"{name}_k1"])
            np.testing.assert_allclose(r[f"{name}_s2"], r[f"{name}_s1"], rtol=1e-9)
            _same_up_to_sign(r[f"{name}_v1"], r[f"{name}_v2"], axis=0, tol=1e-8)
            _same_up_to_sign(r[f"{name}_u1"], r[f"{name}_u2"], axis=0, tol=1e-8)
        for blk in range(1, 4):
            assert abs(float(r[f"pw_err2_{blk}"]) - float(r[f"pw_err1_{blk}"])) <= 1e-10 * fro
            _same_up_to_sign(r[f"pw_Q1_{blk}"], r[f"pw_Q2_{blk}"], axis=0, tol=1e-9)
    # the n-side (items) is replicated: bitwise equal on both ranks
    assert np.array_equal(res[0]["tol_v2"], res[1]["tol_v2"])
