"""Scale-out configuration (BASELINE configs[4]) on one B200.

8,000,000 users x 1,000,000 items, 2.0e9 ratings (rank-64 model, Zipf(1.2)
items, half stars), generated on the device; adaptive QB with block size
64, p = 2 (passes = 6), k capped at 512.  ``--scale f`` keeps the items and
scales users and ratings by f (the dense item-side operand, 1e6 x 64
doubles = 512 MB, stays out of L2 either way, so the SpMM gathers are
HBM-bound).  The CSR is fp64 values / int32 indices (12 B per rating; the
config names fp32 values -- this path computes in the reference's fp64).

Reports one JSON line: time to k = 512 (device-timed), per-block times, the
SpMM launches' time and bytes -- algorithmic HBM bytes (CSR stream + X + Y)
and gathered bytes -- against the measured HBM peak, and the CPU oracle
timed on a 1/64 row subsample (first two blocks, with the GPU's result on
the same subsample checked against it).

  python tools/scaleout.py [--scale 1.0] [--no-oracle]      (GPU box)
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2009_02251_b200 as P  # noqa: E402
from paper_2009_02251_b200 import kernels as K, synth  # noqa: E402

B, PASSES, K_CAP = 64, 6, 512


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--sub", type=int, default=64, help="oracle row subsample 1/sub")
    ap.add_argument("--precision", choices=("fp64", "fp32"), default="fp64",
                    help="fp32: the SpMMs gather float copies of their dense operand")
    args = ap.parse_args()
    dev = torch.device("cuda")
    cfg = synth.CONFIGS["c4_2b"]
    t = time.perf_counter()
    A = synth.generate_device(cfg, dev, scale=args.scale)
    d = A.device()
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t
    mem_gen = torch.cuda.max_memory_allocated() / 2**30
    torch.cuda.reset_peak_memory_stats()
    m, n = A.shape
    # QB to k = 512 (warm-up: one block on a fresh stream, then the timed run)
    g = P.qb_pass_blocks(A, B, PASSES, P.GaussianStream(1), max_rank=K_CAP, precision=args.precision)
    next(g).err
    del g
    torch.cuda.synchronize()
    K.PROFILE = []
    ev = [torch.cuda.Event(enable_timing=True)]
    ev[0].record()
    errs, ranks = [], []
    for s in P.qb_pass_blocks(A, B, PASSES, P.GaussianStream(0), max_rank=K_CAP, precision=args.precision):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        ev.append(e)
        ranks.append(s.rank)
        if s.rank >= K_CAP:
            break
    torch.cuda.synchronize()
    total_s = ev[0].elapsed_time(ev[-1]) / 1e3
    block_s = [ev[i].elapsed_time(ev[i + 1]) / 1e3 for i in range(len(ev) - 1)]
    prof = K.profile_summary(K.PROFILE)
    K.PROFILE = None
    s._engine.flush()
    errs = [float(x) for x in s._engine.errs]
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").is_file() else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    c, ms, _, _ = prof.get("spmm", (0, 0.0, 0, 0))
    # per SpMM call: CSR stream + one pass over X + Y (algorithmic HBM bytes);
    # the gathered row bytes (nnz x 8b) are what the kernel actually moves
    # through L2 (X is 512 MB, out of L2: the cold rows come from HBM)
    csr_b = A.nnz * 12
    alg = csr_b + (m + n) * B * 8
    gathered = A.nnz * B * (4 if args.precision == "fp32" else 8)
    per_call_ms = ms / max(c, 1)
    line = {
        "config": f"c4_2b x {args.scale:g}: {m} users x {n} items, {A.nnz} ratings, rank 64, Zipf(1.2), half stars "
                  f"(device-generated)",
        "precision": args.precision,
        "qb": {"block_size": B, "passes": PASSES, "power": (PASSES - 2) // 2, "k_cap": K_CAP, "k": ranks[-1],
               "blocks": len(ranks)},
        "time_to_k_s": round(total_s, 4), "block_s": [round(x, 4) for x in block_s],
        "err_over_frob": [e / d.frob_sq for e in errs][: len(ranks)],
        "spmm": {"calls": c, "ms_per_call": round(per_call_ms, 3), "share_of_qb": round(ms / 1e3 / total_s, 3),
                 "algorithmic_hbm_bytes_per_call": alg,
                 "algorithmic_hbm_GBps": round(alg / (per_call_ms / 1e3) / 1e9, 1),
                 "hbm_frac": round(alg / (per_call_ms / 1e3) / 1e9 / hbm, 4),
                 "gathered_bytes_per_call": gathered,
                 "gathered_GBps": round((csr_b + gathered) / (per_call_ms / 1e3) / 1e9, 1),
                 "gathered_frac_of_hbm_peak": round((csr_b + gathered) / (per_call_ms / 1e3) / 1e9 / hbm, 4),
                 "hbm_peak_GBps": hbm},
        "kernel_ms": {k: round(v[1], 2) for k, v in prof.items()},
        "generate_s": round(gen_s, 1), "peak_mem_GiB": {"generate": round(mem_gen, 1),
                                                         "qb": round(torch.cuda.max_memory_allocated() / 2**30, 1)},
    }
    if not args.no_oracle:
        from oracle import svdrec_oracle as O
        import threadpoolctl
        rows = m // args.sub
        H = A.to_host(0, rows)
        sub_gpu = P.SparseRatings(H.matrix, H.rating_min, H.rating_max)
        t = time.perf_counter()
        o = O.pass_blocks(H.matrix, B, PASSES, O.Stream(0))
        so = [next(o), next(o)]
        cpu_s = time.perf_counter() - t
        gg = P.qb_pass_blocks(sub_gpu, B, PASSES, P.GaussianStream(0))
        sg = [next(gg), next(gg)]
        fro = O.frob2(H.matrix)
        err_dev = max(abs(a.err - b.err) / fro for a, b in zip(sg, so))
        Bg, Bo = sg[1].B, so[1].B
        sgn = np.where(np.sum(Bg * Bo, axis=1, keepdims=True) < 0, -1.0, 1.0)
        b_dev = float(np.abs(Bg * sgn - Bo).max() / np.sqrt(fro))
        info = threadpoolctl.threadpool_info()
        line["cpu_baseline"] = {"value": round(cpu_s, 2), "unit": "s", "kind": "port",
                                "cores": max([i.get("num_threads", 1) for i in info] + [1]),
                                "sample": f"oracle: first 2 QB blocks (b={B}, passes={PASSES}) on rows [0, {rows}) "
                                          f"= 1/{args.sub} of the users, {H.nnz} ratings"}
        line["parity_subsample"] = {"err_rel_diff": err_dev, "B_rows_up_to_sign_max_rel": b_dev,
                                    "bound": "1e-10 (err), 1e-9 (B)"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
