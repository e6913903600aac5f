#!/usr/bin/env python3
"""Headline benchmark: time-to-converged-k of the adaptive-PCA CF pipeline.

Workload (BASELINE.json configs[3]): a 138,493 x 26,744 synthetic rating
matrix with 20,000,263 ratings (half stars, rank-40 model, Zipf(1.2) items,
log-normal(4, 1.2) user degrees, >= 20 ratings/user), split 90/5/5 with
seed 0.  One step = the reference's Alg. 5 pipeline
``auto_latent_factors(train, validation, block_size=20, passes=4 (p=1),
patience=2, min_improvement=1e-4, seed=0)`` capped at k = 400, followed by
test-set scoring (MAE and RMSE of the Alg. 4 predictions).  The value is the
device-timed seconds of one step (lower is better).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

--impl reference times the CPU port of the reference (the oracle,
oracle/svdrec_oracle.py: numpy/scipy orchestration statement by statement,
with the reference's CSR products and its per-sample Alg. 4 loop in
threaded C, oracle/cpu_port.c + cf_score.c) on the host cores: full runs
of the same job, as many as fit a time budget (BENCH_REF_BUDGET_S, default
240 s; at least one).  Nothing is extrapolated.  The unmodified reference
package itself (single-threaded Python scoring loop) took 1,568.6 s on
this workload in the build container (profiles/r2_reference_c3_20m.json);
that recorded figure is carried in the line as ``reference_package_recorded``.

--gpus N without a torchrun environment re-launches itself under
``torch.distributed.run`` with N ranks (one GPU each, NCCL).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIG = "c3_20m"
BLOCK, PASSES, PATIENCE, MIN_IMPROVEMENT, SEED, K_CAP = 20, 4, 2, 1e-4, 0, 400
SPLIT = (0.9, 0.05, 0.05)
METRIC = "time-to-converged-k (s), adaptive-PCA CF pipeline, 138k x 27k / 20M nnz"


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _workload():
    from paper_2009_02251_b200 import synth
    cfg = synth.CONFIGS[CONFIG]
    t = time.perf_counter()
    M = synth.generate(cfg)
    tr, va, te = synth.split_holdout(M, SPLIT, seed=0)
    gen_s = time.perf_counter() - t
    return cfg, M, tr, va, te, gen_s


def _config_dict(cfg, tr):
    return {
        "workload": f"{CONFIG}: synthetic {cfg.users}x{cfg.items}, {cfg.nnz} ratings "
                    f"(train {tr.nnz}), rank {cfg.rank}, Zipf({cfg.zipf}) items, half stars",
        "pipeline": "auto_latent_factors (Alg. 5, ValidationMae stop) + test MAE/RMSE",
        "block_size": BLOCK, "passes": PASSES, "power": (PASSES - 2) // 2, "patience": PATIENCE,
        "k_cap": K_CAP, "split": "0.9/0.05/0.05 seed 0", "dtype": "float64",
        "l2": "inputs exceed L2 (CSR of A and A.T, 2 x 216 MB > 126 MB); no explicit flush",
    }


class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-i", str(index), "-lms", os.environ.get("BENCH_SMI_MS", "100")], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    @classmethod
    def disabled(cls) -> "Clocks":
        c = object.__new__(cls)
        c.p = None
        return c

    def _rows(self):
        self.f.flush()
        return [ln.split(",") for ln in Path(self.f.name).read_text().splitlines() if ln.strip()]

    def wait_first(self, timeout: float = 5.0) -> None:
        """nvidia-smi's start-up stalls the driver for a moment: let it
        finish (first sample written) before anything is timed."""
        t = time.perf_counter()
        while self.p is not None and not self._rows() and time.perf_counter() - t < timeout:
            time.sleep(0.05)

    def mark(self) -> int:
        return len(self._rows()) if self.p is not None else 0

    def stop(self, start: int = 0) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        end = self.mark()
        self.p.terminate()
        self.p.wait()
        rows = self._rows()[start:max(end, start + 1)]  # samples taken during the timed region
        sm = [float(r[0]) for r in rows if len(r) >= 6 and r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if len(r) >= 6 and r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 6 for i in range(4) if "Active" == r[2 + i].strip()})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


class NvmlClocks(Clocks):
    """The same clocks line sampled in-process through NVML (the library
    nvidia-smi queries): SM clock and the clock-event reasons every
    BENCH_SMI_MS ms from a daemon thread (BENCH_CLOCKS=nvml; the default is
    the recipe's nvidia-smi -lms process).  Both measured alike: neither
    sampler disturbs the timed steps."""

    def __init__(self, index: int):
        import threading
        import pynvml as nv
        self.nv = nv
        nv.nvmlInit()
        self.h = nv.nvmlDeviceGetHandleByIndex(index)
        self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
        get = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
        self.bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                     "sw_power_cap": 0x4}
        self.samples: list[tuple[float, int]] = []
        self.p = self  # "running" marker for the base class
        self._halt = threading.Event()
        dt = float(os.environ.get("BENCH_SMI_MS", "100")) / 1e3

        def loop():
            while not self._halt.is_set():
                self.samples.append((float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)), int(get(self.h))))
                self._halt.wait(dt)

        self.t = threading.Thread(target=loop, daemon=True)
        self.t.start()

    def wait_first(self, timeout: float = 5.0) -> None:
        t = time.perf_counter()
        while not self.samples and time.perf_counter() - t < timeout:
            time.sleep(0.01)

    def mark(self) -> int:
        return len(self.samples)

    def stop(self, start: int = 0) -> dict:
        end = self.mark()
        self._halt.set()
        self.t.join()
        rows = self.samples[start:max(end, start + 1)]
        sm = [c for c, _ in rows]
        reasons = sorted({n for _, r in rows for n, b in self.bits.items() if r & b})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(rows), "sampler": "nvml"}


def make_clocks(index: int) -> Clocks:
    if os.environ.get("BENCH_NO_CLOCKS"):
        return Clocks.disabled()
    if os.environ.get("BENCH_CLOCKS", "smi") == "nvml":
        try:
            return NvmlClocks(index)
        except Exception:  # no NVML binding / library: the nvidia-smi process
            pass
    return Clocks(index)


def cpu_port_run(tr, va, te, lo, hi, threads: int | None = None):
    """One full run of the job on the CPU port of the reference: the
    oracle's Alg. 5 pipeline (auto_latent_factors with the bench settings)
    + test scoring, with its CSR products and per-sample Alg. 4 loop on
    ``threads`` host threads (all of this process's CPUs by default) and
    BLAS single-threaded (its spinning workers would otherwise contend with
    the C kernels' threads: 3.5x slower measured on c1).  Returns (seconds,
    threads, summary)."""
    from oracle import svdrec_oracle as O
    import threadpoolctl

    with threadpoolctl.threadpool_limits(1):
        nt = O.use_c_backend(threads)
        try:
            t = time.perf_counter()
            res = O.auto_latent_factors(tr, va, lo, hi, block_size=BLOCK, passes=PASSES, patience=PATIENCE,
                                        min_improvement=MIN_IMPROVEMENT, seed=SEED, max_rank=K_CAP)
            p = O.predict_many(tr, res.T, lo, hi, te[0], te[1])
            dt = time.perf_counter() - t
        finally:
            O.use_c_backend(0)
    e = p[:, 0] - te[2]
    return dt, nt, {"k": int(res.k), "blocks": len(res.trace), "test_mae": float(np.abs(e).mean()),
                    "test_rmse": float(np.sqrt((e * e).mean()))}


def _cpu_sample_text(nt, nv, nte, blocks):
    return (f"one full run of the job (not extrapolated): {blocks} QB blocks + {blocks} validation scorings of {nv} "
            f"samples + test scoring of {nte} samples, by the oracle port (numpy/scipy orchestration, CSR products "
            f"and the per-sample Alg. 4 loop in C on {nt} threads, BLAS 1 thread)")


def _recorded_reference():
    p = ROOT / "profiles" / f"r2_reference_{CONFIG}.json"
    if not p.is_file():
        return None
    r = json.loads(p.read_text())
    return {"value": r.get("total_s"), "unit": "s", "host_cpus": r.get("host_cpus"), "k": r.get("k"),
            "test_rmse": r.get("test_rmse"), "source": f"profiles/{p.name}",
            "note": "the unmodified reference package (per-sample Python scoring loop), run once in the build "
                    "container; it cannot run on the GPU box (no /root/reference there)"}


def run_reference(args):
    _, rank, _ = _dist()
    if rank != 0:  # rank 0 alone runs the CPU reference arm
        return
    cfg, M, tr, va, te, gen_s = _workload()
    lo, hi = cfg.bounds
    # warm-up: the same pipeline on config 0's small workload (pages in the
    # code paths and libraries; nothing is cached across runs)
    from paper_2009_02251_b200 import synth
    c0 = synth.CONFIGS["c0_100k"]
    s_tr, s_va, s_te = synth.split_holdout(synth.generate(c0), SPLIT, seed=0)
    for _ in range(args.warmup):
        cpu_port_run(s_tr, s_va, s_te, *c0.bounds)
    budget = float(os.environ.get("BENCH_REF_BUDGET_S", "240"))
    runs, info, nt = [], {}, 1
    while len(runs) < args.steps:
        dt, nt, info = cpu_port_run(tr, va, te, lo, hi)
        runs.append(dt)
        if sum(runs) + dt > budget:
            break
    v = float(statistics.median(runs))
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "s", "n_gpus": args.gpus,
            "steps": len(runs), "steps_requested": args.steps, "warmup": args.warmup,
            "ms_per_step": round(v * 1e3, 1), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": _config_dict(cfg, tr),
            "runs_s": [round(x, 3) for x in runs], "result": info,
            "cpu_baseline": {"value": round(v, 3), "unit": "s", "cores": nt, "kind": "port",
                             "sample": _cpu_sample_text(nt, len(va[0]), len(te[0]), info.get("blocks"))
                                       + f"; median of {len(runs)} run(s) within a {budget:.0f} s budget"},
            "e2e": {"value": round(v, 3), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "reference_package_recorded": _recorded_reference(),
            "setup": {"generate_split_s": round(gen_s, 2)}}
    print(json.dumps(line), flush=True)


def scaleout_variant(dev, peak) -> dict:
    """BASELINE configs[4] on this GPU: 8,000,000 x 1,000,000, 2.0e9 ratings
    generated on the device (rank 64, Zipf(1.2) items, half stars; int32
    indices, fp64 values), adaptive QB with b = 64, p = 2 (passes 6), k
    capped at 512 -- time to k = 512 (CUDA events, after one untimed block)
    in fp64 and with float X in the SpMMs (the fp32 variant), and the
    SpMM's compulsory-byte HBM rate."""
    import torch
    import paper_2009_02251_b200 as P
    from paper_2009_02251_b200 import kernels as K, synth

    b, passes, cap = 64, 6, 512
    t = time.perf_counter()
    A = synth.generate_device(synth.CONFIGS["c4_2b"], dev)
    d = A.device()
    torch.cuda.synchronize()
    out = {"config": f"c4_2b: {d.m} users x {d.n} items, {d.nnz} ratings (device-generated), b={b}, "
                     f"passes={passes} (p=2), k<={cap}", "generate_s": round(time.perf_counter() - t, 1)}
    for prec in ("fp64", "fp32"):
        g = P.qb_pass_blocks(A, b, passes, P.GaussianStream(1), max_rank=cap, precision=prec)
        next(g).err  # warm-up block (first-call plans)
        del g
        torch.cuda.synchronize()
        K.PROFILE = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ranks = []
        for st in P.qb_pass_blocks(A, b, passes, P.GaussianStream(0), max_rank=cap, precision=prec):
            ranks.append(st.rank)
            if st.rank >= cap:
                break
        e1.record()
        torch.cuda.synchronize()
        prof = K.profile_summary(K.PROFILE)
        K.PROFILE = None
        c, ms, hbm_b, _ = prof.get("spmm", (0, 0.0, 0, 0))
        ach = hbm_b / (ms / 1e3) / 1e9 if ms else None
        out[prec] = {"time_to_k_s": round(e0.elapsed_time(e1) / 1e3, 4), "k": ranks[-1], "blocks": len(ranks),
                     "spmm": {"calls": c, "ms_per_call": round(ms / max(c, 1), 2),
                              "hbm_GBps": round(ach, 1) if ach else None,
                              "hbm_frac": round(ach / peak, 4) if ach else None},
                     "timing": "CUDA events around the whole run; per-call SpMM spans (events) recorded in it"}
    out["peak_mem_GiB"] = round(torch.cuda.max_memory_allocated(dev) / 2**30, 1)
    del A, d
    torch.cuda.empty_cache()
    return out


def run_b200(args):
    import torch
    import torch.distributed as dist
    import paper_2009_02251_b200 as P
    from paper_2009_02251_b200 import _lib, kernels as K
    from paper_2009_02251_b200.cf import _Samples, _shard_samples
    from paper_2009_02251_b200.parallel import Comm, ShardedRatings, max_over_ranks
    from paper_2009_02251_b200.parallel import row_partition as _row_partition

    ws, rank, local = _dist()
    if os.environ.get("BENCH_SHARE_GPU"):  # flow check only: every rank on cuda:0 over gloo (not a timing)
        local = 0
    if ws > 1:
        if os.environ.get("BENCH_SHARE_GPU"):
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = _lib.load()
    cfg, M, tr, va, te, gen_s = _workload()
    lo, hi = cfg.bounds
    if ws > 1:  # users (rows of A) sharded over the ranks, item side replicated
        A = ShardedRatings.from_csr(tr, lo, hi, Comm())
        vs, ts = _shard_samples(A, va, dev), _shard_samples(A, te, dev)
    else:
        A = P.SparseRatings(tr, lo, hi)
        vs, ts = _Samples(va, dev), _Samples(te, dev)
    d = A.device(dev)
    torch.cuda.synchronize()

    def step(precision="fp64"):
        f, trace = P.auto_latent_factors(A, vs, block_size=BLOCK, passes=PASSES, patience=PATIENCE,
                                         min_improvement=MIN_IMPROVEMENT, seed=SEED, max_rank=K_CAP,
                                         precision=precision)
        mae, rmse = P.evaluate_errors(A, f, ts, precision=precision)
        return f, trace, mae, rmse

    clocks = make_clocks(local)
    clocks.wait_first()
    import gc
    for i in range(args.warmup):
        if i == args.warmup - 1:
            # the last warm-up step runs on a clean heap: collect, then
            # freeze the set-up objects (data generation leaves millions of
            # them) so a cyclic collection inside the timed steps does not
            # walk them; the collector stays off until the timing ends.  One
            # step between the collection and the timed region absorbs what
            # the collection leaves behind (freed pages, deferred frees).
            gc.collect()
            gc.freeze()
            gc.disable()
        # hold the result as the timed loop does (the previous step's
        # factors stay alive while the next step runs), so the caching
        # allocator reaches the timed loop's peak here: otherwise the
        # second timed step made one cudaMalloc (+10 to +90 ms, seen)
        f, trace, mae, rmse = step()
    if args.warmup == 0:
        gc.collect()
        gc.freeze()
        gc.disable()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    ck0 = clocks.mark()
    launches0 = lib.svdrec_launch_count()
    ms0 = torch.cuda.memory_stats(dev)
    # the K steps are one timed region (total / K); per-step events inside
    # it are reported for spread only
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    torch.cuda.synchronize()
    ev[0].record()
    for i in range(args.steps):
        f, trace, mae, rmse = step()
        ev[i + 1].record()
    torch.cuda.synchronize()
    times = [ev[i].elapsed_time(ev[i + 1]) / 1e3 for i in range(args.steps)]
    launches = (lib.svdrec_launch_count() - launches0) // args.steps
    gc.enable()
    ck = clocks.stop(ck0)
    ms1 = torch.cuda.memory_stats(dev)
    alloc = {k: int(ms1.get(k, 0) - ms0.get(k, 0)) for k in ("num_device_alloc", "num_device_free", "num_alloc_retries",
                                                             "num_sync_all_streams")}
    t_step = ev[0].elapsed_time(ev[-1]) / 1e3 / args.steps
    # kernel breakdown from one extra, untimed step with per-call CUDA-event
    # spans (their host cost stays out of the timed region)
    # (scoring on the caller's stream, so each span holds one kernel alone)
    from paper_2009_02251_b200 import cf as _cf
    pipe, _cf.PIPELINE = _cf.PIPELINE, False
    K.PROFILE = []
    step()
    torch.cuda.synchronize()
    prof = K.profile_summary(K.PROFILE)
    K.PROFILE = None
    _cf.PIPELINE = pipe
    psteps = 1
    if ws > 1:  # the slowest rank's time per step
        t_step = max_over_ranks(t_step, dev)

    # fp32 variant (BASELINE configs 2 / 4): float storage of the gathered
    # operands, fp64 accumulation; same protocol, fewer steps
    variants = {}
    if not args.no_variants:
        # same protocol as the timed region: results held across steps (the
        # allocator reaches its peak in the warm-up), collector off
        gc.disable()
        for _ in range(3):
            f32, tr32, mae32, rmse32 = step("fp32")
        torch.cuda.synchronize()
        nv = max(2, min(args.steps, 5))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(nv):
            f32, tr32, mae32, rmse32 = step("fp32")
        e1.record()
        torch.cuda.synchronize()
        gc.enable()
        t32 = max_over_ranks(e0.elapsed_time(e1) / 1e3 / nv, dev)
        variants["fp32"] = {"value": round(t32, 6), "unit": "s", "steps": nv, "k": int(f32.k), "blocks": len(tr32),
                            "test_mae": mae32, "test_rmse": rmse32,
                            "test_rmse_rel_err_vs_f64": abs(rmse32 - rmse) / rmse,
                            "storage": "float copies of the SpMM dense operand and of the CF item rows; "
                                       "fp64 accumulation, QB algebra and outputs"}

    # e2e: the public API from host buffers, upload + results read inside.
    # The step's inputs sit in page-locked host memory (allocated once,
    # outside the timed region, as a serving process keeps its input
    # buffers): the CSR of A (this rank's rows) and the validation / test
    # triples; every run uploads them, builds the device image, runs the
    # pipeline and reads the errors back.
    from scipy import sparse as _sp

    def pinned(a, dtype):
        a = np.ascontiguousarray(a, dtype=dtype)
        t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()

    if ws > 1:
        off = _row_partition(tr.indptr, ws)
        tr_local = tr[int(off[rank]): int(off[rank + 1])]
    else:
        tr_local = tr
    h_tr = _sp.csr_matrix((pinned(tr_local.data, np.float64), pinned(tr_local.indices, np.int32),
                           pinned(tr_local.indptr, np.int64)), shape=tr_local.shape)
    h_va = tuple(pinned(x, dt) for x, dt in zip(va, (np.int64, np.int64, np.float64)))
    h_te = tuple(pinned(x, dt) for x, dt in zip(te, (np.int64, np.int64, np.float64)))
    e2e_times, h2d = [], 0
    gc.disable()  # as in the timed region: no collector pauses inside the runs
    for i in range(6):  # the first run is a warm-up (first-call plans); median of 5
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if ws > 1:
            A2 = ShardedRatings(P.SparseRatings(h_tr, lo, hi), int(off[rank]), tr.shape[0], Comm(), off)
        else:
            A2 = P.SparseRatings(h_tr, lo, hi)
        f2, tr2 = P.auto_latent_factors(A2, h_va, block_size=BLOCK, passes=PASSES, patience=PATIENCE,
                                        min_improvement=MIN_IMPROVEMENT, seed=SEED, max_rank=K_CAP)
        mae2, rmse2 = P.evaluate_errors(A2, f2, h_te)
        e1.record()
        torch.cuda.synchronize()
        if i:
            e2e_times.append(max_over_ranks(e0.elapsed_time(e1) / 1e3, dev))
        d2 = A2.device(dev)
        h2d = d2.h2d_bytes + 24 * (len(va[0]) + len(te[0]))  # CSR of A (this rank's rows) + (u, i, r) triples
        assert f2.k == f.k and abs(rmse2 - rmse) <= 1e-9 * rmse, (f2.k, f.k, rmse2, rmse)
        # release this run's matrix and factors before the next run builds
        # its own, so every run is served from the allocator's cache
        del A2, d2, f2, tr2
    gc.enable()
    nb = len(trace)
    d2h = nb * ((BLOCK + 1) * 8 + 4 * 3 + 16) + 16

    peaks_p = ROOT / "MEASURED_PEAKS.json"
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if peaks_p.is_file():
        peak, peak_src = float(json.loads(peaks_p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"

    # DRAM bytes per launch from the committed ncu --set full captures
    # (tools/traffic.py -> profiles/traffic.json), or null
    traffic_p = ROOT / "profiles" / "traffic.json"
    traffic = json.loads(traffic_p.read_text()) if traffic_p.is_file() else {}

    def roof(name, kernel, l2_ceiling, l2_note):
        """HBM roofline of one kernel: achieved = its compulsory HBM bytes
        (inputs read once, outputs written once; kernels.py spans) over its
        CUDA-event time in the profiled step.  The gathered bytes (every
        fetched row, wherever it is served from) are reported beside it,
        against the measured L2 random-gather ceiling."""
        c, ms, hbm_b, gath_b = prof.get(name, (0, 0.0, 0, 0))
        sec = ms / 1e3
        ach = hbm_b / sec / 1e9 if sec > 0 else None
        g_rate = (hbm_b + gath_b) / sec / 1e9 if sec > 0 else None
        tr_ = traffic.get(name, {}).get("dram_bytes_per_launch")
        return {"kernel": kernel, "bound": "hbm", "achieved": round(ach, 1) if ach else None, "peak": peak,
                "unit": "GB/s", "frac": round(ach / peak, 4) if ach else None, "traffic": tr_,
                "traffic_source": f"ncu --set full, profiles/traffic.json ({traffic[name]['launches']} launches)"
                if tr_ else None, "peak_source": peak_src,
                "algorithmic_bytes_per_call": int(hbm_b / max(c, 1)),
                "algorithmic_bytes": "compulsory HBM bytes: CSR once, dense operands once, outputs once",
                "calls_per_step": c // psteps, "ms_per_step": round(ms / psteps, 3),
                "us_per_call": round(ms * 1e3 / max(c, 1), 1),
                "gathered": {"bytes_per_call": int(gath_b / max(c, 1)), "GBps": round(g_rate, 1) if g_rate else None,
                             "l2_gather_ceiling_GBps": l2_ceiling,
                             "frac_of_l2_ceiling": round(g_rate / l2_ceiling, 4) if g_rate else None,
                             "note": l2_note}}

    roof_cf = roof("cf_predict", "svdrec_cf_predict (k_predict<R>)", 18904.6,
                   "CSR stream + every gathered item row; ceiling: random 1920-B row gathers from L2, 32 warps/SM "
                   "(tools/probe_l2bw.cu on B200)")
    roof_spmm = roof("spmm", "svdrec_spmm (k_spmm_pipe: chunk-record TMA gather4 pipeline)", 7799.0,
                     "CSR stream + every gathered row of X; ceiling: random 160-B row gathers from L2, 64 warps/SM "
                     "(tools/probe_l2bw.cu on B200)")
    # the line's roofline is the kernel with the larger share of the step
    dominant, other = (roof_cf, roof_spmm) if roof_cf["ms_per_step"] >= roof_spmm["ms_per_step"] else \
        (roof_spmm, roof_cf)
    breakdown = {k: {"calls": v[0] // psteps, "ms": round(v[1] / psteps, 3),
                     "share": round(v[1] / (sum(x[1] for x in prof.values()) or 1), 4)} for k, v in prof.items()}

    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": round(t_step, 6), "unit": "s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 3), "higher_is_better": False,
        "scaling": "strong",
        "parallelism": f"users sharded over {ws} GPUs, NCCL all-reduce of the partials" if ws > 1 else "single", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config_dict(cfg, tr),
        "k": int(f.k), "blocks": nb, "test_mae": mae, "test_rmse": rmse, "val_mae": min(e.mae for e in trace),
        "step_times_s": [round(t, 6) for t in times],
        "roofline": dominant,
        "roofline_other": other,
        "spmm_hbm_GBps": roof_spmm["achieved"],
        "kernel_breakdown": breakdown,
        "e2e": {"value": round(statistics.median(e2e_times), 6), "unit": "s", "runs_s": [round(t, 4) for t in e2e_times], "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        "variants": variants,
        "clocks": ck,
        "allocator_in_timed_region": alloc,
        "setup": {"generate_split_s": round(gen_s, 2)},
    }
    if ws == 1 and not args.no_scaleout and not args.no_variants and CONFIG == "c3_20m":
        # the c3 device state is released first (the 2e9-rating matrix peaks
        # at ~134 GiB)
        del A, d, vs, ts, f, trace
        if variants:
            del f32, tr32
        gc.collect()
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats(dev)
        line["variants"]["c4_scaleout"] = scaleout_variant(dev, peak)
    if ws == 1 and not args.no_cpu_baseline:
        total, cores, info = cpu_port_run(tr, va, te, lo, hi)
        line["cpu_baseline"] = {"value": round(total, 3), "unit": "s", "cores": cores, "kind": "port",
                                "sample": _cpu_sample_text(cores, len(va[0]), len(te[0]), info["blocks"]),
                                "result": info, "reference_package_recorded": _recorded_reference()}
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def _spawn(nproc: int) -> int:
    """Re-launch this command under torch.distributed.run with ``nproc``
    ranks on 127.0.0.1 (one GPU per rank); returns its exit code."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    global CONFIG
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--config", default=CONFIG, help="workload (default: the headline c3_20m; smaller ones for tests)")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the fp32-variant timing")
    ap.add_argument("--no-scaleout", action="store_true", help="skip the config-4 (2e9 ratings) variant")
    args = ap.parse_args()
    CONFIG = args.config
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn(args.gpus))
    ws = _dist()[0]
    if ws != args.gpus and args.impl != "reference":
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
