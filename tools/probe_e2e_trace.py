"""GPU idle time inside one end-to-end run (pinned host inputs -> device
image -> Alg. 5 pipeline -> test errors), from a torch.profiler (CUPTI)
trace: kernel/memcpy intervals on the device, the gaps between them and
the host ranges (record_function labels) active during each large gap.
python tools/probe_e2e_trace.py   (GPU box)"""
import sys
from pathlib import Path

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile, record_function

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2009_02251_b200 as P  # noqa: E402
from paper_2009_02251_b200 import cf, sparse  # noqa: E402
from scipy import sparse as sp  # noqa: E402

cfg, M, tr, va, te, _ = bench._workload()
lo, hi = cfg.bounds


def pinned(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


h_tr = sp.csr_matrix((pinned(tr.data, np.float64), pinned(tr.indices, np.int32), pinned(tr.indptr, np.int64)),
                     shape=tr.shape)
h_va = tuple(pinned(x, dt) for x, dt in zip(va, (np.int64, np.int64, np.float64)))
h_te = tuple(pinned(x, dt) for x, dt in zip(te, (np.int64, np.int64, np.float64)))

# label the host stages
for owner, name in [(sparse.SparseRatings, "__init__"), (sparse.DeviceRatings, "_init_from"),
                    (sparse.DeviceCSR, "transposed"), (sparse.DeviceCSR, "ranked"), (sparse.DeviceCSR, "__init__"),
                    (cf._Samples, "__init__"), (cf._Samples, "plan_for"), (cf.ValidationMae, "__init__"),
                    (cf.ValidationMae, "submit"), (cf.ValidationMae, "collect")]:
    fn = getattr(owner, name)

    def wrap(fn=fn, label=f"{owner.__name__}.{name}"):
        def w(*a, **k):
            with record_function(label):
                return fn(*a, **k)
        return w
    setattr(owner, name, wrap())


def run():
    A = P.SparseRatings(h_tr, lo, hi)
    f, trace = P.auto_latent_factors(A, h_va, block_size=bench.BLOCK, passes=bench.PASSES, patience=bench.PATIENCE,
                                     min_improvement=bench.MIN_IMPROVEMENT, seed=bench.SEED, max_rank=bench.K_CAP)
    return P.evaluate_errors(A, f, h_te)


run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    with record_function("e2e"):
        run()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
host = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU and
        (e.name.startswith(("SparseRatings", "DeviceRatings", "DeviceCSR", "_Samples", "ValidationMae", "e2e")))]
t0 = min(s for s, _, _ in iv)
t1 = max(e for _, e, _ in iv)
busy, cur_s, cur_e = 0.0, None, None
gaps = []
for s, e, n in iv:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            gaps.append((cur_e, s))
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
e2e = [h for h in host if h.name == "e2e"][0]
print(f"host e2e {(e2e.time_range.end - e2e.time_range.start) / 1e3:.2f} ms | device span {(t1 - t0) / 1e3:.2f} ms | "
      f"device busy {busy / 1e3:.2f} ms | first device op at +{(t0 - e2e.time_range.start) / 1e3:.2f} ms")
big = sorted(gaps, key=lambda g: -(g[1] - g[0]))[:15]
for a, b in sorted(big):
    act = [h.name for h in host if h.time_range.start <= a and h.time_range.end >= b and h.name != "e2e"]
    print(f"  gap +{(a - t0) / 1e3:7.2f} ms  {(b - a) / 1e3:6.2f} ms  host: {', '.join(act[-2:]) or '-'}")
# device time by kernel / copy name
import collections  # noqa: E402
agg = collections.defaultdict(lambda: [0, 0.0])
for s, e, n in iv:
    agg[n[:80]][0] += 1
    agg[n[:80]][1] += (e - s) / 1e3
print("device time by op (ms):")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
    print(f"  {t:8.3f} ms x{c:4d}  {n}")
