"""One bench step under torch.profiler: GPU busy vs idle, biggest idle gaps.

python tools/probe_timeline.py   (GPU box)
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2009_02251_b200 as P  # noqa: E402
from paper_2009_02251_b200.cf import _Samples  # noqa: E402

cfg, M, tr, va, te, _ = bench._workload()
lo, hi = cfg.bounds
A = P.SparseRatings(tr, lo, hi)
dev = torch.device("cuda")
A.device(dev)
vs, ts = _Samples(va, dev), _Samples(te, dev)


def step():
    f, trace = P.auto_latent_factors(A, vs, block_size=bench.BLOCK, passes=bench.PASSES, patience=bench.PATIENCE,
                                     min_improvement=bench.MIN_IMPROVEMENT, seed=bench.SEED, max_rank=bench.K_CAP)
    return P.evaluate_errors(A, f, ts)


for _ in range(3):
    step()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
out = Path("gpurun_out/timeline.json")
prof.export_chrome_trace(str(out))
ev = json.loads(out.read_text())["traceEvents"]
k = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
t0, t1 = k[0]["ts"], k[-1]["ts"] + k[-1]["dur"]
busy = sum(e["dur"] for e in k)
gaps = []
end = k[0]["ts"] + k[0]["dur"]
for a, b in zip(k, k[1:]):
    g = b["ts"] - max(end, a["ts"] + a["dur"])
    end = max(end, b["ts"] + b["dur"])
    if g > 0:
        gaps.append((g, a["name"][:50], b["name"][:50]))
gaps.sort(reverse=True)
print(f"span {(t1 - t0) / 1e3:.2f} ms, kernel busy {busy / 1e3:.2f} ms, idle {sum(g for g, *_ in gaps) / 1e3:.2f} ms "
      f"in {len(gaps)} gaps, {len(k)} GPU ops")
hist = {}
for g, a, b in gaps:
    hist.setdefault((a.split("(")[0], b.split("(")[0]), [0, 0.0])
    hist[(a.split("(")[0], b.split("(")[0])][0] += 1
    hist[(a.split("(")[0], b.split("(")[0])][1] += g
for (a, b), (n, tot) in sorted(hist.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{tot / 1e3:7.3f} ms {n:4d}x  {a} -> {b}")
