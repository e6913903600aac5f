"""Host-side timing probe of the headline pipeline (GPU box)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2009_02251_b200 as P  # noqa: E402
from paper_2009_02251_b200.cf import _Samples  # noqa: E402

cfg, M, tr, va, te, _ = bench._workload()
A = P.SparseRatings(tr, *cfg.bounds)
A.device()
vs, ts = _Samples(va, torch.device("cuda")), _Samples(te, torch.device("cuda"))
torch.cuda.synchronize()
for i in range(6):
    t0 = time.perf_counter()
    f, trace = P.auto_latent_factors(A, vs, block_size=20, passes=4, seed=0, max_rank=400)
    t1 = time.perf_counter()
    m = P.evaluate_errors(A, f, ts)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    st = torch.cuda.memory_stats()
    print(f"run {i}: alf {1e3*(t1-t0):.1f} ms  eval {1e3*(t2-t1):.1f} ms  blocks {len(trace)}  "
          f"cudaMalloc retries {st.get('num_alloc_retries')}  segments {st.get('segment.all.current')}  "
          f"reserved {st.get('reserved_bytes.all.current')/1e9:.2f} GB", flush=True)
