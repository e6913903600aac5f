"""Multi-process plumbing for N > 1 GPUs (one process per GPU).

Round 1 runs the pipeline as independent replicas: the QB factorisation of
one rating matrix has no partition whose parts are independent (every
block's sketch needs the whole matrix), so ``bench.py --gpus N`` runs N
full replicas and reports the slowest one; the row-sharded engine with its
real exchange steps (all-reduce of the n x b partials of A.T products and of
the small Gram / projection partials) is the next scope row.
What is shared is exercised here and in ``tests/test_parallel.py`` with
``gloo`` on CPU: rank discovery from the torchrun environment and the
device-side max-over-ranks of a timing.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_ranks() -> tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def max_over_ranks(value: float, device: torch.device | None = None) -> float:
    """The maximum of ``value`` over all ranks (every rank gets it); the
    timing rule for multi-GPU numbers (slowest rank).  Identity when no
    process group is initialised."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or torch.device("cpu"))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    return float(t.item())
