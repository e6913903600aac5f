"""N > 1 plumbing on CPU: world_size-2 gloo process group (no GPU)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    from paper_2009_02251_b200 import parallel
    ws, r, lr = parallel.env_ranks()
    dist.init_process_group("gloo", rank=r, world_size=ws)
    try:
        got = parallel.max_over_ranks(1.5 + rank)  # rank 1 is the slowest
        out[rank] = got
        assert (ws, r, lr) == (world, rank, rank)
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    port = _free_port()
    out = torch.zeros(2, dtype=torch.float64).share_memory_()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out.tolist() == [2.5, 2.5]


def test_max_over_ranks_single_process():
    from paper_2009_02251_b200 import parallel
    assert not dist.is_initialized()
    assert parallel.max_over_ranks(3.25) == 3.25
