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


def test_row_partition_balances_nonzeros():
    import numpy as np
    from paper_2009_02251_b200.parallel import row_partition
    rng = np.random.default_rng(0)
    deg = np.maximum(1, rng.lognormal(3, 1.2, 5000).astype(np.int64))
    indptr = np.concatenate([[0], np.cumsum(deg)])
    for world in (1, 2, 3, 8):
        off = row_partition(indptr, world)
        assert off[0] == 0 and off[-1] == deg.size and np.all(np.diff(off) >= 1)
        load = indptr[off[1:]] - indptr[off[:-1]] + 16 * np.diff(off)
        assert load.max() <= (indptr[-1] + 16 * deg.size) / world + deg.max() + 16
    # tiny: every rank still gets a row
    off = row_partition(np.array([0, 100, 100, 100]), 3)
    assert off.tolist() == [0, 1, 2, 3]
    with pytest.raises(ValueError):
        row_partition(np.array([0, 1]), 2)


def test_local_samples_rebases_users():
    import numpy as np
    from paper_2009_02251_b200.parallel import local_samples
    u, i, r = local_samples([(0, 1, 3.0), (5, 2, 4.0), (7, 0, 1.0), (4, 4, 2.5)], 4, 7)
    assert u.tolist() == [1, 0] and i.tolist() == [2, 4] and r.tolist() == [4.0, 2.5]
    u, i, r = local_samples((np.array([3, 9]), np.array([1, 1]), np.array([2.0, 3.0])), 0, 5)
    assert u.tolist() == [3]


def _comm_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2009_02251_b200.parallel import Comm
        c = Comm()
        assert (c.world, c.rank, c.backend) == (world, rank, "gloo")
        t = torch.full((2, 3), float(rank + 1), dtype=torch.float64)
        c.all_reduce_(t)  # the n x b / k x b / Gram partial sums of the sharded engine
        assert torch.equal(t, torch.full((2, 3), 3.0, dtype=torch.float64))
        rows = torch.arange(3 * (rank + 1), dtype=torch.float64).reshape(rank + 1, 3) + 100 * rank
        g = c.gather_rows(rows, [1, 2])  # ragged shards
        out[rank] = float(g.sum())
        assert g.shape == (3, 3) and g[0].tolist() == [0.0, 1.0, 2.0] and g[2].tolist() == [103.0, 104.0, 105.0]
    finally:
        dist.destroy_process_group()


def test_comm_gloo_world2():
    port = _free_port()
    out = torch.zeros(2, dtype=torch.float64).share_memory_()
    mp.spawn(_comm_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] == out[1]


def test_comm_single_process_is_identity():
    from paper_2009_02251_b200.parallel import Comm
    c = Comm()
    t = torch.ones(3)
    assert c.world == 1 and c.all_reduce_(t) is t and c.gather_rows(t.view(3, 1), [3]) is not None
