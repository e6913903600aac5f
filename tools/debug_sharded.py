"""Debug: step through one sharded QB block on 2 gloo ranks sharing cuda:0."""
import os, sys
import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))


def w(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2009_02251_b200 as P
    from paper_2009_02251_b200 import kernels as K
    from paper_2009_02251_b200.parallel import Comm, ShardedRatings
    from paper_2009_02251_b200.rsvd import _QbEngine
    import inputs
    _, A0 = inputs.rand_sparse(310, 190, 0.09, seed=11)
    A = P.SparseRatings(A0, 0.5, 5.0)
    comm = Comm()
    S = ShardedRatings.from_full(A, comm)
    E = _QbEngine.create(S, 10, P.GaussianStream(5), 400)
    F = _QbEngine.create(A, 10, P.GaussianStream(5), 400)
    print(rank, type(E).__name__, S.row0, S.row1, S.frob_sq, F.frob, flush=True)
    g = lambda t: comm.gather_rows(t, S.counts).cpu().numpy()
    om = E.normal(190, 10, E.yn); om1 = F.normal(190, 10, F.yn)
    print(rank, "om", np.abs(om.cpu().numpy() - om1.cpu().numpy()).max(), flush=True)
    y = E.A_mul(om, E.ym); y1 = F.A_mul(om1, F.ym)
    print(rank, "Aom", np.abs(g(y) - y1.cpu().numpy()).max(), flush=True)
    yy = y.clone()
    G = K.gram(yy); Gl = G.clone(); comm.all_reduce_(G)
    G1 = K.gram(y1)
    print(rank, "gram local vs full", np.abs(G.cpu().numpy() - G1.cpu().numpy()).max(), np.abs(G1.cpu().numpy()).max(), flush=True)
    E.lu(y); F.lu(y1)
    r = E.AT_mul(y, E.yn); r1 = F.AT_mul(y1, F.yn)
    # compare spans: project r1 onto r
    a, b = r.cpu().numpy(), r1.cpu().numpy()
    qa = np.linalg.qr(a)[0]
    print(rank, "span(A.T ql) residual", np.linalg.norm(b - qa @ (qa.T @ b)) / np.linalg.norm(b), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    mp.spawn(w, args=(2, 29533), nprocs=2, join=True)
