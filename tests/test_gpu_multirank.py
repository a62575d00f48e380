"""The column-sharded full Hessian with the LIBRARY in several ranks (-m gpu).

SURVEY.md 8(e) / PAPER.md:351-352 ("compute the reduced Hessian slice by slice,
in an embarrassingly parallel fashion"): every rank loads the grid, runs the
fused rh_reduced_hessian(transposed=1) on its contiguous column shard
(paper_2201_00241_b200/parallel.py ShardedHessian.reduced), and one all-gather
assembles H^T.  The gathered result must equal the 1-rank Hessian BITWISE
(per-column arithmetic order is fixed).

This box has one GPU: the ranks share cuda:0 and talk over gloo (the gather
stages through host memory there); on an 8-GPU node bench.py runs the same
ShardedHessian path over NCCL.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
rh = pytest.importorskip("paper_2201_00241_b200")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, name, N, out_dir):
    import torch.distributed as dist
    import gridgen
    import paper_2201_00241_b200 as rhl
    from oracle import powerflow as pf
    from paper_2201_00241_b200.parallel import ShardedHessian
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = pf.backout_loads(gridgen.make_grid(name))
        ctx = rhl.RedHess(0)
        ctx.load_grid(g)
        x, p = ctx.state_vectors(g)
        xd = torch.from_numpy(x).cuda()
        pd = torch.from_numpy(p).cuda()
        sh = ShardedHessian(ctx)
        for _ in range(3):                      # uncaptured, captured, replayed graph
            grad, HT = sh.reduced(xd, pd, N)
        torch.cuda.synchronize()
        np.save(os.path.join(out_dir, f"shard{rank}.npy"), sh.H_local[: sh.j1 - sh.j0].cpu().numpy())
        if rank == 0:
            np.save(os.path.join(out_dir, "HT.npy"), HT.cpu().numpy())
            np.save(os.path.join(out_dir, "grad.npy"), grad.cpu().numpy())
            np.save(os.path.join(out_dir, "range.npy"), np.array([sh.j0, sh.j1, sh.c]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world,N", [("case118", 3, 64), ("case2869pegase", 2, 512),
                                          ("case9241pegase", 2, 1024)])
def test_library_sharded_gather_equals_one_rank(tmp_path, name, world, N):
    import torch.multiprocessing as mp
    import gridgen
    from oracle import powerflow as pf
    out = str(tmp_path)
    mp.start_processes(_rank_main, args=(world, _free_port(), name, N, out), nprocs=world,
                       start_method="spawn")
    HT = np.load(os.path.join(out, "HT.npy"))
    grad = np.load(os.path.join(out, "grad.npy"))
    g = pf.backout_loads(gridgen.make_grid(name))
    ctx = rh.RedHess(0)
    ctx.load_grid(g)
    x, p = ctx.state_vectors(g)
    g1, H1 = ctx.reduced_hessian(torch.from_numpy(x).cuda(), torch.from_numpy(p).cuda(), N)
    H1 = H1.cpu().numpy()
    assert HT.shape == H1.shape
    np.testing.assert_array_equal(HT.T, H1)
    np.testing.assert_array_equal(grad, g1.cpu().numpy())
    # each rank's slab is its own contiguous range of columns
    c = -(-ctx.n_p // world)
    for r in range(world):
        j0, j1 = min(ctx.n_p, r * c), min(ctx.n_p, (r + 1) * c)
        np.testing.assert_array_equal(np.load(os.path.join(out, f"shard{r}.npy")).T, H1[:, j0:j1])
