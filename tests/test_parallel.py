"""Multi-rank host logic of the column-sharded full Hessian (
paper_2201_00241_b200/parallel.py) on CPU: world_size 2 over gloo.  Each rank
computes its column shard with the ORACLE (test infrastructure standing in for
the library's kernels, which need a GPU) and the package's gather assembles
H^T; it must equal the oracle's full Hessian exactly (a gather moves bytes)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gridgen
from oracle import powerflow as pf
from oracle import reduction as red
from paper_2201_00241_b200.parallel import column_shard, gather_columns


def test_column_shard_partition():
    for n_p in (1, 5, 107, 519, 1019, 2889):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                j0, j1, c = column_shard(n_p, world, r)
                assert 0 <= j0 <= j1 <= n_p and j1 - j0 <= c and c == -(-n_p // world)
                seen.extend(range(j0, j1))
            assert seen == list(range(n_p))   # contiguous, disjoint, complete, rank order


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, name, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = pf.backout_loads(gridgen.make_grid(name))
        L = pf.Layout(g)
        x, p = pf.state_vectors(g, L)
        _, lam = red.reduced_gradient(g, x, p, L)
        ops = red.operators(g, x, p, lam, L)
        n_p = L.n_p
        j0, j1, c = column_shard(n_p, world, rank)
        H_local = torch.zeros((c, n_p), dtype=torch.float64)
        if j1 > j0:
            W = np.zeros((n_p, j1 - j0))
            W[np.arange(j0, j1), np.arange(j1 - j0)] = 1.0
            H_local[: j1 - j0] = torch.from_numpy(red.hvp_batch(ops, W).T.copy())
        _, HT = gather_columns(H_local, n_p)
        if rank == 0:
            np.save(out_path, HT.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("case9", 2), ("case118", 2)])
def test_gloo_sharded_full_hessian(tmp_path, name, world):
    out = str(tmp_path / "HT.npy")
    mp.start_processes(_rank_main, args=(world, _free_port(), name, out), nprocs=world, start_method="spawn")
    HT = np.load(out)
    g = pf.backout_loads(gridgen.make_grid(name))
    L = pf.Layout(g)
    x, p = pf.state_vectors(g, L)
    _, lam = red.reduced_gradient(g, x, p, L)
    H = red.full_hessian(red.operators(g, x, p, lam, L), L.n_p)
    assert HT.shape == H.shape
    np.testing.assert_array_equal(HT.T, H)
