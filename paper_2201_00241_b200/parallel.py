"""Multi-GPU full reduced Hessian: the column shard of SURVEY.md 8(e).

The columns of grad^2_pp F (the Cartesian direction blocks) are independent
("compute the reduced Hessian slice by slice, in an
embarrassingly parallel fashion").  Rank g of G owns the
contiguous columns [g c, min((g + 1) c, n_p)) with c = ceil(n_p / G); grid,
analysis, state, factors and lambda are replicated (the refactorization is
deterministic, so every rank holds bitwise-identical factors).  Each rank writes
its columns TRANSPOSED (rh_hessian_columns(..., transposed=1)), so its shard is
one contiguous [c][n_p] slab, and ONE all-gather over the process group (NCCL
on GPUs) yields [G c][n_p] whose first n_p rows are H^T: the raw, unsymmetrized
columns of H as rows (R18), no reorder kernel.  The last shard is
zero-padded to c rows.

Host logic only (partition, buffers, the collective); the columns come from
the library's kernels.
"""
from __future__ import annotations


def column_shard(n_p: int, world: int, rank: int):
    """(j0, j1, c): rank's contiguous column range and the padded shard height."""
    c = (n_p + world - 1) // world
    return min(n_p, rank * c), min(n_p, (rank + 1) * c), c


def gather_columns(H_local, n_p: int, group=None, out=None):
    """All-gather the ranks' transposed column slabs [c][n_p] into [world c][n_p].

    Returns (Hall, HT) with HT = Hall[:n_p] = H^T (row j = column j of H)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    c = H_local.shape[0]
    if out is None:
        out = torch.empty((world * c, n_p), dtype=H_local.dtype, device=H_local.device)
    if H_local.is_cuda and dist.get_backend(group) == "gloo":
        # gloo (ranks sharing one GPU in the tests) gathers host tensors: stage
        # through host memory; NCCL gathers device memory directly
        tmp = torch.empty((world * c, n_p), dtype=H_local.dtype)
        dist.all_gather_into_tensor(tmp, H_local.cpu(), group=group)
        out.copy_(tmp)
    else:
        dist.all_gather_into_tensor(out, H_local, group=group)
    return out, out[:n_p]


class ShardedHessian:
    """Per-rank buffers and one call for the sharded full Hessian of a context."""

    def __init__(self, ctx, group=None):
        import torch
        import torch.distributed as dist
        self.ctx = ctx
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        n_p = ctx.n_p
        self.j0, self.j1, self.c = column_shard(n_p, self.world, self.rank)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.H_local = torch.zeros((self.c, n_p), dtype=torch.float64, device=dev)
        self.H_all = torch.zeros((self.world * self.c, n_p), dtype=torch.float64, device=dev)

    def local_columns(self, N: int):
        """This rank's columns (transposed slab); no communication."""
        if self.j1 > self.j0:
            self.ctx.hessian_columns(self.j0, self.j1, N, H=self.H_local[:self.j1 - self.j0], transposed=True)
        return self.H_local

    def reduced(self, x, p, N: int, grad=None):
        """State + reduced gradient + this rank's columns in one library call
        (rh_reduced_hessian, transposed slab), then the one all-gather.
        Returns (grad, H^T) with H^T [n_p][n_p] (row j = column j of H)."""
        rows = self.j1 - self.j0
        grad, _ = self.ctx.reduced_hessian(x, p, N, j0=self.j0, j1=self.j1, grad=grad,
                                           H=self.H_local[:rows] if rows else self.H_local,
                                           transposed=True)
        if self.world == 1:
            return grad, self.H_local[:self.ctx.n_p]
        _, HT = gather_columns(self.H_local, self.ctx.n_p, self.group, out=self.H_all)
        return grad, HT

    def full(self, N: int):
        """Every rank's columns, gathered: returns H^T ([n_p][n_p], row j = column j of H)."""
        self.local_columns(N)
        if self.world == 1:
            return self.H_local[:self.ctx.n_p]
        _, HT = gather_columns(self.H_local, self.ctx.n_p, self.group, out=self.H_all)
        return HT
