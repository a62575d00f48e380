"""Run a few Alg. 2 batches on one case (for ncu).
    python tools/prof_hvp.py [case] [N] [reps] [random|cartesian]

The LAST batch runs between cudaProfilerStart/Stop, so
`ncu --profile-from-start off ...` captures exactly one complete batch: every
kernel of it (random W: k_blk x4, k_sep_gather x2, k_sep_gemm x2, k_for,
k_muladd; cartesian = the full Hessian's columns 0..N-1: also k_batch_plan)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gridgen  # noqa
import paper_2201_00241_b200 as rh  # noqa

name = sys.argv[1] if len(sys.argv) > 1 else "case9241pegase"
N = int(sys.argv[2]) if len(sys.argv) > 2 else gridgen.CONFIG_N.get(name, 256)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
kind = sys.argv[4] if len(sys.argv) > 4 else "random"
g = gridgen.make_grid(name)
ctx = rh.RedHess(0)
ctx.load_grid(g)
x, p = ctx.state_vectors(g)
ctx.set_state(torch.from_numpy(x).cuda(), torch.from_numpy(p).cuda())
ctx.reduced_gradient()
W = torch.randn(ctx.n_p, N, dtype=torch.float64, device="cuda")
HW = torch.empty_like(W)
Nc = min(N, ctx.n_p)
Hc = torch.empty((ctx.n_p, Nc), dtype=torch.float64, device="cuda")


def one():
    if kind == "cartesian":
        ctx.hessian_columns(0, Nc, N, H=Hc)
    else:
        ctx.hvp(W, HW)


for _ in range(max(0, reps - 1)):
    one()
torch.cuda.synchronize()
torch.cuda.profiler.start()
one()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", kind, ctx.get_info())
