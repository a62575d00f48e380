"""Run a few HVP batches on one case (for ncu).  python tools/prof_hvp.py [case] [N] [reps]

The LAST batch runs between cudaProfilerStart/Stop, so
`ncu --profile-from-start off ...` captures exactly one complete Alg. 2 batch
(every kernel of it: k_blk x4, k_sep_gather x2, k_sep_gemm x2, k_for, k_muladd)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gridgen  # noqa
import paper_2201_00241_b200 as rh  # noqa

name = sys.argv[1] if len(sys.argv) > 1 else "case9241pegase"
N = int(sys.argv[2]) if len(sys.argv) > 2 else gridgen.CONFIG_N.get(name, 256)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
g = gridgen.make_grid(name)
ctx = rh.RedHess(0)
ctx.load_grid(g)
x, p = ctx.state_vectors(g)
ctx.set_state(torch.from_numpy(x).cuda(), torch.from_numpy(p).cuda())
ctx.reduced_gradient()
W = torch.randn(ctx.n_p, N, dtype=torch.float64, device="cuda")
HW = torch.empty_like(W)
for _ in range(max(0, reps - 1)):
    ctx.hvp(W, HW)
torch.cuda.synchronize()
torch.cuda.profiler.start()
ctx.hvp(W, HW)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", ctx.get_info())
