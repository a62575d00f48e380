"""Run a few HVP batches on one case (for ncu).  python tools/prof_hvp.py [case] [N] [reps]"""
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
for _ in range(reps):
    ctx.hvp(W, HW)
torch.cuda.synchronize()
print("ok", ctx.get_info())
