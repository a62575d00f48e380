"""set_state + reduced gradient a few times (for an ncu launch list).  python tools/prof_state.py [case] [reps]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gridgen  # noqa
import paper_2201_00241_b200 as rh  # noqa

name = sys.argv[1] if len(sys.argv) > 1 else "case9241pegase"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = gridgen.make_grid(name)
ctx = rh.RedHess(0)
ctx.load_grid(g)
x, p = ctx.state_vectors(g)
xd, pd = torch.from_numpy(x).cuda(), torch.from_numpy(p).cuda()
for _ in range(reps):
    ctx.set_state(xd, pd)
    ctx.reduced_gradient()
torch.cuda.synchronize()
print("ok")
