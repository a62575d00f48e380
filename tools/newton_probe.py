import sys, os, numpy as np, torch
sys.path.insert(0, "/root/repo")
import gridgen, paper_2201_00241_b200 as rh
from oracle import powerflow as pf
for name, amp in (("case2869pegase", 0.01), ("case9241pegase", 0.01), ("case9241pegase", 0.001)):
    g = pf.backout_loads(gridgen.make_grid(name)) if name != "case9241pegase" else gridgen.make_grid(name)
    ctx = rh.RedHess(0); ctx.load_grid(g)
    x, p = ctx.state_vectors(g)
    x0 = x + amp * np.random.default_rng(7).standard_normal(x.size)
    xd = torch.from_numpy(x0).cuda()
    try:
        print(name, amp, ctx.newton(xd, torch.from_numpy(p).cuda(), maxit=12), flush=True)
    except Exception as e:
        print(name, amp, e, flush=True)
