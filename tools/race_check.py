"""Race check (diagnostic): many back-to-back fused calls, eager (a fresh output buffer each
time: no graph) and graph-replayed, must all be bitwise equal to the first.
    python tools/race_check.py [case] [N] [reps]"""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import gridgen, paper_2201_00241_b200 as rh
from oracle import powerflow as pf
case = sys.argv[1] if len(sys.argv) > 1 else "case9241pegase"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 100
g = pf.backout_loads(gridgen.make_grid(case))
ctx = rh.RedHess(0); ctx.load_grid(g)
x, p = ctx.state_vectors(g)
xd, pd = torch.from_numpy(x).cuda(), torch.from_numpy(p).cuda()
g0, H0 = ctx.reduced_hessian(xd, pd, N)
H0 = H0.cpu().numpy(); g0 = g0.cpu().numpy()
bad = 0
for r in range(reps):                          # eager: new buffers each call
    gf, Hf = ctx.reduced_hessian(xd, pd, N)
    bad += not (np.array_equal(Hf.cpu().numpy(), H0) and np.array_equal(gf.cpu().numpy(), g0))
gf = torch.empty_like(torch.from_numpy(g0)).cuda(); Hf = torch.empty_like(torch.from_numpy(H0)).cuda()
for r in range(reps):                          # fixed buffers: captured, then replayed
    ctx.reduced_hessian(xd, pd, N, grad=gf, H=Hf)
    bad += not (np.array_equal(Hf.cpu().numpy(), H0) and np.array_equal(gf.cpu().numpy(), g0))
print(case, "N", N, "calls", 2 * reps, "mismatches", bad)
