"""Experiment: nonzero separator rows per chunk of the first Cartesian batch (RH_DEBUG=16384 printf)."""
import sys
sys.path.insert(0, ".")
import torch, gridgen, paper_2201_00241_b200 as rh
g = gridgen.make_grid("case9241pegase")
c = rh.RedHess(0)
c.load_grid(g)
x, p = c.state_vectors(g)
c.set_state(torch.from_numpy(x).cuda(), torch.from_numpy(p).cuda())
c.reduced_gradient()
H = torch.empty((2889, 963), dtype=torch.float64, device="cuda")
c.hessian_columns(0, 963, 1024, H=H)
torch.cuda.synchronize()
