"""Stage timeline of the fused state + gradient + Hessian call (RH_DEBUG=1024 marks)."""
import sys
import torch
sys.path.insert(0, ".")
import gridgen
import paper_2201_00241_b200 as rh
from bench import backout_loads_lib

case = sys.argv[1] if len(sys.argv) > 1 else "case9241pegase"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
g = gridgen.make_grid(case)
ctx = rh.RedHess(0)
n_x, n_p = ctx.load_grid(g)
x_np, p_np = ctx.state_vectors(g)
x = torch.from_numpy(x_np).cuda(); p = torch.from_numpy(p_np).cuda()
backout_loads_lib(rh, ctx, g, x, p)
H = torch.empty((n_p, n_p), dtype=torch.float64, device="cuda")
for it in range(4):
    print("run", it, file=sys.stderr)
    ctx.reduced_hessian(x, p, N, H=H, transposed=True)
