"""Exercise every entry point on small grids (for compute-sanitizer memcheck /
racecheck runs): state, gradient, HVP, full Hessian, fused call + graph replay,
host call, Newton, tracking step, dense SPD solve, colored Jacobians."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import gridgen
import paper_2201_00241_b200 as rh
from bench import backout_loads_lib

for name in (sys.argv[1:] or ["case9", "case118"]):
    g = gridgen.make_grid(name)
    c = rh.RedHess(0)
    n_x, n_p = c.load_grid(g)
    x_np, p_np = c.state_vectors(g)
    x = torch.from_numpy(x_np).cuda()
    p = torch.from_numpy(p_np).cuda()
    backout_loads_lib(rh, c, g, x, p)
    c.set_state(x, p)
    grad, lam = c.reduced_gradient()
    W = torch.randn(n_p, 37, dtype=torch.float64, device="cuda")
    c.hvp(W)
    c.hvp_stages(W)
    c.full_hessian(16)
    grad2 = torch.empty(n_p, dtype=torch.float64, device="cuda")
    H = torch.empty((n_p, n_p), dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    for _ in range(3):
        c.reduced_hessian(x, p, 16, grad=grad2, H=H, stream=s)
    s.synchronize()
    c.reduced_hessian_host(x_np, p_np, 16)
    xw = x + 1e-6 * torch.randn_like(x)
    try:
        c.newton(xw, p)
    except rh.RHError as e:   # the default synthetic grids can be near voltage collapse
        print(name, "newton:", e)
    c.set_jacobian_mode(rh.JAC_COLORED)
    c.set_state(x, p)
    c.compressed_jacobian()
    c.set_jacobian_mode(rh.JAC_ANALYTIC)
    A = torch.randn(40, 40, dtype=torch.float64, device="cuda")
    A = A @ A.T + 40 * torch.eye(40, dtype=torch.float64, device="cuda")
    c.dense_spd_solve(A, torch.randn(40, dtype=torch.float64, device="cuda"))
    Pd = torch.from_numpy(np.asarray(g.Pd) * 1.01).cuda()
    Qd = torch.from_numpy(np.asarray(g.Qd) * 1.01).cuda()
    try:
        c.tracking_step(x.clone(), p.clone(), 16, Pd=Pd, Qd=Qd)
    except rh.RHError as e:
        print(name, "tracking:", e)
    torch.cuda.synchronize()
    print(name, "ok", c.launch_count(), "launches")
