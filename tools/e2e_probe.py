"""e2e diagnostics: D2H bandwidth (pinned, 1D and 2D column blocks) and the
distribution of rh_reduced_hessian_host times on case9241 (N = 1024)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import gridgen
import paper_2201_00241_b200 as rh
from bench import backout_loads_lib

n = 2889
Hd = torch.randn(n, n, dtype=torch.float64, device="cuda")
Hh = torch.empty(n, n, dtype=torch.float64).pin_memory()
for _ in range(2):
    Hh.copy_(Hd)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    Hh.copy_(Hd)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 5
print(f"D2H 1D {n*n*8/1e6:.1f} MB: {dt*1e3:.3f} ms = {n*n*8/dt/1e9:.1f} GB/s")
t0 = time.perf_counter()
for _ in range(5):
    for a in range(0, n, 1024):
        Hh[:, a:a + 1024].copy_(Hd[:, a:a + 1024], non_blocking=True)
    torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 5
print(f"D2H 2D column blocks: {dt*1e3:.3f} ms = {n*n*8/dt/1e9:.1f} GB/s")

grid = gridgen.make_grid("case9241pegase")
ctx = rh.RedHess(0)
ctx.load_grid(grid)
x_np, p_np = ctx.state_vectors(grid)
x = torch.from_numpy(x_np).cuda(); p = torch.from_numpy(p_np).cuda()
backout_loads_lib(rh, ctx, grid, x, p)
x_h = torch.from_numpy(x_np).pin_memory(); p_h = torch.from_numpy(p_np).pin_memory()
H_h = torch.empty((n, n), dtype=torch.float64).pin_memory(); g_h = torch.empty(n, dtype=torch.float64).pin_memory()
for NB in [int(a) for a in (sys.argv[1:] or ["1024"])]:
    for _ in range(3):
        ctx.reduced_hessian_host(x_h.numpy(), p_h.numpy(), NB, grad=g_h.numpy(), H=H_h.numpy())
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        ctx.reduced_hessian_host(x_h.numpy(), p_h.numpy(), NB, grad=g_h.numpy(), H=H_h.numpy())
        ts.append((time.perf_counter() - t0) * 1e3)
    print("N=%d e2e ms: median %.3f min %.3f max %.3f" % (NB, np.median(ts), np.min(ts), np.max(ts)))
