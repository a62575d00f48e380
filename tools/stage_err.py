"""Per-stage GPU-vs-oracle error on one case (diagnostic).  python tools/stage_err.py case [lossless]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gridgen  # noqa
import paper_2201_00241_b200 as rh  # noqa
from oracle import powerflow as pf, reduction as red  # noqa

name = sys.argv[1]
lossless = len(sys.argv) > 2
g = pf.backout_loads(gridgen.make_grid(name, lossless=lossless))
L = pf.Layout(g)
x, p = pf.state_vectors(g, L)
grad, lam = red.reduced_gradient(g, x, p, L)
ops = red.operators(g, x, p, lam, L)
ctx = rh.RedHess(0)
ctx.load_grid(g)
xd, pd = torch.from_numpy(x).cuda(), torch.from_numpy(p).cuda()
ctx.set_state(xd, pd)
gd, ld = ctx.reduced_gradient()
print("lambda rel err", np.abs(ld.cpu().numpy() - lam).max() / np.abs(lam).max())
cols = list(range(0, L.n_p, max(1, L.n_p // 64)))
W = np.zeros((L.n_p, len(cols)))
W[cols, np.arange(len(cols))] = 1.0
tr = {}
HWo = red.hvp_batch(ops, W, tr)
HW, Z, Yx, Psi = (t.cpu().numpy() for t in ctx.hvp_stages(torch.from_numpy(W).cuda()))
for nm, a, b in (("Z", Z, tr["Z"]), ("Yx", Yx, tr["Yx"]), ("Psi", Psi, tr["Psi"]), ("HW", HW, HWo)):
    print(nm, "max|.|", np.abs(b).max(), "abs err", np.abs(a - b).max(), "rel", np.abs(a - b).max() / np.abs(b).max())
Yx_from_gpuZ = ops.Hxx @ Z + ops.Hxp @ W
print("FoR only: Yx(gpu) vs Hxx Zgpu + Hxp W", np.abs(Yx - Yx_from_gpuZ).max() / np.abs(Yx_from_gpuZ).max())
Psi_from_gpuYx = -ops.solve_T(Yx)
print("solve_T only", np.abs(Psi - Psi_from_gpuYx).max() / np.abs(Psi_from_gpuYx).max())
Z_o = -ops.solve(ops.Gp @ W)
print("solve only", np.abs(Z - Z_o).max() / np.abs(Z_o).max())
Yp_o = ops.Hpx @ Z + ops.Hpp @ W
HW_from = Yp_o + ops.Gp.T @ Psi
print("muladd only", np.abs(HW - HW_from).max() / np.abs(HW_from).max())
if lossless:
    c2 = np.zeros(L.n_bus); c2[g.gen_bus] = g.c2; npv = len(L.pv)
    Hc = np.zeros((L.n_p, L.n_p)); Hc[:npv, :npv] = 2 * c2[L.ref] + np.diag(2 * c2[L.pv])
    print("closed form: gpu", np.abs(HW - Hc[:, cols]).max() / np.abs(Hc).max(), "oracle",
          np.abs(HWo - Hc[:, cols]).max() / np.abs(Hc).max())
