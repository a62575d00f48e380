import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gridgen, paper_2201_00241_b200 as rh  # noqa
name = sys.argv[1] if len(sys.argv) > 1 else "case9241pegase"
g = gridgen.make_grid(name, lossless=True)
ctx = rh.RedHess(0); ctx.load_grid(g)
x, p = ctx.state_vectors(g)
ctx.set_state(torch.from_numpy(x).cuda(), torch.from_numpy(p).cuda())
ctx.reduced_gradient()
xb, xk, pb, pk = ctx.orderings()
c2 = np.zeros(g.n_bus); c2[g.gen_bus] = g.c2
ref = int(np.flatnonzero(g.bus_type == gridgen.REF)[0])
pgm = pk == rh.KIND_PG
Hc = np.zeros((ctx.n_p, ctx.n_p)); Hc[np.ix_(pgm, pgm)] = 2 * c2[ref] + np.diag(2 * c2[pb[pgm]])
for N in (1024, 256, 64, 8, 1):
    H = ctx.full_hessian(N).cpu().numpy()
    E = np.abs(H - Hc)
    i, j = np.unravel_index(np.argmax(E), E.shape)
    colmax = E.max(axis=0)
    bad = np.flatnonzero(colmax > 1e-10)
    print(N, "maxerr", E.max(), "at", (i, j), "kinds", pk[i], pk[j], "bus", pb[i], pb[j], "nbadcols", bad.size, bad[:10])
W = torch.zeros(ctx.n_p, 64, dtype=torch.float64, device="cuda")
cols = np.arange(64) * 45
W[cols, torch.arange(64)] = 1.0
HW = ctx.hvp(W).cpu().numpy()
print("hvp sampled", np.abs(HW - Hc[:, cols]).max())
