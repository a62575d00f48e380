#!/bin/bash
# e2e (rh_reduced_hessian_host, pinned) per config
OUT=gpurun_out/${1:-e2esweep}; mkdir -p $OUT
timeout 600 python - > $OUT/e2e.txt 2>&1 <<'PY'
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import gridgen, paper_2201_00241_b200 as rh
from bench import backout_loads_lib
for case in ["case118", "case1354pegase", "case2869pegase", "case9241pegase"]:
    N = gridgen.CONFIG_N[case]
    g = gridgen.make_grid(case); ctx = rh.RedHess(0); n_x, n_p = ctx.load_grid(g)
    x_np, p_np = ctx.state_vectors(g)
    x = torch.from_numpy(x_np).cuda(); p = torch.from_numpy(p_np).cuda()
    backout_loads_lib(rh, ctx, g, x, p)
    x_h = torch.from_numpy(x_np).pin_memory(); p_h = torch.from_numpy(p_np).pin_memory()
    H_h = torch.empty((n_p, n_p), dtype=torch.float64).pin_memory(); g_h = torch.empty(n_p, dtype=torch.float64).pin_memory()
    for _ in range(3): ctx.reduced_hessian_host(x_h.numpy(), p_h.numpy(), N, grad=g_h.numpy(), H=H_h.numpy())
    ts = []
    for _ in range(20):
        t0 = time.perf_counter(); ctx.reduced_hessian_host(x_h.numpy(), p_h.numpy(), N, grad=g_h.numpy(), H=H_h.numpy()); ts.append((time.perf_counter() - t0) * 1e3)
    print(case, "N", N, "e2e ms median %.3f min %.3f" % (np.median(ts), np.min(ts)), flush=True)
PY
cat $OUT/e2e.txt
