"""Time rh_dense_spd_solve (tracking Step 2) at the tracking sizes; run under ncu
for per-kernel durations (k_chol, k_chol_bwd)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2201_00241_b200 as rh

ctx = rh.RedHess(0)
for n in [int(a) for a in (sys.argv[1:] or ["259", "1444", "2889"])]:
    rng = np.random.default_rng(n)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    H = torch.from_numpy((Q * np.linspace(1, 10, n)) @ Q.T).cuda()
    g = torch.from_numpy(rng.standard_normal(n)).cuda()
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        ctx.dense_spd_solve(H, g, d)
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.dense_spd_solve(H, g, d)
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"n={n}: dense_spd_solve {np.median(ts):.3f} ms (wall, incl. sync)", flush=True)
