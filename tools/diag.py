"""GPU diagnostics: parity margins and a quick per-stage timing probe.

    python tools/diag.py [case ...]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gridgen  # noqa: E402
import paper_2201_00241_b200 as rh  # noqa: E402
from oracle import powerflow as pf  # noqa: E402
from oracle import reduction as red  # noqa: E402


def ev_time(fn, reps=5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return min(ts), float(np.median(ts))


def main(cases, parity=True):
    for name in cases:
        g = pf.backout_loads(gridgen.make_grid(name))
        ctx = rh.RedHess(0)
        ctx.load_grid(g)
        info = ctx.get_info()
        x, p = ctx.state_vectors(g)
        xd = torch.from_numpy(x).cuda()
        pd = torch.from_numpy(p).cuda()
        ctx.set_state(xd, pd)
        ctx.reduced_gradient()
        N = gridgen.CONFIG_N.get(name, 256)
        H = ctx.full_hessian(N)
        torch.cuda.synchronize()
        Hn = H.cpu().numpy()
        line = (f"{name}: n_x={info['n_x']} n_p={info['n_p']} nnzLU={info['nnz_LU']} lev={info['levels_fwd']} "
                f"blocks={info['n_blocks']} sep={info['sep_rows']} seglev={info['seg_levels']} ")
        if parity and info["n_x"] < 10000:
            L = pf.Layout(g)
            xo, po = pf.state_vectors(g, L)
            t0 = time.time()
            grad, lam = red.reduced_gradient(g, xo, po, L)
            ops = red.operators(g, xo, po, lam, L)
            Ho = red.full_hessian(ops, N)
            to = time.time() - t0
            den = np.max(np.abs(Ho), axis=0)
            colerr = np.max(np.max(np.abs(Hn - Ho), axis=0) / den)
            ents = []
            for fl in (1e-6, 1e-5, 1e-4, 1e-3):
                m = np.abs(Ho) >= fl * np.max(np.abs(Ho))
                ents.append(np.max(np.abs(Hn - Ho)[m] / np.abs(Ho)[m]))
            line += f"colerr={colerr:.2e} entry(1e-6..1e-3)={['%.1e' % v for v in ents]} oracle={to:.2f}s "
        line += f"asym={np.max(np.abs(Hn - Hn.T)) / np.max(np.abs(Hn)):.1e}"
        print(line, flush=True)
        t_state = ev_time(lambda: ctx.set_state(xd, pd))
        ctx.reduced_gradient()
        t_grad = ev_time(lambda: ctx.reduced_gradient())
        Hbuf = torch.empty_like(H)
        t_full = ev_time(lambda: ctx.full_hessian(N, Hbuf))
        W = torch.randn(info["n_p"], N, dtype=torch.float64, device="cuda")
        HW = torch.empty_like(W)
        t_hvp = ev_time(lambda: ctx.hvp(W, HW))
        ctx.set_timing(True)
        ctx.hvp(W, HW)
        st = ctx.stage_times()
        ctx.set_timing(False)
        print(f"   set_state {t_state[0]:.3f} ms, grad {t_grad[0]:.3f} ms, full H (N={N}) {t_full[0]:.3f} ms, "
              f"hvp(N={N}) {t_hvp[0]:.3f} ms -> {N / t_hvp[0] * 1e3:.3e} HVP/s; stages A_L/B_LU/A_U/FoR/A_Ut/B_UtLt/A_Lt/MulAdd "
              f"{['%.3f' % v for v in st[:8]]}", flush=True)


if __name__ == "__main__":
    cases = sys.argv[1:] or ["case9", "case118", "case1354pegase", "case2869pegase", "case9241pegase"]
    main(cases)
