"""Step timing probe (device events): the fused rh_reduced_hessian call (graph
replay) per config, with and without the Cartesian L-tile mask, and the
per-stage times of one Cartesian batch vs one random-W batch.

    python tools/step_probe.py [case ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gridgen  # noqa: E402
import paper_2201_00241_b200 as rh  # noqa: E402
from oracle import powerflow as pf  # noqa: E402


def ev_time(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts)), float(min(ts))


def run(name, N, modes=("mask", "nomask")):
    g = pf.backout_loads(gridgen.make_grid(name))
    out = {}
    Href = None
    for mode in modes:
        if mode == "nomask":
            os.environ["RH_NO_MASK"] = "1"
        else:
            os.environ.pop("RH_NO_MASK", None)
        ctx = rh.RedHess(0)
        ctx.load_grid(g)
        x, p = ctx.state_vectors(g)
        xd, pd = torch.from_numpy(x).cuda(), torch.from_numpy(p).cuda()
        grad = torch.empty(ctx.n_p, dtype=torch.float64, device="cuda")
        H = torch.empty((ctx.n_p, ctx.n_p), dtype=torch.float64, device="cuda")
        HT = torch.empty((ctx.n_p, ctx.n_p), dtype=torch.float64, device="cuda")
        out[mode + "_fused"] = ev_time(lambda: ctx.reduced_hessian(xd, pd, N, grad=grad, H=H))
        out[mode + "_fusedT"] = ev_time(lambda: ctx.reduced_hessian(xd, pd, N, grad=grad, H=HT, transposed=True))
        Hn = H.cpu().numpy()
        if Href is None:
            Href = Hn
        else:
            out["mask_vs_nomask_equal"] = bool(np.array_equal(Href, Hn))
        assert np.array_equal(HT.cpu().numpy().T, Hn)
        ctx.set_state(xd, pd)
        ctx.reduced_gradient()
        ctx.set_timing(True)
        HcT = torch.empty((min(N, ctx.n_p), ctx.n_p), dtype=torch.float64, device="cuda")
        ctx.hessian_columns(0, min(N, ctx.n_p), N, H=HcT, transposed=True)   # the step's layout
        out[mode + "_cart_stages"] = [round(float(v), 4) for v in ctx.stage_times()[:9]]
        W = torch.randn(ctx.n_p, N, dtype=torch.float64, device="cuda")
        ctx.hvp(W)
        out[mode + "_randW_stages"] = [round(float(v), 4) for v in ctx.stage_times()[:9]]
        ctx.set_timing(False)
    os.environ.pop("RH_NO_MASK", None)
    print(name, N, out, flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    modes = ("mask", "nomask")
    if args and args[0] == "--mask-only":
        modes = ("mask",)
        args = args[1:]
    cases = args or ["case118", "case1354pegase", "case2869pegase", "case9241pegase"]
    tag = os.environ.get("PROBE_TAG", "")
    for c in cases:
        if tag:
            print("variant", tag, end=": ")
        run(c, int(os.environ.get("PROBE_N", 0)) or gridgen.CONFIG_N.get(c, 256), modes)
