"""GPU parity of NEXT-4, Jacobians by column coloring + forward mode
(PAPER.md:440-468, 694-713), against oracle/coloring.py and the oracle's
reduced Hessian, through the C ABI (-m gpu)."""
import numpy as np
import pytest

import gridgen
from oracle import coloring as col
from oracle import powerflow as pf
from oracle import reduction as red

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
rh = pytest.importorskip("paper_2201_00241_b200")


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _np(t):
    return t.detach().cpu().numpy()


def col_rel_err(A, B):
    den = np.maximum(np.max(np.abs(B), axis=0), 1e-300)
    return float(np.max(np.max(np.abs(A - B), axis=0) / den))


CASES = [("case9", dict(tap_line=True)), ("case118", dict(tap_line=True)), ("case1354pegase", {})]


@pytest.mark.parametrize("name,kw", CASES, ids=[c[0] for c in CASES])
def test_compressed_jacobian_matches_oracle(name, kw):
    g = pf.backout_loads(gridgen.make_grid(name, **kw))
    L = pf.Layout(g)
    ctx = rh.RedHess(0)
    ctx.load_grid(g)
    x, p = ctx.state_vectors(g)
    ctx.set_state(_dev(x), _dev(p))
    colors, nc = ctx.coloring()
    JS = _np(ctx.compressed_jacobian())
    JSo = col.compressed_jacobian(g, x, p, colors.astype(np.int64), L)
    assert JS.shape == JSo.shape == (L.n_x, nc)
    err = col_rel_err(JS, JSo)
    print(f"{name}: {nc} colors, compressed Jacobian col rel err {err:.2e}")
    assert err <= 1e-13


@pytest.mark.parametrize("name,kw,N", [("case9", dict(tap_line=True), 5), ("case118", dict(tap_line=True), 64),
                                       ("case1354pegase", {}, 256)])
def test_colored_mode_hessian_matches_oracle(name, kw, N):
    g = pf.backout_loads(gridgen.make_grid(name, **kw))
    L = pf.Layout(g)
    x, p = pf.state_vectors(g, L)
    grad, lam = red.reduced_gradient(g, x, p, L)
    Ho = red.full_hessian(red.operators(g, x, p, lam, L), N)
    out = {}
    for mode in (rh.JAC_ANALYTIC, rh.JAC_COLORED):
        ctx = rh.RedHess(0)
        ctx.load_grid(g)
        ctx.set_jacobian_mode(mode)
        gd, H = ctx.reduced_hessian(_dev(x), _dev(p), N)
        out[mode] = (_np(gd), _np(H))
    gc, Hc = out[rh.JAC_COLORED]
    ga, Ha = out[rh.JAC_ANALYTIC]
    assert np.max(np.abs(gc - grad)) <= 1e-10 * np.max(np.abs(grad))
    assert col_rel_err(Hc, Ho) <= 1e-9
    assert col_rel_err(Hc, Ha) <= 1e-11          # same J up to rounding


def test_colored_mode_newton_and_case9241():
    g = pf.backout_loads(gridgen.make_grid("case9241pegase"))
    ctx = rh.RedHess(0)
    ctx.load_grid(g)
    ctx.set_jacobian_mode(rh.JAC_COLORED)
    x, p = ctx.state_vectors(g)
    xd = _dev(x + 1e-3 * np.random.default_rng(7).standard_normal(x.size))
    steps, res = ctx.newton(xd, _dev(p))
    assert res <= 1e-10 and np.max(np.abs(_np(xd) - x)) <= 1e-10
    _, Hc = ctx.reduced_hessian(_dev(x), _dev(p), 1024)
    ctx.set_jacobian_mode(rh.JAC_ANALYTIC)
    _, Ha = ctx.reduced_hessian(_dev(x), _dev(p), 1024)
    err = col_rel_err(_np(Hc), _np(Ha))
    print(f"case9241 colored vs analytic Hessian: {err:.2e}; Newton {steps} steps, resid {res:.1e}")
    assert err <= 1e-10
