"""GPU parity on every input class the C ABI accepts, and at the north-star size.

  * the 2-bus toy (n_pv = 0, n_p = 1) against the golden closed-form value
    H = 0.47346713984 (tests/golden/spec_worked_values.json),
    the operating point solved on the device by rh_newton;
  * grids with parallel lines (rh_grid: "parallel lines add", R1), a
    phase-shifting transformer, and no PQ bus at all (n_pq = 0, R24) against
    the oracle (which tests/test_oracle.py pins on the same grids by
    complex-step through complex Newton);
  * ALL 2889 columns of case9241pegase's grad^2 F through the fused
    rh_reduced_hessian call at N = 1024 -- the CUDA-graph path bench.py times
    -- against the oracle's full Hessian, element by element (north star:
    "full reduced Hessian of a 9241-bus-shaped grid matching the CPU oracle").

Tolerances: tests/parity.py (R21, revised r02).
"""
import json
import os

import numpy as np
import pytest

import gridgen
import pins
from oracle import powerflow as pf
from oracle import reduction as red
from parity import TOL_H, check_hessian, col_rel_err

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
rh = pytest.importorskip("paper_2201_00241_b200")

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _np(t):
    return t.detach().cpu().numpy()


def test_two_bus_golden_on_gpu():
    """n_pv = 0: x = (theta_2, v_2), p = (v_1), one 2x2 unit, no separator.
    rh_newton solves the power flow from the generator's start; the fused call
    then gives the 1x1 reduced Hessian; both must match the closed form."""
    ex = json.load(open(os.path.join(GOLD, "spec_worked_values.json")))["two_bus_hessian"]
    g = gridgen.two_bus(R=ex["R"], X=ex["X"], P=ex["P"], Q=ex["Q"], Pd1=ex["Pd1"], c2=ex["c2"], c1=ex["c1"],
                        v1=ex["v1"])
    Hc, s = pins.two_bus_closed_form(ex["R"], ex["X"], ex["P"], ex["Q"], ex["Pd1"], ex["c2"], ex["c1"], ex["v1"])
    ctx = rh.RedHess(0)
    assert ctx.load_grid(g) == (2, 1)
    x, p = ctx.state_vectors(g)
    xd, pd = _dev(x), _dev(p)
    ctx.newton(xd, pd)
    xs = _np(xd)
    xb, xk, _, _ = ctx.orderings()
    v2 = xs[xk == rh.KIND_V][0]
    assert abs(v2 * v2 - ex["s"]) <= 1e-12
    grad, H = ctx.reduced_hessian(xd, pd, 1)
    H = _np(H)
    assert H.shape == (1, 1)
    assert abs(H[0, 0] - Hc) <= 1e-11 * abs(Hc)
    assert abs(H[0, 0] - ex["H"]) <= ex["rtol"] * ex["H"]
    # and through the separate calls, any batch width
    ctx.set_state(xd, pd)
    ctx.reduced_gradient()
    assert np.array_equal(_np(ctx.full_hessian(4)), H)


VARIANTS = {
    "parallel+shift": dict(name="case9", kw=dict(parallel_lines=3, phase_shift=0.08, tap_line=True), N=5),
    "parallel118": dict(name="case118", kw=dict(parallel_lines=6, phase_shift=-0.05), N=64),
    "no_pq": dict(name="allpv", kw=dict(shape=(12, 17, 11)), N=8),
    "no_pq_300": dict(name="allpv300", kw=dict(shape=(300, 420, 299)), N=128),
    "parallel1354": dict(name="case1354pegase", kw=dict(parallel_lines=40, phase_shift=0.1), N=256),
}


@pytest.fixture(scope="module", params=sorted(VARIANTS), ids=sorted(VARIANTS))
def variant(request):
    v = VARIANTS[request.param]
    g = pf.backout_loads(gridgen.make_grid(v["name"], **v["kw"]))
    L = pf.Layout(g)
    x, p = pf.state_vectors(g, L)
    grad, lam = red.reduced_gradient(g, x, p, L)
    ops = red.operators(g, x, p, lam, L)
    return request.param, v["N"], g, L, x, p, grad, lam, ops


def test_variant_parity(variant):
    key, N, g, L, x, p, grad, lam, ops = variant
    ctx = rh.RedHess(0)
    assert ctx.load_grid(g) == (L.n_x, L.n_p)
    # the library's orderings equal the oracle's (R5), so vectors are exchangeable
    xb, xk, pb, pk = ctx.orderings()
    assert np.array_equal(xb, L.x_bus) and np.array_equal(pb, L.p_bus)
    xd, pd = _dev(x), _dev(p)
    # residual at the solved point, then the fused call (state + gradient + H)
    ctx.set_state(xd, pd)
    res, f = ctx.residual()
    assert np.max(np.abs(_np(res))) <= 1e-11
    assert abs(_np(f)[0] - pf.objective(g, x, p, L)) <= 1e-12 * abs(pf.objective(g, x, p, L))
    for _ in range(3):                      # uncaptured, captured, replayed graph
        gd, H = ctx.reduced_hessian(xd, pd, N)
    assert np.max(np.abs(_np(gd) - grad)) <= 1e-10 * np.max(np.abs(grad))
    Ho = red.full_hessian(ops, N)
    check_hessian(_np(H), Ho, f"variant {key} N={N} (fused, graph replay)", ops, N, red.full_hessian)
    # Alg. 2 intermediates on random directions
    ctx.set_state(xd, pd)
    ctx.reduced_gradient()
    W = gridgen.random_W(L.n_p, 7, seed=3)
    trace = {}
    HWo = red.hvp_batch(ops, W, trace)
    HW, Z, Yx, Psi = (_np(t) for t in ctx.hvp_stages(_dev(W)))
    assert col_rel_err(Z, trace["Z"]) <= 1e-10
    assert col_rel_err(Yx, trace["Yx"]) <= 1e-10
    assert col_rel_err(Psi, trace["Psi"]) <= 1e-10
    assert col_rel_err(HW, HWo) <= TOL_H


def test_variant_lossless_closed_form_parallel_lines():
    """Lossless closed form on a case2869-shaped grid WITH
    parallel lines: H_PgPg = 2 c2_ref 11^T + diag(2 c2), v rows/cols = 0."""
    g = gridgen.make_grid("case2869pegase", lossless=True, parallel_lines=60)
    ctx = rh.RedHess(0)
    ctx.load_grid(g)
    x, p = ctx.state_vectors(g)
    _, H = ctx.reduced_hessian(_dev(x), _dev(p), 512)
    H = _np(H)
    xb, xk, pb, pk = ctx.orderings()
    c2 = np.zeros(g.n_bus)
    c2[g.gen_bus] = g.c2
    pgm = pk == rh.KIND_PG
    Hc = np.zeros_like(H)
    Hc[np.ix_(pgm, pgm)] = 2 * c2[g.ref] + np.diag(2 * c2[pb[pgm]])
    assert np.max(np.abs(H - Hc)) <= 1e-9 * np.max(np.abs(Hc))


@pytest.fixture(scope="module")
def case9241():
    g = pf.backout_loads(gridgen.make_grid("case9241pegase"))
    L = pf.Layout(g)
    x, p = pf.state_vectors(g, L)
    grad, lam = red.reduced_gradient(g, x, p, L)
    ops = red.operators(g, x, p, lam, L)
    Ho = red.full_hessian(ops, 1024)
    return g, L, x, p, grad, Ho, ops


def test_case9241_all_columns_fused_graph_path(case9241):
    """Every one of the 2889 columns of case9241pegase's grad^2 F, produced by the
    fused rh_reduced_hessian call at N = 1024 after its CUDA graph was captured
    (the launch configuration bench.py times), vs the oracle element by element."""
    g, L, x, p, grad, Ho, ops = case9241
    ctx = rh.RedHess(0)
    ctx.load_grid(g)
    xd, pd = _dev(x), _dev(p)
    gbuf = torch.empty(L.n_p, dtype=torch.float64, device="cuda")
    Hbuf = torch.empty((L.n_p, L.n_p), dtype=torch.float64, device="cuda")
    outs = []
    for _ in range(3):                      # uncaptured, captured, replayed
        ctx.reduced_hessian(xd, pd, 1024, grad=gbuf, H=Hbuf)
        outs.append(_np(Hbuf).copy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    H = outs[2]
    assert np.max(np.abs(_np(gbuf) - grad)) <= 1e-10 * np.max(np.abs(grad))
    check_hessian(H, Ho, "case9241pegase all 2889 columns, N=1024 (fused, graph replay)", ops, 1024,
                  red.full_hessian)
    # the transposed shard layout the multi-GPU path uses, same graph machinery
    j0, j1 = 1000, 1362
    gt, Ht = ctx.reduced_hessian(xd, pd, 1024, j0=j0, j1=j1, transposed=True)
    assert np.array_equal(_np(Ht).T, H[:, j0:j1])


def test_newton_replay_clears_multipliers():
    """a replayed Newton graph must invalidate lambda: rh_newton, then
    rh_reduced_gradient, then a second rh_newton (graph replay, ends in
    RH_E_NOCONV) -> rh_hvp must refuse with RH_E_ORDER, not use the old tape."""
    g = pf.backout_loads(gridgen.make_grid("case118"))
    ctx = rh.RedHess(0)
    ctx.load_grid(g)
    x, p = ctx.state_vectors(g)
    x0 = x + 1e-3 * np.random.default_rng(5).standard_normal(x.size)
    xd, pd = _dev(x0), _dev(p)
    ctx.newton(xd, pd)
    ctx.reduced_gradient()
    W = _dev(np.ones((ctx.n_p, 2)))
    ctx.hvp(W)
    with pytest.raises(rh.RHError) as e:
        ctx.newton(_dev(x0), pd, tol=0.0, extra=0, maxit=4)
    assert e.value.code == rh.RH_E_NOCONV
    with pytest.raises(rh.RHError) as e:
        ctx.hvp(W)
    assert e.value.code == rh.RH_E_ORDER


def test_binding_rejects_bad_buffers():
    """every caller buffer is validated before the C call."""
    g = pf.backout_loads(gridgen.make_grid("case9"))
    ctx = rh.RedHess(0)
    ctx.load_grid(g)
    x, p = ctx.state_vectors(g)
    xd, pd = _dev(x), _dev(p)
    ctx.set_state(xd, pd)
    ctx.reduced_gradient()
    with pytest.raises(ValueError):
        ctx.hvp(_dev(np.ones((ctx.n_p - 1, 2))))                          # too few rows
    with pytest.raises(ValueError):
        ctx.hvp(_dev(np.ones((ctx.n_p, 3))), HW=_dev(np.ones((ctx.n_p, 2))))
    with pytest.raises(TypeError):
        ctx.hvp(torch.ones((ctx.n_p, 2), dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        ctx.hvp(_dev(np.ones((2, ctx.n_p))).t())                          # column-major view
    with pytest.raises(ValueError):
        ctx.full_hessian(5, H=_dev(np.ones((ctx.n_p, ctx.n_p - 1))))
    with pytest.raises(ValueError):
        ctx.hessian_columns(0, 3, 5, H=_dev(np.ones((ctx.n_p, 2))))
    with pytest.raises(ValueError):
        ctx.hessian_columns(2, ctx.n_p + 1, 5)
    with pytest.raises(TypeError):
        ctx.reduced_hessian_host(x.astype(np.float32), p, 5)
    with pytest.raises(ValueError):
        ctx.reduced_hessian_host(x, p, 5, H=np.empty((ctx.n_p, ctx.n_p - 1)))
    with pytest.raises(TypeError):
        ctx.reduced_hessian_host(x, p, 5, H=np.empty((ctx.n_p, 2 * ctx.n_p))[:, ::2])
    with pytest.raises(ValueError):
        ctx.dense_spd_solve(torch.eye(3, dtype=torch.float64), _dev(np.ones(3)))   # host H
    # the valid calls still work
    assert ctx.hvp(_dev(np.ones((ctx.n_p, 2)))).shape == (ctx.n_p, 2)
