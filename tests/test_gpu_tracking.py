"""GPU parity of the real-time tracking step
against oracle/tracking.py, through the C ABI (-m gpu).

Tolerances: the dense solve's d is compared in max-norm relative to |d|_inf;
both sides carry rounding ~ cond(H) eps, so the bar is 1e-12 for the
well-conditioned synthetic matrices (cond <= 10) and 1e-8 for reduced Hessians
(cond ~1e3..1e4 on the synthetic grids, times the 1e-9 Hessian bar of R21 would
be looser; observed errors are printed by -s).  The tau / attempt sequence of
the shift rule (R-T4) is compared exactly on matrices whose eigenvalues keep the
decisions away from their thresholds.
"""
import numpy as np
import pytest

import gridgen
from oracle import powerflow as pf
from oracle import tracking as trk

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
rh = pytest.importorskip("paper_2201_00241_b200")


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _np(t):
    return t.detach().cpu().numpy()


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def _spd(n, seed, lo=1.0, hi=10.0, skew=0.0):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    H = (Q * np.linspace(lo, hi, n)) @ Q.T
    if skew:
        K = rng.standard_normal((n, n))
        H = H + skew * (K - K.T)      # only (H + H^T)/2 may matter (R-T1)
    return H, rng.standard_normal(n)


@pytest.fixture(scope="module")
def ctx():
    return rh.RedHess(0)


@pytest.mark.parametrize("n", [1, 2, 5, 31, 32, 33, 63, 64, 65, 100, 259, 700])
def test_dense_spd_solve_matches_oracle(ctx, n):
    H, g = _spd(n, seed=n, skew=0.3)
    d_o, tau_o, att_o = trk.spd_solve(H, g)
    d, tau, att = ctx.dense_spd_solve(_dev(H), _dev(g))
    assert (tau, att) == (tau_o, att_o) == (0.0, 1)
    err = _rel(_np(d), d_o)
    print(f"n={n}: rel err {err:.2e}")
    assert err <= 1e-12


def test_dense_spd_solve_padded_ld_and_p_update(ctx):
    n = 77
    H, g = _spd(n, seed=5)
    Hp = np.zeros((n + 3, n + 9))
    Hp[:n, :n] = H
    p0 = np.linspace(0, 1, n)
    p = _dev(p0)
    d_o, _, _ = trk.spd_solve(H, g)
    Hd = _dev(Hp)
    d, _, _ = ctx.dense_spd_solve(Hd[:n + 3], _dev(g), p=p, alpha=0.5)
    assert _rel(_np(d), d_o) <= 1e-12
    np.testing.assert_allclose(_np(p), p0 + 0.5 * d_o, rtol=0, atol=1e-12 * np.max(np.abs(d_o)))


def test_dense_spd_solve_shift_rule(ctx):
    # diag(2, -1): 22 attempts, tau = 2^20 1e-6 (closed form, R-T4)
    H = np.diag([2.0, -1.0])
    g = np.array([1.0, 1.0])
    d, tau, att = ctx.dense_spd_solve(_dev(H), _dev(g))
    assert att == 22 and tau == 1e-6 * 2 ** 20
    np.testing.assert_allclose(_np(d), [-1.0 / (2.0 + tau), -1.0 / (tau - 1.0)], rtol=1e-13)
    # a larger indefinite matrix, lambda_min = -0.3: same shift sequence as the oracle
    Hn, gn = _spd(90, seed=9, lo=-0.3, hi=5.0)
    d_o, tau_o, att_o = trk.spd_solve(Hn, gn)
    d, tau, att = ctx.dense_spd_solve(_dev(Hn), _dev(gn))
    assert (tau, att) == (tau_o, att_o) and att > 1
    assert _rel(_np(d), d_o) <= 1e-11


def test_dense_spd_solve_zero_rhs_and_not_pd(ctx):
    H, _ = _spd(40, seed=2)
    d, _, _ = ctx.dense_spd_solve(_dev(H), torch.zeros(40, dtype=torch.float64, device="cuda"))
    assert torch.all(d == 0)                      # fixed point: g = 0 -> d = 0 exactly
    with pytest.raises(rh.RHError) as ei:
        ctx.dense_spd_solve(_dev(np.diag([1.0, -1e30])), _dev(np.ones(2)))
    assert ei.value.code == rh.RH_E_NOTPD


def test_dense_spd_solve_large(ctx):
    # the tracking bench's sizes: n_pv = 1444 (case9241 generator set points), n_p = 2889
    for n in (1444, 2889):
        H, g = _spd(n, seed=n)
        d_o, _, _ = trk.spd_solve(H, g)
        d, tau, att = ctx.dense_spd_solve(_dev(H), _dev(g))
        assert att == 1
        err = _rel(_np(d), d_o)
        print(f"n={n}: rel err {err:.2e}")
        assert err <= 1e-11


def _tracking_case(name, kw=None, costs=False):
    """The tracking workload (DESIGN.md R-T5): smooth-voltage grid, loads backed
    out; with costs=True also c1 backed out so p is stationary on the set points."""
    g = pf.backout_loads(gridgen.tracking_grid(name, **(kw or {})))
    L = pf.Layout(g)
    if costs:
        x, p = pf.state_vectors(g, L)
        g = trk.backout_costs(g, x, p, 0, int(np.sum(L.p_kind == 2)), L)
    c = rh.RedHess(0)
    c.load_grid(g)
    x, p = c.state_vectors(g)
    return g, L, c, x, p


@pytest.mark.parametrize("name,kw,free,N,costs", [
    ("case9", dict(tap_line=True), "all", 5, False),
    ("case118", dict(tap_line=True), "all", 64, False),
    ("case118", dict(tap_line=True), "pg", 64, True),
    ("case1354pegase", {}, "pg", 256, True),
    ("case1354pegase", {}, "pg", 100, False),
])
def test_tracking_step_matches_oracle(name, kw, free, N, costs):
    g, L, c, x, p = _tracking_case(name, kw, costs)
    n_pv = int(np.sum(L.p_kind == 2))
    j1 = L.n_p if free == "all" else n_pv
    Pd, Qd = gridgen.load_scenario(g, 60, amp=0.05, kind="sin", seed=4)
    p_o, x_o, info_o = trk.tracking_step(g, p, x, Pd[3], Qd[3], 0, j1, N=N, L=L)
    xd, pd = _dev(x), _dev(p)
    grad, H, d, info = c.tracking_step(xd, pd, N, Pd=_dev(Pd[3]), Qd=_dev(Qd[3]), j0=0, j1=j1)
    ex = float(np.max(np.abs(_np(xd) - x_o)))
    eg = _rel(_np(grad), info_o["grad"])
    HT = _np(H)                                   # row k = column k of H_t
    eH = max(_rel(HT[k], info_o["H"][:, k]) for k in range(j1))
    ed = _rel(_np(d), info_o["d"])
    ep = float(np.max(np.abs(_np(pd) - p_o)))
    print(f"{name}/{free}: x {ex:.1e} grad {eg:.1e} H {eH:.1e} d {ed:.1e} p {ep:.1e} info {info}")
    assert ex <= 1e-10
    assert eg <= 1e-10
    assert eH <= 1e-9
    assert ed <= 1e-8
    assert ep <= 1e-8 * max(1.0, np.max(np.abs(info_o["d"])))
    assert info["tau"] == info_o["tau"] and info["attempts"] == info_o["attempts"]
    assert abs(info["F"] - info_o["F"]) <= 1e-10 * abs(info_o["F"])
    assert info["resid"] <= 1e-9
    assert np.all(_np(pd)[j1:] == p[j1:])          # controls outside [j0, j1) untouched (R-T2)


def test_tracking_trace_matches_oracle():
    # five consecutive minutes of +-5 % sinusoidal loads on case118 (generator set points)
    g, L, c, x, p = _tracking_case("case118", dict(tap_line=True), costs=True)
    n_pv = int(np.sum(L.p_kind == 2))
    Pd, Qd = gridgen.load_scenario(g, 60, amp=0.05, kind="sin", seed=1)
    xo, po = x.copy(), p.copy()
    xd, pd = _dev(x), _dev(p)
    for t in range(5):
        po, xo, info_o = trk.tracking_step(g, po, xo, Pd[t], Qd[t], 0, n_pv, N=64, L=L)
        _, _, d, info = c.tracking_step(xd, pd, 64, Pd=_dev(Pd[t]), Qd=_dev(Qd[t]), j0=0, j1=n_pv)
        assert _rel(_np(d), info_o["d"]) <= 1e-8, t
    assert float(np.max(np.abs(_np(pd) - po))) <= 1e-8
    assert float(np.max(np.abs(_np(xd) - xo))) <= 1e-9


def test_tracking_step_full_size_case9241():
    # BASELINE.json's largest grid, in the bench's configuration (N = 1024, set points free)
    g, L, c, x, p = _tracking_case("case9241pegase", costs=True)
    n_pv = int(np.sum(L.p_kind == 2))
    Pd, Qd = gridgen.load_scenario(g, 60, amp=0.05, kind="sin", seed=4)
    p_o, x_o, info_o = trk.tracking_step(g, p, x, Pd[0], Qd[0], 0, n_pv, N=1024, L=L)
    xd, pd = _dev(x), _dev(p)
    grad, H, d, info = c.tracking_step(xd, pd, 1024, Pd=_dev(Pd[0]), Qd=_dev(Qd[0]), j0=0, j1=n_pv)
    HT = _np(H)
    eH = max(_rel(HT[k], info_o["H"][:, k]) for k in range(0, n_pv, 37))
    ed = _rel(_np(d), info_o["d"])
    print(f"case9241: H {eH:.1e} d {ed:.1e} info {info}")
    assert float(np.max(np.abs(_np(xd) - x_o))) <= 1e-10
    assert _rel(_np(grad), info_o["grad"]) <= 1e-10
    assert eH <= 1e-9
    assert ed <= 1e-8
    assert info["tau"] == info_o["tau"] == 0.0


def test_tracking_step_voltage_block_and_single_control():
    # free range not starting at 0 (the voltage set points [n_pv, n_p)) and a single
    # free control: the [j0, j1) block of the transposed columns, p untouched outside
    g, L, c, x, p = _tracking_case("case118", dict(tap_line=True))
    n_pv = int(np.sum(L.p_kind == 2))
    Pd, Qd = gridgen.load_scenario(g, 60, amp=0.05, kind="sin", seed=5)
    for j0, j1 in ((n_pv, L.n_p), (3, 4)):
        p_o, x_o, info_o = trk.tracking_step(g, p, x, Pd[2], Qd[2], j0, j1, N=64, L=L)
        xd, pd = _dev(x), _dev(p)
        grad, H, d, info = c.tracking_step(xd, pd, 64, Pd=_dev(Pd[2]), Qd=_dev(Qd[2]), j0=j0, j1=j1)
        assert (info["tau"], info["attempts"]) == (info_o["tau"], info_o["attempts"])
        assert _rel(_np(d), info_o["d"]) <= 1e-8
        pn = _np(pd)
        assert np.all(pn[:j0] == p[:j0]) and np.all(pn[j1:] == p[j1:])
        assert float(np.max(np.abs(pn - p_o))) <= 1e-8 * max(1.0, float(np.max(np.abs(info_o["d"]))))
