"""Pins of oracle/tracking.py (the real-time tracking step).

What pins it (none of these retypes its formulas):
  * Step 2 on matrices with closed-form inverses: tridiag(-1, 2, -1) and an
    indefinite diagonal (the tau-doubling count and the regularized solution
    in closed form, R-T4).
  * the fixed point g = 0 => d = 0 exactly (SPEC.md tracking invariants);
  * the descent property g^T d < 0 whenever tau = 0;
  * the second-order model: F(p + s d) - F(p) - s g^T d - s^2/2 d^T H d = O(s^3)
    with F evaluated independently by the Newton projection;
  * with constant loads the tracking iteration IS Newton's method on F: the
    gradient norm contracts quadratically to the rounding floor.
"""
import numpy as np
import pytest

import gridgen
from oracle import powerflow as pf
from oracle import reduction as red
from oracle import tracking as trk


def solved(name, **kw):
    return pf.backout_loads(gridgen.make_grid(name, **kw))


@pytest.fixture(scope="module")
def case118():
    return solved("case118", tap_line=True)


def test_spd_solve_tridiagonal_closed_form():
    # T = tridiag(-1, 2, -1): (T^-1)_ij = min(i,j) (n + 1 - max(i,j)) / (n + 1), 1-based
    n = 7
    T = 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    i = np.arange(1, n + 1)
    Tinv = np.minimum.outer(i, i) * (n + 1 - np.maximum.outer(i, i)) / (n + 1)
    g = np.linspace(-1.0, 2.0, n)
    d, tau, tries = trk.spd_solve(T, g)
    assert tau == 0.0 and tries == 1
    np.testing.assert_allclose(d, -Tinv @ g, rtol=0, atol=1e-13)


def test_spd_solve_symmetrizes():
    # only (H + H^T)/2 matters (R-T1): an antisymmetric part changes nothing
    n = 5
    T = 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    K = np.triu(np.arange(n * n, dtype=float).reshape(n, n), 1)
    g = np.arange(n, dtype=float) - 2.0
    d0, _, _ = trk.spd_solve(T, g)
    d1, _, _ = trk.spd_solve(T + K - K.T, g)
    np.testing.assert_allclose(d1, d0, rtol=0, atol=1e-14)


def test_spd_solve_indefinite_tau_doubling():
    # diag(2, -1): fails until tau > 1; tau = 1e-6 * 2^k first exceeds 1 at k = 20,
    # so attempts = 1 (tau = 0) + 21 (k = 0..20), d = -(g1 / (2 + tau), g2 / (tau - 1))
    H = np.diag([2.0, -1.0])
    g = np.array([1.0, 1.0])
    d, tau, tries = trk.spd_solve(H, g)
    assert tries == 22
    assert tau == pytest.approx(1e-6 * 2 ** 20, rel=1e-15)
    np.testing.assert_allclose(d, [-1.0 / (2.0 + tau), -1.0 / (tau - 1.0)], rtol=1e-14)


def test_spd_solve_gives_up():
    with pytest.raises(np.linalg.LinAlgError):
        trk.spd_solve(np.diag([1.0, -1e30]), np.ones(2), max_tries=10)


def test_fixed_point_zero_gradient():
    H = np.array([[4.0, 1.0], [1.0, 3.0]])
    d, _, _ = trk.spd_solve(H, np.zeros(2))
    assert np.all(d == 0.0)


def test_load_scenario_bounds_and_seed():
    g = gridgen.make_grid("case118")
    for kind in ("sin", "walk"):
        Pd, Qd = gridgen.load_scenario(g, 30, amp=0.05, kind=kind, seed=3)
        assert Pd.shape == (30, g.Pd.shape[0]) and Qd.shape == Pd.shape
        base = np.abs(np.asarray(g.Pd))[None, :]
        assert np.all(np.abs(Pd - np.asarray(g.Pd)[None, :]) <= 0.05 * base + 1e-15)
        Pd2, _ = gridgen.load_scenario(g, 30, amp=0.05, kind=kind, seed=3)
        assert np.array_equal(Pd, Pd2)
    Pd0, _ = gridgen.load_scenario(g, 10, amp=0.0)
    assert np.array_equal(Pd0, np.repeat(np.asarray(g.Pd, float)[None, :], 10, 0))


def _newton_on_F(grid, steps, j1):
    L = pf.Layout(grid)
    x, p = pf.state_vectors(grid, L)
    out = []
    for _ in range(steps):
        p, x, info = trk.tracking_step(grid, p, x, grid.Pd, grid.Qd, 0, j1, N=64, L=L)
        out.append((np.max(np.abs(info["grad"][:j1])), info))
    return out, p, x


def test_constant_loads_is_newton_on_F(case118):
    # constant loads: p_{t+1} = p_t - H^-1 g is Newton's method on F over the
    # generator set points (R-T2): quadratic contraction of |g| to the floor
    L = pf.Layout(case118)
    n_pv = int(np.sum(L.p_kind == 2))
    out, _, _ = _newton_on_F(case118, 7, n_pv)
    gn = [o[0] for o in out]
    assert gn[-1] < 1e-9 * gn[0]
    # quadratic phase: |g_{t+1}| <= C |g_t|^2 once |g_t| < 1
    for a, b in zip(gn[:-1], gn[1:]):
        if 1e-6 < a < 1.0:
            assert b <= 10.0 * a * a, (a, b)
    for _, info in out:
        if info["tau"] == 0.0 and np.max(np.abs(info["d"])) > 0:
            assert info["grad"][:n_pv] @ info["d"] < 0.0   # descent


def test_second_order_model(case118):
    # F(p + s d) - F(p) - s g^T d - s^2/2 d^T H d = O(s^3); F by the Newton
    # projection (independent of Alg. 2), on the literal free set [0, n_p)
    L = pf.Layout(case118)
    x, p = pf.state_vectors(case118, L)
    _, x1, info = trk.tracking_step(case118, p, x, case118.Pd, case118.Qd, 0, L.n_p, N=64, L=L)
    d = info["d"] * 1e-2 / np.max(np.abs(info["d"]))     # scale the step into the Taylor regime
    g = info["grad"]
    H = 0.5 * (info["H"] + info["H"].T)
    F0 = red.reduced_objective(case118, p, x1, L)
    errs = []
    for s in (1.0, 0.5, 0.25):
        Fs = red.reduced_objective(case118, p + s * d, x1, L)
        errs.append(Fs - F0 - s * g @ d - 0.5 * s * s * d @ H @ d)
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 6.0 < r1 < 10.0 and 6.0 < r2 < 10.0, errs
    # and the full step solves the model: Hs d = -g
    np.testing.assert_allclose(H @ info["d"], -g, rtol=0, atol=1e-9 * np.max(np.abs(g)))


def test_tracking_trace_follows_the_optimum(case118):
    # +-5 % sinusoidal loads (T = 60, first 4 minutes) from the Newton-converged
    # point: every step is PD (tau = 0) and one step lands much closer to the
    # optimum p*_t of the new loads than p_t was (p*_t: Newton on F at w_t, the
    # offline comparison of PAPER.md:980-984)
    L = pf.Layout(case118)
    n_pv = int(np.sum(L.p_kind == 2))
    _, p, x = _newton_on_F(case118, 6, n_pv)
    Pd, Qd = gridgen.load_scenario(case118, 60, amp=0.05, kind="sin", seed=1)
    for t in range(4):
        p_next, x, info = trk.tracking_step(case118, p, x, Pd[t], Qd[t], 0, n_pv, N=64, L=L)
        assert info["tau"] == 0.0
        ps, xs = p_next.copy(), x.copy()
        for _ in range(6):
            ps, xs, inf2 = trk.tracking_step(case118, ps, xs, Pd[t], Qd[t], 0, n_pv, N=64, L=L)
        assert np.max(np.abs(inf2["grad"][:n_pv])) < 1e-9
        dev0, dev1 = np.max(np.abs(p - ps)), np.max(np.abs(p_next - ps))
        assert dev1 < 0.1 * dev0 and dev1 < 50.0 * dev0 * dev0, (t, dev0, dev1)   # Newton: quadratic
        p = p_next


def test_backout_costs_makes_p_stationary():
    g = pf.backout_loads(gridgen.tracking_grid("case118"))
    L = pf.Layout(g)
    n_pv = int(np.sum(L.p_kind == 2))
    x, p = pf.state_vectors(g, L)
    g0, _ = red.reduced_gradient(g, x, p, L)
    g2 = trk.backout_costs(g, x, p, 0, n_pv, L)
    grad, _ = red.reduced_gradient(g2, x, p, L)
    assert np.max(np.abs(grad[:n_pv])) <= 1e-12 * np.max(np.abs(g0[:n_pv]))
    np.testing.assert_array_equal(grad[n_pv:], g0[n_pv:])     # the v controls do not see c1
    # the Newton step from a stationary point with unchanged loads is zero
    _, _, info = trk.tracking_step(g2, p, x, g2.Pd, g2.Qd, 0, n_pv, N=64, L=L)
    assert np.max(np.abs(info["d"])) <= 1e-10


def test_tracking_grid_is_well_conditioned_for_load_changes():
    # +-5 % per-bus-phase loads keep the power flow solvable from the base state
    # on the PEGASE1354-shaped tracking grid (the paper's Table 3 case)
    g = pf.backout_loads(gridgen.tracking_grid("case1354pegase"))
    L = pf.Layout(g)
    x, p = pf.state_vectors(g, L)
    Pd, Qd = gridgen.load_scenario(g, 60, amp=0.05, kind="sin", seed=4)
    for t in (0, 15, 30):
        xt = pf.newton(trk.with_loads(g, Pd[t], Qd[t]), p, x, L)
        assert np.max(np.abs(pf.residual(trk.with_loads(g, Pd[t], Qd[t]), xt, p, L))) < 1e-10


def test_run_tracking_constant_loads_is_newton_on_F(case118):
    """run_tracking over a CONSTANT load series is Newton's method on F over the
    free set points (PAPER.md:962-975 with w_t = w): the trace's |g_t| contracts
    quadratically to the rounding floor, every step is PD (tau = 0), |d_t|
    contracts with it, and p_t is the iterate (p_0 first)."""
    L = pf.Layout(case118)
    x, p = pf.state_vectors(case118, L)
    n_pv = int(np.sum(L.p_kind == 2))
    T = 6
    Pd = np.repeat(np.asarray(case118.Pd, float)[None, :], T, 0)
    Qd = np.repeat(np.asarray(case118.Qd, float)[None, :], T, 0)
    tr = trk.run_tracking(case118, p, x, Pd, Qd, 0, n_pv, N=64, L=L)
    assert [e["t"] for e in tr] == list(range(T))
    assert np.array_equal(tr[0]["p"], p)
    gn = [e["grad_inf"] for e in tr]
    assert gn[-1] < 1e-9 * gn[0]
    for a, b in zip(gn[:-1], gn[1:]):
        if 1e-6 < a < 1.0:
            assert b <= 10.0 * a * a, (a, b)
    assert all(e["tau"] == 0.0 for e in tr)
    dn = [e["d_inf"] for e in tr]
    assert dn[-1] < 1e-6 * dn[0]
    # only the free range moves
    assert np.array_equal(tr[-1]["p"][n_pv:], p[n_pv:])
