"""Pins of the CPU oracle (-m "not gpu").

Each test checks the oracle against something other than itself: worked
values (tests/golden/), closed forms, complex-step / finite-difference
derivatives of lower-order (already pinned) quantities, brute-force tensors,
or invariants that the mathematics fixes.  A deliberately broken variant
(negative control) must fail the same pins.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp

import gridgen
import pins
from oracle import powerflow as pf
from oracle import reduction as red

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


def solved(name, **kw):
    return pf.backout_loads(gridgen.make_grid(name, **kw))


@pytest.fixture(scope="module")
def case9():
    return solved("case9", tap_line=True)


@pytest.fixture(scope="module")
def case118():
    return solved("case118", tap_line=True)


# ---------------------------------------------------------------- inputs / dims

def test_table1_dimensions():
    gold = _load("table1_dims.json")["cases"]
    for name, d in gold.items():
        g = gridgen.make_grid(name)
        L = pf.Layout(g)
        assert (g.n_bus, g.n_line, L.n_x, L.n_p) == (d["n_v"], d["n_e"], d["n_x"], d["n_p"]), name


def test_spec_admittance_values():
    for ex in _load("spec_worked_values.json")["admittance"]:
        yff, yft, ytf, ytt = gridgen.branch_admittance(ex["r"], ex["x"])
        want = complex(*ex["Y_ft"])
        assert abs(complex(yft) - want) <= ex["rtol"] * abs(want) + 1e-15
        assert abs(complex(ytf) - want) <= ex["rtol"] * abs(want) + 1e-15
        if "Y_ff" in ex:
            assert abs(complex(yff) - complex(*ex["Y_ff"])) <= 1e-12


def test_batch_count_reading():
    ex = _load("spec_worked_values.json")["batches"]
    assert red.n_batches(ex["n_p"], ex["N"]) == ex["n_batches"]
    assert red.n_batches(5, 5) == 1          # R10: div(5,5)+1 would give 2
    assert red.n_batches(2889, 1024) == 3


def test_orderings_two_bus():
    # 2-bus toy -> x = (theta_2, v_2), p = (v_1)
    L = pf.Layout(gridgen.two_bus())
    assert list(L.x_bus) == [1, 1] and list(L.x_kind) == [0, 1]
    assert list(L.p_bus) == [0] and list(L.p_kind) == [1]


def test_orderings_R5(case118):
    L = pf.Layout(case118)
    npv, npq = len(L.pv), len(L.pq)
    assert np.all(np.diff(L.x_bus[:npv]) > 0) and np.all(np.diff(L.x_bus[npv:npv + npq]) > 0)
    assert np.all(case118.bus_type[L.x_bus[:npv]] == gridgen.PV)
    assert np.all(case118.bus_type[L.x_bus[npv:]] == gridgen.PQ)
    assert np.all(L.p_kind[:npv] == 2) and np.all(L.p_kind[npv:] == 1)
    assert L.ref in set(L.p_bus[npv:].tolist())


# ---------------------------------------------------------------- g, f

def _lossless_flat_grid():
    # flat profile, no shunts/charging, zero loads, zero generation
    g = gridgen.make_grid("case118")
    yff, yft, ytf, ytt = gridgen.branch_admittance(np.full(g.n_line, 0.01), np.full(g.n_line, 0.1))
    g.G_ft, g.B_ft, g.G_tf, g.B_tf = yft.real, yft.imag, ytf.real, ytf.imag
    diag = np.zeros(g.n_bus, complex)
    np.add.at(diag, g.line_f, yff)
    np.add.at(diag, g.line_t, ytt)
    g.G_ii, g.B_ii = diag.real, diag.imag
    g.theta[:] = 0.0
    g.v[:] = 1.0
    g.Pg[:] = 0.0
    g.Pd[:] = 0.0
    g.Qd[:] = 0.0
    return g


def test_flat_profile_residual_zero():
    # flat profile, zero loads/generation, no shunts -> g = 0
    g = _lossless_flat_grid()
    x, p = pf.state_vectors(g)
    assert np.max(np.abs(pf.residual(g, x, p))) < 1e-12


def test_two_bus_injection_value():
    ex = _load("spec_worked_values.json")["two_bus_injection"]
    yff, yft, ytf, ytt = gridgen.branch_admittance(0.0, ex["x"])
    g = gridgen.two_bus()
    g.G_ft[:], g.B_ft[:], g.G_tf[:], g.B_tf[:] = yft.real, yft.imag, ytf.real, ytf.imag
    g.G_ii[:] = [yff.real, ytt.real]
    g.B_ii[:] = [yff.imag, ytt.imag]
    P, Q = pf.injections(g, np.array([0.0, ex["theta2"]]), np.array([1.0, 1.0]))
    assert abs(P[1] - ex["P2_inj"]) <= ex["rtol"] * abs(ex["P2_inj"])


def test_objective_linear_cost():
    # single non-REF generator c1=1, Pg=0.5, REF cost zero -> f = 0.5
    g = gridgen.make_grid("case9")
    g.c2[:] = 0
    g.c1[:] = 0
    g.c0[:] = 0
    L = pf.Layout(g)
    k = int(np.flatnonzero(g.gen_bus == L.pv[0])[0])
    g.c1[k] = 1.0
    g.Pg[k] = 0.5
    x, p = pf.state_vectors(g, L)
    assert abs(pf.objective(g, x, p, L) - 0.5) < 1e-15


@pytest.mark.parametrize("name", ["case9", "case118"])
def test_jacobians_complex_step(name):
    g = solved(name, tap_line=True)
    L = pf.Layout(g)
    x, p = pf.state_vectors(g, L)
    J, Gp = pf.jacobians(g, x, p, L)
    Jcs = pins.cs_columns(lambda xc: pf.residual(g, xc, p, L), x)
    Gcs = pins.cs_columns(lambda pc: pf.residual(g, x, pc, L), p)
    assert np.max(np.abs(J.toarray() - Jcs)) <= 1e-13 * np.max(np.abs(Jcs))
    assert np.max(np.abs(Gp.toarray() - Gcs)) <= 1e-13 * np.max(np.abs(Gcs))


def test_dot_product_test(case118):
    # lambda^T (J v) == (J^T lambda)^T v
    L = pf.Layout(case118)
    x, p = pf.state_vectors(case118, L)
    J, Gp = pf.jacobians(case118, x, p, L)
    rng = np.random.default_rng(0)
    lam, v = rng.standard_normal(L.n_x), rng.standard_normal(L.n_x)
    assert abs(lam @ (J @ v) - (J.T @ lam) @ v) <= 1e-12 * abs(lam @ (J @ v))


def test_objective_gradients_complex_step(case118):
    L = pf.Layout(case118)
    x, p = pf.state_vectors(case118, L)
    gx, gp, _ = pf.objective_gradients(case118, x, p, L)
    gx_cs = pins.cs_columns(lambda xc: np.atleast_1d(pf.objective(case118, xc, p, L)), x)[0]
    gp_cs = pins.cs_columns(lambda pc: np.atleast_1d(pf.objective(case118, x, pc, L)), p)[0]
    assert np.max(np.abs(gx - gx_cs)) <= 1e-13 * np.max(np.abs(gx_cs))
    assert np.max(np.abs(gp - gp_cs)) <= 1e-13 * np.max(np.abs(gp_cs))


# ---------------------------------------------------------------- second order

def _lagrangian_gradient(g, L, lam):
    """grad l = grad f + [J G_p]^T lambda, complex-safe (built from pinned pieces)."""
    def fun(u):
        x, p = u[:L.n_x], u[L.n_x:]
        J, Gp = pf.jacobians(g, x, p, L)
        gx, gp, _ = pf.objective_gradients(g, x, p, L)
        return np.concatenate([gx + J.T @ lam, gp + Gp.T @ lam])
    return fun


@pytest.mark.parametrize("name", ["case9", "case118"])
def test_lagrangian_hessian_complex_step(name):
    g = solved(name, tap_line=True)
    L = pf.Layout(g)
    x, p = pf.state_vectors(g, L)
    lam = np.random.default_rng(1).standard_normal(L.n_x)
    H = sp.bmat([list(pf.lagrangian_hessian(g, x, p, lam, L)[:2]),
                 list(pf.lagrangian_hessian(g, x, p, lam, L)[2:])]).toarray()
    Hcs = pins.cs_columns(_lagrangian_gradient(g, L, lam), np.concatenate([x, p]))
    assert np.max(np.abs(H - Hcs)) <= 1e-13 * np.max(np.abs(Hcs))


def test_lagrangian_hessian_brute_force_tensor(case9):
    # dense third-order tensor contraction, what the method avoids
    L = pf.Layout(case9)
    x, p = pf.state_vectors(case9, L)
    lam = np.random.default_rng(2).standard_normal(L.n_x)
    H = sp.bmat([list(pf.lagrangian_hessian(case9, x, p, lam, L)[:2]),
                 list(pf.lagrangian_hessian(case9, x, p, lam, L)[2:])]).toarray()
    Hbf = pins.brute_force_lagrangian_hessian(case9, x, p, lam, L)
    assert np.max(np.abs(H - Hbf)) <= 1e-13 * np.max(np.abs(Hbf))
    assert np.max(np.abs(H - H.T)) <= 1e-14 * np.max(np.abs(H))


# ---------------------------------------------------------------- reduced gradient

def test_reduced_gradient_complex_step(case118):
    L = pf.Layout(case118)
    x, p = pf.state_vectors(case118, L)
    grad, lam = red.reduced_gradient(case118, x, p, L)
    F = lambda pc: np.atleast_1d(red.reduced_objective(case118, pc, x.astype(complex), L))
    gcs = pins.cs_columns(F, p)[0]
    assert np.max(np.abs(grad - gcs)) <= 1e-12 * np.max(np.abs(gcs))


def test_reduced_gradient_lossless_closed_form():
    # all conductances zero: dF/dPg_k = 2c2_k Pg_k + c1_k - (2c2_ref Pg_ref + c1_ref); v entries 0
    g = solved("case118", lossless=True)
    L = pf.Layout(g)
    x, p = pf.state_vectors(g, L)
    grad, _ = red.reduced_gradient(g, x, p, L)
    _, _, mu_ref = pf.objective_gradients(g, x, p, L)
    c2 = np.zeros(L.n_bus)
    c1 = np.zeros(L.n_bus)
    c2[g.gen_bus], c1[g.gen_bus] = g.c2, g.c1
    want = np.zeros(L.n_p)
    for k in range(L.n_p):
        if L.p_kind[k] == 2:
            b = L.p_bus[k]
            want[k] = 2 * c2[b] * p[k] + c1[b] - mu_ref
    assert np.max(np.abs(grad - want)) <= 1e-11 * np.max(np.abs(want))


# ---------------------------------------------------------------- reduced Hessian

def test_two_bus_closed_form_golden():
    ex = _load("spec_worked_values.json")["two_bus_hessian"]
    Hc, s = pins.two_bus_closed_form(ex["R"], ex["X"], ex["P"], ex["Q"], ex["Pd1"], ex["c2"], ex["c1"], ex["v1"])
    assert abs(s - ex["s"]) <= 1e-12 and abs(Hc - ex["H"]) <= ex["rtol"] * ex["H"]
    g = gridgen.two_bus(R=ex["R"], X=ex["X"], P=ex["P"], Q=ex["Q"], Pd1=ex["Pd1"], c2=ex["c2"],
                        c1=ex["c1"], v1=ex["v1"])
    L = pf.Layout(g)
    x, p = pf.state_vectors(g, L)
    x = pf.newton(g, p, x, L)
    g.theta[1], g.v[1] = x[0], x[1]
    assert abs(x[1] ** 2 - ex["s"]) <= 1e-12
    H = red.reduced_hessian(g)
    assert H.shape == (1, 1)
    assert abs(H[0, 0] - Hc) <= 1e-12 * abs(Hc)


@pytest.mark.parametrize("name", ["case9", "case118"])
def test_hessian_complex_step_all_columns(name):
    g = solved(name, tap_line=True)
    H = red.reduced_hessian(g, N=16)
    Hcs, _ = pins.cs_reduced_hessian(g)
    assert np.max(np.abs(H - Hcs)) <= 1e-12 * np.max(np.abs(Hcs))


@pytest.mark.slow
def test_hessian_complex_step_case1354_sampled():
    g = solved("case1354pegase")
    L = pf.Layout(g)
    cols = list(range(0, L.n_p, 37)) + [L.n_p - 1]
    H = red.reduced_hessian(g, N=256)
    Hcs, _ = pins.cs_reduced_hessian(g, cols=cols)
    err = np.max(np.abs(H[:, cols] - Hcs), axis=0) / np.max(np.abs(Hcs), axis=0)
    assert np.max(err) <= 1e-11


def test_hessian_finite_difference(case9):
    H = red.reduced_hessian(case9)
    Hfd = pins.fd_reduced_hessian(case9)
    assert np.max(np.abs(H - Hfd)) <= 1e-6 * np.max(np.abs(H))


def test_hessian_dense_definition(case118):
    L = pf.Layout(case118)
    x, p = pf.state_vectors(case118, L)
    _, lam = red.reduced_gradient(case118, x, p, L)
    ops = red.operators(case118, x, p, lam, L)
    H = red.full_hessian(ops, 32)
    assert np.max(np.abs(H - red.dense_definition(ops))) <= 1e-12 * np.max(np.abs(H))


@pytest.mark.parametrize("name", ["case118", "case1354pegase"])
def test_lossless_closed_form(name):
    # G == 0 => H_PgPg = 2 c2_ref 11^T + diag(2 c2), v rows/cols == 0
    g = solved(name, lossless=True)
    L = pf.Layout(g)
    H = red.reduced_hessian(g, N=256)
    c2 = np.zeros(L.n_bus)
    c2[g.gen_bus] = g.c2
    npv = len(L.pv)
    Hc = np.zeros_like(H)
    Hc[:npv, :npv] = 2 * c2[L.ref] + np.diag(2 * c2[L.pv])
    assert np.max(np.abs(H - Hc)) <= 1e-10 * np.max(np.abs(Hc))


def test_zero_objective_gives_zero_hessian(case9):
    g = case9.copy()
    g.c2[:] = 0
    g.c1[:] = 0
    g.c0[:] = 0
    assert np.max(np.abs(red.reduced_hessian(g))) == 0.0


def test_pv_only_costs_give_diagonal(case118):
    g = case118.copy()
    L = pf.Layout(g)
    kref = int(np.flatnonzero(g.gen_bus == L.ref)[0])
    g.c2[kref] = 0
    g.c1[kref] = 0
    H = red.reduced_hessian(g)
    c2 = np.zeros(L.n_bus)
    c2[g.gen_bus] = g.c2
    want = np.zeros_like(H)
    npv = len(L.pv)
    want[np.arange(npv), np.arange(npv)] = 2 * c2[L.pv]
    assert np.max(np.abs(H - want)) <= 1e-14


def test_spec_linear_quadratic_toy():
    # g = x - A p, f = 1/2|x|^2 + 1/2|p|^2  =>  grad^2 F = A^T A + I
    rng = np.random.default_rng(3)
    nx, npp = 7, 4
    A = rng.standard_normal((nx, npp))
    ops = red.Operators(J=sp.eye(nx), Gp=-A, Hxx=sp.eye(nx), Hxp=sp.csr_matrix((nx, npp)),
                        Hpx=sp.csr_matrix((npp, nx)), Hpp=sp.eye(npp))
    H = red.full_hessian(ops, 3)
    assert np.max(np.abs(H - (A.T @ A + np.eye(npp)))) <= 1e-13


def test_symmetry_linearity_batch_invariance(case118):
    L = pf.Layout(case118)
    x, p = pf.state_vectors(case118, L)
    _, lam = red.reduced_gradient(case118, x, p, L)
    ops = red.operators(case118, x, p, lam, L)
    H1 = red.full_hessian(ops, 1)
    H64 = red.full_hessian(ops, 64)
    Hs = red.full_hessian(ops, 0, sequential=True)
    scale = np.max(np.abs(H64))
    assert np.max(np.abs(H64 - H1)) <= 1e-13 * scale
    assert np.max(np.abs(H64 - Hs)) <= 1e-13 * scale
    assert np.max(np.abs(H64 - H64.T)) <= 1e-13 * scale
    rng = np.random.default_rng(4)
    W = rng.standard_normal((L.n_p, 5))
    a, b = 2.5, -0.75
    lhs = red.hvp_batch(ops, a * W[:, :1] + b * W[:, 1:2])
    rhs = a * red.hvp_batch(ops, W[:, :1]) + b * red.hvp_batch(ops, W[:, 1:2])
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.max(np.abs(rhs))
    assert np.max(np.abs(red.hvp_batch(ops, W) - H64 @ W)) <= 1e-12 * np.max(np.abs(H64 @ W))


def test_symmetry_any_lambda(case118):
    # H(lambda) = S^T grad^2 l(lambda) S is symmetric for any lambda (R16)
    L = pf.Layout(case118)
    x, p = pf.state_vectors(case118, L)
    lam = np.random.default_rng(5).standard_normal(L.n_x)
    H = red.full_hessian(red.operators(case118, x, p, lam, L), 107)
    assert np.max(np.abs(H - H.T)) <= 1e-12 * np.max(np.abs(H))


def test_affine_in_lambda(case118):
    L = pf.Layout(case118)
    x, p = pf.state_vectors(case118, L)
    rng = np.random.default_rng(6)
    l1, l2 = rng.standard_normal(L.n_x), rng.standard_normal(L.n_x)
    H = lambda lam: red.full_hessian(red.operators(case118, x, p, lam, L), 107)
    Hm = H(0.5 * (l1 + l2))
    assert np.max(np.abs(Hm - 0.5 * (H(l1) + H(l2)))) <= 1e-12 * np.max(np.abs(Hm))


def test_angle_shift_invariance():
    g0 = solved("case118")
    g1 = g0.copy()
    g1.theta = g0.theta + 0.3
    g1.theta_ref = g0.theta_ref + 0.3
    H0 = red.reduced_hessian(g0)
    H1 = red.reduced_hessian(g1)
    assert np.max(np.abs(H0 - H1)) <= 1e-12 * np.max(np.abs(H0))


def test_bus_permutation_equivariance():
    g0 = solved("case118", tap_line=True)
    perm = np.random.default_rng(7).permutation(g0.n_bus)
    g1 = gridgen.permute_buses(g0, perm)
    L0, L1 = pf.Layout(g0), pf.Layout(g1)
    H0, H1 = red.reduced_hessian(g0), red.reduced_hessian(g1)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.shape[0])
    # p entry k of g1 is (kind, bus perm[b1]) in g0's labelling
    key0 = {(int(k), int(b)): i for i, (b, k) in enumerate(zip(L0.p_bus, L0.p_kind))}
    q = np.array([key0[(int(k), int(perm[b]))] for b, k in zip(L1.p_bus, L1.p_kind)])
    assert np.max(np.abs(H1 - H0[np.ix_(q, q)])) <= 1e-12 * np.max(np.abs(H0))


def test_negative_control_broken_projection(monkeypatch, case9):
    """A sign error in the tensor projection (drop the theta_i-v_j cross term)
    must be caught by the complex-step pin."""
    good = red.reduced_hessian(case9)
    Hcs, _ = pins.cs_reduced_hessian(case9)
    assert np.max(np.abs(good - Hcs)) <= 1e-12 * np.max(np.abs(Hcs))
    orig = pf.bus_hessian

    def broken(grid, th, v, muP, muQ):
        H = orig(grid, th, v, muP, muQ).tolil()
        n = th.shape[0]
        ref = int(np.flatnonzero(grid.bus_type == gridgen.REF)[0])
        k = next(k for k in range(grid.n_line) if ref not in (grid.line_f[k], grid.line_t[k]))
        i, j = int(grid.line_f[k]), int(grid.line_t[k])
        assert H[i, n + j] != 0
        H[i, n + j] = -H[i, n + j]
        H[n + j, i] = -H[n + j, i]
        return H.tocsr()
    monkeypatch.setattr(pf, "bus_hessian", broken)
    bad = red.reduced_hessian(case9)
    assert np.max(np.abs(bad - Hcs)) > 1e-8 * np.max(np.abs(Hcs))


def test_unsolved_point_hessian_is_shifted_problem():
    """R17: at an unsolved point the path returns grad^2 F of the problem whose
    loads are shifted by -g(x,p); loads enter only through Pg_ref."""
    g0 = gridgen.make_grid("case118")       # random loads: g != 0
    L = pf.Layout(g0)
    x, p = pf.state_vectors(g0, L)
    assert np.max(np.abs(pf.residual(g0, x, p, L))) > 1e-3
    H0 = red.reduced_hessian(g0)
    g1 = pf.backout_loads(g0)               # same Pd_ref, shifted others
    assert g1.Pd[L.ref] == g0.Pd[L.ref]
    H1 = red.reduced_hessian(g1)
    assert np.max(np.abs(H0 - H1)) <= 1e-13 * np.max(np.abs(H0))
    assert math.isfinite(float(np.max(H0)))


# ---------------------------------------------------------------- input classes the ABI accepts
# (include/redhess.h rh_grid: parallel lines add, phase shifters, n_pq = 0; R1, R24)

VARIANTS = {
    "parallel+shift": dict(name="case9", kw=dict(parallel_lines=3, phase_shift=0.08, tap_line=True)),
    "parallel118": dict(name="case118", kw=dict(parallel_lines=6, phase_shift=-0.05)),
    "no_pq": dict(name="allpv", kw=dict(shape=(12, 17, 11))),
}


def variant_grid(key):
    v = VARIANTS[key]
    return solved(v["name"], **v["kw"])


def test_variant_grids_have_their_feature():
    g = variant_grid("parallel+shift")
    pairs = [tuple(sorted(e)) for e in zip(g.line_f.tolist(), g.line_t.tolist())]
    assert len(set(pairs)) == len(pairs) - 3                       # three doubled corridors
    # phase shifter: Y_tf != Y_ft (a tap alone keeps G_ft = G_tf, B_ft = B_tf)
    assert abs(g.G_ft[1] - g.G_tf[1]) > 1e-3
    L = pf.Layout(variant_grid("no_pq"))
    assert L.n_x == 11 and L.n_p == 23


@pytest.mark.parametrize("key", sorted(VARIANTS))
def test_variant_residual_zero_and_jacobian_complex_step(key):
    g = variant_grid(key)
    L = pf.Layout(g)
    x, p = pf.state_vectors(g, L)
    assert np.max(np.abs(pf.residual(g, x, p, L))) <= 1e-12
    J, Gp = pf.jacobians(g, x, p, L)
    Jcs = pins.cs_columns(lambda xc: pf.residual(g, xc, p.astype(np.complex128), L), x)
    Gcs = pins.cs_columns(lambda pc: pf.residual(g, x.astype(np.complex128), pc, L), p)
    assert np.max(np.abs(J.toarray() - Jcs)) <= 1e-13 * np.max(np.abs(Jcs))
    assert np.max(np.abs(Gp.toarray() - Gcs)) <= 1e-13 * max(1.0, np.max(np.abs(Gcs)))


@pytest.mark.parametrize("key", sorted(VARIANTS))
def test_variant_hessian_complex_step(key):
    """H by Alg. 2 vs complex-step of the reduced gradient through complex Newton
    (SURVEY.md 8(c) pin (1)) on grids with parallel lines, a phase shifter and no
    PQ bus: the oracle is pinned on every input class the GPU tests feed it."""
    g = variant_grid(key)
    H = red.reduced_hessian(g, N=16)
    Hcs, _ = pins.cs_reduced_hessian(g)
    assert np.max(np.abs(H - Hcs)) <= 1e-12 * np.max(np.abs(Hcs))


def test_oracle_pivot_order_floor():
    """The oracle's Alg. 2 with two SuperLU column orderings (COLAMD, MMD on
    A^T + A) agrees per column to rounding: the reference the GPU is held to is
    stable, and tests/parity.py's 'oracle floor' is a rounding floor, not a
    second answer."""
    from parity import col_rel_err, oracle_alt_ordering
    g = solved("case1354pegase")
    L = pf.Layout(g)
    x, p = pf.state_vectors(g, L)
    _, lam = red.reduced_gradient(g, x, p, L)
    ops = red.operators(g, x, p, lam, L)
    H1 = red.full_hessian(ops, 256)
    H2 = oracle_alt_ordering(ops, 256, red.full_hessian)
    assert col_rel_err(H2, H1) <= 1e-10
