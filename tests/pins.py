"""Independent references used to PIN the oracle (tests only).

Nothing here re-types the oracle's Hessian arithmetic: the references are
  * complex-step derivatives (Im f(x + i h e_k) / h, h = 1e-30) of lower-order
    oracle quantities that are themselves pinned one level down,
  * complex Newton solves of g(x, p) = 0,
  * closed forms derived by hand (2-bus, lossless grid),
  * brute-force dense third-order tensors on tiny grids.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import powerflow as pf

H_CS = 1e-30


def cs_columns(fun, x0, cols=None, h=H_CS):
    """Complex-step Jacobian columns of a complex-safe vector function."""
    x0 = np.asarray(x0, dtype=np.float64)
    cols = range(x0.shape[0]) if cols is None else cols
    out = []
    for k in cols:
        xc = x0.astype(np.complex128)
        xc[k] += 1j * h
        out.append(np.imag(np.asarray(fun(xc))) / h)
    return np.array(out).T


def complex_reduced_gradient(grid, x0, p, L):
    """grad_p F at a (complex) p through a complex Newton solve: every step is
    analytic, so Im(.)/h of it is the exact derivative (SURVEY.md 8(c) pin (1))."""
    x = pf.newton(grid, p, x0.astype(np.complex128), L)
    J, Gp = pf.jacobians(grid, x, p, L)
    gx, gp, _ = pf.objective_gradients(grid, x, p, L)
    lam = -spla.spsolve(sp.csc_matrix(J).T.tocsc(), gx)   # plain transpose, no conj
    return gp + Gp.T @ lam


def cs_reduced_hessian(grid, cols=None, h=H_CS):
    """Columns of grad^2 F by complex-step of the reduced gradient."""
    L = pf.Layout(grid)
    x0, p0 = pf.state_vectors(grid, L)
    x0 = pf.newton(grid, p0, x0, L)
    return cs_columns(lambda pc: complex_reduced_gradient(grid, x0, pc, L), p0, cols, h), x0


def fd_reduced_hessian(grid, cols=None, h=1e-5):
    """Central finite differences of the reduced gradient."""
    from oracle import reduction as red
    L = pf.Layout(grid)
    x0, p0 = pf.state_vectors(grid, L)
    x0 = pf.newton(grid, p0, x0, L)
    cols = range(L.n_p) if cols is None else cols
    out = []
    for k in cols:
        gs = []
        for sgn in (1, -1):
            p = p0.copy()
            p[k] += sgn * h
            x = pf.newton(grid, p, x0, L)
            gs.append(red.reduced_gradient(grid, x, p, L)[0])
        out.append((gs[0] - gs[1]) / (2 * h))
    return np.array(out).T


def two_bus_closed_form(R, X, P, Q, Pd1, c2, c1, v1):
    """H = d2F/dv1^2 for the 2-bus toy of SURVEY.md 8(c) (derived by hand).

    u = v1^2, a = u - 2(RP + XQ), D = a^2 - 4|Z|^2|S|^2, s = v2^2 = (a + sqrt D)/2,
    Pg = Pd1 + P + R|S|^2/s, H = (2 c2 Pg + c1) Pg_vv + 2 c2 Pg_v^2.
    """
    Z2 = R * R + X * X
    S2 = P * P + Q * Q
    u = v1 * v1
    a = u - 2 * (R * P + X * Q)
    D = a * a - 4 * Z2 * S2
    sD = np.sqrt(D)
    s = 0.5 * (a + sD)
    s_u = 0.5 * (1 + a / sD)
    s_uu = -2 * Z2 * S2 * D ** -1.5
    s_v = 2 * v1 * s_u
    s_vv = 4 * v1 * v1 * s_uu + 2 * s_u
    Pg = Pd1 + P + R * S2 / s
    Pg_s = -R * S2 / s ** 2
    Pg_ss = 2 * R * S2 / s ** 3
    Pg_v = Pg_s * s_v
    Pg_vv = Pg_ss * s_v ** 2 + Pg_s * s_vv
    return (2 * c2 * Pg + c1) * Pg_vv + 2 * c2 * Pg_v ** 2, s


def brute_force_lagrangian_hessian(grid, x, p, lam, L):
    """Dense third-order tensor T[r, a, b] = d2 g_r / du_a du_b (u = (x, p)) by
    complex-step of the pinned Jacobian columns, contracted as
    sum_r lam_r T_r + grad^2 f (f's Hessian by complex-step of its pinned
    gradient).  This is what the method avoids forming."""
    nx, npp = L.n_x, L.n_p
    u0 = np.concatenate([x, p])

    def jac_full(u):
        J, Gp = pf.jacobians(grid, u[:nx], u[nx:], L)
        return np.hstack([J.toarray(), Gp.toarray()])

    n = nx + npp
    T = np.zeros((nx, n, n))
    for b in range(n):
        uc = u0.astype(np.complex128)
        uc[b] += 1j * H_CS
        T[:, :, b] = np.imag(jac_full(uc)) / H_CS

    def grad_f(u):
        gx, gp, _ = pf.objective_gradients(grid, u[:nx], u[nx:], L)
        return np.concatenate([gx, gp])

    Hf = cs_columns(grad_f, u0)
    return np.einsum("r,rab->ab", lam, T) + Hf
