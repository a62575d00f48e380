"""Oracle: the real-time tracking step (TEST INFRASTRUCTURE ONLY).

Follows PAPER.md section 6.3 (Eq. nonlinearoptreduced_time,
Eq. qp_rto):
  Step 1: for new loads w_t = (Pd_t, Qd_t), the reduced gradient
          g_t = grad_p F(p_t; w_t) and the reduced Hessian H_t by Alg. 2, at
          x(p_t; w_t) from the Newton projection;
  Step 2: H_t d_t = -g_t by a dense Cholesky factorization,
          p_{t+1} = p_t + d_t.
Readings:
  R-T1  H_t is symmetrized, (H + H^T) / 2, before the factorization (the raw
        columns of Alg. 2 are symmetric only up to rounding, R18).
  R-T2  the free controls are a contiguous range [j0, j1) of p; d is zero
        outside it and Step 2 solves the [j0, j1) block.  [0, n_p) is the
        paper's literal step; [0, n_pv) (the generator set points, voltage
        magnitudes held at their set points) is the bench's.
  R-T4  not positive definite -> (H + tau I) with tau = 1e-6, doubling, up to
        64 attempts ("regularized solve ... tau doubling from 1e-6").
The Cholesky factor and the triangular solves are library routines
(numpy.linalg.cholesky, scipy.linalg.solve_triangular).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from . import powerflow as pf
from . import reduction as red

TAU0 = 1e-6
MAX_TRIES = 64


def with_loads(grid, Pd, Qd):
    """The grid with loads w_t = (Pd, Qd)."""
    g = grid.copy()
    g.Pd = np.array(Pd, dtype=np.float64)
    g.Qd = np.array(Qd, dtype=np.float64)
    return g


def backout_costs(grid, x, p, j0, j1, L=None):
    """Copy of grid whose linear costs c1 make p stationary on the free
    generator set points [j0, j1) (DESIGN.md R-T5): c1_gen -= grad_p F.  Exact,
    because dF/dPg_i contains c1_i with coefficient 1 and nothing else depends
    on it (R4)."""
    L = L or pf.Layout(grid)
    grad, _ = red.reduced_gradient(grid, x, p, L)
    g2 = grid.copy()
    c1 = np.array(grid.c1, dtype=np.float64)
    for k in range(j0, j1):
        if L.p_kind[k] != 2:
            raise ValueError("cost back-out needs Pg controls only")
        c1[L.gen_of_bus[L.p_bus[k]]] -= grad[k]
    g2.c1 = c1
    return g2


def spd_solve(H, g, tau0=TAU0, max_tries=MAX_TRIES):
    """Step 2 (Eq. qp_rto): d with (Hs + tau I) d = -g, Hs = (H + H^T)/2 (R-T1),
    by Cholesky Hs + tau I = L L^T, L y = -g, L^T d = y.  tau = 0 first, then
    tau0, 2 tau0, ... while the factorization fails (R-T4).
    Returns (d, tau, attempts)."""
    H = np.asarray(H, dtype=np.float64)
    n = H.shape[0]
    Hs = 0.5 * (H + H.T)
    tau = 0.0
    for attempt in range(1, max_tries + 1):
        try:
            Lc = np.linalg.cholesky(Hs + tau * np.eye(n))
        except np.linalg.LinAlgError:
            tau = tau0 if tau == 0.0 else 2.0 * tau
            continue
        y = sla.solve_triangular(Lc, -np.asarray(g, np.float64), lower=True)
        d = sla.solve_triangular(Lc.T, y, lower=False)
        return d, tau, attempt
    raise np.linalg.LinAlgError("not positive definite after %d regularized attempts" % max_tries)


def tracking_step(grid, p_t, x_prev, Pd_t, Qd_t, j0=0, j1=None, N=None, alpha=1.0, L=None):
    """One tracking update (Steps 1-2) on the free range [j0, j1).

    Returns (p_next, x_t, info) with info = dict(F, grad, H (columns j0..j1 of
    H_t, n_p x (j1-j0)), d (length j1-j0), tau, attempts, newton_x)."""
    L = L or pf.Layout(grid)
    j1 = L.n_p if j1 is None else j1
    g = with_loads(grid, Pd_t, Qd_t)
    x = pf.newton(g, p_t, x_prev, L)                               # x(p_t; w_t)
    grad, lam = red.reduced_gradient(g, x, p_t, L)                 # g_t
    H = red.full_hessian(red.operators(g, x, p_t, lam, L), N or L.n_p)   # H_t (Alg. 2)
    d, tau, tries = spd_solve(H[j0:j1, j0:j1], grad[j0:j1])        # Eq. qp_rto
    p_next = np.array(p_t, dtype=np.float64)
    p_next[j0:j1] += alpha * d
    info = dict(F=pf.objective(g, x, p_t, L), grad=grad, H=H[:, j0:j1], d=d, tau=tau, attempts=tries)
    return p_next, x, info


def run_tracking(grid, p0, x0, Pd, Qd, j0=0, j1=None, N=None, L=None):
    """Iterate tracking_step over the load series.
    Returns a list of per-step dicts (p_t, F, |g|_inf, |d|_inf, tau)."""
    L = L or pf.Layout(grid)
    p, x = np.array(p0, np.float64), np.array(x0, np.float64)
    trace = []
    for t in range(np.asarray(Pd).shape[0]):
        p_next, x, info = tracking_step(grid, p, x, Pd[t], Qd[t], j0, j1, N, L=L)
        trace.append(dict(t=t, p=p, F=info["F"], grad_inf=float(np.max(np.abs(info["grad"][j0:j1]))),
                          d_inf=float(np.max(np.abs(info["d"]))), tau=info["tau"]))
        p = p_next
    return trace
