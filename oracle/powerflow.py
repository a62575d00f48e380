"""Oracle: AC power-flow model in bus-row form (TEST INFRASTRUCTURE ONLY).

Follows PAPER.md section 3.1 (Eq. powerflow; Eq. powerflowvec,
PAPER.md:225-239), section 3.3 (Eq. lagrangian) and the
readings R1-R6 of DESIGN.md:

  R1  Ybus convention: P_i = sum_{j in row i of Ybus} v_i v_j (G_ij cos th_ij + B_ij sin th_ij),
      Q_i = sum_j v_i v_j (G_ij sin th_ij - B_ij cos th_ij), the diagonal included.
  R2  g = [P_pv - Pg + Pd_pv ; P_pq + Pd_pq ; Q_pq + Qd_pq].
  R3  p = (Pg over PV buses, v over {REF} u PV buses);  n_p = 2 n_pv + 1.
  R4  f = sum_gen c2 Pg^2 + c1 Pg + c0 with Pg_ref = P_ref + Pd_ref.
  R5  x = (theta_pv asc, theta_pq asc, v_pq asc); p = (Pg_pv asc, v_{ref u pv} asc).
  R6  theta_ref is a constant, not in x.

Everything here is complex-safe (analytic in theta, v, p) so that complex-step
differentiation through it is exact: no abs(), no conj(), transposes are plain.
Every matrix is assembled term by term from one Ybus entry at a time ("bus-row
form"); the CUDA path uses a per-line form with hoisted coefficients instead.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

PQ, PV, REF = 1, 2, 3


# ----------------------------------------------------------------------------
# orderings (R5)
# ----------------------------------------------------------------------------

class Layout:
    """Index maps between bus quantities and positions in x, p (R3, R5).

    kind codes: 0 = theta, 1 = v, 2 = Pg.
    """

    def __init__(self, grid):
        bt = np.asarray(grid.bus_type)
        n = bt.shape[0]
        self.n_bus = n
        refs = np.flatnonzero(bt == REF)
        if refs.shape[0] != 1:
            raise ValueError("exactly one REF bus required")
        self.ref = int(refs[0])
        pv = np.flatnonzero(bt == PV)
        pq = np.flatnonzero(bt == PQ)
        self.pv, self.pq = pv, pq
        self.n_x = pv.shape[0] + 2 * pq.shape[0]
        vbuses = np.sort(np.concatenate([[self.ref], pv]))
        self.n_p = pv.shape[0] + vbuses.shape[0]
        # x = (theta_pv, theta_pq, v_pq)
        self.x_bus = np.concatenate([pv, pq, pq]).astype(np.int64)
        self.x_kind = np.concatenate([np.zeros(pv.size + pq.size), np.ones(pq.size)]).astype(np.int64)
        # p = (Pg_pv, v over {ref} u pv)  (R3)
        self.p_bus = np.concatenate([pv, vbuses]).astype(np.int64)
        self.p_kind = np.concatenate([2 * np.ones(pv.size), np.ones(vbuses.size)]).astype(np.int64)
        # bus-space variable index: theta_b -> b, v_b -> n + b
        self.th_x = -np.ones(n, np.int64)
        self.v_x = -np.ones(n, np.int64)
        self.v_p = -np.ones(n, np.int64)
        self.pg_p = -np.ones(n, np.int64)
        for k, (b, kind) in enumerate(zip(self.x_bus, self.x_kind)):
            (self.th_x if kind == 0 else self.v_x)[b] = k
        for k, (b, kind) in enumerate(zip(self.p_bus, self.p_kind)):
            (self.pg_p if kind == 2 else self.v_p)[b] = k
        # residual rows are aligned with x: row k is P_b if x_kind[k]==0 else Q_b
        # selection matrices from bus space (2n) to x and p
        nx, npp = self.n_x, self.n_p
        rows_x = np.where(self.x_kind == 0, self.x_bus, n + self.x_bus)
        self.Ex = sp.csr_matrix((np.ones(nx), (rows_x, np.arange(nx))), shape=(2 * n, nx))
        vmask = self.p_kind == 1
        self.Ep = sp.csr_matrix((np.ones(int(vmask.sum())),
                                 (n + self.p_bus[vmask], np.flatnonzero(vmask))), shape=(2 * n, npp))
        self.Sg = self.Ex.T.tocsr()  # selects g rows (P_b / Q_b) from bus-space rows
        # generators
        gb = np.asarray(grid.gen_bus)
        if np.unique(gb).shape[0] != gb.shape[0]:
            raise ValueError("at most one generator per bus (R25)")
        self.gen_of_bus = -np.ones(n, np.int64)
        self.gen_of_bus[gb] = np.arange(gb.shape[0])
        if np.any((bt[gb] != PV) & (bt[gb] != REF)):
            raise ValueError("generator on a PQ bus")


def state_vectors(grid, layout: Layout | None = None):
    """x and p from bus-level theta, v and generator Pg (R5)."""
    L = layout or Layout(grid)
    th, v = np.asarray(grid.theta), np.asarray(grid.v)
    x = np.where(L.x_kind == 0, th[L.x_bus], v[L.x_bus]).astype(np.float64)
    p = np.empty(L.n_p)
    for k, (b, kind) in enumerate(zip(L.p_bus, L.p_kind)):
        if kind == 2:
            gi = L.gen_of_bus[b]
            p[k] = grid.Pg[gi] if gi >= 0 else 0.0
        else:
            p[k] = v[b]
    return x, p


def bus_state(grid, L: Layout, x, p):
    """(theta, v, Pg_by_bus) over all buses from x, p; complex-safe."""
    dt = np.result_type(x, p, np.float64)
    n = L.n_bus
    th = np.zeros(n, dtype=dt)
    th[L.ref] = grid.theta_ref
    v = np.zeros(n, dtype=dt)
    pg = np.zeros(n, dtype=dt)
    for k in range(L.n_x):
        (th if L.x_kind[k] == 0 else v)[L.x_bus[k]] = x[k]
    for k in range(L.n_p):
        (pg if L.p_kind[k] == 2 else v)[L.p_bus[k]] = p[k]
    return th, v, pg


# ----------------------------------------------------------------------------
# Ybus entries, one term per (row i, col j) entry, diagonal included (R1)
# ----------------------------------------------------------------------------

def ybus_terms(grid):
    """COO list of Ybus entries: row i, col j, G_ij, B_ij (R1).

    Off-diagonal entries come from lines (row f: Y_ft, row t: Y_tf); parallel
    lines stay separate terms (they add).  Diagonal entries are (G_ii, B_ii).
    """
    f = np.asarray(grid.line_f, np.int64)
    t = np.asarray(grid.line_t, np.int64)
    n = np.asarray(grid.bus_type).shape[0]
    I = np.concatenate([f, t, np.arange(n)])
    J = np.concatenate([t, f, np.arange(n)])
    G = np.concatenate([grid.G_ft, grid.G_tf, grid.G_ii]).astype(np.float64)
    B = np.concatenate([grid.B_ft, grid.B_tf, grid.B_ii]).astype(np.float64)
    return I, J, G, B


def injections(grid, th, v):
    """P_i, Q_i of Eq. powerflow with the Ybus diagonal (R1)."""
    I, J, G, B = ybus_terms(grid)
    dt = np.result_type(th, v, np.float64)
    n = th.shape[0]
    tij = th[I] - th[J]
    c, s = np.cos(tij), np.sin(tij)
    vv = v[I] * v[J]
    P = np.zeros(n, dtype=dt)
    Q = np.zeros(n, dtype=dt)
    np.add.at(P, I, vv * (G * c + B * s))
    np.add.at(Q, I, vv * (G * s - B * c))
    return P, Q


def _pg_ref(grid, L, P):
    return P[L.ref] + grid.Pd[L.ref]


def residual(grid, x, p, L: Layout | None = None):
    """g(x,p) of Eq. powerflowvec (reading R2); rows aligned with x."""
    L = L or Layout(grid)
    th, v, pg = bus_state(grid, L, x, p)
    P, Q = injections(grid, th, v)
    Pd, Qd = np.asarray(grid.Pd), np.asarray(grid.Qd)
    g = np.where(L.x_kind == 0, P[L.x_bus] + Pd[L.x_bus] - pg[L.x_bus], Q[L.x_bus] + Qd[L.x_bus])
    return g


def _cost_by_bus(grid, L):
    n = L.n_bus
    c2 = np.zeros(n)
    c1 = np.zeros(n)
    c0 = np.zeros(n)
    gb = np.asarray(grid.gen_bus)
    c2[gb], c1[gb], c0[gb] = grid.c2, grid.c1, grid.c0
    return c2, c1, c0


def objective(grid, x, p, L: Layout | None = None):
    """f = sum_gen c2 Pg^2 + c1 Pg + c0, Pg_ref = P_ref + Pd_ref (R4)."""
    L = L or Layout(grid)
    th, v, pg = bus_state(grid, L, x, p)
    P, _ = injections(grid, th, v)
    c2, c1, c0 = _cost_by_bus(grid, L)
    pgb = pg.copy()
    pgb[L.ref] = _pg_ref(grid, L, P)
    has = L.gen_of_bus >= 0
    return np.sum((c2 * pgb ** 2 + c1 * pgb + c0)[has])


# ----------------------------------------------------------------------------
# first derivatives (bus space: rows [P_0..P_n-1, Q_0..], cols [th_0.., v_0..])
# ----------------------------------------------------------------------------

def bus_jacobian(grid, th, v):
    """d(P,Q)/d(theta,v) over all buses, accumulated term by term."""
    I, J, G, B = ybus_terms(grid)
    n = th.shape[0]
    off = I != J
    tij = th[I] - th[J]
    c, s = np.cos(tij), np.sin(tij)
    vv = v[I] * v[J]
    rows, cols, vals = [], [], []

    def add(r, cidx, val):
        rows.append(r)
        cols.append(cidx)
        vals.append(val)

    Io, Jo = I[off], J[off]
    co, so, vvo, Go, Bo = c[off], s[off], vv[off], G[off], B[off]
    # P term v_i v_j (G c + B s)
    add(Io, Io, vvo * (-Go * so + Bo * co))          # d/d th_i
    add(Io, Jo, vvo * (Go * so - Bo * co))           # d/d th_j
    add(Io, n + Io, v[Jo] * (Go * co + Bo * so))     # d/d v_i
    add(Io, n + Jo, v[Io] * (Go * co + Bo * so))     # d/d v_j
    # Q term v_i v_j (G s - B c)
    add(n + Io, Io, vvo * (Go * co + Bo * so))
    add(n + Io, Jo, -vvo * (Go * co + Bo * so))
    add(n + Io, n + Io, v[Jo] * (Go * so - Bo * co))
    add(n + Io, n + Jo, v[Io] * (Go * so - Bo * co))
    # diagonal terms v_i^2 G_ii and -v_i^2 B_ii
    Id = I[~off]
    add(Id, n + Id, 2 * v[Id] * G[~off])
    add(n + Id, n + Id, -2 * v[Id] * B[~off])
    r = np.concatenate(rows)
    cc = np.concatenate(cols)
    vals = np.concatenate(vals)
    return sp.csr_matrix((vals, (r, cc)), shape=(2 * n, 2 * n))


def jacobians(grid, x, p, L: Layout | None = None):
    """J = grad_x g (n_x x n_x) and G_p = grad_p g (n_x x n_p)."""
    L = L or Layout(grid)
    th, v, _ = bus_state(grid, L, x, p)
    Jb = bus_jacobian(grid, th, v)
    J = (L.Sg @ Jb @ L.Ex).tocsr()
    Gp = (L.Sg @ Jb @ L.Ep).tolil()
    for k in range(L.n_p):
        if L.p_kind[k] == 2:  # dg[P_b]/dPg_b = -1
            Gp[L.th_x[L.p_bus[k]], k] = -1.0
    return J, Gp.tocsr()


def ref_gradient_bus(grid, th, v, L):
    """grad of P_ref over bus space (2n), complex-safe."""
    Jb = bus_jacobian(grid, th, v)
    return np.asarray(Jb[L.ref].toarray()).ravel()


def objective_gradients(grid, x, p, L: Layout | None = None):
    """grad_x f, grad_p f and f'(Pg_ref) (R4)."""
    L = L or Layout(grid)
    th, v, pg = bus_state(grid, L, x, p)
    P, _ = injections(grid, th, v)
    c2, c1, _ = _cost_by_bus(grid, L)
    pgr = _pg_ref(grid, L, P)
    mu_ref = 2 * c2[L.ref] * pgr + c1[L.ref]
    gref = ref_gradient_bus(grid, th, v, L)
    gx = mu_ref * (L.Ex.T @ gref)
    gp = mu_ref * (L.Ep.T @ gref)
    gp = np.asarray(gp, dtype=np.result_type(gp, pg))
    for k in range(L.n_p):
        if L.p_kind[k] == 2:
            b = L.p_bus[k]
            gp[k] = gp[k] + 2 * c2[b] * pg[b] + c1[b]
    return gx, gp, mu_ref


# ----------------------------------------------------------------------------
# second derivatives: Lagrangian Hessian (Eq. ADreduction 423-429)
# ----------------------------------------------------------------------------

def bus_multipliers(grid, x, p, lam, L: Layout | None = None):
    """Reverse seeds mu over bus outputs (P_b, Q_b): mu = lambda on g rows,
    mu_P,ref = f'(Pg_ref) from the objective (R4, R22)."""
    L = L or Layout(grid)
    n = L.n_bus
    _, _, mu_ref = objective_gradients(grid, x, p, L)
    muP = np.zeros(n, dtype=np.result_type(lam, mu_ref))
    muQ = np.zeros(n, dtype=muP.dtype)
    for k in range(L.n_x):
        (muP if L.x_kind[k] == 0 else muQ)[L.x_bus[k]] = lam[k]
    muP[L.ref] = mu_ref
    return muP, muQ


def bus_hessian(grid, th, v, muP, muQ):
    """sum_b muP_b d2P_b + muQ_b d2Q_b over bus space (2n x 2n), assembled term by term.

    Term T = v_i v_j (alpha c + beta s), D = -alpha s + beta c, P: (alpha,beta)=(G,B),
    Q: (alpha,beta)=(-B,G):  T_thi thi = T_thj thj = -T, T_thi thj = T,
    T_thi vi = v_j D, T_thi vj = v_i D, T_thj vi = -v_j D, T_thj vj = -v_i D,
    T_vi vj = alpha c + beta s; diagonal: d2/dv_i^2 = 2 G_ii (P), -2 B_ii (Q).
    """
    I, J, G, B = ybus_terms(grid)
    n = th.shape[0]
    off = I != J
    Io, Jo = I[off], J[off]
    Go, Bo = G[off], B[off]
    tij = th[Io] - th[Jo]
    c, s = np.cos(tij), np.sin(tij)
    alpha = muP[Io] * Go - muQ[Io] * Bo
    beta = muP[Io] * Bo + muQ[Io] * Go
    acbs = alpha * c + beta * s
    D = -alpha * s + beta * c
    T = v[Io] * v[Jo] * acbs
    ti, tj, vi, vj = Io, Jo, n + Io, n + Jo
    r, cc, vals = [], [], []

    def sym(a, b, val):
        r.append(a)
        cc.append(b)
        vals.append(val)
        r.append(b)
        cc.append(a)
        vals.append(val)

    def dia(a, val):
        r.append(a)
        cc.append(a)
        vals.append(val)

    dia(ti, -T)
    dia(tj, -T)
    sym(ti, tj, T)
    sym(ti, vi, v[Jo] * D)
    sym(ti, vj, v[Io] * D)
    sym(tj, vi, -v[Jo] * D)
    sym(tj, vj, -v[Io] * D)
    sym(vi, vj, acbs)
    Id = I[~off]
    dia(n + Id, 2 * muP[Id] * G[~off] - 2 * muQ[Id] * B[~off])
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(r), np.concatenate(cc))),
                         shape=(2 * n, 2 * n))


def lagrangian_hessian(grid, x, p, lam, L: Layout | None = None):
    """grad^2 l over (x, p), l = f + lambda^T g (Eq. lagrangian).

    Returns (Hxx, Hxp, Hpx, Hpp) as sparse matrices.  Contains
    lambda^T grad^2 g + grad^2 f: the REF-generation objective gives
    f'(Pg_ref) grad^2 P_ref (inside the mu seeds) + f''(Pg_ref) grad P_ref grad P_ref^T,
    and the Pg costs give diag(2 c2).
    """
    L = L or Layout(grid)
    th, v, _ = bus_state(grid, L, x, p)
    muP, muQ = bus_multipliers(grid, x, p, lam, L)
    Hb = bus_hessian(grid, th, v, muP, muQ)
    c2, _, _ = _cost_by_bus(grid, L)
    gref = ref_gradient_bus(grid, th, v, L)
    gref_s = sp.csr_matrix(gref.reshape(1, -1))
    Hb = Hb + 2 * c2[L.ref] * (gref_s.T @ gref_s)
    E = sp.hstack([L.Ex, L.Ep]).tocsr()
    H = (E.T @ Hb @ E).tolil()
    for k in range(L.n_p):
        if L.p_kind[k] == 2:
            H[L.n_x + k, L.n_x + k] += 2 * c2[L.p_bus[k]]
    H = H.tocsr()
    nx = L.n_x
    return H[:nx, :nx], H[:nx, nx:], H[nx:, :nx], H[nx:, nx:]


# ----------------------------------------------------------------------------
# Newton projection x(p) and load back-out
# ----------------------------------------------------------------------------

def newton(grid, p, x0, L: Layout | None = None, tol=1e-11, extra=2, maxit=40):
    """x_{k+1} = x_k - J_k^{-1} g(x_k, p); complex-safe.

    Stops `extra` iterations after max|dx| <= tol (quadratic convergence makes
    those last steps land on the rounding floor; the imaginary part of a
    complex-step perturbation converges with the same iteration)."""
    L = L or Layout(grid)
    x = np.array(x0, dtype=np.result_type(x0, p, np.float64))
    left = None
    for _ in range(maxit):
        g = residual(grid, x, p, L)
        J, _ = jacobians(grid, x, p, L)
        dx = spla.spsolve(J.tocsc(), g)
        x = x - dx
        if left is None and np.max(np.abs(dx.real)) <= tol:
            left = extra
        if left is not None:
            if left == 0:
                return x
            left -= 1
    raise RuntimeError("Newton did not converge")


def backout_loads(grid, L: Layout | None = None):
    """Return a copy of grid whose loads make g(x,p) = 0 at its bus state
    (SURVEY.md 8(d) 'Loads are backed out'): Pd = Pg - P (PV), Pd = -P (PQ),
    Qd = -Q (PQ).  REF/PV Qd and Pd_ref are kept."""
    L = L or Layout(grid)
    x, p = state_vectors(grid, L)
    th, v, pg = bus_state(grid, L, x, p)
    P, Q = injections(grid, th, v)
    g2 = grid.copy()
    Pd = np.array(grid.Pd, dtype=np.float64)
    Qd = np.array(grid.Qd, dtype=np.float64)
    Pd[L.pv] = pg[L.pv] - P[L.pv]
    Pd[L.pq] = -P[L.pq]
    Qd[L.pq] = -Q[L.pq]
    g2.Pd, g2.Qd = Pd, Qd
    return g2
