"""Oracle: Jacobians by column coloring + forward-mode differentiation
(TEST INFRASTRUCTURE ONLY).

Follows PAPER.md section 4 ("Sparse Jacobian Accumulation";
PAPER.md:694-713, "Forward Evaluation of Sparse Jacobians"): the columns of the
sparse Jacobian are compressed by a column coloring, one tangent direction per
color is propagated through the residual g(x, p) in forward mode (c seeds
instead of n), and the Jacobian is read back from the compressed product.

Readings (DESIGN.md R-C1..R-C3):
  R-C1  the columns colored are those of [grad_x g | grad_p g] (x entries in x
        order, then p entries in p order), so that one pass yields J and G_p.
  R-C2  the structural pattern comes from the topology: a theta_o or v_o column
        has the P / Q rows (those that exist, R2) of o and of its neighbours;
        a Pg_o column has the row P_o.  Two columns conflict iff their row sets
        intersect; colors are assigned greedily in column order, each column
        taking the smallest color unused by its conflicting predecessors (the
        paper does not name its coloring algorithm).
  R-C3  the forward-mode tangents are evaluated by the complex step,
        Im g(x + i h s_x, p + i h s_p) / h with h = 1e-30: exact to rounding for
        the complex-safe residual of oracle.powerflow (no subtraction), i.e. the
        same numbers a dual-number evaluation produces.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import powerflow as pf

H_STEP = 1e-30


def column_rows(grid, L=None):
    """Structural row sets (residual row indices, rows aligned with x, R5) of every
    column of [J | G_p] (R-C2).  Returns a list of sorted int arrays, n_x + n_p long."""
    L = L or pf.Layout(grid)
    n = L.n_bus
    nbrs = [set() for _ in range(n)]
    for f, t in zip(np.asarray(grid.line_f), np.asarray(grid.line_t)):
        nbrs[int(f)].add(int(t))
        nbrs[int(t)].add(int(f))

    def rows_of_bus_var(o):
        rows = []
        for b in sorted({o} | nbrs[o]):
            if L.th_x[b] >= 0:
                rows.append(int(L.th_x[b]))
            if L.v_x[b] >= 0:
                rows.append(int(L.v_x[b]))
        return np.array(sorted(rows), dtype=np.int64)

    out = []
    for b in L.x_bus:
        out.append(rows_of_bus_var(int(b)))
    for b, kind in zip(L.p_bus, L.p_kind):
        if kind == 2:                       # Pg_b: dg[P_b]/dPg_b = -1 only
            out.append(np.array([int(L.th_x[b])], dtype=np.int64))
        else:                               # v_b of a REF / PV bus
            out.append(rows_of_bus_var(int(b)))
    return out


def greedy_coloring(col_rows, n_rows):
    """Smallest-available-color greedy coloring of the column intersection graph
    in column order (R-C2).  Returns int array of colors (0-based)."""
    row_cols = [[] for _ in range(n_rows)]
    colors = -np.ones(len(col_rows), dtype=np.int64)
    for j, rows in enumerate(col_rows):
        used = set()
        for r in rows:
            for k in row_cols[r]:
                used.add(int(colors[k]))
        c = 0
        while c in used:
            c += 1
        colors[j] = c
        for r in rows:
            row_cols[r].append(j)
    return colors


def seed_matrices(colors, n_x, n_p):
    """S_x [n_x][c], S_p [n_p][c]: S[j, color(j)] = 1 (Fig. coloring)."""
    c = int(colors.max()) + 1 if colors.size else 0
    S = np.zeros((n_x + n_p, c))
    S[np.arange(n_x + n_p), colors] = 1.0
    return S[:n_x], S[n_x:]


def compressed_jacobian(grid, x, p, colors, L=None):
    """JS [n_x][c] = [J | G_p] S, one forward-mode tangent per color (R-C3)."""
    L = L or pf.Layout(grid)
    Sx, Sp = seed_matrices(colors, L.n_x, L.n_p)
    JS = np.zeros((L.n_x, Sx.shape[1]))
    for k in range(Sx.shape[1]):
        g = pf.residual(grid, x + 1j * H_STEP * Sx[:, k], p + 1j * H_STEP * Sp[:, k], L)
        JS[:, k] = g.imag / H_STEP
    return JS


def decompress(JS, col_rows, colors, n_x, n_p):
    """J [n_x][n_x], G_p [n_x][n_p] (CSR) with entry (r, j) = JS[r, color(j)] on the
    structural pattern ("compresses independent columns")."""
    rows, cols, vals = [], [], []
    for j, rr in enumerate(col_rows):
        rows.append(rr)
        cols.append(np.full(rr.shape[0], j))
        vals.append(JS[rr, colors[j]])
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = np.concatenate(vals)
    M = sp.csr_matrix((vals, (rows, cols)), shape=(n_x, n_x + n_p))
    return M[:, :n_x].tocsr(), M[:, n_x:].tocsr()


def colored_jacobians(grid, x, p, L=None):
    """(J, G_p, colors) by coloring + forward mode."""
    L = L or pf.Layout(grid)
    cr = column_rows(grid, L)
    colors = greedy_coloring(cr, L.n_x)
    JS = compressed_jacobian(grid, x, p, colors, L)
    J, Gp = decompress(JS, cr, colors, L.n_x, L.n_p)
    return J, Gp, colors
