"""Pins of oracle/coloring.py (Jacobians by column coloring + forward mode,
PAPER.md:440-468, 694-713).  The decompressed Jacobians must equal the analytic
ones of oracle.powerflow (themselves pinned by complex-step derivatives in
test_oracle.py); the coloring must be structurally orthogonal; the structural
pattern must contain the numeric one."""
import numpy as np
import pytest

import gridgen
from oracle import coloring as col
from oracle import powerflow as pf


def _grid(name, **kw):
    return pf.backout_loads(gridgen.make_grid(name, **kw))


@pytest.mark.parametrize("name,kw", [("case9", dict(tap_line=True)), ("case118", dict(tap_line=True)),
                                     ("case1354pegase", {})])
def test_colored_jacobians_equal_analytic(name, kw):
    g = _grid(name, **kw)
    L = pf.Layout(g)
    x, p = pf.state_vectors(g, L)
    J, Gp, colors = col.colored_jacobians(g, x, p, L)
    Ja, Gpa = pf.jacobians(g, x, p, L)
    for A, B in ((J, Ja), (Gp, Gpa)):
        D = (A - B).toarray() if A.shape[0] < 3000 else (A - B)
        err = abs(D).max() / abs(B).max()
        assert err <= 1e-13, err
    # far fewer seeds than columns
    assert colors.max() + 1 < (L.n_x + L.n_p) / 4 or L.n_x < 50


@pytest.mark.parametrize("name", ["case9", "case118", "case2869pegase"])
def test_coloring_is_structurally_orthogonal_and_greedy(name):
    g = gridgen.make_grid(name)
    L = pf.Layout(g)
    cr = col.column_rows(g, L)
    colors = col.greedy_coloring(cr, L.n_x)
    owner = {}
    for j, rows in enumerate(cr):
        for r in rows:
            key = (int(r), int(colors[j]))
            assert key not in owner, (j, owner.get(key))   # same color, shared row
            owner[key] = j
    # greedy: every column with color c > 0 conflicts with an earlier column of each color < c
    row_cols = {}
    for j, rows in enumerate(cr):
        for r in rows:
            row_cols.setdefault(int(r), []).append(j)
    for j in np.random.default_rng(0).choice(len(cr), 200, replace=True) if len(cr) > 200 else range(len(cr)):
        earlier = {int(colors[k]) for r in cr[j] for k in row_cols[int(r)] if k < j}
        assert all(c in earlier for c in range(int(colors[j])))
    # lower bound: a row's columns all need distinct colors
    assert colors.max() + 1 >= max(len(v) for v in row_cols.values())


def test_structural_pattern_contains_numeric_pattern():
    g = _grid("case118", tap_line=True)
    L = pf.Layout(g)
    x, p = pf.state_vectors(g, L)
    Ja, Gpa = pf.jacobians(g, x, p, L)
    M = np.hstack([Ja.toarray(), Gpa.toarray()])
    S = np.zeros_like(M, dtype=bool)
    for j, rows in enumerate(col.column_rows(g, L)):
        S[rows, j] = True
    assert not np.any((M != 0) & ~S)
    # at a generic state every structural entry is numerically nonzero
    assert np.all(M[S] != 0)


def test_seed_count_equals_tangent_count_two_bus():
    # 2-bus toy: x = (theta_2, v_2) share both rows -> 2 colors; p = (v_1) conflicts with both
    g = gridgen.two_bus()
    L = pf.Layout(g)
    cr = col.column_rows(g, L)
    colors = col.greedy_coloring(cr, L.n_x)
    assert colors.tolist() == [0, 1, 2]
