"""C-ABI library: load, exports, host-side setup logic (-m "not gpu").

No compute calls here (no GPU): a host-only context (device = -1) runs the
grid validation and the symbolic analysis, which are checked against the
oracle's orderings and against SciPy's static-pivot LU pattern.
"""
import re
import os

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import gridgen
from oracle import powerflow as pf

rh = pytest.importorskip("paper_2201_00241_b200")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "redhess.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    declared = sorted(set(re.findall(r"\b(rh_[a-z_0-9]+)\s*\(", hdr)))
    assert declared, "no declarations found"
    lib = rh.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(rh.EXPORTS) == declared


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", rh.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("name", ["case9", "case118", "case1354pegase"])
def test_orderings_match_oracle(name):
    g = gridgen.make_grid(name)
    c = rh.RedHess(-1)
    nx, npp = c.load_grid(g)
    L = pf.Layout(g)
    assert (nx, npp) == (L.n_x, L.n_p)
    xb, xk, pb, pk = c.orderings()
    assert (xb == L.x_bus).all() and (xk == L.x_kind).all()
    assert (pb == L.p_bus).all() and (pk == L.p_kind).all()


@pytest.mark.parametrize("name", ["case9", "case118", "case1354pegase"])
def test_symbolic_factor(name):
    g = pf.backout_loads(gridgen.make_grid(name, tap_line=True))
    c = rh.RedHess(-1)
    c.load_grid(g)
    S = c.symbolic()
    info = c.get_info()
    nx = c.n_x
    perm = S["perm"]
    assert sorted(perm.tolist()) == list(range(nx))
    L = pf.Layout(g)
    x, p = pf.state_vectors(g, L)
    J, _ = pf.jacobians(g, x, p, L)
    Jp = J[perm][:, perm].tocsr()
    F = sp.csr_matrix((np.ones(S["colidx"].shape[0]), S["colidx"], S["rowptr"]), shape=(nx, nx))
    # the J pattern is contained in the L+U pattern, which is structurally symmetric
    Jb = (abs(Jp) > 0).astype(int)
    assert (Jb - Jb.multiply(F)).nnz == 0
    assert (F - F.T).nnz == 0
    assert info["nnz_J"] == J.nnz and info["nnz_LU"] == F.nnz
    # SuperLU with the same (natural) ordering and static diagonal pivots must
    # produce a pattern contained in ours (numerical cancellation may drop entries)
    lu = spla.splu(Jp.tocsc(), permc_spec="NATURAL", diag_pivot_thresh=0.0,
                   options=dict(SymmetricMode=True))
    assert (lu.perm_r == np.arange(nx)).all()
    LU = (abs(lu.L) + abs(lu.U)).tocsr()
    LUb = (LU > 0).astype(int)
    assert (LUb - LUb.multiply(F)).nnz == 0
    # and the fill is exact symbolically: same count up to numerical zeros
    assert LU.nnz >= 0.95 * F.nnz
    # level sets: every dependency sits at a strictly lower level
    lf, lb = S["level_fwd"], S["level_bwd"]
    Fc = F.tocoo()
    lower = Fc.col < Fc.row
    assert np.all(lf[Fc.col[lower]] < lf[Fc.row[lower]])
    upper = Fc.col > Fc.row
    assert np.all(lb[Fc.col[upper]] < lb[Fc.row[upper]])
    assert info["levels_fwd"] == lf.max() + 1 and info["levels_bwd"] == lb.max() + 1


def _bad(grid, **kw):
    g = grid.copy()
    for k, v in kw.items():
        setattr(g, k, v)
    return g


def test_grid_validation_errors():
    g = gridgen.make_grid("case9")
    c = rh.RedHess(-1)
    bt = g.bus_type.copy()
    bt[4] = gridgen.REF
    cases = {
        "two REF": _bad(g, bus_type=bt),
        "no REF": _bad(g, bus_type=np.where(g.bus_type == gridgen.REF, gridgen.PV, g.bus_type).astype(np.int32)),
        "f == t": _bad(g, line_t=np.where(np.arange(g.n_line) == 0, g.line_f, g.line_t).astype(np.int32)),
        "bus out of range": _bad(g, line_t=np.where(np.arange(g.n_line) == 0, 99, g.line_t).astype(np.int32)),
        "gen on PQ": _bad(g, gen_bus=np.array([0, 1, 4], np.int32)),
        "two gens on a bus": _bad(g, gen_bus=np.array([0, 1, 1], np.int32)),
    }
    for what, bad in cases.items():
        with pytest.raises(rh.RHError) as ei:
            c.load_grid(bad)
        assert ei.value.code == rh.RH_E_GRID, what
    # disconnected: drop the only line of a spur bus
    spur = np.array([k for k in range(g.n_line) if 2 in (g.line_f[k], g.line_t[k])])
    keep = np.setdiff1d(np.arange(g.n_line), spur)
    bad = _bad(g, line_f=g.line_f[keep], line_t=g.line_t[keep], G_ft=g.G_ft[keep], B_ft=g.B_ft[keep],
               G_tf=g.G_tf[keep], B_tf=g.B_tf[keep])
    with pytest.raises(rh.RHError) as ei:
        c.load_grid(bad)
    assert ei.value.code == rh.RH_E_GRID and "connected" in str(ei.value)


def test_degenerate_two_bus_and_no_pq():
    c = rh.RedHess(-1)
    assert c.load_grid(gridgen.two_bus()) == (2, 1)
    g = gridgen.make_grid("case9")
    g.bus_type = np.where(g.bus_type == gridgen.PQ, gridgen.PV, g.bus_type).astype(np.int32)
    g.gen_bus = np.flatnonzero(g.bus_type != gridgen.PQ).astype(np.int32)
    g.c2 = np.ones(g.gen_bus.shape[0])
    g.c1 = np.ones(g.gen_bus.shape[0])
    g.c0 = np.zeros(g.gen_bus.shape[0])
    g.Pg = np.ones(g.gen_bus.shape[0])
    nx, npp = c.load_grid(g)
    assert nx == 8 and npp == 17


def test_host_only_context_refuses_compute():
    c = rh.RedHess(-1)
    c.load_grid(gridgen.make_grid("case9"))
    x = np.zeros(c.n_x)
    p = np.ones(c.n_p)
    with pytest.raises(rh.RHError) as ei:
        c.reduced_hessian_host(x, p, 5)
    assert ei.value.code == rh.RH_E_NODEV


@pytest.mark.parametrize("name", ["case9", "case118", "case1354pegase", "case9241pegase"])
def test_coloring_matches_oracle(name):
    # NEXT-4: the host analysis colors [J | G_p] exactly as oracle/coloring.py (R-C1, R-C2)
    from oracle import coloring as col
    from oracle import powerflow as pf
    g = gridgen.make_grid(name)
    ctx = rh.RedHess(-1)
    ctx.load_grid(g)
    colors, nc = ctx.coloring()
    L = pf.Layout(g)
    co = col.greedy_coloring(col.column_rows(g, L), L.n_x)
    assert nc == int(co.max()) + 1
    assert np.array_equal(colors, co.astype(np.int32))


def test_host_buffers_validated_before_the_call():
    """reduced_hessian_host checks dtype, contiguity and shape of every
    host buffer before libredhess sees it (a float32 / short / strided array
    would be read or written past its end by the C call)."""
    c = rh.RedHess(-1)
    c.load_grid(gridgen.make_grid("case9"))
    x = np.zeros(c.n_x)
    p = np.ones(c.n_p)
    bad = [dict(x=x.astype(np.float32)), dict(x=x[:-1]), dict(p=np.ones(2 * c.n_p)[::2]),
           dict(H=np.empty((c.n_p, c.n_p - 1))), dict(grad=np.empty(c.n_p + 1)),
           dict(H=np.empty((c.n_p, c.n_p), dtype=np.float32))]
    for kw in bad:
        args = dict(x=x, p=p)
        args.update(kw)
        xx, pp = args.pop("x"), args.pop("p")
        with pytest.raises((TypeError, ValueError)):
            c.reduced_hessian_host(xx, pp, 5, **args)
