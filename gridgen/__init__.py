"""Seeded synthetic power-grid generator (INPUTS ONLY).

This module is shared by the CPU oracle tests and by the CUDA path's tests and
bench.  It holds none of the method's arithmetic: no power injections, no
residual, no Jacobian, no Hessian.  It only draws a topology, line impedances,
a bus-type partition, bus-level state (theta, v, Pg), loads, costs and seed
blocks W -- the recipe of SURVEY.md section 8(d) -- and converts branch
impedances to Ybus entries with the standard MATPOWER branch model
("build_admittance"; pinned by tests/test_oracle.py::test_spec_admittance_values against
SPEC.md:67-68's worked values 1/(j0.1) = -j10 and -1/(0.01+j0.1)).

Shapes follow PAPER.md:846-853 (Table 1): for each case the generator
reproduces n_v, n_e and, through the partition, n_x = n_pv + 2 n_pq and
n_p = 2 n_pv + 1.

Bus type codes follow MATPOWER: 1 = PQ, 2 = PV, 3 = REF.
"""
from __future__ import annotations

import dataclasses
import numpy as np

PQ, PV, REF = 1, 2, 3

# (n_v, n_e, n_pv) -- PAPER.md:848-853 (Table 1) and BASELINE.json configs[0]
CASES = {
    "case9": (9, 9, 2),
    "case118": (118, 186, 53),
    "case300": (300, 411, 68),
    "case1354pegase": (1354, 1991, 259),
    "case2869pegase": (2869, 4582, 509),
    "case9241pegase": (9241, 16049, 1444),
    "case30000goc": (30000, 35393, 2277),
}
# BASELINE.json "configs" order -> seed = 220100241 + index
CONFIG_ORDER = ["case9", "case118", "case1354pegase", "case2869pegase", "case9241pegase"]
CONFIG_N = {"case9": 5, "case118": 64, "case1354pegase": 256, "case2869pegase": 512,
            "case9241pegase": 1024}
SEED_BASE = 220100241


def case_seed(name: str) -> int:
    if name in CONFIG_ORDER:
        return SEED_BASE + CONFIG_ORDER.index(name)
    return SEED_BASE + 100 + sorted(CASES).index(name)


@dataclasses.dataclass
class Grid:
    """A grid in the C-ABI's terms (include/redhess.h, struct rh_grid) plus a
    bus-level operating point.  All arrays are numpy; indices are 0-based."""
    name: str
    bus_type: np.ndarray     # int32 [n_bus]
    G_ii: np.ndarray         # f64 [n_bus]  Ybus diagonal (real)
    B_ii: np.ndarray         # f64 [n_bus]  Ybus diagonal (imag)
    Pd: np.ndarray           # f64 [n_bus]
    Qd: np.ndarray           # f64 [n_bus]
    line_f: np.ndarray       # int32 [n_line]
    line_t: np.ndarray       # int32 [n_line]
    G_ft: np.ndarray         # f64 [n_line]  Ybus[f,t] real
    B_ft: np.ndarray         # f64 [n_line]  Ybus[f,t] imag
    G_tf: np.ndarray         # f64 [n_line]  Ybus[t,f] real
    B_tf: np.ndarray         # f64 [n_line]  Ybus[t,f] imag
    gen_bus: np.ndarray      # int32 [n_gen]
    c2: np.ndarray           # f64 [n_gen]
    c1: np.ndarray           # f64 [n_gen]
    c0: np.ndarray           # f64 [n_gen]
    theta_ref: float
    # operating point (bus level)
    theta: np.ndarray        # f64 [n_bus] (theta[ref] == theta_ref)
    v: np.ndarray            # f64 [n_bus]
    Pg: np.ndarray           # f64 [n_gen] (entry of the REF generator is ignored)

    @property
    def n_bus(self):
        return int(self.bus_type.shape[0])

    @property
    def n_line(self):
        return int(self.line_f.shape[0])

    @property
    def n_gen(self):
        return int(self.gen_bus.shape[0])

    @property
    def n_pv(self):
        return int(np.sum(self.bus_type == PV))

    @property
    def n_pq(self):
        return int(np.sum(self.bus_type == PQ))

    @property
    def ref(self):
        return int(np.flatnonzero(self.bus_type == REF)[0])

    def copy(self) -> "Grid":
        return dataclasses.replace(self, **{f.name: (getattr(self, f.name).copy()
                                                     if isinstance(getattr(self, f.name), np.ndarray)
                                                     else getattr(self, f.name))
                                            for f in dataclasses.fields(self)})


def branch_admittance(r, x, b=0.0, tap=1.0, shift=0.0):
    """MATPOWER branch pi-model: returns (Y_ff, Y_ft, Y_tf, Y_tt).

    ys = 1/(r + jx); t = tap * exp(j shift); Y_tt = ys + j b/2;
    Y_ff = Y_tt / |t|^2; Y_ft = -ys / conj(t); Y_tf = -ys / t.
    """
    r = np.asarray(r, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    ys = 1.0 / (r + 1j * x)
    t = np.asarray(tap, dtype=np.float64) * np.exp(1j * np.asarray(shift, dtype=np.float64))
    ytt = ys + 0.5j * np.asarray(b, dtype=np.float64)
    yff = ytt / (t * np.conj(t))
    yft = -ys / np.conj(t)
    ytf = -ys / t
    return yff, yft, ytf, ytt


def _assemble_ybus_terms(n_bus, f, t, r, x, b, tap, shift, gsh, bsh):
    yff, yft, ytf, ytt = branch_admittance(r, x, b, tap, shift)
    diag = np.zeros(n_bus, dtype=np.complex128)
    np.add.at(diag, f, yff)
    np.add.at(diag, t, ytt)
    diag += gsh + 1j * bsh
    return diag, yft, ytf


# --------------------------------------------------------------------------
# topology
# --------------------------------------------------------------------------

def _case9_topology():
    # IEEE case9 shape (MATPOWER topology recalled, unverified):
    # lines 1-4, 4-5, 5-6, 3-6, 6-7, 7-8, 8-2, 8-9, 9-4 ; gens at 1 (REF), 2, 3.
    lines = [(1, 4), (4, 5), (5, 6), (3, 6), (6, 7), (7, 8), (8, 2), (8, 9), (9, 4)]
    f = np.array([a - 1 for a, _ in lines], dtype=np.int32)
    t = np.array([b - 1 for _, b in lines], dtype=np.int32)
    bus_type = np.full(9, PQ, dtype=np.int32)
    bus_type[0] = REF
    bus_type[1] = PV
    bus_type[2] = PV
    return f, t, bus_type, None


def _geometric_topology(n_v, n_e, rng, k=12):
    from scipy.spatial import cKDTree
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import minimum_spanning_tree, connected_components

    pts = rng.random((n_v, 2))
    kk = min(k + 1, n_v)
    tree = cKDTree(pts)
    dist, idx = tree.query(pts, k=kk)
    src = np.repeat(np.arange(n_v), kk - 1)
    dst = idx[:, 1:].reshape(-1)
    d = dist[:, 1:].reshape(-1)
    a = np.minimum(src, dst)
    bb = np.maximum(src, dst)
    key = a.astype(np.int64) * n_v + bb
    key, first = np.unique(key, return_index=True)
    a, bb, d = a[first], bb[first], d[first]
    d = np.maximum(d, 1e-12)
    G = coo_matrix((d, (a, bb)), shape=(n_v, n_v)).tocsr()
    ncomp, lab = connected_components(G, directed=False)
    extra_a, extra_b, extra_d = [], [], []
    if ncomp > 1:  # join components through nearest pairs (rare with k=12)
        for c in range(1, ncomp):
            ia = np.flatnonzero(lab == 0)
            ib = np.flatnonzero(lab == c)
            dd = np.linalg.norm(pts[ia][:, None, :] - pts[ib][None, :, :], axis=2)
            p, q = np.unravel_index(np.argmin(dd), dd.shape)
            u, w = sorted((int(ia[p]), int(ib[q])))
            extra_a.append(u)
            extra_b.append(w)
            extra_d.append(max(dd[p, q], 1e-12))
            lab[lab == c] = 0
        a = np.concatenate([a, extra_a]).astype(np.int64)
        bb = np.concatenate([bb, extra_b]).astype(np.int64)
        d = np.concatenate([d, extra_d])
        G = coo_matrix((d, (a, bb)), shape=(n_v, n_v)).tocsr()
    mst = minimum_spanning_tree(G).tocoo()
    tf = np.minimum(mst.row, mst.col)
    tt = np.maximum(mst.row, mst.col)
    tree_keys = set((tf.astype(np.int64) * n_v + tt).tolist())
    all_keys = a.astype(np.int64) * n_v + bb
    nontree = np.array([i for i, kk_ in enumerate(all_keys) if kk_ not in tree_keys], dtype=np.int64)
    n_extra = n_e - (n_v - 1)
    if n_extra < 0:
        raise ValueError("n_e < n_v - 1")
    n_short = int(round(0.7 * n_extra))
    order = nontree[np.argsort(d[nontree], kind="stable")]
    short = order[:n_short]
    rest = order[n_short:]
    n_rand = n_extra - n_short
    if n_rand > rest.shape[0]:
        raise ValueError("not enough kNN candidate lines")
    rand = rng.choice(rest, size=n_rand, replace=False) if n_rand > 0 else np.zeros(0, np.int64)
    sel = np.concatenate([short, rand])
    f = np.concatenate([tf, a[sel]]).astype(np.int32)
    t = np.concatenate([tt, bb[sel]]).astype(np.int32)
    perm = rng.permutation(f.shape[0])
    return f[perm], t[perm], None, pts


def _dc_angles(n_bus, f, t, x, ref, rng, max_diff=0.25):
    """DC power-flow angles B' theta = P -- used only to draw a
    realistic operating point; not part of the method."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    bl = 1.0 / x
    Bp = sp.coo_matrix((np.concatenate([-bl, -bl, bl, bl]),
                        (np.concatenate([f, t, f, t]), np.concatenate([t, f, f, t]))),
                       shape=(n_bus, n_bus)).tocsc()
    P = rng.standard_normal(n_bus)
    P -= P.mean()
    keep = np.array([i for i in range(n_bus) if i != ref])
    th = np.zeros(n_bus)
    th[keep] = spla.spsolve(Bp[keep][:, keep].tocsc(), P[keep])
    dmax = np.max(np.abs(th[f] - th[t]))
    if dmax > 0:
        th *= max_diff / dmax
    th -= th[ref]
    return th


def make_grid(name: str = "case118", seed: int | None = None, *, lossless: bool = False,
              tap_line: bool = False, theta_ref: float = 0.0, shape=None, parallel_lines: int = 0,
              phase_shift: float = 0.0) -> Grid:
    """Draw a synthetic grid shaped like `name` (Table 1).

    lossless=True zeroes every conductance (G_ft = G_tf = G_ii = 0, no phase
    shift) -- the closed-form test case of SURVEY.md 8(c).
    tap_line=True gives one line an off-nominal tap (1.05) so that
    Y_ft != Y_tf and Y_ff != Y_tt.
    parallel_lines=k appends k extra lines between the end buses of existing
    lines (every other one reversed, f <-> t), each with its own impedance:
    their Ybus entries add (include/redhess.h, rh_grid; R1).
    phase_shift=phi gives one line (index 1) a phase-shifting transformer of
    angle phi rad, so that Y_ft and Y_tf differ by more than a conjugate tap.
    shape=(n_v, n_e, n_pv) overrides the case's counts; n_pv = n_v - 1 gives a
    grid without PQ buses (n_pq = 0, R24).
    """
    if shape is None:
        n_v, n_e, n_pv = CASES[name]
    else:
        n_v, n_e, n_pv = shape
    if seed is None:
        seed = case_seed(name) if name in CASES else SEED_BASE + 999
    rng = np.random.default_rng(seed)
    if name == "case9" and shape is None:
        f, t, bus_type, _ = _case9_topology()
    else:
        f, t, _, _ = _geometric_topology(n_v, n_e, rng)
        bus_type = np.full(n_v, PQ, dtype=np.int32)
        picks = rng.choice(n_v, size=n_pv + 1, replace=False)
        bus_type[picks[0]] = REF
        bus_type[picks[1:]] = PV
    if parallel_lines:
        prng = np.random.default_rng(seed + 7)
        dup = prng.choice(f.shape[0], size=parallel_lines, replace=False)
        rev = (np.arange(parallel_lines) % 2) == 1
        f, t = (np.concatenate([f, np.where(rev, t[dup], f[dup])]).astype(np.int32),
                np.concatenate([t, np.where(rev, f[dup], t[dup])]).astype(np.int32))
    n_line = f.shape[0]
    r = rng.uniform(0.002, 0.05, n_line)
    x = r * rng.uniform(3.0, 10.0, n_line)
    b = rng.uniform(0.0, 0.05, n_line)
    tap = np.ones(n_line)
    if tap_line:
        tap[0] = 1.05
    shift = np.zeros(n_line)
    if phase_shift and not lossless:
        shift[1 % n_line] = phase_shift
    bsh = np.where(rng.random(n_v) < 0.05, rng.uniform(0.0, 0.02, n_v), 0.0)
    gsh = np.zeros(n_v)
    if lossless:
        r = np.zeros(n_line)
    diag, yft, ytf = _assemble_ybus_terms(n_v, f, t, r, x, b, tap, shift, gsh, bsh)
    G_ii, B_ii = diag.real.copy(), diag.imag.copy()
    G_ft, B_ft, G_tf, B_tf = yft.real.copy(), yft.imag.copy(), ytf.real.copy(), ytf.imag.copy()
    if lossless:
        G_ii[:] = 0.0
        G_ft[:] = 0.0
        G_tf[:] = 0.0
    ref = int(np.flatnonzero(bus_type == REF)[0])
    theta = _dc_angles(n_v, f, t, x, ref, rng) + theta_ref
    v = rng.uniform(0.95, 1.05, n_v)
    gen_bus = np.flatnonzero((bus_type == PV) | (bus_type == REF)).astype(np.int32)
    n_gen = gen_bus.shape[0]
    Pg = rng.uniform(0.1, 1.0, n_gen)
    c2 = rng.uniform(0.5, 2.0, n_gen)
    c1 = rng.uniform(5.0, 20.0, n_gen)
    c0 = np.zeros(n_gen)
    Pd = rng.uniform(0.0, 0.5, n_v)
    Qd = rng.uniform(-0.1, 0.3, n_v)
    return Grid(name=name, bus_type=bus_type.astype(np.int32), G_ii=G_ii, B_ii=B_ii, Pd=Pd, Qd=Qd,
                line_f=f.astype(np.int32), line_t=t.astype(np.int32), G_ft=G_ft, B_ft=B_ft,
                G_tf=G_tf, B_tf=B_tf, gen_bus=gen_bus, c2=c2, c1=c1, c0=c0,
                theta_ref=float(theta_ref), theta=theta, v=v, Pg=Pg)


def two_bus(R=0.02, X=0.1, P=0.5, Q=0.2, Pd1=0.1, c2=1.5, c1=10.0, v1=1.02,
            theta2=-0.05, v2=1.0) -> Grid:
    """2-bus toy of SURVEY.md 8(c): bus 0 REF (load Pd1), bus 1 PQ (load P + jQ),
    one line Z = R + jX, no charging, no shunt.  x = (theta_2, v_2), p = (v_1)."""
    yff, yft, ytf, ytt = branch_admittance(R, X)
    return Grid(name="two_bus", bus_type=np.array([REF, PQ], np.int32),
                G_ii=np.array([yff.real, ytt.real]), B_ii=np.array([yff.imag, ytt.imag]),
                Pd=np.array([Pd1, P]), Qd=np.array([0.0, Q]),
                line_f=np.array([0], np.int32), line_t=np.array([1], np.int32),
                G_ft=np.array([yft.real]), B_ft=np.array([yft.imag]),
                G_tf=np.array([ytf.real]), B_tf=np.array([ytf.imag]),
                gen_bus=np.array([0], np.int32), c2=np.array([c2]), c1=np.array([c1]),
                c0=np.array([0.0]), theta_ref=0.0,
                theta=np.array([0.0, theta2]), v=np.array([v1, v2]), Pg=np.array([0.0]))


def random_W(n_p: int, N: int, seed: int) -> np.ndarray:
    """Seed block W ~ N(0,1), shape [n_p][N] (batch index fastest)."""
    return np.random.default_rng(seed).standard_normal((n_p, N))


def permute_buses(grid: Grid, perm: np.ndarray) -> Grid:
    """Relabel buses: new bus k is old bus perm[k]."""
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.shape[0])
    g = grid.copy()
    for name in ("bus_type", "G_ii", "B_ii", "Pd", "Qd", "theta", "v"):
        setattr(g, name, getattr(grid, name)[perm].copy())
    g.line_f = inv[grid.line_f].astype(np.int32)
    g.line_t = inv[grid.line_t].astype(np.int32)
    g.gen_bus = inv[grid.gen_bus].astype(np.int32)
    return g


def load_scenario(grid: Grid, T: int, amp: float = 0.05, kind: str = "sin", seed: int = 0,
                  sigma: float = 0.2):
    """Seeded load time series w_t = (Pd_t, Qd_t), t = 0..T-1, for the tracking
    workload (loads "updated every minute"; the paper does
    not give their evolution, DESIGN.md R-T3).  Every load stays within
    +-amp of its base value: Pd_t[b] = Pd[b] (1 + amp s_t[b]), s_t[b] in [-1, 1].

      kind "sin":  s_t[b] = sin(2 pi t / T + phi_b), phi_b ~ U(0, 2 pi) (per-bus
                   phases: the net load change stays small, so the slack bus can
                   carry it on the synthetic grids)
      kind "walk": s_t[b] = clip(s_{t-1}[b] + sigma N(0,1), -1, 1), s_{-1} = 0
    Returns (Pd [T][n_bus], Qd [T][n_bus]) float64."""
    rng = np.random.default_rng(seed)
    n = np.asarray(grid.Pd).shape[0]
    tt = np.arange(T, dtype=np.float64)[:, None]
    if kind == "sin":
        phi = rng.uniform(0.0, 2.0 * np.pi, n)[None, :]
        s = np.sin(2.0 * np.pi * tt / T + phi)
    elif kind == "walk":
        s = np.zeros((T, n))
        cur = np.zeros(n)
        for k in range(T):
            cur = np.clip(cur + sigma * rng.standard_normal(n), -1.0, 1.0)
            s[k] = cur
    else:
        raise ValueError("kind must be 'sin' or 'walk'")
    Pd = np.asarray(grid.Pd, np.float64)[None, :] * (1.0 + amp * s)
    Qd = np.asarray(grid.Qd, np.float64)[None, :] * (1.0 + amp * s)
    return Pd, Qd


def tracking_grid(name: str = "case118", seed: int | None = None, **kw) -> Grid:
    """Grid for the tracking workload: make_grid(name) with a
    smooth voltage profile -- PQ buses at 1.0, PV set points ~ U(1.0, 1.04), REF
    at 1.02 -- instead of independent U(0.95, 1.05) magnitudes, whose reactive
    flows put the backed-out operating point next to voltage collapse (DESIGN.md
    R-T5).  Loads and linear costs are backed out by the caller (the operating
    point is then a power-flow solution and p is stationary for the base loads)."""
    g = make_grid(name, seed, **kw)
    rng = np.random.default_rng((case_seed(name) if name in CASES else SEED_BASE + 999) + 17
                                if seed is None else seed + 17)
    bt = np.asarray(g.bus_type)
    v = np.ones(bt.shape[0])
    pv = np.flatnonzero(bt == PV)
    v[pv] = rng.uniform(1.0, 1.04, pv.shape[0])
    v[bt == REF] = 1.02
    g.v = v
    return g
