"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle (-m gpu).

Tolerance (BASELINE.json north_star, R21 revised r02): tests/parity.py
-- per-column max-norm relative error <= 1e-9 (primary); entrywise <= 1e-9 on
entries >= 1e-4 max|H|, and at SURVEY R21's 1e-6 floor either <= 1e-9 or
within 4x the oracle's own pivot-order floor.  Intermediates (g, J-based quantities, Z, Y_x, Psi) use
1e-11 relative to the block's max.  Integer outputs (orderings, sizes) are
compared exactly.
"""
import numpy as np
import pytest

import gridgen
from oracle import powerflow as pf
from oracle import reduction as red
from parity import check_hessian

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
rh = pytest.importorskip("paper_2201_00241_b200")

TOL_H = 1e-9


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _np(t):
    return t.detach().cpu().numpy()


def col_rel_err(A, B):
    den = np.maximum(np.max(np.abs(B), axis=0), 1e-300)
    return float(np.max(np.max(np.abs(A - B), axis=0) / den))


def setup(grid):
    ctx = rh.RedHess(0)
    ctx.load_grid(grid)
    x, p = ctx.state_vectors(grid)
    xd, pd = _dev(x), _dev(p)
    ctx.set_state(xd, pd)
    return ctx, x, p


CASES = [("case9", dict(tap_line=True)), ("case118", dict(tap_line=True)), ("case1354pegase", {}),
         ("case2869pegase", {})]


@pytest.fixture(scope="module", params=CASES, ids=[c[0] for c in CASES])
def solved_case(request):
    name, kw = request.param
    g = pf.backout_loads(gridgen.make_grid(name, **kw))
    L = pf.Layout(g)
    x, p = pf.state_vectors(g, L)
    grad, lam = red.reduced_gradient(g, x, p, L)
    ops = red.operators(g, x, p, lam, L)
    return name, g, L, x, p, grad, lam, ops


def test_residual_objective(solved_case):
    name, g, L, x, p, *_ = solved_case
    g2 = gridgen.make_grid(name)        # unsolved point: g != 0
    ctx, x2, p2 = setup(g2)
    gd, fd = ctx.residual()
    want = pf.residual(g2, x2, p2)
    assert np.max(np.abs(_np(gd) - want)) <= 1e-12 * max(1.0, np.max(np.abs(want)))
    fw = pf.objective(g2, x2, p2)
    assert abs(_np(fd)[0] - fw) <= 1e-12 * abs(fw)


def test_reduced_gradient(solved_case):
    name, g, L, x, p, grad, lam, ops = solved_case
    ctx, *_ = setup(g)
    gd, ld = ctx.reduced_gradient()
    assert np.max(np.abs(_np(ld) - lam)) <= 1e-10 * np.max(np.abs(lam))
    assert np.max(np.abs(_np(gd) - grad)) <= 1e-10 * np.max(np.abs(grad))


def test_hvp_stages_random_W(solved_case):
    name, g, L, x, p, grad, lam, ops = solved_case
    ctx, *_ = setup(g)
    ctx.reduced_gradient()
    for N in (1, 3, 37, 70):
        W = gridgen.random_W(L.n_p, N, seed=N)
        trace = {}
        HWo = red.hvp_batch(ops, W, trace)
        HW, Z, Yx, Psi = (_np(t) for t in ctx.hvp_stages(_dev(W)))
        assert col_rel_err(Z, trace["Z"]) <= 1e-10, "Z"
        assert col_rel_err(Yx, trace["Yx"]) <= 1e-10, "Yx"
        assert col_rel_err(Psi, trace["Psi"]) <= 1e-10, "Psi"
        assert col_rel_err(HW, HWo) <= TOL_H, "HW"
        HW2 = _np(ctx.hvp(_dev(W)))       # fused kernel == staged kernels bitwise
        assert np.array_equal(HW2, HW)


def test_full_hessian_parity(solved_case):
    name, g, L, x, p, grad, lam, ops = solved_case
    ctx, *_ = setup(g)
    ctx.reduced_gradient()
    N = {"case9": 5, "case118": 64, "case1354pegase": 256, "case2869pegase": 512}[name]
    H = _np(ctx.full_hessian(N))
    Ho = red.full_hessian(ops, N)
    check_hessian(H, Ho, f"{name} N={N} (separate calls)", ops, N, red.full_hessian)
    # batch invariance: bitwise identical across N (fixed per-column arithmetic order)
    for N2 in (1, 7, L.n_p):
        assert np.array_equal(_np(ctx.full_hessian(N2)), H), N2
    # transposed shard layout
    j0, j1 = L.n_p // 3, L.n_p // 3 + min(50, L.n_p - L.n_p // 3)
    Ht = _np(ctx.hessian_columns(j0, j1, 16, transposed=True))
    assert np.array_equal(Ht.T, H[:, j0:j1])


def test_cartesian_separator_paths(solved_case, monkeypatch):
    """The Cartesian batches' L-side separator product over T's nonzero rows only
    (k_sep_spmm, the default) and the dense S^-1 GEMM (RH_NO_SPMM), and the masked
    vs dense L sweep (RH_NO_MASK): each matches the oracle at the parity bar, and
    the mask on/off is bitwise ("Cartesian batches")."""
    name, g, L, x, p, grad, lam, ops = solved_case
    ctx, *_ = setup(g)
    ctx.reduced_gradient()
    N = {"case9": 5, "case118": 64, "case1354pegase": 256, "case2869pegase": 512}[name]
    H = _np(ctx.full_hessian(N))
    Ho = red.full_hessian(ops, N)
    monkeypatch.setenv("RH_NO_SPMM", "1")
    Hg = _np(ctx.full_hessian(N))
    assert col_rel_err(Hg, Ho) <= TOL_H
    assert col_rel_err(Hg, H) <= 1e-12     # two summation orders of the same product
    monkeypatch.delenv("RH_NO_SPMM")
    monkeypatch.setenv("RH_NO_MASK", "1")   # dense L sweep + dense separator GEMM
    Hd = _np(ctx.full_hessian(N))
    assert np.array_equal(Hd, Hg)
    monkeypatch.delenv("RH_NO_MASK")
    assert np.array_equal(_np(ctx.full_hessian(N)), H)


def test_split_u_sweep_forced(solved_case, monkeypatch):
    """The split U sweep of Cartesian batches (Z^0 swept
    without the separator, spikes per block, k_spike's DMMA product) and the pruned
    L^T sweep, forced on the small configs (RH_SPIKE=1; by default only grids with
    n_x >= 8192 take it): the oracle's Hessian at the parity bar, the unsplit path
    within rounding, bitwise N invariance, mask on/off bitwise (both with the dense
    separator product), and the fused call bitwise equal to the separate calls."""
    name, g, L, x, p, grad, lam, ops = solved_case
    N = {"case9": 5, "case118": 64, "case1354pegase": 256, "case2869pegase": 512}[name]
    ctx0, *_ = setup(g)
    ctx0.reduced_gradient()
    H0 = _np(ctx0.full_hessian(N))              # default path (unsplit on these grids)
    monkeypatch.setenv("RH_SPIKE", "1")
    ctx, *_ = setup(g)                          # the split is chosen when the grid is loaded
    ctx.reduced_gradient()
    H = _np(ctx.full_hessian(N))
    Ho = red.full_hessian(ops, N)
    check_hessian(H, Ho, f"{name} N={N} (split U sweep)", ops, N, red.full_hessian)
    assert col_rel_err(H, H0) <= 1e-11        # the same solve, two summation orders
    for N2 in (7, L.n_p):
        assert np.array_equal(_np(ctx.full_hessian(N2)), H), N2
    monkeypatch.setenv("RH_NO_SPMM", "1")       # the dense separator product, as without the mask
    Hg = _np(ctx.full_hessian(N))
    monkeypatch.setenv("RH_NO_MASK", "1")       # every tile live: Z^0 swept everywhere
    assert np.array_equal(_np(ctx.full_hessian(N)), Hg)
    monkeypatch.delenv("RH_NO_MASK")
    monkeypatch.delenv("RH_NO_SPMM")
    xd, pd = _dev(x), _dev(p)
    gf = torch.empty(L.n_p, dtype=torch.float64, device="cuda")
    Hf = torch.empty((L.n_p, L.n_p), dtype=torch.float64, device="cuda")
    for _ in range(3):                          # uncaptured, captured, replayed
        ctx.reduced_hessian(xd, pd, N, grad=gf, H=Hf)
        assert np.array_equal(_np(Hf), H)


def test_plan_cache_other_ranges(solved_case):
    """Cartesian batch plans are cached per (workspace, column range) and skipped by
    later calls and graph replays of the same range: a call on other ranges in
    between (rebuilding the plans) must not leave a replayed graph with stale plans."""
    name, g, L, x, p, *_ = solved_case
    N = {"case9": 5, "case118": 64, "case1354pegase": 256, "case2869pegase": 512}[name]
    ctx, *_ = setup(g)
    ctx.reduced_gradient()
    H = _np(ctx.full_hessian(N))
    xd, pd = _dev(x), _dev(p)
    gf = torch.empty(L.n_p, dtype=torch.float64, device="cuda")
    Hf = torch.empty((L.n_p, L.n_p), dtype=torch.float64, device="cuda")
    for _ in range(3):                           # uncaptured, captured, replayed
        ctx.reduced_hessian(xd, pd, N, grad=gf, H=Hf)
        assert np.array_equal(_np(Hf), H)
    j0, j1 = L.n_p // 5, L.n_p // 5 + min(37, L.n_p - L.n_p // 5)
    assert np.array_equal(_np(ctx.hessian_columns(j0, j1, max(1, N // 3))), H[:, j0:j1])
    for _ in range(3):
        ctx.reduced_hessian(xd, pd, N, grad=gf, H=Hf)
        assert np.array_equal(_np(Hf), H)


def test_set_multipliers_any_lambda(solved_case):
    name, g, L, x, p, *_ = solved_case
    if name not in ("case9", "case118"):
        pytest.skip("small cases only")
    ctx, *_ = setup(g)
    lam = np.random.default_rng(9).standard_normal(L.n_x)
    ctx.set_multipliers(_dev(lam))
    H = _np(ctx.full_hessian(32))
    Ho = red.full_hessian(red.operators(g, x, p, lam, L), 32)
    assert col_rel_err(H, Ho) <= TOL_H


def test_end_to_end_host_call(solved_case):
    name, g, L, x, p, grad, lam, ops = solved_case
    ctx = rh.RedHess(0)
    ctx.load_grid(g)
    gh, H = ctx.reduced_hessian_host(x, p, 64)
    assert np.max(np.abs(gh - grad)) <= 1e-10 * np.max(np.abs(grad))
    assert col_rel_err(H, red.full_hessian(ops, 64)) <= TOL_H


@pytest.mark.parametrize("name", ["case1354pegase", "case2869pegase", "case9241pegase"])
def test_lossless_closed_form_gpu(name):
    # no oracle needed: H_PgPg = 2 c2_ref 11^T + diag(2 c2), v rows/cols == 0
    g = gridgen.make_grid(name, lossless=True)
    ctx, x, p = setup(g)
    ctx.reduced_gradient()
    N = gridgen.CONFIG_N.get(name, 256)
    H = _np(ctx.full_hessian(N))
    xb, xk, pb, pk = ctx.orderings()
    c2 = np.zeros(g.n_bus)
    c2[g.gen_bus] = g.c2
    ref = int(np.flatnonzero(g.bus_type == gridgen.REF)[0])
    pgm = pk == rh.KIND_PG
    Hc = np.zeros_like(H)
    Hc[np.ix_(pgm, pgm)] = 2 * c2[ref] + np.diag(2 * c2[pb[pgm]])
    # 1e-9 = the north-star bar; the oracle itself deviates 2.6e-10 on case9241 (conditioning)
    assert np.max(np.abs(H - Hc)) <= 1e-9 * np.max(np.abs(Hc))


def test_case9241_repeated_fused_calls():
    """Uncaptured fused calls back to back (each with its own output buffers, so no
    graph): the per-state spike sweep on its own stream, the early L / Z^0 sweeps on the
    side stream and the cached batch plans must give bitwise the same Hessian every
    time (r02: a ticket counter shared by the spike sweep and workspace 0's Z^0 sweep
    raced once the cached plans removed the plan kernel's latency)."""
    g = pf.backout_loads(gridgen.make_grid("case9241pegase"))
    ctx = rh.RedHess(0)
    ctx.load_grid(g)
    x, p = ctx.state_vectors(g)
    xd, pd = _dev(x), _dev(p)
    outs = []
    for _ in range(4):
        gf, Hf = ctx.reduced_hessian(xd, pd, 1024)
        outs.append((_np(gf), _np(Hf)))
    for gf, Hf in outs[1:]:
        assert np.array_equal(Hf, outs[0][1]) and np.array_equal(gf, outs[0][0])
    ctx.set_state(xd, pd)
    ctx.reduced_gradient()
    assert np.array_equal(_np(ctx.full_hessian(1024)), outs[0][1])


def test_case9241_sampled_columns_vs_oracle():
    """Full size of the north-star config, in the launch configuration the bench
    uses (N = 1024): sampled columns checked against the oracle one by one."""
    g = pf.backout_loads(gridgen.make_grid("case9241pegase"))
    L = pf.Layout(g)
    x, p = pf.state_vectors(g, L)
    grad, lam = red.reduced_gradient(g, x, p, L)
    ops = red.operators(g, x, p, lam, L)
    ctx, *_ = setup(g)
    gd, _ = ctx.reduced_gradient()
    assert np.max(np.abs(_np(gd) - grad)) <= 1e-10 * np.max(np.abs(grad))
    H = _np(ctx.full_hessian(1024))
    cols = sorted(set(np.random.default_rng(0).choice(L.n_p, 24, replace=False).tolist() + [0, L.n_p - 1]))
    W = np.zeros((L.n_p, len(cols)))
    W[cols, np.arange(len(cols))] = 1.0
    Ho = red.hvp_batch(ops, W)
    assert col_rel_err(H[:, cols], Ho) <= TOL_H
    # symmetry diagnostic (R18): raw columns, symmetric to rounding
    assert np.max(np.abs(H - H.T)) <= 1e-9 * np.max(np.abs(H))


def test_call_order_errors():
    g = gridgen.make_grid("case9")
    ctx = rh.RedHess(0)
    ctx.load_grid(g)
    W = _dev(np.ones((ctx.n_p, 2)))
    with pytest.raises(rh.RHError) as ei:
        ctx.hvp(W)
    assert ei.value.code == rh.RH_E_ORDER
    x, p = ctx.state_vectors(g)
    ctx.set_state(_dev(x), _dev(p))
    with pytest.raises(rh.RHError) as ei:
        ctx.hvp(W)
    assert ei.value.code == rh.RH_E_ORDER
    ctx.reduced_gradient()
    ctx.hvp(W)
    assert ctx.launch_count() > 0


def test_singular_pivot_reported():
    # v = 0 at every PQ bus makes every Q-row of J vanish -> zero pivots
    g = gridgen.make_grid("case118")
    ctx = rh.RedHess(0)
    ctx.load_grid(g)
    x, p = ctx.state_vectors(g)
    xb, xk, pb, pk = ctx.orderings()
    x[xk == rh.KIND_V] = 0.0
    x[xk == rh.KIND_THETA] = 0.0
    with pytest.raises(rh.RHError) as ei:
        ctx.set_state(_dev(x), _dev(p))
    assert ei.value.code in (rh.RH_E_SINGULAR,)


def test_fused_reduced_hessian_matches_separate_calls(solved_case):
    """rh_reduced_hessian (first block sweeps overlapping the separator's
    refactorization) == rh_set_state + rh_reduced_gradient + rh_hessian_columns,
    bitwise (same kernels, same per-column arithmetic order)."""
    name, g, L, x, p, grad, lam, ops = solved_case
    ctx = rh.RedHess(0)
    ctx.load_grid(g)
    xd, pd = _dev(x), _dev(p)
    N = {"case9": 2, "case118": 40, "case1354pegase": 200, "case2869pegase": 400}[name]
    gf, Hf = ctx.reduced_hessian(xd, pd, N)
    ctx.set_state(xd, pd)
    gs, _ = ctx.reduced_gradient()
    Hs = ctx.full_hessian(N)
    assert np.array_equal(_np(gf), _np(gs))
    assert np.array_equal(_np(Hf), _np(Hs))
    assert col_rel_err(_np(Hf), red.full_hessian(ops, N)) <= TOL_H
    j0, j1 = L.n_p // 4, L.n_p // 4 + max(1, L.n_p // 3)
    _, Ht = ctx.reduced_hessian(xd, pd, N, j0=j0, j1=j1, transposed=True)
    assert np.array_equal(_np(Ht).T, _np(Hs)[:, j0:j1])


def test_newton_projection_matches_oracle(solved_case):
    """rh_newton vs the oracle's Newton from the same x0 and
    the same stopping rule: same solution, same step count (+-1), and the state
    it leaves behind gives the oracle's reduced gradient at x(p)."""
    name, g, L, x, p, grad, lam, ops = solved_case
    rng = np.random.default_rng(42)
    x0 = x + 0.01 * rng.standard_normal(x.size)   # perturbed angles and voltages
    xo = pf.newton(g, p, x0, L)
    ctx = rh.RedHess(0)
    ctx.load_grid(g)
    xd = _dev(x0)
    steps, res = ctx.newton(xd, _dev(p))
    xg = _np(xd)
    assert np.max(np.abs(xg - xo)) <= 1e-10 * max(1.0, np.max(np.abs(xo))), name
    assert res <= 1e-10
    gd, _ = ctx.reduced_gradient()
    go, _ = red.reduced_gradient(g, xo, p, L)
    assert np.max(np.abs(_np(gd) - go)) <= 1e-9 * np.max(np.abs(go))


def test_newton_from_unsolved_point():
    """From the generator's unsolved point (loads not backed out, g != 0):
    both Newtons converge to the same x(p) of the grid's own loads."""
    g2 = gridgen.make_grid("case118", tap_line=True)
    L = pf.Layout(g2)
    x0, p = pf.state_vectors(g2, L)
    xo = pf.newton(g2, p, x0, L)
    ctx = rh.RedHess(0)
    ctx.load_grid(g2)
    xd = _dev(x0)
    steps, res = ctx.newton(xd, _dev(p))
    assert np.max(np.abs(_np(xd) - xo)) <= 1e-10 * max(1.0, np.max(np.abs(xo)))
    assert res <= 1e-10 and steps >= 3
    with pytest.raises(rh.RHError) as e:   # one step cannot satisfy a zero tolerance with extra steps
        ctx.newton(_dev(x0), _dev(p), tol=0.0, extra=2, maxit=1)
    assert e.value.code == rh.RH_E_NOCONV


def test_two_kernel_assembly_matches_serial(monkeypatch):
    """The line + bus assembly kernels (grids without parallel lines) agree with the
    bus-serial k_assemble to rounding: same per-bus summation order, but the serial
    kernel contracts v_o (G c + B s) into its running sum with an FMA."""
    g = pf.backout_loads(gridgen.make_grid("case1354pegase"))
    ctx = rh.RedHess(0)
    ctx.load_grid(g)
    x, p = ctx.state_vectors(g)
    out = []
    for serial in (False, True):
        if serial:
            monkeypatch.setenv("RH_ASM_SERIAL", "1")
        gd, H = ctx.reduced_hessian(_dev(x), _dev(p), 256)
        res, f = ctx.residual()
        out.append((_np(gd), _np(H), _np(res)))
    (g0, H0, r0), (g1, H1, r1) = out
    assert np.max(np.abs(g0 - g1)) <= 1e-12 * np.max(np.abs(g1))
    assert np.max(np.abs(r0 - r1)) <= 1e-12 * np.max(np.abs(g.Pd)) + 1e-13
    assert col_rel_err(H0, H1) <= 1e-10      # rounding amplified by the solves (R21)


@pytest.mark.parametrize("own_stream", [False, True])
def test_fused_call_graph_replay(own_stream):
    """rh_reduced_hessian captures a CUDA graph on the second identical call and
    replays it afterwards: results must equal an uncaptured context's, also after
    the inputs change in place (the graph reads the buffers, not their values)."""
    g = pf.backout_loads(gridgen.make_grid("case1354pegase"))
    ctx, ref = rh.RedHess(0), rh.RedHess(0)
    ctx.load_grid(g)
    ref.load_grid(g)
    x, p = ctx.state_vectors(g)
    xd, pd = _dev(x), _dev(p)
    grad = torch.empty(ctx.n_p, dtype=torch.float64, device="cuda")
    H = torch.empty((ctx.n_p, ctx.n_p), dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream() if own_stream else torch.cuda.current_stream()
    outs = []
    with torch.cuda.stream(s):
        for it in range(4):
            if it == 3:   # new point, same buffers
                xd.add_(1e-3 * torch.from_numpy(np.random.default_rng(1).standard_normal(x.size)).cuda())
            ctx.reduced_hessian(xd, pd, 256, grad=grad, H=H, stream=s)
            s.synchronize()
            outs.append((_np(grad).copy(), _np(H).copy()))
    for a, b in outs[1:3]:
        pass
    assert np.array_equal(outs[0][1], outs[1][1]) and np.array_equal(outs[0][1], outs[2][1])
    import os
    os.environ["RH_NO_GRAPH"] = "1"
    try:
        gr, Hr = ref.reduced_hessian(xd, pd, 256)
    finally:
        del os.environ["RH_NO_GRAPH"]
    assert np.array_equal(_np(Hr), outs[3][1]) and np.array_equal(_np(gr), outs[3][0])
    # after graph replays, separate calls on the same state (the bench's order): a
    # random-W batch (dense separator GEMM on S^-T, formed on the fused call's
    # gradient stream) equals the uncaptured context's
    W = _dev(np.random.default_rng(3).standard_normal((ctx.n_p, 64)))
    with torch.cuda.stream(s):
        HW = ctx.hvp(W, stream=s)
        s.synchronize()
    assert np.array_equal(_np(HW), _np(ref.hvp(W)))


def test_host_call_graph_replay():
    """rh_reduced_hessian_host replays a CUDA graph from the third identical call
    (pinned buffers): equal to the first call and to the device call."""
    g = pf.backout_loads(gridgen.make_grid("case1354pegase"))
    ctx = rh.RedHess(0)
    ctx.load_grid(g)
    x, p = ctx.state_vectors(g)
    xh = torch.from_numpy(x).pin_memory()
    ph = torch.from_numpy(p).pin_memory()
    Hh = torch.empty((ctx.n_p, ctx.n_p), dtype=torch.float64).pin_memory()
    gh = torch.empty(ctx.n_p, dtype=torch.float64).pin_memory()
    outs = []
    for it in range(4):
        if it == 3:
            xh.add_(1e-3 * torch.from_numpy(np.random.default_rng(2).standard_normal(x.size)))
        ctx.reduced_hessian_host(xh.numpy(), ph.numpy(), 256, grad=gh.numpy(), H=Hh.numpy())
        outs.append((gh.numpy().copy(), Hh.numpy().copy()))
    assert all(np.array_equal(outs[0][1], o[1]) and np.array_equal(outs[0][0], o[0]) for o in outs[1:3])
    ref = rh.RedHess(0)
    ref.load_grid(g)
    gr, Hr = ref.reduced_hessian(_dev(xh.numpy()), _dev(p), 256)
    assert np.array_equal(_np(Hr), outs[3][1]) and np.array_equal(_np(gr), outs[3][0])


def test_empty_and_degenerate_ranges():
    """Empty inputs: an HVP with N = 0, an empty column range, the fused call with
    j0 == j1 (state + gradient only), a 0 x 0 dense solve; and N > n_p (one batch
    wider than the Hessian) against the default batching, bitwise."""
    g = pf.backout_loads(gridgen.make_grid("case118", tap_line=True))
    ctx, x, p = setup(g)
    ctx.reduced_gradient()
    W0 = torch.empty((ctx.n_p, 0), dtype=torch.float64, device="cuda")
    assert ctx.hvp(W0).shape == (ctx.n_p, 0)
    H0 = torch.empty((ctx.n_p, 1), dtype=torch.float64, device="cuda")
    ctx.hessian_columns(5, 5, 16, H=H0)                      # nothing to do, no error
    gd, _ = ctx.reduced_hessian(_dev(x), _dev(p), 16, j0=7, j1=7, H=H0)
    L = pf.Layout(g)
    grad_o, _ = red.reduced_gradient(g, x, p, L)
    assert np.max(np.abs(_np(gd) - grad_o)) <= 1e-10 * np.max(np.abs(grad_o))
    d, tau, att = ctx.dense_spd_solve(torch.empty((0, 0), dtype=torch.float64, device="cuda"),
                                      torch.empty(0, dtype=torch.float64, device="cuda"))
    assert d.numel() == 0 and att == 0
    ctx.set_state(_dev(x), _dev(p))
    ctx.reduced_gradient()
    Hwide = _np(ctx.full_hessian(4 * ctx.n_p))
    assert np.array_equal(Hwide, _np(ctx.full_hessian(64)))
