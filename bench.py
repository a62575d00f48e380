#!/usr/bin/env python
"""Benchmark: full reduced Hessian (arXiv 2201.00241, Alg. 2 over all column
batches) on a synthetic grid shaped like BASELINE.json's configs.

One STEP = one pass of the whole hot path:
rh_set_state (state, assembly, numeric refactorization) + rh_reduced_gradient
(first-order adjoint, hoisted FoR tape) + all ceil(n_p/N) HVP batches of the
full grad^2 F.  Multi-GPU (torchrun): the columns are sharded contiguously
over ranks and gathered with one NCCL all-gather.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--case NAME] [--N WIDTH]
    python bench.py --impl reference ...     # the CPU oracle, timed on host cores

Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "full reduced-Hessian time (ms) and batched HVPs/s vs grid size, 1/2/4/8 B200"
UNIT = "HVP/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--case", default="case9241pegase")
    ap.add_argument("--N", type=int, default=0, help="batch width (default: BASELINE config's N)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-cols", type=int, default=2048, help="oracle sample columns for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    return ap.parse_args()


def workload_name(case, N):
    return f"{case}-shaped synthetic grid, full grad^2_pp F, batch N={N}"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------- oracle (CPU)
# The CPU oracle as it stands (oracle/, never tuned for this), timed on the
# host cores.  Two modes (SURVEY.md 8(d) "How the oracle is timed alongside"):
#   * single core: setup (state + gradient, assembly + SuperLU factorization),
#     Alg. 2 on Cartesian batches with a per-stage breakdown (the Fig. 6 analog,
#     PAPER.md:920-936), and Alg. 1 one column at a time ("N=1 corresponds to
#     the CPU implementation");
#   * all cores: a process pool over contiguous column ranges, every worker
#     single-threaded with its own setup and factorization; one pool pass is a
#     REAL full Hessian (no extrapolation).

_POOL = {}


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _oracle_setup(grid, timers=None):
    from oracle import powerflow as pf
    from oracle import reduction as red
    t0 = time.perf_counter()
    L = pf.Layout(grid)
    x, p = pf.state_vectors(grid, L)
    grad, lam = red.reduced_gradient(grid, x, p, L)            # lambda + grad_p F
    t1 = time.perf_counter()
    ops = red.operators(grid, x, p, lam, L)                    # J, G_p, Lagrangian Hessian, SuperLU
    t2 = time.perf_counter()
    if timers is not None:
        timers["state_gradient"] = timers.get("state_gradient", 0.0) + (t1 - t0)
        timers["assembly_factorization"] = timers.get("assembly_factorization", 0.0) + (t2 - t1)
    return L, ops


def _oracle_columns(ops, n_p, j0, j1, N, timers=None):
    from oracle import reduction as red
    acc = 0.0
    for a in range(j0, j1, N):
        b = min(j1, a + N)
        W = np.zeros((n_p, b - a))
        W[np.arange(a, b), np.arange(b - a)] = 1.0
        acc += float(red.hvp_batch(ops, W, timers=timers).sum())
    return acc


def _pool_init(case):
    from threadpoolctl import threadpool_limits
    import gridgen
    from oracle import powerflow as pf
    _POOL["limits"] = threadpool_limits(1)
    _POOL["grid"] = pf.backout_loads(gridgen.make_grid(case))


def _pool_task(args):
    j0, j1, N = args
    t0 = time.perf_counter()
    L, ops = _oracle_setup(_POOL["grid"])
    t1 = time.perf_counter()
    chk = _oracle_columns(ops, L.n_p, j0, j1, N)
    return t1 - t0, time.perf_counter() - t1, chk


class OraclePool:
    """All-cores oracle: `workers` single-threaded processes, each with its own
    grid copy (built once, outside any timing), setup and factorization."""

    def __init__(self, case, n_p, workers):
        import multiprocessing as mpx
        self.n_p, self.workers = n_p, max(1, min(workers, n_p))
        self.pool = mpx.get_context("spawn").Pool(self.workers, initializer=_pool_init, initargs=(case,))

    def full_hessian(self, N):
        """One real full Hessian: setup on every worker + its contiguous column range.
        Returns (wall seconds, max worker setup seconds, checksum)."""
        c = -(-self.n_p // self.workers)
        tasks = [(j0, min(self.n_p, j0 + c), min(N, c)) for j0 in range(0, self.n_p, c)]
        t0 = time.perf_counter()
        res = self.pool.map(_pool_task, tasks, chunksize=1)
        wall = time.perf_counter() - t0
        return wall, max(r[0] for r in res), sum(r[2] for r in res)

    def close(self):
        self.pool.terminate()
        self.pool.join()


def oracle_single_core(grid, n_cols, N, alg1_cols=8):
    """Single-threaded oracle on a bounded sample: setup + n_cols Cartesian
    columns by Alg. 2 (batches of N, per-stage timers) + alg1_cols columns by
    Alg. 1.  Returns a dict; full-Hessian figures are EXTRAPOLATED and say so."""
    from threadpoolctl import threadpool_limits
    from oracle import reduction as red
    with threadpool_limits(1):
        st = {}
        t0 = time.perf_counter()
        L, ops = _oracle_setup(grid, st)
        t_setup = time.perf_counter() - t0
        n_cols = min(n_cols, L.n_p)
        t1 = time.perf_counter()
        _oracle_columns(ops, L.n_p, 0, n_cols, N, st)
        t_cols = time.perf_counter() - t1
        k = min(alg1_cols, L.n_p)
        t2 = time.perf_counter()
        for j in range(k):
            e = np.zeros(L.n_p)
            e[j] = 1.0
            red.hvp_sequential(ops, e)
        t_alg1 = (time.perf_counter() - t2) / k
    per_col = t_cols / n_cols
    t_full = t_setup + per_col * L.n_p
    return {"cores": 1, "setup_s": t_setup, "alg2_per_column_s": per_col, "alg2_columns": n_cols, "N": N,
            "alg1_per_column_s": t_alg1, "alg1_columns": k,
            "stages_s": {kk: float(v) for kk, v in st.items()},
            "full_hessian_s_extrapolated": t_full, "hvps_per_s_extrapolated": L.n_p / t_full,
            "alg1_full_hessian_s_extrapolated": t_setup + t_alg1 * L.n_p,
            "spent_s": t_setup + t_cols + t_alg1 * k}


def run_reference(args):
    """--impl reference: the oracle as it stands, on the host cores.  One step =
    one REAL full Hessian (setup on every worker + all n_p Cartesian columns)
    through the all-cores process pool; ms_per_step is the time it ran."""
    rank, world, _ = dist_env()
    if world > 1 and rank != 0:
        return 0
    import gridgen
    from oracle import powerflow as pf
    case = args.case
    N = args.N or gridgen.CONFIG_N.get(case, 256)
    grid = pf.backout_loads(gridgen.make_grid(case))   # the same solved operating point as our arm
    from oracle import powerflow as pf2
    n_p = pf2.Layout(grid).n_p
    cores = host_cores()
    pool = OraclePool(case, n_p, cores)
    try:
        walls = []
        for i in range(args.warmup + args.steps):
            wall, t_setup, _ = pool.full_hessian(N)
            if i >= args.warmup:
                walls.append(wall)
    finally:
        pool.close()
    t = float(np.median(walls))
    v = n_p / t
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": workload_name(case, N), "case": case, "N": N},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": pool.workers, "host_cores": cores, "kind": "oracle",
                         "sample": f"per step: one full grad^2 F of {case} (all {n_p} Cartesian columns, Alg. 2) "
                                   f"by {pool.workers} single-threaded oracle processes over contiguous column "
                                   f"ranges, each with its own setup + SuperLU factorization; not extrapolated"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    return 0


# ---------------------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([s.strip() for s in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = []
        mx = 0.0
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                mx = max(mx, float(s[1]))
                for n, v in zip(names, s[2:6]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------- ours

def backout_loads_lib(rh, ctx, grid, x, p):
    """Make (x, p) a power-flow solution: shift the loads by the library's own
    residual g(x, p) (g is linear in Pd, Qd, R2) and reload the grid."""
    ctx.set_state(x, p)
    g_res, _ = ctx.residual()
    g_np = g_res.cpu().numpy()
    xb, xk, _, _ = ctx.orderings()
    grid.Pd = grid.Pd.copy()
    grid.Qd = grid.Qd.copy()
    th_rows = xk == rh.KIND_THETA
    grid.Pd[xb[th_rows]] -= g_np[th_rows]
    grid.Qd[xb[~th_rows]] -= g_np[~th_rows]
    ctx.load_grid(grid)


PAPER_TABLE3 = {"case": "case1354pegase", "N": 256, "gpu_s": [0.05, 0.05, 0.10], "cpu_s": [1.41, 0.81, 2.22],
                "hardware": "V100 / Xeon (PAPER.md Table 3)"}


def tracking_bench(rh, gridgen, dev, case, N, minutes, warm=2, T=60):
    """Real-time tracking (Table 3): one
    rh_tracking_step per minute of a +-5 % per-bus-phase load series (seed 4),
    free controls = the generator set points (R-T2), from the optimum of the
    base loads (loads and linear costs backed out with the library's residual
    and reduced gradient, R-T5).  Step 1 = loads + Newton x(p_t; w_t) + g_t +
    H_t columns; Step 2 = dense Cholesky solve + p update (CUDA events on the
    stream, host syncs inside included)."""
    import torch
    grid = gridgen.tracking_grid(case)
    ctx = rh.RedHess(dev.index)
    n_x, n_p = ctx.load_grid(grid)
    x_np, p_np = ctx.state_vectors(grid)
    x = torch.from_numpy(x_np).to(dev)
    p = torch.from_numpy(p_np).to(dev)
    backout_loads_lib(rh, ctx, grid, x, p)
    _, _, pb, pk = ctx.orderings()
    n_pv = int(np.sum(pk == rh.KIND_PG))
    assert np.all(pk[:n_pv] == rh.KIND_PG)
    ctx.set_state(x, p)
    grad = torch.empty(n_p, dtype=torch.float64, device=dev)
    ctx.reduced_gradient(grad)
    g_np = grad.cpu().numpy()
    gen_of_bus = {int(b): i for i, b in enumerate(grid.gen_bus)}
    grid.c1 = np.array(grid.c1, dtype=np.float64)
    for k in range(n_pv):                       # dF/dPg_k contains c1 with coefficient 1
        grid.c1[gen_of_bus[int(pb[k])]] -= g_np[k]
    ctx.load_grid(grid)
    Pd, Qd = gridgen.load_scenario(grid, T, amp=0.05, kind="sin", seed=4)
    Pd_d = torch.from_numpy(Pd).to(dev)
    Qd_d = torch.from_numpy(Qd).to(dev)
    H = torch.empty((n_pv, n_p), dtype=torch.float64, device=dev)
    d = torch.empty(n_pv, dtype=torch.float64, device=dev)
    recs = []
    for t in range(warm + minutes):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, _, _, info = ctx.tracking_step(x, p, N, Pd=Pd_d[t % T], Qd=Qd_d[t % T], j0=0, j1=n_pv, grad=grad, H=H,
                                          d=d)
        wall = (time.perf_counter() - t0) * 1e3
        if t >= warm:
            recs.append((info, wall))
    med = lambda k: float(np.median([r[0][k] for r in recs]))
    return {"case": case, "N": N, "n_free": n_pv, "n_p": n_p, "minutes": minutes,
            "ms_step1": med("ms_step1"), "ms_step2": med("ms_step2"),
            "ms_total": float(np.median([r[0]["ms_step1"] + r[0]["ms_step2"] for r in recs])),
            "wall_ms": float(np.median([r[1] for r in recs])),
            "newton_steps": med("newton_steps"), "max_tau": float(max(r[0]["tau"] for r in recs)),
            "max_abs_d": float(d.abs().max().item()),
            "workload": "tracking_grid (smooth voltages), loads + c1 backed out at the base point, "
                        "+-5 % per-bus-phase sinusoidal loads (seed 4), free = Pg set points"}


def lib_cj(ctx, JS):
    """rh_compressed_jacobian into a preallocated device buffer."""
    import paper_2201_00241_b200 as rh
    rc = rh.lib().rh_compressed_jacobian(ctx._h, JS.data_ptr(), rh._stream(None))
    if rc:
        raise rh.RHError(rc, rh.lib().rh_last_error(ctx._h).decode())


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    import gridgen
    import paper_2201_00241_b200 as rh

    rank, world, local = dist_env()
    if world > 1:
        # one rank per GPU; BENCH_DIST_BACKEND=gloo (ranks sharing a GPU) is a
        # plumbing check of the sharded path on a 1-GPU box, not a measurement
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        dev_idx = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(dev_idx)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_idx))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    case = args.case
    N = args.N or gridgen.CONFIG_N.get(case, 256)
    grid = gridgen.make_grid(case)
    ctx = rh.RedHess(dev.index)
    n_x, n_p = ctx.load_grid(grid)
    info = ctx.get_info()
    x_np, p_np = ctx.state_vectors(grid)
    stream = torch.cuda.current_stream()
    x = torch.from_numpy(x_np).to(dev)
    p = torch.from_numpy(p_np).to(dev)
    # solved operating point: back the loads out with the library's own residual
    # (loads enter the path only through Pd_ref, R17)
    backout_loads_lib(rh, ctx, grid, x, p)
    ctx.set_state(x, p)
    g_res, _ = ctx.residual()
    resid_inf = float(g_res.abs().max().item())
    torch.cuda.synchronize()

    from paper_2201_00241_b200.parallel import ShardedHessian, gather_columns
    sh = ShardedHessian(ctx)                 # column shard of SURVEY.md 8(e), transposed slabs
    j0, j1, cpad = sh.j0, sh.j1, sh.c
    Hloc, Hall = sh.H_local, sh.H_all
    grad = torch.empty(n_p, dtype=torch.float64, device=dev)
    flush = None if args.no_flush else torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

    def step(timed):
        # one pass of the path: state + refactorization + reduced gradient + this
        # rank's Hessian columns (rh_reduced_hessian: the first block sweeps
        # overlap the separator's refactorization), then the all-gather
        if timed:
            ev[0].record(stream)
        ctx.reduced_hessian(x, p, N, j0=j0, j1=j1, grad=grad, H=Hloc[:j1 - j0], transposed=True)
        if timed:
            ev[2].record(stream)
        if world > 1:
            gather_columns(Hloc, n_p, out=Hall)   # one NCCL all-gather
        if timed:
            ev[3].record(stream)

    def pre_only():   # breakdown: state + refactorization + gradient alone
        ctx.set_state(x, p)
        ctx.reduced_gradient(grad)

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    clocks = ClockSampler(dev.index)
    clocks.start()
    time.sleep(0.3)
    launches0 = ctx.launch_count()
    t_step, t_hess, t_pre = [], [], []
    for _ in range(args.steps):
        if flush is not None:
            flush.fill_(1.0)          # L2 flush (256 MB > 126 MB L2), outside the timed region
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        step(True)
        torch.cuda.synchronize()
        t_step.append(ev[0].elapsed_time(ev[3]))
        t_hess.append(ev[0].elapsed_time(ev[2]))
        torch.cuda.synchronize()
        ev[0].record(stream)
        pre_only()
        ev[1].record(stream)
        torch.cuda.synchronize()
        t_pre.append(ev[0].elapsed_time(ev[1]))
    launches = (ctx.launch_count() - launches0) / args.steps
    clk = clocks.stop()
    tt = torch.tensor([sum(t_step), sum(t_hess), sum(t_pre)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms_step = tt[0].item() / args.steps
    ms_hess = tt[1].item() / args.steps
    ms_pre = tt[2].item() / args.steps

    # ---- batched HVP throughput (random W, width N, weak scaling: each GPU its own W)
    W = torch.from_numpy(gridgen.random_W(n_p, N, seed=1 + rank)).to(dev)
    HW = torch.empty_like(W)
    for _ in range(3):
        ctx.hvp(W, HW)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    hv = []
    for _ in range(reps):
        if flush is not None:
            flush.fill_(1.0)
        torch.cuda.synchronize()
        e0.record(stream)
        ctx.hvp(W, HW)
        e1.record(stream)
        torch.cuda.synchronize()
        hv.append(e0.elapsed_time(e1))
    t_hvp = torch.tensor([float(np.median(hv))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_hvp, op=dist.ReduceOp.MAX)
    hvps = world * N / (t_hvp.item() * 1e-3)

    # ---- end to end through the public API with host buffers
    x_h = torch.from_numpy(x_np).pin_memory()
    p_h = torch.from_numpy(p_np).pin_memory()
    H_h = torch.empty((cpad * world, n_p), dtype=torch.float64).pin_memory()
    g_h = torch.empty(n_p, dtype=torch.float64).pin_memory()
    h2d = (n_x + n_p) * 8
    d2h = (n_p + n_p * n_p) * 8
    if world == 1:
        def e2e_once():
            ctx.reduced_hessian_host(x_h.numpy(), p_h.numpy(), N, grad=g_h.numpy(), H=H_h.numpy())
    else:
        def e2e_once():
            x.copy_(x_h, non_blocking=True)
            p.copy_(p_h, non_blocking=True)
            ctx.set_state(x, p)
            ctx.reduced_gradient(grad)
            sh.full(N)
            g_h.copy_(grad, non_blocking=True)
            H_h.copy_(Hall, non_blocking=True)
            torch.cuda.synchronize()
    for _ in range(2):
        e2e_once()
    te = []
    for _ in range(max(5, args.steps)):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        e2e_once()
        te.append(time.perf_counter() - t0)
    t_e2e = torch.tensor([float(np.median(te))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    e2e_val = n_p / t_e2e.item()

    # ---- multi-GPU projection on this GPU: one rank's contiguous column shard of a
    # G-GPU run, timed alone (the replicated state + gradient
    # included; the all-gather, tens of microseconds over NVLink, is not)
    shards = {}
    if world == 1:
        ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for G in (2, 4, 8):
            c = -(-n_p // G)
            Hs = torch.empty((c, n_p), dtype=torch.float64, device=dev)
            ts = []
            for rep in range(8):
                if flush is not None:
                    flush.fill_(1.0)
                torch.cuda.synchronize()
                ev_a.record(stream)
                ctx.reduced_hessian(x, p, N, j0=0, j1=c, grad=grad, H=Hs, transposed=True)
                ev_b.record(stream)
                torch.cuda.synchronize()
                if rep >= 3:
                    ts.append(ev_a.elapsed_time(ev_b))
            shards[str(G)] = {"columns": c, "ms": float(np.median(ts)),
                              "projected_hvps_per_s": n_p / (float(np.median(ts)) * 1e-3)}

    # ---- roofline of the dominant kernels: the block triangular solves (k_blk,
    # the bus-unit block sweeps, and on Cartesian batches k_spike, the U sweep's
    # spike product; ~55 % of an Alg. 2 batch).  Algorithmic bytes = SURVEY.md
    # 8(d)'s M2 share of the two solve stages, per HVP
    #   [SpMul + L + U]  reads w (n_p), writes z (n_x)
    #   [U^T + L^T]      reads y_x (n_x), writes psi (n_x)
    # = (3 n_x + n_p) * 8 B, credited in full to the 4 block-solve stages of a
    # batch (L [+ U0], U [k_spike on Cartesian batches], U^T, L^T; the separator
    # kernels get none): per stage (3 n_x + n_p) 8 N / 4.
    # Per-stage device times: CUDA events the library records around each
    # kernel of a batch, on the stream the kernels run on (rh_set_timing).
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "B200_PROFILING.md fallback"
    names = ["A_L", "B_LU", "A_U", "FoR", "A_Ut", "B_UtLt", "A_Lt", "MulAdd"]
    ns = info["sep_rows"]
    m2_hvp = (6 * n_x + 5 * n_p) * 8                  # SURVEY.md 8(d) model M2, whole path
    solve_m2_hvp = (3 * n_x + n_p) * 8                # its solve-stage share
    for_m2_hvp = 2 * (n_x + n_p) * 8                  # its FoR share: reads z, w; writes y_x, y_p
    kblk_bytes = solve_m2_hvp * N / 4.0

    def stage_roofline(kind):
        """Per-stage device times of one Alg. 2 batch of width N (CUDA events the library
        records around each kernel, on the stream they run on): kind 'cartesian' = the
        full Hessian's first N columns written as a transposed slab (what the timed step
        runs), 'random' = W ~ N(0, 1)."""
        Hc = torch.empty((min(N, n_p), n_p), dtype=torch.float64, device=dev)   # transposed slab, as the step
        ctx.set_timing(True)
        st_ = np.zeros(9)
        reps_t = 5
        for _ in range(reps_t):
            if flush is not None:
                flush.fill_(1.0)
            if kind == "cartesian":
                ctx.hessian_columns(0, min(N, n_p), N, H=Hc, transposed=True)
            else:
                ctx.hvp(W, HW)
            st_ += ctx.stage_times()
        ctx.set_timing(False)
        st_ /= reps_t
        seg = st_[[0, 2, 4, 6]]                        # A_L, A_U, A_Ut, A_Lt
        lm = float(seg.mean())
        ach = kblk_bytes / (lm * 1e-3) / 1e9 if lm > 0 else None
        bm = float(st_[:8].sum())
        cols = min(N, n_p)
        pg = m2_hvp * cols / (bm * 1e-3) / 1e9 if bm > 0 else None
        fg = for_m2_hvp * cols / (st_[3] * 1e-3) / 1e9 if st_[3] > 0 else None
        return {"kind": kind, "achieved": ach, "frac": (ach / peak) if ach else None, "launch_ms": lm,
                "stage_ms": {k: float(v) for k, v in zip(names, st_[:8])}, "batch_ms": bm,
                "k_blk_share_of_batch": float(seg.sum() / bm) if bm > 0 else None,
                "path_m2_gbs": pg, "path_m2_frac": (pg / peak) if pg else None,
                "for_m2_gbs": fg, "for_m2_frac": (fg / peak) if fg else None, "columns": cols,
                "launch_ms_each": [float(v) for v in seg]}

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "B200_PROFILING.md fallback"
    rl_cart = stage_roofline("cartesian")
    rl_rand = stage_roofline("random")
    cols_local = j1 - j0
    step_gbs = m2_hvp * cols_local / (ms_step * 1e-3) / 1e9 if ms_step > 0 else None
    seg_ms = np.array(rl_rand["launch_ms_each"])
    # secondary, per-launch read + write of the block rows each k_blk launch moves
    # (A_L reads W and G_p only and writes Z's block rows; the others read and write them)
    rw_bytes = np.array([(n_x - ns) * N * 8 + n_p * N * 8] + [2.0 * (n_x - ns) * N * 8] * 3)
    rw_gbs = float(np.mean(rw_bytes / (seg_ms * 1e-3) / 1e9)) if np.all(seg_ms > 0) else None
    traffic, ncu_share, ncu_rec = None, None, {}
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        ncu_rec = prof.get(f"{case}:N={N}:cartesian", {})
        traffic = ncu_rec.get("solve_dram_bytes_per_stage", ncu_rec.get("k_blk_dram_bytes_per_launch"))
        ncu_share = ncu_rec.get("solve_time_share", ncu_rec.get("k_blk_time_share"))
    except Exception:
        pass
    achieved = rl_cart["achieved"]
    roofline = {
        "bound": "hbm", "kernel": "block triangular solves: k_blk (bus-unit sweeps L, U0, U^T, L^T) + k_spike "
                                  "(the U sweep's spike product on Cartesian batches)",
        "achieved": achieved, "peak": peak, "peak_source": peak_src, "unit": "GB/s",
        "frac": (achieved / peak) if achieved else None, "traffic": traffic,
        "algorithmic_bytes_per_launch": kblk_bytes,
        "model": "SURVEY.md 8(d) M2 solve-stage share: (3 n_x + n_p) * 8 B per HVP over the 4 block-solve "
                 "stages of a batch (L + U0, U = k_spike, U^T, L^T), / their mean event time in a Cartesian batch "
                 "(the full Hessian's first N columns, the batches the timed step runs; CUDA events, L2 flushed)",
        "launch_ms": rl_cart["launch_ms"], "stage_ms": rl_cart["stage_ms"], "batch_ms": rl_cart["batch_ms"],
        "k_blk_share_of_batch": rl_cart["k_blk_share_of_batch"], "k_blk_share_of_batch_ncu": ncu_share,
        "traffic_over_algorithmic": (traffic / kblk_bytes) if traffic else None,
        "path_m2_gbs": rl_cart["path_m2_gbs"], "path_m2_frac": rl_cart["path_m2_frac"],
        "path_model": "M2 (6 n_x + 5 n_p) * 8 B per HVP (SURVEY.md 8(d)) / stage-timed batch (sum of its "
                      "kernels' event times)",
        "for_m2_frac": rl_cart["for_m2_frac"],
        "for_model": "k_for's M2 share 2 (n_x + n_p) * 8 B per HVP / its event time",
        "step_m2_gbs": step_gbs, "step_m2_frac": (step_gbs / peak) if step_gbs else None,
        "step_model": "M2 bytes of all this rank's columns / ms_per_step (state + refactorization + gradient "
                      "included in the time, not in the bytes)",
        "random_W": {k: v for k, v in rl_rand.items() if k != "launch_ms_each"},
        "kblk_rw_gbs": rw_gbs, "kblk_rw_frac": (rw_gbs / peak) if rw_gbs else None,
        "kblk_rw_model": "random W: block rows each launch moves: A_L (n_x - n_sep) N 8 + n_p N 8 (W), "
                         "A_U / A_Ut / A_Lt 2 (n_x - n_sep) N 8",
        "ncu": {k: ncu_rec.get(k) for k in ("round", "batch_us_serialized", "k_blk_dram_over_m2", "solve_dram_over_m2",
                                            "solve_kernels", "stages")}
        if ncu_rec else None,
    }

    # ---- Newton projection x(p) from a perturbed solution
    x_pert = x + 1e-3 * torch.from_numpy(np.random.default_rng(7).standard_normal(n_x)).to(dev)
    xw = torch.empty_like(x)
    newton_ms, newton_steps, newton_res, newton_fail = [], 0, None, None
    for rep in range(4):
        xw.copy_(x_pert)
        torch.cuda.synchronize()
        t0n = time.perf_counter()
        try:
            newton_steps, newton_res = ctx.newton(xw, p)
        except rh.RHError as e:   # report, do not lose the headline line
            newton_fail = str(e)
            break
        torch.cuda.synchronize()
        if rep:
            newton_ms.append((time.perf_counter() - t0n) * 1e3)
    newton_err = float((xw - x).abs().max().item())
    ctx.set_state(x, p)
    ctx.reduced_gradient(grad)

    # ---- NEXT-4: Jacobians by coloring + forward mode (PAPER.md 4) vs analytic assembly
    colors, ncolors = ctx.coloring()
    JSb = torch.empty((n_x, max(1, ncolors)), dtype=torch.float64, device=dev)
    ej0, ej1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    jv, st_ms = [], {}
    for _ in range(3):
        lib_cj(ctx, JSb)
    for _ in range(10):
        torch.cuda.synchronize()
        ej0.record(stream)
        lib_cj(ctx, JSb)
        ej1.record(stream)
        torch.cuda.synchronize()
        jv.append(ej0.elapsed_time(ej1))
    for mode in (rh.JAC_ANALYTIC, rh.JAC_COLORED):
        ctx.set_jacobian_mode(mode)
        ts = []
        for rep in range(6):
            torch.cuda.synchronize()
            ej0.record(stream)
            ctx.reduced_hessian(x, p, N, j0, j1, grad, H=Hloc[:j1 - j0], transposed=True)
            ej1.record(stream)
            torch.cuda.synchronize()
            if rep:
                ts.append(ej0.elapsed_time(ej1))
        st_ms[mode] = float(np.median(ts))
    ctx.set_jacobian_mode(rh.JAC_ANALYTIC)
    ctx.set_state(x, p)
    ctx.reduced_gradient(grad)
    jac_colored = {"ncolors": ncolors, "columns": n_x + n_p, "compressed_jacobian_ms": float(np.median(jv)),
                   "step_ms_analytic": st_ms[rh.JAC_ANALYTIC], "step_ms_colored": st_ms[rh.JAC_COLORED],
                   "note": "k_jvp_colored (one forward-mode tangent per color) timed alone; steps = the fused "
                           "state + gradient + Hessian call (L2 not flushed) in each Jacobian mode"}

    # ---- real-time tracking: the paper's Table 3 case, and this case
    tracking = None
    if world == 1:
        tracking = {"table3": tracking_bench(rh, gridgen, dev, "case1354pegase", 256, 10),
                    "paper": PAPER_TABLE3}
        if case != "case1354pegase":
            try:
                tracking[case] = tracking_bench(rh, gridgen, dev, case, N, 5)
            except rh.RHError as e:
                tracking[case] = {"error": str(e)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sc = oracle_single_core(grid, args.cpu_cols, N)
        cores = host_cores()
        pool = OraclePool(case, n_p, cores)
        try:
            pool.full_hessian(N)                       # warm the workers (imports, first factorization)
            wall, t_setup_w, _ = pool.full_hessian(N)
        finally:
            pool.close()
        cpu = {"value": n_p / wall, "unit": UNIT, "cores": pool.workers, "host_cores": cores, "kind": "oracle",
               "sample": f"one real full grad^2 F of {case} ({n_p} Cartesian columns, Alg. 2) by {pool.workers} "
                         f"single-threaded oracle processes (own setup + SuperLU each), {wall:.2f} s; plus a "
                         f"single-core sample: setup + {sc['alg2_columns']} columns (Alg. 2, batch {N}) and "
                         f"{sc['alg1_columns']} columns by Alg. 1",
               "full_hessian_s": wall, "worker_setup_s": t_setup_w, "single_core": sc}

    if rank == 0:
        out = {
            "metric": METRIC, "value": n_p / (ms_step * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(case, N), "case": case, "n_bus": info["n_bus"],
                       "n_line": info["n_line"], "n_x": n_x, "n_p": n_p, "N": N,
                       "batches_per_rank": -(-max(cols_local, 1) // N), "parallelism": f"columns{world}",
                       "l2": "flushed (256 MB write) between timed steps" if flush is not None else "not flushed",
                       "nnz_LU": info["nnz_LU"], "levels": info["levels_fwd"], "blocks": info["n_blocks"],
                       "separator_rows": info["sep_rows"],
                       "residual_inf": resid_inf},
            "full_hessian_ms": ms_step, "state_grad_hessian_columns_ms": ms_hess,
            "state_refactor_grad_ms": ms_pre, "hessian_batches_ms_est": ms_hess - ms_pre,
            "batched_hvps_per_s": hvps, "batched_hvp_ms": t_hvp.item(),
            "gpu_launches": launches,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": t_e2e.item() * 1e3},
            "roofline": roofline,
            "newton": {"ms": float(np.median(newton_ms)) if newton_ms else None, "steps": newton_steps,
                       "resid_inf": newton_res, "error": newton_fail,
                       "max_abs_x_err": newton_err,
                       "start": "solved x + 1e-3 N(0,1) (seed 7; from 1e-2 the oracle diverges too on case9241); tol 1e-11, 2 extra steps (oracle rule); host wall clock incl. one max|dx| readback per step"},
            "shard_projection": {"per_rank": shards,
                                 "note": "one rank's shard [0, ceil(n_p/G)) of the G-GPU column split, fused call "
                                         "(state + refactorization + gradient replicated), timed alone on this GPU; "
                                         "no all-gather"} if shards else None,
            "tracking": tracking,
            "jacobian_colored": jac_colored,
            "cpu_baseline": cpu,
            "clocks": {k: clk[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
