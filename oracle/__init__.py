"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct fp64 NumPy/SciPy implementation of what the
batched adjoint-adjoint reduced-Hessian path computes (arXiv 2201.00241,
PAPER.md sections 3-4).  It is the parity reference for the CUDA path and is
itself pinned by tests/test_oracle_*.py against closed forms, complex-step
derivatives, finite differences, brute-force tensors and invariants.

Rules:
  * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
    --impl reference legs may import anything under oracle/.
  * It shares no code with paper_2201_00241_b200/ (the CUDA path) and imports
    nothing from it; the only shared module is gridgen/ (seeded inputs).
  * Every function cites the PAPER.md passage it follows.

Modules:
  powerflow  -- orderings, injections, g, f, J, G_p, grad f, Lagrangian Hessian,
                Newton, load back-out (PAPER.md 3.1-3.3, Eq. powerflow,
                Eq. powerflowvec, Eq. lagrangian)
  reduction  -- reduced gradient, Alg. 1, Alg. 2, full Hessian, dense definition
                (PAPER.md 3.3, 4.1-4.3, Eq. socadjoint, Eq. hessvecprod)
  coloring   -- Jacobians by column coloring + forward mode (PAPER.md 4,
                PAPER.md:440-468, 694-713)
  tracking   -- the real-time tracking step: Newton, g_t, H_t, dense Cholesky
                solve of Eq. qp_rto (PAPER.md 6.3)
"""
from . import coloring, powerflow, reduction, tracking  # noqa: F401
