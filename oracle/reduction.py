"""Oracle: reduced gradient and adjoint-adjoint reduced Hessian (TEST INFRASTRUCTURE ONLY).

Follows PAPER.md:
  * section 3.3, Eq. reduced_gradient:
        lambda = -(grad_x g)^{-T} grad_x f^T,  grad_p F = grad_p f + lambda^T grad_p g
  * section 4.1, Eq. socadjoint / Eq. hessvecprod, readings R7, R8:
        J z = -G_p w ;  J^T psi = -H_xp w - H_xx z ;  H w = H_pp w + H_px z + G_p^T psi
  * Alg. 1: SpMul, SparseSolve, TensorProjection, SparseSolve^T, MulAdd
  * Alg. 2: the same on an n_p x N block W
  * full Hessian by ceil(n_p / N) Cartesian batches (reading R10)

Linear algebra: SuperLU (scipy.sparse.linalg.splu, partial pivoting, no
iterative refinement -- reading R15).  The tensor projection (Eq. reduction,
PAPER.md:550-566) is a plain sparse matrix product with the assembled
Lagrangian Hessian of oracle.powerflow.lagrangian_hessian.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import powerflow as pf


class Operators:
    """The linear operators of one operating point: J, G_p and the blocks of
    the Lagrangian Hessian.  Generic: Alg. 1/2 below only use these fields,
    so the SPEC toy g = x - A p can be fed directly."""

    def __init__(self, J, Gp, Hxx, Hxp, Hpx, Hpp):
        self.J = sp.csc_matrix(J)
        self.Gp = sp.csr_matrix(Gp)
        self.Hxx, self.Hxp, self.Hpx, self.Hpp = (sp.csr_matrix(Hxx), sp.csr_matrix(Hxp),
                                                  sp.csr_matrix(Hpx), sp.csr_matrix(Hpp))
        # SuperLU with partial pivoting (R15); one factorization serves both solves
        self.lu = spla.splu(self.J, permc_spec="COLAMD")

    def solve(self, B):
        return self.lu.solve(np.asarray(B, dtype=np.float64))

    def solve_T(self, B):
        return self.lu.solve(np.asarray(B, dtype=np.float64), trans="T")


def reduced_gradient(grid, x, p, L=None):
    """(grad_p F, lambda) by the first-order adjoint method."""
    L = L or pf.Layout(grid)
    J, Gp = pf.jacobians(grid, x, p, L)
    gx, gp, _ = pf.objective_gradients(grid, x, p, L)
    lam = -spla.splu(sp.csc_matrix(J)).solve(np.asarray(gx, np.float64), trans="T")
    grad = gp + Gp.T @ lam
    return np.asarray(grad), lam


def operators(grid, x, p, lam, L=None) -> Operators:
    L = L or pf.Layout(grid)
    J, Gp = pf.jacobians(grid, x, p, L)
    Hxx, Hxp, Hpx, Hpp = pf.lagrangian_hessian(grid, x, p, lam, L)
    return Operators(J, Gp, Hxx, Hxp, Hpx, Hpp)


def hvp_batch(ops: Operators, W, trace: dict | None = None, timers: dict | None = None):
    """Alg. 2, parallel reduction, W of shape [n_p][N].
    `timers` (optional, bench.py's per-stage CPU breakdown only) accumulates
    wall seconds per Alg. 2 stage; it does not change the arithmetic."""
    W = np.asarray(W, dtype=np.float64)
    if W.ndim == 1:
        W = W[:, None]
    tick = _Ticker(timers)
    B = ops.Gp @ W                                  # SpMul
    tick("SpMul")
    Z = -ops.solve(B)                               # BatchSparseSolve   J Z = -B   (601)
    tick("SparseSolve")
    Yx = ops.Hxx @ Z + ops.Hxp @ W                  # BatchTensorProjection  (602, Eq. reduction)
    Yp = ops.Hpx @ Z + ops.Hpp @ W
    tick("TensorProjection")
    Psi = -ops.solve_T(Yx)                          # BatchSparseSolve^T  J^T Psi = -Yx (603)
    tick("SparseSolveT")
    HW = Yp + ops.Gp.T @ Psi                        # SpMulAdd      (604)
    tick("SpMulAdd")
    if trace is not None:
        trace.update(B=B, Z=Z, Yx=Yx, Yp=Yp, Psi=Psi)
    return np.asarray(HW)


class _Ticker:
    """Accumulates wall time between calls into a dict (no-op without one)."""

    def __init__(self, timers):
        import time
        self.t = timers
        self.clock = time.perf_counter
        self.last = self.clock() if timers is not None else 0.0

    def __call__(self, name):
        if self.t is None:
            return
        now = self.clock()
        self.t[name] = self.t.get(name, 0.0) + (now - self.last)
        self.last = now


def hvp_sequential(ops: Operators, w):
    """Alg. 1, one Hessian-vector product."""
    w = np.asarray(w, dtype=np.float64).ravel()
    b = ops.Gp @ w                                  # SpMul
    z = -ops.solve(b)                               # SparseSolve
    yx = ops.Hxx @ z + ops.Hxp @ w                  # TensorProjection
    yp = ops.Hpx @ z + ops.Hpp @ w
    psi = -ops.solve_T(yx)                          # SparseSolve^T
    return np.asarray(yp + ops.Gp.T @ psi)          # MulAdd


def n_batches(n_p: int, N: int) -> int:
    """ceil(n_p / N) (reading R10 of PAPER.md:780, 890's div(n, N) + 1)."""
    return max(1, math.ceil(n_p / N))


def full_hessian(ops: Operators, N: int, sequential: bool = False):
    """grad^2 F by Cartesian column batches.
    H[:, j] is the HVP with e_j."""
    n_p = ops.Gp.shape[1]
    H = np.zeros((n_p, n_p))
    if sequential:
        for j in range(n_p):
            e = np.zeros(n_p)
            e[j] = 1.0
            H[:, j] = hvp_sequential(ops, e)
        return H
    for b in range(n_batches(n_p, N)):
        j0, j1 = b * N, min(n_p, (b + 1) * N)
        W = np.zeros((n_p, j1 - j0))
        W[np.arange(j0, j1), np.arange(j1 - j0)] = 1.0
        H[:, j0:j1] = hvp_batch(ops, W)
    return H


def dense_definition(ops: Operators):
    """H = S^T grad^2 l S with S = [-J^{-1} G_p ; I] (plain definition)."""
    Jd = ops.J.toarray()
    Gd = ops.Gp.toarray()
    n_p = Gd.shape[1]
    S = np.vstack([-np.linalg.solve(Jd, Gd), np.eye(n_p)])
    Hl = np.block([[ops.Hxx.toarray(), ops.Hxp.toarray()], [ops.Hpx.toarray(), ops.Hpp.toarray()]])
    return S.T @ Hl @ S


def reduced_hessian(grid, N: int | None = None, L=None, lam=None, sequential=False):
    """Convenience: full reduced Hessian at the grid's bus state with the true
    first-order adjoint (or a given lam, reading R16)."""
    L = L or pf.Layout(grid)
    x, p = pf.state_vectors(grid, L)
    if lam is None:
        _, lam = reduced_gradient(grid, x, p, L)
    ops = operators(grid, x, p, lam, L)
    return full_hessian(ops, N or L.n_p, sequential=sequential)


def reduced_objective(grid, p, x0, L=None):
    """F(p) = f(x(p), p) with x(p) from the Newton projection
    (Eq. nonlinearoptreduced)."""
    L = L or pf.Layout(grid)
    x = pf.newton(grid, p, x0, L)
    return pf.objective(grid, x, p, L)
