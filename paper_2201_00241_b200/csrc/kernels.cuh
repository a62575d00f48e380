// Device kernels of the batched adjoint-adjoint reduced Hessian (sm_100a, fp64).
//
// Layout of the batched blocks: the n_x x N blocks Z
// and Psi live in library scratch, tiled by columns: tile t holds columns
// [t*T, t*T+T) of all n_x (permuted) rows, element (row r, col c) at
// X[(t * n_x + r) * T + c].  One CTA owns one column tile for the whole HVP,
// so the entire Alg. 2 pipeline runs without any
// inter-CTA synchronization: columns are independent ("slice by slice, in an
// embarrassingly parallel fashion").
#pragma once

#include <cstdint>

namespace rh {

constexpr int kThreads = 256;

struct DSweep {
  int nlev;
  const int *__restrict__ lev_ptr;   // [nlev+1]
  const int *__restrict__ rows;      // [n] level order
  const int *__restrict__ rptr;      // [n+1]
  const int *__restrict__ col;       // [nnz]
  const double *__restrict__ val;    // [nnz]
  const double *__restrict__ dinv;   // [n] (null: unit diagonal)
};

enum : int {
  PH_L = 1,        // SpMul (B = G_p W) fused into the forward L sweep: L Z' = -P B
  PH_U = 2,        // backward U sweep: Z' = U^{-1} Z'
  PH_FOR = 4,      // BatchTensorProjection by forward-over-reverse (bus-centric)
  PH_UT = 8,       // forward U^T sweep on -Y_x
  PH_LT = 16,      // backward L^T sweep -> Psi'
  PH_MULADD = 32,  // SpMulAdd HW = Y_p + G_p^T Psi
  PH_ALL = 63
};

struct HvpParams {
  int n_x, n_p, n_bus, N;
  const double *W;  // [n_p][ldw] or null with ident_j0 >= 0 (Cartesian block e_{j0..})
  long long ldw;
  double *HW;
  long long ldhw;
  int ident_j0;
  int transposed;   // HW element (row i, col k) at k*ldhw + i instead of i*ldhw + k
  double *X1, *X2;  // tiled scratch
  DSweep L, U, Ut, Lt;
  const int *gp_rptr, *gp_col;
  const double *gp_val;
  const int *gpc_ptr, *gpc_row;
  const double *gpc_val;
  const int *bl_ptr, *bl_line, *bl_end;
  const int *o_dth_src, *o_dv_src;   // per incident slot: delta sources of the other end
  const int *dth_src, *dv_src, *yth_dst, *yv_dst, *pg_p;
  const double4 *coef;               // per line (K, a_i, a_j, m)
  const double *dcoef;               // per bus 2 (G_ii mu_P - B_ii mu_Q)
  const double *refg_th, *refg_v;    // grad P_ref over bus theta / v
  const double *c2b;                 // per-bus c2
  const int *near_ref;
  int n_near_ref;
  double f2ref;                      // f''(Pg_ref) = 2 c2_ref
};

}  // namespace rh
