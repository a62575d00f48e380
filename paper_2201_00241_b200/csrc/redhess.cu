// B200-native batched adjoint-adjoint reduced Hessian: device kernels + C ABI.
// Everything on the hot path is a hand-written sm_100a fp64 kernel in this
// file; the host only runs the one-time symbolic analysis (analysis.cpp).
//
// Citations are PAPER.md line numbers (arXiv 2201.00241) or DESIGN.md readings.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/redhess.h"
#include "analysis.hpp"
#include "kernels.cuh"

using namespace rh;

// ============================================================================
// device helpers
// ============================================================================

__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ============================================================================
// state kernels: bus state, line trig, injections, g,
// J and G_p assembly (Appendix A identities), grad P_ref
// ============================================================================

// x, p -> bus-level theta, v, Pg (R5 orderings)
__global__ void k_bus_state(int n_x, int n_p, const int *x_bus, const int *x_kind, const int *p_bus,
                            const int *p_kind, const double *x, const double *p, double *th, double *v,
                            double *pgb, int ref, double theta_ref) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n_x) {
    const int b = x_bus[k];
    if (x_kind[k] == RH_KIND_THETA)
      th[b] = x[k];
    else
      v[b] = x[k];
  } else if (k < n_x + n_p) {
    const int q = k - n_x;
    const int b = p_bus[q];
    if (p_kind[q] == RH_KIND_PG)
      pgb[b] = p[q];
    else
      v[b] = p[q];
  } else if (k == n_x + n_p) {
    th[ref] = theta_ref;
  }
}

// per line: c = cos(th_f - th_t), s = sin(th_f - th_t) (trig once per line)
__global__ void k_line_trig(int m, const int *lf, const int *lt, const double *th, double2 *cs) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= m) return;
  double s, c;
  sincos(th[lf[l]] - th[lt[l]], &s, &c);
  cs[l] = make_double2(c, s);
}

struct AsmParams {
  int n_bus, ref;
  const int *bus_type, *bl_ptr, *bl_line, *bl_other, *bl_end;
  const double *G_ii, *B_ii, *Pd, *Qd, *G_ft, *B_ft, *G_tf, *B_tf;
  const double *th, *v, *pgb;
  const double2 *cs;
  const int *th_x, *v_x;
  const int *diag_pos, *slot_pos;
  const int *gp_self_pos, *gp_pg_pos, *gp_slot_pos;
  double *P, *Q, *g, *F_val, *gp_val, *refg_th, *refg_v;
};

// Bus-centric assembly (race-free: bus b owns rows P_b, Q_b).  Eq. powerflow
// with the Ybus diagonal (R1); g per Eq. powerflowvec
// (R2); J / G_p entries per SURVEY.md Appendix A.
__global__ void k_assemble(AsmParams a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.n_bus) return;
  const double vb = a.v[b];
  const int s0 = a.bl_ptr[b], s1 = a.bl_ptr[b + 1];
  double P = 0.0, Q = 0.0;
  for (int s = s0; s < s1; ++s) {
    const int l = a.bl_line[s], o = a.bl_other[s];
    const double2 cs = a.cs[l];
    const bool from = a.bl_end[s] == 0;
    const double G = from ? a.G_ft[l] : a.G_tf[l];
    const double B = from ? a.B_ft[l] : a.B_tf[l];
    const double c = cs.x, sn = from ? cs.y : -cs.y;   // cos/sin(th_b - th_o)
    const double vo = a.v[o];
    P += vo * (G * c + B * sn);
    Q += vo * (G * sn - B * c);
  }
  const double Gbb = a.G_ii[b], Bbb = a.B_ii[b];
  P = vb * P + vb * vb * Gbb;
  Q = vb * Q - vb * vb * Bbb;
  a.P[b] = P;
  a.Q[b] = Q;
  const int t = a.bus_type[b];
  if (b == a.ref) {
    // grad P_ref over (theta_o, v_o) of the neighbours and v_ref (theta_ref constant)
    for (int s = s0; s < s1; ++s) {
      const int l = a.bl_line[s], o = a.bl_other[s];
      const double2 cs = a.cs[l];
      const bool from = a.bl_end[s] == 0;
      const double G = from ? a.G_ft[l] : a.G_tf[l];
      const double B = from ? a.B_ft[l] : a.B_tf[l];
      const double c = cs.x, sn = from ? cs.y : -cs.y;
      a.refg_th[o] += vb * a.v[o] * (G * sn - B * c);
      a.refg_v[o] += vb * (G * c + B * sn);
    }
    a.refg_v[b] += P / vb + Gbb * vb;
    return;
  }
  const int rP = a.th_x[b];
  const int rQ = a.v_x[b];
  a.g[rP] = P + a.Pd[b] - (t == RH_PV ? a.pgb[b] : 0.0);
  if (rQ >= 0) a.g[rQ] = Q + a.Qd[b];
  // diagonal block
  const int *dp = a.diag_pos + 4 * b;
  a.F_val[dp[0]] += -Q - Bbb * vb * vb;            // dP_b/dth_b
  if (rQ >= 0) {
    a.F_val[dp[1]] += P / vb + Gbb * vb;            // dP_b/dv_b
    a.F_val[dp[2]] += P - Gbb * vb * vb;            // dQ_b/dth_b
    a.F_val[dp[3]] += Q / vb - Bbb * vb;            // dQ_b/dv_b
  } else {
    a.gp_val[a.gp_self_pos[b]] += P / vb + Gbb * vb; // dP_b/dv_b, v_b in p (PV)
    a.gp_val[a.gp_pg_pos[b]] = -1.0;                  // dP_b/dPg_b
  }
  for (int s = s0; s < s1; ++s) {
    const int l = a.bl_line[s], o = a.bl_other[s];
    const double2 cs = a.cs[l];
    const bool from = a.bl_end[s] == 0;
    const double G = from ? a.G_ft[l] : a.G_tf[l];
    const double B = from ? a.B_ft[l] : a.B_tf[l];
    const double c = cs.x, sn = from ? cs.y : -cs.y;
    const double vo = a.v[o];
    const double gsbc = G * sn - B * c, gcbs = G * c + B * sn;
    const double dPth = vb * vo * gsbc, dPv = vb * gcbs;
    const double dQth = -vb * vo * gcbs, dQv = vb * gsbc;
    const int *sp = a.slot_pos + 4 * s;
    if (sp[0] >= 0) a.F_val[sp[0]] += dPth;
    if (sp[1] >= 0) a.F_val[sp[1]] += dPv;
    if (sp[2] >= 0) a.F_val[sp[2]] += dQth;
    if (sp[3] >= 0) a.F_val[sp[3]] += dQv;
    const int *gs = a.gp_slot_pos + 2 * s;
    if (gs[0] >= 0) a.gp_val[gs[0]] += dPv;
    if (gs[1] >= 0) a.gp_val[gs[1]] += dQv;
  }
}

// f (R4) and the REF multiplier seed mu_ref = f'(Pg_ref) (R22).  One block.
// scal[0] = P_ref, scal[1] = Pg_ref, scal[2] = mu_ref, scal[3] = f
__global__ void k_objective(int n_bus, int ref, const int *has_gen, const double *c2b, const double *c1b,
                            const double *c0b, const double *pgb, const double *P, const double *Pd,
                            double *scal) {
  __shared__ double red[kThreads];
  const double pg_ref = P[ref] + Pd[ref];
  double acc = 0.0;
  for (int b = threadIdx.x; b < n_bus; b += blockDim.x) {
    if (!has_gen[b]) continue;
    const double pg = b == ref ? pg_ref : pgb[b];
    acc += (c2b[b] * pg + c1b[b]) * pg + c0b[b];
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    scal[0] = P[ref];
    scal[1] = pg_ref;
    scal[2] = 2.0 * c2b[ref] * pg_ref + c1b[ref];
    scal[3] = red[0];
  }
}

// ============================================================================
// numeric refactorization on the fixed pattern (
// PAPER.md:764-767).  Up-looking Doolittle, one warp per row, rows taken in
// forward-level (topological) order from a ticket counter; a row waits on
// per-row completion flags of the rows it depends on (no grid barrier; the
// ticket order makes the wait deadlock-free).  Static diagonal pivots (R15).
// ============================================================================

__global__ void __launch_bounds__(kThreads) k_refactor(int nx, const int *__restrict__ order,
                                                       const int *__restrict__ rowptr,
                                                       const int *__restrict__ colidx,
                                                       const int *__restrict__ diag, double *val, int *flags,
                                                       int epoch, int *ticket, int *status, double pivtol) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    int t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= nx) return;
    const int i = order[t];
    const int rb = rowptr[i], re = rowptr[i + 1], dpos = diag[i];
    double amax = 0.0;
    for (int e = rb + lane; e < re; e += 32) amax = fmax(amax, fabs(val[e]));
    amax = warp_max(amax);
    for (int e = rb + lane; e < dpos; e += 32) {
      const int k = colidx[e];
      while (ld_acquire(flags + k) != epoch) {
      }
    }
    __syncwarp();
    __threadfence();  // invalidate stale L1 lines before reading other rows
    for (int e = rb; e < dpos; ++e) {
      const int k = colidx[e];
      const int dk = diag[k];
      const double lik = val[e] / val[dk];
      __syncwarp();
      if (lane == 0) val[e] = lik;
      const int ub = dk + 1, ue = rowptr[k + 1];
      for (int u = ub + lane; u < ue; u += 32) {
        const int j = colidx[u];
        // binary search j in row i (j > k, present by construction of the fill)
        int lo = e + 1, hi = re - 1;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (colidx[mid] < j)
            lo = mid + 1;
          else
            hi = mid;
        }
        val[lo] -= lik * val[u];
      }
      __syncwarp();
    }
    if (lane == 0) {
      const double piv = val[dpos];
      if (!(fabs(piv) > pivtol * amax)) atomicMax(status, i + 1);
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release(flags + i, epoch);
  }
}

// copy factor values into the four sweep value arrays + inverted pivots,
// and G_p values into CSC order
__global__ void k_gather_vals(int n, const int *__restrict__ src, const double *__restrict__ F, double *dst) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) dst[e] = F[src[e]];
}
__global__ void k_gather_inv(int n, const int *__restrict__ src, const double *__restrict__ F, double *dst) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) dst[e] = 1.0 / F[src[e]];
}

// ============================================================================
// batched sweeps: one CTA walks all levels of its
// column tile with CTA barriers only.  Each row slot is T threads (one per
// column of the tile); rows of one level are independent.
// ============================================================================

template <int T, bool DIAG>
__device__ __forceinline__ void sweep_inplace(const DSweep &S, double *__restrict__ X) {
  const int c = threadIdx.x % T;
  const int slot = threadIdx.x / T;
  constexpr int nslots = kThreads / T;
  for (int lv = 0; lv < S.nlev; ++lv) {
    const int beg = S.lev_ptr[lv], end = S.lev_ptr[lv + 1];
    for (int q = beg + slot; q < end; q += nslots) {
      const int r = S.rows[q];
      const int e0 = S.rptr[q], e1 = S.rptr[q + 1];
      double acc = X[r * T + c];
      for (int e = e0; e < e1; ++e) acc -= S.val[e] * X[S.col[e] * T + c];
      if (DIAG) acc *= S.dinv[q];
      X[r * T + c] = acc;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ double load_W(const HvpParams &h, int row, int col) {
  if (col >= h.N) return 0.0;
  if (h.ident_j0 >= 0) return row == h.ident_j0 + col ? 1.0 : 0.0;
  return h.W[(long long)row * h.ldw + col];
}

__device__ __forceinline__ long long hw_index(const HvpParams &h, int row, int col) {
  return h.transposed ? (long long)col * h.ldhw + row : (long long)row * h.ldhw + col;
}

// forward L sweep with the SpMul fused into the right-hand side:
// row r of -B = -(G_p W)[r] is formed on the fly
template <int T>
__device__ __forceinline__ void sweep_L_spmul(const HvpParams &h, double *__restrict__ X, int col0) {
  const int c = threadIdx.x % T;
  const int slot = threadIdx.x / T;
  constexpr int nslots = kThreads / T;
  const int col = col0 + c;
  const DSweep &S = h.L;
  for (int lv = 0; lv < S.nlev; ++lv) {
    const int beg = S.lev_ptr[lv], end = S.lev_ptr[lv + 1];
    for (int q = beg + slot; q < end; q += nslots) {
      const int r = S.rows[q];
      double acc = 0.0;
      const int g0 = h.gp_rptr[r], g1 = h.gp_rptr[r + 1];
      for (int e = g0; e < g1; ++e) acc -= h.gp_val[e] * load_W(h, h.gp_col[e], col);
      const int e0 = S.rptr[q], e1 = S.rptr[q + 1];
      for (int e = e0; e < e1; ++e) acc -= S.val[e] * X[S.col[e] * T + c];
      X[r * T + c] = acc;
    }
    __syncthreads();
  }
}

template <int T>
__device__ __forceinline__ double delta_src(const HvpParams &h, const double *__restrict__ X1, int src, int c,
                                            int col) {
  if (src >= 0) return X1[src * T + c];
  if (src == -1) return 0.0;
  return load_W(h, -(src + 2), col);
}

// BatchTensorProjection (Eq. so_model)
// by hand-written forward-over-reverse on the line graph, hoisted tape:
// per line (K, a_i, a_j, m) is column independent (computed once per state
// and lambda by k_coefs); per column it is 8 FMAs per line end.  Bus-centric
// gather ("edges then nodes") without atomics.
template <int T>
__device__ __forceinline__ void tensor_projection(const HvpParams &h, const double *__restrict__ X1,
                                                  double *__restrict__ X2, int col0, double *s_ref) {
  const int c = threadIdx.x % T;
  const int slot = threadIdx.x / T;
  constexpr int nslots = kThreads / T;
  const int col = col0 + c;
  // s = grad P_ref . delta per column (REF objective rank-1 term, R22)
  if (slot == 0) {
    double s = 0.0;
    for (int q = 0; q < h.n_near_ref; ++q) {
      const int b = h.near_ref[q];
      s += h.refg_th[b] * delta_src<T>(h, X1, h.dth_src[b], c, col) +
           h.refg_v[b] * delta_src<T>(h, X1, h.dv_src[b], c, col);
    }
    s_ref[c] = h.f2ref * s;
  }
  __syncthreads();
  const double sr = s_ref[c];
  for (int b = slot; b < h.n_bus; b += nslots) {
    const double dth_b = delta_src<T>(h, X1, h.dth_src[b], c, col);
    const double dv_b = delta_src<T>(h, X1, h.dv_src[b], c, col);
    double yth = sr * h.refg_th[b];
    double yv = h.dcoef[b] * dv_b + sr * h.refg_v[b];
    const int s0 = h.bl_ptr[b], s1 = h.bl_ptr[b + 1];
    for (int s = s0; s < s1; ++s) {
      const double4 k = h.coef[h.bl_line[s]];
      const double dth_o = delta_src<T>(h, X1, h.o_dth_src[s], c, col);
      const double dv_o = delta_src<T>(h, X1, h.o_dv_src[s], c, col);
      if (h.bl_end[s] == 0) {  // b is the from-end i
        const double D = dth_b - dth_o;
        yth += k.x * D + k.y * dv_b + k.z * dv_o;
        yv += k.y * D + k.w * dv_o;
      } else {                 // b is the to-end j
        const double D = dth_o - dth_b;
        yth -= k.x * D + k.y * dv_o + k.z * dv_b;
        yv += k.z * D + k.w * dv_o;
      }
    }
    const int dt = h.yth_dst[b];
    if (dt >= 0) X2[dt * T + c] = -yth;
    const int dv = h.yv_dst[b];
    if (dv >= 0) {
      X2[dv * T + c] = -yv;
    } else if (col < h.N) {
      h.HW[hw_index(h, -(dv + 2), col)] = yv;
    }
    const int pg = h.pg_p[b];
    if (pg >= 0 && col < h.N) h.HW[hw_index(h, pg, col)] = 2.0 * h.c2b[b] * load_W(h, pg, col);
  }
  __syncthreads();
}

// SpMulAdd HW = Y_p + G_p^T Psi, by p column (CSC of G_p)
template <int T>
__device__ __forceinline__ void spmuladd(const HvpParams &h, const double *__restrict__ X2, int col0) {
  const int c = threadIdx.x % T;
  const int slot = threadIdx.x / T;
  constexpr int nslots = kThreads / T;
  const int col = col0 + c;
  if (col >= h.N) return;
  for (int cp = slot; cp < h.n_p; cp += nslots) {
    const long long idx = hw_index(h, cp, col);
    double acc = h.HW[idx];
    for (int q = h.gpc_ptr[cp]; q < h.gpc_ptr[cp + 1]; ++q) acc += h.gpc_val[q] * X2[h.gpc_row[q] * T + c];
    h.HW[idx] = acc;
  }
}

// The fused HVP: one CTA per column tile runs Alg. 2 end to end
// -- no stage boundaries, no host syncs (cf. the two
// explicit synchronizations of PAPER.md:798-805).  PHASES selects a subset
// for the staged (per-stage timing / parity) mode.
template <int T>
__global__ void __launch_bounds__(kThreads) k_hvp(HvpParams h, int phases) {
  __shared__ double s_ref[T];
  const int tile = blockIdx.x;
  const int col0 = tile * T;
  double *X1 = h.X1 + (long long)tile * h.n_x * T;
  double *X2 = h.X2 + (long long)tile * h.n_x * T;
  if (phases & PH_L) sweep_L_spmul<T>(h, X1, col0);
  if (phases & PH_U) sweep_inplace<T, true>(h.U, X1);
  if (phases & PH_FOR) tensor_projection<T>(h, X1, X2, col0, s_ref);
  if (phases & PH_UT) sweep_inplace<T, true>(h.Ut, X2);
  if (phases & PH_LT) sweep_inplace<T, false>(h.Lt, X2);
  if (phases & PH_MULADD) spmuladd<T>(h, X2, col0);
}

// ============================================================================
// first-order adjoint + reduced gradient, single column
// ============================================================================

// rhs of J^T lambda = -grad_x f:  X'[pinv[k]] = -mu_ref * dP_ref/dx_k
__global__ void k_grad_rhs(int n_x, const int *x_bus, const int *x_kind, const int *pinv, const double *refg_th,
                           const double *refg_v, const double *scal, double *X) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_x) return;
  const int b = x_bus[k];
  const double g = x_kind[k] == RH_KIND_THETA ? refg_th[b] : refg_v[b];
  X[pinv[k]] = -scal[2] * g;
}

__global__ void __launch_bounds__(kThreads) k_solve_T1(DSweep Ut, DSweep Lt, double *X) {
  sweep_inplace<1, true>(Ut, X);
  sweep_inplace<1, false>(Lt, X);
}

__global__ void k_grad_out(int n_x, int n_p, const int *pinv, const int *p_bus, const int *p_kind,
                           const double *c2b, const double *c1b, const double *p, const double *refg_v,
                           const double *scal, const int *gpc_ptr, const int *gpc_row, const double *gpc_val,
                           const double *X, double *lam, double *grad) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n_x) lam[k] = X[pinv[k]];
  if (k < n_p) {
    const int b = p_bus[k];
    double acc = p_kind[k] == RH_KIND_PG ? 2.0 * c2b[b] * p[k] + c1b[b] : scal[2] * refg_v[b];
    for (int q = gpc_ptr[k]; q < gpc_ptr[k + 1]; ++q) acc += gpc_val[q] * X[gpc_row[q]];
    grad[k] = acc;
  }
}

// Hoisted forward-over-reverse tape: bus multipliers
// mu_P = lambda on P rows, mu_Q = lambda on Q rows, mu_P,ref = f'(Pg_ref);
// per line (K, a_i, a_j, m); per bus the diagonal 2 (G_ii mu_P - B_ii mu_Q).
__global__ void k_mu(int n_bus, int ref, const int *th_x, const int *v_x, const double *lam, const double *scal,
                     double *muP, double *muQ) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n_bus) return;
  muP[b] = b == ref ? scal[2] : lam[th_x[b]];
  muQ[b] = v_x[b] >= 0 ? lam[v_x[b]] : 0.0;
}

__global__ void k_coefs(int m, int n_bus, const int *lf, const int *lt, const double *G_ft, const double *B_ft,
                        const double *G_tf, const double *B_tf, const double *G_ii, const double *B_ii,
                        const double2 *cs, const double *v, const double *muP, const double *muQ, double4 *coef,
                        double *dcoef) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l < m) {
    const int i = lf[l], j = lt[l];
    const double Pi = muP[i], Qi = muQ[i], Pj = muP[j], Qj = muQ[j];
    // outputs P_i:(G_ft,B_ft) Q_i:(-B_ft,G_ft) P_j:(G_tf,-B_tf) Q_j:(-B_tf,-G_tf)
    const double alpha = Pi * G_ft[l] - Qi * B_ft[l] + Pj * G_tf[l] - Qj * B_tf[l];
    const double beta = Pi * B_ft[l] + Qi * G_ft[l] - Pj * B_tf[l] - Qj * G_tf[l];
    const double c = cs[l].x, s = cs[l].y;
    const double E = alpha * c + beta * s;
    const double D = -alpha * s + beta * c;
    const double vi = v[i], vj = v[j];
    coef[l] = make_double4(-vi * vj * E, vj * D, vi * D, E);
  }
  if (l < n_bus) dcoef[l] = 2.0 * (G_ii[l] * muP[l] - B_ii[l] * muQ[l]);
}

// natural-order copy of a tiled block: out[k][col] = sgn * X[tile][pinv[k]][c]
__global__ void k_untile(int n_x, int N, int T, const int *pinv, const double *X, double sgn, double *out,
                         long long ld) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)n_x * N) return;
  const int k = (int)(idx / N), col = (int)(idx % N);
  const int tile = col / T, c = col % T;
  out[(long long)k * ld + col] = sgn * X[((long long)tile * n_x + pinv[k]) * T + c];
}

// ============================================================================
// context
// ============================================================================

namespace {

template <class T>
T *dalloc_copy(const std::vector<T> &v, std::vector<void *> &pool) {
  T *p = nullptr;
  size_t bytes = std::max<size_t>(1, v.size()) * sizeof(T);
  if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
  pool.push_back(p);
  if (!v.empty()) cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return p;
}
template <class T>
T *dalloc(size_t n, std::vector<void *> &pool) {
  T *p = nullptr;
  if (cudaMalloc(&p, std::max<size_t>(1, n) * sizeof(T)) != cudaSuccess) return nullptr;
  pool.push_back(p);
  return p;
}

struct DevSweepStore {
  DSweep d{};
  int *src = nullptr, *diag_src = nullptr;
  int nnz = 0, n = 0;
  double *dinv_mut = nullptr, *val_mut = nullptr;
};

}  // namespace

struct rh_ctx {
  int device = -1;
  bool host_only = true;
  bool loaded = false, has_state = false, has_mult = false;
  std::string err;
  Analysis A;
  std::vector<void *> pool;   // grid-lifetime device buffers
  long long launches = 0;
  int epoch = 0;
  bool timing = false;
  float stage_ms[6] = {0, 0, 0, 0, 0, 0};

  // device grid + analysis
  int *bus_type, *lf, *lt, *bl_ptr, *bl_line, *bl_other, *bl_end, *has_gen;
  double *G_ii, *B_ii, *Pd, *Qd, *G_ft, *B_ft, *G_tf, *B_tf, *c2b, *c1b, *c0b;
  int *x_bus, *x_kind, *p_bus, *p_kind, *th_x, *v_x, *pinv;
  int *F_rowptr, *F_col, *F_diag, *fact_order;
  double *F_val;
  int *flags, *ticket, *status;
  int *diag_pos, *slot_pos, *gp_rptr, *gp_col, *gp_self_pos, *gp_pg_pos, *gp_slot_pos;
  double *gp_val;
  int *gpc_ptr, *gpc_pos, *gpc_row;
  double *gpc_val;
  DevSweepStore sL, sU, sUt, sLt;
  int *dth_src, *dv_src, *yth_dst, *yv_dst, *o_dth_src, *o_dv_src, *pg_p, *near_ref;
  // state
  double *x, *p, *th, *v, *pgb, *P, *Q, *g, *refg_th, *refg_v, *scal;
  double2 *cs;
  double *lam, *muP, *muQ, *dcoef, *X1col;
  double4 *coef;
  // workspace
  double *X1 = nullptr, *X2 = nullptr;
  size_t ws_elems = 0;
  double *Wtmp = nullptr;
  size_t wtmp_elems = 0;

  void free_all() {
    for (void *q : pool) cudaFree(q);
    pool.clear();
    if (X1) cudaFree(X1);
    if (X2) cudaFree(X2);
    if (Wtmp) cudaFree(Wtmp);
    X1 = X2 = Wtmp = nullptr;
    ws_elems = wtmp_elems = 0;
  }
};

namespace {

int fail(rh_ctx *c, int code, const std::string &msg) {
  if (c) c->err = msg;
  return code;
}

#define RH_CUDA(ctx, call)                                                                 \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) return fail(ctx, RH_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define RH_LAUNCHED(ctx)                                                                   \
  do {                                                                                     \
    (ctx)->launches++;                                                                     \
    cudaError_t e_ = cudaGetLastError();                                                   \
    if (e_ != cudaSuccess) return fail(ctx, RH_E_CUDA, std::string("launch: ") + cudaGetErrorString(e_)); \
  } while (0)

inline int nblk(long long n, int t = kThreads) { return (int)((n + t - 1) / t); }

int upload(rh_ctx *c) {
  const Analysis &A = c->A;
  auto &P = c->pool;
  bool ok = true;
  auto chk = [&](const void *q) { ok = ok && q != nullptr; };
#define UP(dst, vec) chk(c->dst = dalloc_copy(vec, P))
  UP(bus_type, A.bus_type); UP(lf, A.line_f); UP(lt, A.line_t); UP(bl_ptr, A.bl_ptr);
  UP(bl_line, A.bl_line); UP(bl_other, A.bl_other); UP(bl_end, A.bl_end); UP(has_gen, A.has_gen);
  UP(G_ii, A.G_ii); UP(B_ii, A.B_ii); UP(Pd, A.Pd); UP(Qd, A.Qd); UP(G_ft, A.G_ft); UP(B_ft, A.B_ft);
  UP(G_tf, A.G_tf); UP(B_tf, A.B_tf); UP(c2b, A.c2b); UP(c1b, A.c1b); UP(c0b, A.c0b);
  UP(x_bus, A.x_bus); UP(x_kind, A.x_kind); UP(p_bus, A.p_bus); UP(p_kind, A.p_kind);
  UP(th_x, A.th_x); UP(v_x, A.v_x); UP(pinv, A.pinv);
  UP(F_rowptr, A.F_rowptr); UP(F_col, A.F_col); UP(F_diag, A.F_diag); UP(fact_order, A.fact_order);
  UP(diag_pos, A.diag_pos); UP(slot_pos, A.slot_pos); UP(gp_rptr, A.gp_rptr); UP(gp_col, A.gp_col);
  UP(gp_self_pos, A.gp_self_pos); UP(gp_pg_pos, A.gp_pg_pos); UP(gp_slot_pos, A.gp_slot_pos);
  UP(gpc_ptr, A.gpc_ptr); UP(gpc_pos, A.gpc_pos); UP(gpc_row, A.gpc_row);
  UP(dth_src, A.dth_src); UP(dv_src, A.dv_src); UP(yth_dst, A.yth_dst); UP(yv_dst, A.yv_dst);
  UP(pg_p, A.pg_p); UP(near_ref, A.near_ref);
#undef UP
  std::vector<int32_t> odth(2 * A.n_line), odv(2 * A.n_line);
  for (int s = 0; s < 2 * A.n_line; ++s) {
    odth[s] = A.dth_src[A.bl_other[s]];
    odv[s] = A.dv_src[A.bl_other[s]];
  }
  chk(c->o_dth_src = dalloc_copy(odth, P));
  chk(c->o_dv_src = dalloc_copy(odv, P));
  const int nx = A.n_x, np_ = A.n_p, nb = A.n_bus, m = A.n_line;
  const size_t nF = A.F_col.size();
  chk(c->F_val = dalloc<double>(nF, P));
  chk(c->flags = dalloc<int>(nx, P));
  chk(c->ticket = dalloc<int>(1, P));
  chk(c->status = dalloc<int>(1, P));
  chk(c->gp_val = dalloc<double>(A.gp_col.size(), P));
  chk(c->gpc_val = dalloc<double>(A.gp_col.size(), P));
  auto mk = [&](DevSweepStore &S, const Sweep &H) {
    S.n = nx;
    S.nnz = (int)H.col.size();
    S.d.nlev = H.nlev();
    int *lp, *rw, *rp, *cl;
    chk(lp = dalloc_copy(H.lev_ptr, P));
    chk(rw = dalloc_copy(H.rows, P));
    chk(rp = dalloc_copy(H.rptr, P));
    chk(cl = dalloc_copy(H.col, P));
    chk(S.src = dalloc_copy(H.src, P));
    chk(S.diag_src = dalloc_copy(H.diag_src, P));
    chk(S.val_mut = dalloc<double>(H.col.size(), P));
    S.d.lev_ptr = lp;
    S.d.rows = rw;
    S.d.rptr = rp;
    S.d.col = cl;
    S.d.val = S.val_mut;
    if (H.diag_src.empty() || H.diag_src[0] < 0) {
      S.d.dinv = nullptr;
    } else {
      chk(S.dinv_mut = dalloc<double>(nx, P));
      S.d.dinv = S.dinv_mut;
    }
  };
  mk(c->sL, A.sL);
  mk(c->sU, A.sU);
  mk(c->sUt, A.sUt);
  mk(c->sLt, A.sLt);
  chk(c->x = dalloc<double>(nx, P));
  chk(c->p = dalloc<double>(np_, P));
  chk(c->th = dalloc<double>(nb, P));
  chk(c->v = dalloc<double>(nb, P));
  chk(c->pgb = dalloc<double>(nb, P));
  chk(c->P = dalloc<double>(nb, P));
  chk(c->Q = dalloc<double>(nb, P));
  chk(c->g = dalloc<double>(nx, P));
  chk(c->refg_th = dalloc<double>(nb, P));
  chk(c->refg_v = dalloc<double>(nb, P));
  chk(c->scal = dalloc<double>(8, P));
  chk(c->cs = dalloc<double2>(m, P));
  chk(c->lam = dalloc<double>(nx, P));
  chk(c->muP = dalloc<double>(nb, P));
  chk(c->muQ = dalloc<double>(nb, P));
  chk(c->dcoef = dalloc<double>(nb, P));
  chk(c->X1col = dalloc<double>(nx, P));
  chk(c->coef = dalloc<double4>(m, P));
  if (!ok) return fail(c, RH_E_NOMEM, "device allocation failed while loading the grid");
  cudaError_t e = cudaMemset(c->flags, 0, sizeof(int) * nx);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return fail(c, RH_E_CUDA, std::string("upload: ") + cudaGetErrorString(e));
  c->epoch = 0;
  return RH_OK;
}

int pick_T(int N) {
  // columns per CTA: keep >= ~148 CTAs when N allows (148 SMs), T in {1..32}
  if (N >= 148 * 16) return 16;
  if (N >= 148 * 8) return 8;
  if (N >= 148 * 4) return 4;
  if (N >= 148 * 2) return 2;
  return 1;
}

int ensure_ws(rh_ctx *c, int N, int T) {
  const size_t ntiles = (size_t)((N + T - 1) / T);
  const size_t need = ntiles * T * (size_t)c->A.n_x;
  if (need <= c->ws_elems) return RH_OK;
  if (c->X1) cudaFree(c->X1);
  if (c->X2) cudaFree(c->X2);
  c->X1 = c->X2 = nullptr;
  c->ws_elems = 0;
  if (cudaMalloc(&c->X1, need * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&c->X2, need * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    return fail(c, RH_E_NOMEM, "workspace allocation failed");
  }
  c->ws_elems = need;
  return RH_OK;
}

HvpParams make_params(rh_ctx *c) {
  HvpParams h{};
  const Analysis &A = c->A;
  h.n_x = A.n_x;
  h.n_p = A.n_p;
  h.n_bus = A.n_bus;
  h.X1 = c->X1;
  h.X2 = c->X2;
  h.L = c->sL.d;
  h.U = c->sU.d;
  h.Ut = c->sUt.d;
  h.Lt = c->sLt.d;
  h.gp_rptr = c->gp_rptr;
  h.gp_col = c->gp_col;
  h.gp_val = c->gp_val;
  h.gpc_ptr = c->gpc_ptr;
  h.gpc_row = c->gpc_row;
  h.gpc_val = c->gpc_val;
  h.bl_ptr = c->bl_ptr;
  h.bl_line = c->bl_line;
  h.bl_end = c->bl_end;
  h.o_dth_src = c->o_dth_src;
  h.o_dv_src = c->o_dv_src;
  h.dth_src = c->dth_src;
  h.dv_src = c->dv_src;
  h.yth_dst = c->yth_dst;
  h.yv_dst = c->yv_dst;
  h.pg_p = c->pg_p;
  h.coef = c->coef;
  h.dcoef = c->dcoef;
  h.refg_th = c->refg_th;
  h.refg_v = c->refg_v;
  h.c2b = c->c2b;
  h.near_ref = c->near_ref;
  h.n_near_ref = (int)A.near_ref.size();
  h.f2ref = 2.0 * A.c2b[A.ref];
  return h;
}

void launch_hvp(int T, const HvpParams &h, int phases, int ntiles, cudaStream_t st) {
  switch (T) {
    case 1: k_hvp<1><<<ntiles, kThreads, 0, st>>>(h, phases); break;
    case 2: k_hvp<2><<<ntiles, kThreads, 0, st>>>(h, phases); break;
    case 4: k_hvp<4><<<ntiles, kThreads, 0, st>>>(h, phases); break;
    case 8: k_hvp<8><<<ntiles, kThreads, 0, st>>>(h, phases); break;
    case 16: k_hvp<16><<<ntiles, kThreads, 0, st>>>(h, phases); break;
    default: k_hvp<32><<<ntiles, kThreads, 0, st>>>(h, phases); break;
  }
}

int check_ready(rh_ctx *c, bool need_mult) {
  if (!c) return RH_E_ARG;
  if (c->host_only) return fail(c, RH_E_NODEV, "host-only context (device = -1)");
  if (!c->loaded) return fail(c, RH_E_ORDER, "no grid loaded (call rh_load_grid)");
  if (!c->has_state) return fail(c, RH_E_ORDER, "no state (call rh_set_state)");
  if (need_mult && !c->has_mult)
    return fail(c, RH_E_ORDER, "no multipliers (call rh_reduced_gradient or rh_set_multipliers)");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, RH_E_CUDA, "cudaSetDevice failed");
  return RH_OK;
}

// multipliers -> FoR tape (mu, per-line coefficients, bus diagonal)
int build_tape(rh_ctx *c, cudaStream_t st) {
  const Analysis &A = c->A;
  k_mu<<<nblk(A.n_bus), kThreads, 0, st>>>(A.n_bus, A.ref, c->th_x, c->v_x, c->lam, c->scal, c->muP, c->muQ);
  RH_LAUNCHED(c);
  k_coefs<<<nblk(std::max(A.n_line, A.n_bus)), kThreads, 0, st>>>(
      A.n_line, A.n_bus, c->lf, c->lt, c->G_ft, c->B_ft, c->G_tf, c->B_tf, c->G_ii, c->B_ii, c->cs, c->v,
      c->muP, c->muQ, c->coef, c->dcoef);
  RH_LAUNCHED(c);
  c->has_mult = true;
  return RH_OK;
}

// one Alg. 2 batch; W == nullptr with ident_j0 >= 0 for a Cartesian block
int hvp_impl(rh_ctx *c, const double *W, long long ldw, int ident_j0, double *HW, long long ldhw,
             int transposed, int N, cudaStream_t st, double *Zo = nullptr, double *Yxo = nullptr,
             double *Psio = nullptr, long long ldz = 0) {
  if (N <= 0) return RH_OK;
  const int T = pick_T(N);
  int rc = ensure_ws(c, N, T);
  if (rc) return rc;
  HvpParams h = make_params(c);
  h.N = N;
  h.W = W;
  h.ldw = ldw;
  h.ident_j0 = ident_j0;
  h.HW = HW;
  h.ldhw = ldhw;
  h.transposed = transposed;
  const int ntiles = (N + T - 1) / T;
  const bool staged = c->timing || Zo || Yxo || Psio;
  if (!staged) {
    launch_hvp(T, h, PH_ALL, ntiles, st);
    RH_LAUNCHED(c);
    return RH_OK;
  }
  const int ph[5] = {PH_L, PH_U, PH_FOR, PH_UT | PH_LT, PH_MULADD};
  cudaEvent_t ev[6];
  if (c->timing)
    for (auto &e : ev) cudaEventCreate(&e);
  const int nx = c->A.n_x;
  const long long tot = (long long)nx * N;
  for (int s = 0; s < 5; ++s) {
    if (c->timing) cudaEventRecord(ev[s], st);
    if (s == 3 && Yxo) {  // Y_x before the transposed solve: X2 holds -Y_x
      k_untile<<<nblk(tot), kThreads, 0, st>>>(nx, N, T, c->pinv, c->X2, -1.0, Yxo, ldz);
      RH_LAUNCHED(c);
    }
    launch_hvp(T, h, ph[s], ntiles, st);
    RH_LAUNCHED(c);
    if (s == 1 && Zo) {
      k_untile<<<nblk(tot), kThreads, 0, st>>>(nx, N, T, c->pinv, c->X1, 1.0, Zo, ldz);
      RH_LAUNCHED(c);
    }
    if (s == 3 && Psio) {
      k_untile<<<nblk(tot), kThreads, 0, st>>>(nx, N, T, c->pinv, c->X2, 1.0, Psio, ldz);
      RH_LAUNCHED(c);
    }
  }
  if (c->timing) {
    cudaEventRecord(ev[5], st);
    cudaEventSynchronize(ev[5]);
    float t[5];
    for (int s = 0; s < 5; ++s) cudaEventElapsedTime(&t[s], ev[s], ev[s + 1]);
    // {L+SpMul, U, FoR, U^T+L^T (reported in slot 3, slot 4 = MulAdd), total}
    c->stage_ms[0] = t[0];
    c->stage_ms[1] = t[1];
    c->stage_ms[2] = t[2];
    c->stage_ms[3] = t[3];
    c->stage_ms[4] = t[4];
    c->stage_ms[5] = t[0] + t[1] + t[2] + t[3] + t[4];
    for (auto &e : ev) cudaEventDestroy(e);
  }
  return RH_OK;
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================

extern "C" {

int rh_create(int device, rh_ctx **out) {
  if (!out) return RH_E_ARG;
  *out = nullptr;
  rh_ctx *c = new rh_ctx();
  c->device = device;
  c->host_only = device < 0;
  if (!c->host_only) {
    int nd = 0;
    if (cudaGetDeviceCount(&nd) != cudaSuccess || device >= nd) {
      cudaGetLastError();
      delete c;
      return RH_E_NODEV;
    }
    if (cudaSetDevice(device) != cudaSuccess) {
      delete c;
      return RH_E_CUDA;
    }
  }
  *out = c;
  return RH_OK;
}

int rh_destroy(rh_ctx *c) {
  if (!c) return RH_E_ARG;
  if (!c->host_only) {
    cudaSetDevice(c->device);
    c->free_all();
  }
  delete c;
  return RH_OK;
}

const char *rh_last_error(const rh_ctx *c) { return c ? c->err.c_str() : "null context"; }

int rh_load_grid(rh_ctx *c, const rh_grid *g, int32_t *n_x, int32_t *n_p) {
  if (!c || !g) return fail(c, RH_E_ARG, "null argument");
  if (!c->host_only) {
    if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, RH_E_CUDA, "cudaSetDevice failed");
    c->free_all();
  }
  c->loaded = c->has_state = c->has_mult = false;
  std::string msg = analyze(*g, c->A);
  if (!msg.empty()) return fail(c, RH_E_GRID, msg);
  if (!c->host_only) {
    int rc = upload(c);
    if (rc) return rc;
  }
  c->loaded = true;
  if (n_x) *n_x = c->A.n_x;
  if (n_p) *n_p = c->A.n_p;
  c->err.clear();
  return RH_OK;
}

int rh_get_info(const rh_ctx *c, rh_info *info) {
  if (!c || !info) return RH_E_ARG;
  if (!c->loaded) return RH_E_ORDER;
  const Analysis &A = c->A;
  info->n_bus = A.n_bus;
  info->n_line = A.n_line;
  info->n_x = A.n_x;
  info->n_p = A.n_p;
  info->nnz_J = A.nnz_J;
  info->nnz_Gp = (int)A.gp_col.size();
  info->nnz_LU = (int)A.F_col.size();
  info->levels_fwd = A.nlev_fwd;
  info->levels_bwd = A.nlev_bwd;
  info->max_level_rows = A.max_level_rows;
  info->workspace_bytes = (int64_t)c->ws_elems * 2 * (int64_t)sizeof(double);
  return RH_OK;
}

int rh_orderings(const rh_ctx *c, int32_t *x_bus, int32_t *x_kind, int32_t *p_bus, int32_t *p_kind) {
  if (!c) return RH_E_ARG;
  if (!c->loaded) return RH_E_ORDER;
  const Analysis &A = c->A;
  if (x_bus) std::copy(A.x_bus.begin(), A.x_bus.end(), x_bus);
  if (x_kind) std::copy(A.x_kind.begin(), A.x_kind.end(), x_kind);
  if (p_bus) std::copy(A.p_bus.begin(), A.p_bus.end(), p_bus);
  if (p_kind) std::copy(A.p_kind.begin(), A.p_kind.end(), p_kind);
  return RH_OK;
}

int rh_symbolic(const rh_ctx *c, int32_t *perm, int32_t *lu_rowptr, int32_t *lu_colidx, int32_t *level_fwd,
                int32_t *level_bwd) {
  if (!c) return RH_E_ARG;
  if (!c->loaded) return RH_E_ORDER;
  const Analysis &A = c->A;
  if (perm) std::copy(A.perm.begin(), A.perm.end(), perm);
  if (lu_rowptr) std::copy(A.F_rowptr.begin(), A.F_rowptr.end(), lu_rowptr);
  if (lu_colidx) std::copy(A.F_col.begin(), A.F_col.end(), lu_colidx);
  if (level_fwd) std::copy(A.lev_fwd.begin(), A.lev_fwd.end(), level_fwd);
  if (level_bwd) std::copy(A.lev_bwd.begin(), A.lev_bwd.end(), level_bwd);
  return RH_OK;
}

int rh_set_state(rh_ctx *c, const double *x, const double *p, void *stream) {
  if (!c || !x || !p) return fail(c, RH_E_ARG, "null argument");
  if (c->host_only) return fail(c, RH_E_NODEV, "host-only context (device = -1)");
  if (!c->loaded) return fail(c, RH_E_ORDER, "no grid loaded");
  RH_CUDA(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  const Analysis &A = c->A;
  const int nx = A.n_x, np_ = A.n_p, nb = A.n_bus, m = A.n_line;
  c->has_state = c->has_mult = false;
  RH_CUDA(c, cudaMemcpyAsync(c->x, x, sizeof(double) * nx, cudaMemcpyDeviceToDevice, st));
  RH_CUDA(c, cudaMemcpyAsync(c->p, p, sizeof(double) * np_, cudaMemcpyDeviceToDevice, st));
  RH_CUDA(c, cudaMemsetAsync(c->F_val, 0, sizeof(double) * A.F_col.size(), st));
  RH_CUDA(c, cudaMemsetAsync(c->gp_val, 0, sizeof(double) * A.gp_col.size(), st));
  RH_CUDA(c, cudaMemsetAsync(c->refg_th, 0, sizeof(double) * nb, st));
  RH_CUDA(c, cudaMemsetAsync(c->refg_v, 0, sizeof(double) * nb, st));
  RH_CUDA(c, cudaMemsetAsync(c->ticket, 0, sizeof(int), st));
  RH_CUDA(c, cudaMemsetAsync(c->status, 0, sizeof(int), st));
  k_bus_state<<<nblk(nx + np_ + 1), kThreads, 0, st>>>(nx, np_, c->x_bus, c->x_kind, c->p_bus, c->p_kind, c->x,
                                                      c->p, c->th, c->v, c->pgb, A.ref, A.theta_ref);
  RH_LAUNCHED(c);
  k_line_trig<<<nblk(m), kThreads, 0, st>>>(m, c->lf, c->lt, c->th, c->cs);
  RH_LAUNCHED(c);
  AsmParams a{};
  a.n_bus = nb;
  a.ref = A.ref;
  a.bus_type = c->bus_type;
  a.bl_ptr = c->bl_ptr;
  a.bl_line = c->bl_line;
  a.bl_other = c->bl_other;
  a.bl_end = c->bl_end;
  a.G_ii = c->G_ii;
  a.B_ii = c->B_ii;
  a.Pd = c->Pd;
  a.Qd = c->Qd;
  a.G_ft = c->G_ft;
  a.B_ft = c->B_ft;
  a.G_tf = c->G_tf;
  a.B_tf = c->B_tf;
  a.th = c->th;
  a.v = c->v;
  a.pgb = c->pgb;
  a.cs = c->cs;
  a.th_x = c->th_x;
  a.v_x = c->v_x;
  a.diag_pos = c->diag_pos;
  a.slot_pos = c->slot_pos;
  a.gp_self_pos = c->gp_self_pos;
  a.gp_pg_pos = c->gp_pg_pos;
  a.gp_slot_pos = c->gp_slot_pos;
  a.P = c->P;
  a.Q = c->Q;
  a.g = c->g;
  a.F_val = c->F_val;
  a.gp_val = c->gp_val;
  a.refg_th = c->refg_th;
  a.refg_v = c->refg_v;
  k_assemble<<<nblk(nb, 128), 128, 0, st>>>(a);
  RH_LAUNCHED(c);
  k_objective<<<1, kThreads, 0, st>>>(nb, A.ref, c->has_gen, c->c2b, c->c1b, c->c0b, c->pgb, c->P, c->Pd,
                                      c->scal);
  RH_LAUNCHED(c);
  // numeric refactorization
  c->epoch += 1;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
  const int fblocks = std::min(nsm * 4, std::max(1, nblk((long long)nx * 32)));
  k_refactor<<<fblocks, kThreads, 0, st>>>(nx, c->fact_order, c->F_rowptr, c->F_col, c->F_diag, c->F_val,
                                           c->flags, c->epoch, c->ticket, c->status, 1e-14);
  RH_LAUNCHED(c);
  for (DevSweepStore *S : {&c->sL, &c->sU, &c->sUt, &c->sLt}) {
    if (S->nnz > 0) {
      k_gather_vals<<<nblk(S->nnz), kThreads, 0, st>>>(S->nnz, S->src, c->F_val, S->val_mut);
      RH_LAUNCHED(c);
    }
    if (S->dinv_mut) {
      k_gather_inv<<<nblk(S->n), kThreads, 0, st>>>(S->n, S->diag_src, c->F_val, S->dinv_mut);
      RH_LAUNCHED(c);
    }
  }
  const int ngp = (int)A.gp_col.size();
  if (ngp > 0) {
    k_gather_vals<<<nblk(ngp), kThreads, 0, st>>>(ngp, c->gpc_pos, c->gp_val, c->gpc_val);
    RH_LAUNCHED(c);
  }
  int status = 0;
  RH_CUDA(c, cudaMemcpyAsync(&status, c->status, sizeof(int), cudaMemcpyDeviceToHost, st));
  RH_CUDA(c, cudaStreamSynchronize(st));
  if (status != 0) {
    char buf[160];
    snprintf(buf, sizeof buf, "refactorization: pivot of permuted row %d below 1e-14 * row max", status - 1);
    return fail(c, RH_E_SINGULAR, buf);
  }
  c->has_state = true;
  return RH_OK;
}

int rh_residual(rh_ctx *c, double *g, double *f, void *stream) {
  int rc = check_ready(c, false);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (g) RH_CUDA(c, cudaMemcpyAsync(g, c->g, sizeof(double) * c->A.n_x, cudaMemcpyDeviceToDevice, st));
  if (f) RH_CUDA(c, cudaMemcpyAsync(f, c->scal + 3, sizeof(double), cudaMemcpyDeviceToDevice, st));
  return RH_OK;
}

int rh_reduced_gradient(rh_ctx *c, double *grad_p, double *lambda_out, void *stream) {
  int rc = check_ready(c, false);
  if (rc) return rc;
  if (!grad_p) return fail(c, RH_E_ARG, "grad_p is null");
  cudaStream_t st = (cudaStream_t)stream;
  const Analysis &A = c->A;
  k_grad_rhs<<<nblk(A.n_x), kThreads, 0, st>>>(A.n_x, c->x_bus, c->x_kind, c->pinv, c->refg_th, c->refg_v,
                                                c->scal, c->X1col);
  RH_LAUNCHED(c);
  k_solve_T1<<<1, kThreads, 0, st>>>(c->sUt.d, c->sLt.d, c->X1col);
  RH_LAUNCHED(c);
  k_grad_out<<<nblk(std::max(A.n_x, A.n_p)), kThreads, 0, st>>>(
      A.n_x, A.n_p, c->pinv, c->p_bus, c->p_kind, c->c2b, c->c1b, c->p, c->refg_v, c->scal, c->gpc_ptr, c->gpc_row,
      c->gpc_val, c->X1col, c->lam, grad_p);
  RH_LAUNCHED(c);
  if (lambda_out)
    RH_CUDA(c, cudaMemcpyAsync(lambda_out, c->lam, sizeof(double) * A.n_x, cudaMemcpyDeviceToDevice, st));
  return build_tape(c, st);
}

int rh_set_multipliers(rh_ctx *c, const double *lambda, void *stream) {
  int rc = check_ready(c, false);
  if (rc) return rc;
  if (!lambda) return fail(c, RH_E_ARG, "lambda is null");
  cudaStream_t st = (cudaStream_t)stream;
  RH_CUDA(c, cudaMemcpyAsync(c->lam, lambda, sizeof(double) * c->A.n_x, cudaMemcpyDeviceToDevice, st));
  return build_tape(c, st);
}

int rh_hvp(rh_ctx *c, const double *W, int64_t ldw, double *HW, int64_t ldhw, int32_t N, void *stream) {
  int rc = check_ready(c, true);
  if (rc) return rc;
  if (N < 0 || (N > 0 && (!W || !HW)) || ldw < N || ldhw < N) return fail(c, RH_E_ARG, "bad W/HW/N/ld");
  return hvp_impl(c, W, ldw, -1, HW, ldhw, 0, N, (cudaStream_t)stream);
}

int rh_hvp_stages(rh_ctx *c, const double *W, int64_t ldw, double *HW, int64_t ldhw, int32_t N, double *Z,
                  double *Yx, double *Psi, int64_t ldz, void *stream) {
  int rc = check_ready(c, true);
  if (rc) return rc;
  if (N <= 0 || !W || !HW || ldw < N || ldhw < N || ((Z || Yx || Psi) && ldz < N))
    return fail(c, RH_E_ARG, "bad W/HW/N/ld");
  return hvp_impl(c, W, ldw, -1, HW, ldhw, 0, N, (cudaStream_t)stream, Z, Yx, Psi, ldz);
}

int rh_hessian_columns(rh_ctx *c, int32_t j0, int32_t j1, int32_t N, double *H, int64_t ldh, int32_t transposed,
                       void *stream) {
  int rc = check_ready(c, true);
  if (rc) return rc;
  const int np_ = c->A.n_p;
  if (j0 < 0 || j1 > np_ || j0 > j1 || N <= 0 || !H) return fail(c, RH_E_ARG, "bad column range / N / H");
  if ((!transposed && ldh < j1 - j0) || (transposed && ldh < np_)) return fail(c, RH_E_ARG, "ldh too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int ncols = j1 - j0;
  const int nb = (ncols + N - 1) / N;
  for (int b = 0; b < nb; ++b) {
    // balanced batches of width <= N (SURVEY.md 8(d) batch plan)
    const int a0 = (int)((long long)ncols * b / nb), a1 = (int)((long long)ncols * (b + 1) / nb);
    double *out = transposed ? H + (long long)a0 * ldh : H + a0;
    rc = hvp_impl(c, nullptr, 0, j0 + a0, out, ldh, transposed, a1 - a0, st);
    if (rc) return rc;
  }
  return RH_OK;
}

int rh_full_hessian(rh_ctx *c, int32_t N, double *H, void *stream) {
  int rc = check_ready(c, true);
  if (rc) return rc;
  return rh_hessian_columns(c, 0, c->A.n_p, N, H, c->A.n_p, 0, stream);
}

int rh_reduced_hessian_host(rh_ctx *c, const double *x, const double *p, int32_t N, double *grad_p, double *H) {
  if (!c || !x || !p || !H) return fail(c, RH_E_ARG, "null argument");
  if (c->host_only) return fail(c, RH_E_NODEV, "host-only context (device = -1)");
  if (!c->loaded) return fail(c, RH_E_ORDER, "no grid loaded");
  RH_CUDA(c, cudaSetDevice(c->device));
  const Analysis &A = c->A;
  const size_t nx = A.n_x, np_ = A.n_p;
  double *dx = nullptr, *dp = nullptr, *dg = nullptr, *dH = nullptr;
  cudaStream_t st = nullptr;
  RH_CUDA(c, cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  int rc = RH_OK;
  do {
    if (cudaMallocAsync(&dx, nx * 8, st) || cudaMallocAsync(&dp, np_ * 8, st) ||
        cudaMallocAsync(&dg, np_ * 8, st) || cudaMallocAsync(&dH, np_ * np_ * 8, st)) {
      rc = fail(c, RH_E_NOMEM, "allocation failed");
      break;
    }
    if (cudaMemcpyAsync(dx, x, nx * 8, cudaMemcpyHostToDevice, st) ||
        cudaMemcpyAsync(dp, p, np_ * 8, cudaMemcpyHostToDevice, st)) {
      rc = fail(c, RH_E_CUDA, "H2D copy failed");
      break;
    }
    if ((rc = rh_set_state(c, dx, dp, st))) break;
    if ((rc = rh_reduced_gradient(c, dg, nullptr, st))) break;
    if ((rc = rh_full_hessian(c, N, dH, st))) break;
    if ((grad_p && cudaMemcpyAsync(grad_p, dg, np_ * 8, cudaMemcpyDeviceToHost, st)) ||
        cudaMemcpyAsync(H, dH, np_ * np_ * 8, cudaMemcpyDeviceToHost, st)) {
      rc = fail(c, RH_E_CUDA, "D2H copy failed");
      break;
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) rc = fail(c, RH_E_CUDA, "stream sync failed");
  } while (0);
  cudaFreeAsync(dx, st);
  cudaFreeAsync(dp, st);
  cudaFreeAsync(dg, st);
  cudaFreeAsync(dH, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  return rc;
}

int64_t rh_launch_count(const rh_ctx *c) { return c ? c->launches : 0; }

int rh_set_timing(rh_ctx *c, int enable) {
  if (!c) return RH_E_ARG;
  c->timing = enable != 0;
  return RH_OK;
}

int rh_stage_times(const rh_ctx *c, float *ms_out) {
  if (!c || !ms_out) return RH_E_ARG;
  for (int i = 0; i < 6; ++i) ms_out[i] = c->stage_ms[i];
  return RH_OK;
}

}  // extern "C"
