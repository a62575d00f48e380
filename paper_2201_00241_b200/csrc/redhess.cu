// B200-native batched adjoint-adjoint reduced Hessian: device kernels + C ABI.
// Everything on the hot path is a hand-written sm_100a fp64 kernel in this
// file; the host only runs the one-time symbolic analysis (analysis.cpp).
//
// Citations are PAPER.md line numbers (arXiv 2201.00241) or DESIGN.md readings.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <cmath>
#include <numeric>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/redhess.h"
#include "analysis.hpp"
#include "kernels.cuh"
#include "devutil.cuh"
#include "dense.hpp"

using namespace rh;

// ============================================================================
// device helpers
// ============================================================================


__device__ __forceinline__ int ld_acquire_cta_shared(const int *p) {
  int v;
  asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_shared(int *p, int v) {
  asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}

__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ============================================================================
// state kernels: bus state, line trig, injections, g,
// J and G_p assembly (Appendix A identities), grad P_ref
// ============================================================================

// (k_state_prep: x, p -> bus-level theta, v, Pg (R5 orderings); per
// line c = cos(th_f - th_t), s = sin(th_f - th_t), trig once per line)

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
  const int *bl_bus;    // two-kernel path: owner bus of each incidence
  double *tP, *tQ;      // two-kernel path: per-incidence injection terms
  int n_inc;
};

// Bus-centric assembly (race-free: bus b owns rows P_b, Q_b).  Eq. powerflow
// with the Ybus diagonal (R1); g per Eq. powerflowvec
// (R2); J / G_p entries per SURVEY.md Appendix A.
// Two-kernel assembly (grids without parallel lines, A.asm_unique): every J /
// G_p line slot and REF-gradient entry has one incidence, so the line kernel
// stores it directly, and the bus kernel sums its incidences' injection terms in
// the same order as k_assemble (equal to rounding: k_assemble contracts each term
// into its running sum with an FMA), with much shorter dependent chains.
__global__ void k_asm_lines(AsmParams a) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.n_inc) return;
  const int b = a.bl_bus[s], l = a.bl_line[s], o = a.bl_other[s];
  const double vb = a.v[b], vo = a.v[o];
  const double2 cs = a.cs[l];
  const bool from = a.bl_end[s] == 0;
  const double G = from ? a.G_ft[l] : a.G_tf[l];
  const double B = from ? a.B_ft[l] : a.B_tf[l];
  const double c = cs.x, sn = from ? cs.y : -cs.y;   // cos/sin(th_b - th_o)
  const double gsbc = G * sn - B * c, gcbs = G * c + B * sn;
  a.tP[s] = vo * gcbs;
  a.tQ[s] = vo * gsbc;
  if (b == a.ref) {
    a.refg_th[o] = vb * vo * gsbc;
    a.refg_v[o] = vb * gcbs;
    return;
  }
  const double dPth = vb * vo * gsbc, dPv = vb * gcbs;
  const double dQth = -vb * vo * gcbs, dQv = vb * gsbc;
  const int4 sp = *reinterpret_cast<const int4 *>(a.slot_pos + 4 * s);
  if (sp.x >= 0) a.F_val[sp.x] = dPth;
  if (sp.y >= 0) a.F_val[sp.y] = dPv;
  if (sp.z >= 0) a.F_val[sp.z] = dQth;
  if (sp.w >= 0) a.F_val[sp.w] = dQv;
  const int2 gs = *reinterpret_cast<const int2 *>(a.gp_slot_pos + 2 * s);
  if (gs.x >= 0) a.gp_val[gs.x] = dPv;
  if (gs.y >= 0) a.gp_val[gs.y] = dQv;
}
__global__ void k_asm_buses(AsmParams a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.n_bus) return;
  const double vb = a.v[b];
  double P = 0.0, Q = 0.0;
  for (int s = a.bl_ptr[b]; s < a.bl_ptr[b + 1]; ++s) {
    P += a.tP[s];
    Q += a.tQ[s];
  }
  const double Gbb = a.G_ii[b], Bbb = a.B_ii[b];
  P = vb * P + vb * vb * Gbb;
  Q = vb * Q - vb * vb * Bbb;
  a.P[b] = P;
  a.Q[b] = Q;
  if (b == a.ref) {
    a.refg_v[b] += P / vb + Gbb * vb;
    return;
  }
  const int t = a.bus_type[b];
  const int rP = a.th_x[b];
  const int rQ = a.v_x[b];
  a.g[rP] = P + a.Pd[b] - (t == RH_PV ? a.pgb[b] : 0.0);
  if (rQ >= 0) a.g[rQ] = Q + a.Qd[b];
  const int4 dp = *reinterpret_cast<const int4 *>(a.diag_pos + 4 * b);
  a.F_val[dp.x] += -Q - Bbb * vb * vb;
  if (rQ >= 0) {
    a.F_val[dp.y] += P / vb + Gbb * vb;
    a.F_val[dp.z] += P - Gbb * vb * vb;
    a.F_val[dp.w] += Q / vb - Bbb * vb;
  } else {
    a.gp_val[a.gp_self_pos[b]] += P / vb + Gbb * vb;
    a.gp_val[a.gp_pg_pos[b]] = -1.0;
  }
}

__global__ void k_assemble(AsmParams a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.n_bus) return;
  const double vb = a.v[b];
  const int s0 = a.bl_ptr[b], s1 = a.bl_ptr[b + 1];
  const bool isref = b == a.ref;
  // one pass over the bus's lines: injections P, Q and the off-diagonal
  // derivatives (which do not depend on P, Q); same per-slot order as before
  double P = 0.0, Q = 0.0;
  for (int s = s0; s < s1; ++s) {
    const int l = a.bl_line[s], o = a.bl_other[s];
    const double2 cs = a.cs[l];
    const bool from = a.bl_end[s] == 0;
    const double G = from ? a.G_ft[l] : a.G_tf[l];
    const double B = from ? a.B_ft[l] : a.B_tf[l];
    const double c = cs.x, sn = from ? cs.y : -cs.y;   // cos/sin(th_b - th_o)
    const double vo = a.v[o];
    const double gsbc = G * sn - B * c, gcbs = G * c + B * sn;
    P += vo * gcbs;
    Q += vo * gsbc;
    if (isref) {   // grad P_ref over (theta_o, v_o) of the neighbours (theta_ref constant)
      a.refg_th[o] += vb * vo * gsbc;
      a.refg_v[o] += vb * gcbs;
      continue;
    }
    const double dPth = vb * vo * gsbc, dPv = vb * gcbs;
    const double dQth = -vb * vo * gcbs, dQv = vb * gsbc;
    const int4 sp = *reinterpret_cast<const int4 *>(a.slot_pos + 4 * s);
    if (sp.x >= 0) a.F_val[sp.x] += dPth;
    if (sp.y >= 0) a.F_val[sp.y] += dPv;
    if (sp.z >= 0) a.F_val[sp.z] += dQth;
    if (sp.w >= 0) a.F_val[sp.w] += dQv;
    const int2 gs = *reinterpret_cast<const int2 *>(a.gp_slot_pos + 2 * s);
    if (gs.x >= 0) a.gp_val[gs.x] += dPv;
    if (gs.y >= 0) a.gp_val[gs.y] += dQv;
  }
  const double Gbb = a.G_ii[b], Bbb = a.B_ii[b];
  P = vb * P + vb * vb * Gbb;
  Q = vb * Q - vb * vb * Bbb;
  a.P[b] = P;
  a.Q[b] = Q;
  if (isref) {
    a.refg_v[b] += P / vb + Gbb * vb;   // and v_ref
    return;
  }
  const int t = a.bus_type[b];
  const int rP = a.th_x[b];
  const int rQ = a.v_x[b];
  a.g[rP] = P + a.Pd[b] - (t == RH_PV ? a.pgb[b] : 0.0);
  if (rQ >= 0) a.g[rQ] = Q + a.Qd[b];
  // diagonal block
  const int4 dp = *reinterpret_cast<const int4 *>(a.diag_pos + 4 * b);
  a.F_val[dp.x] += -Q - Bbb * vb * vb;            // dP_b/dth_b
  if (rQ >= 0) {
    a.F_val[dp.y] += P / vb + Gbb * vb;            // dP_b/dv_b
    a.F_val[dp.z] += P - Gbb * vb * vb;            // dQ_b/dth_b
    a.F_val[dp.w] += Q / vb - Bbb * vb;            // dQ_b/dv_b
  } else {
    a.gp_val[a.gp_self_pos[b]] += P / vb + Gbb * vb; // dP_b/dv_b, v_b in p (PV)
    a.gp_val[a.gp_pg_pos[b]] = -1.0;                  // dP_b/dPg_b
  }
}

// f (R4) and the REF multiplier seed mu_ref = f'(Pg_ref) (R22).  One block.
// scal[0] = P_ref, scal[1] = Pg_ref, scal[2] = mu_ref, scal[3] = f
// NEXT-4: forward-mode tangents of the residual, one
// direction per column color.  Thread (bus b, color c): the seed of a bus
// variable is 1 iff its column has color c; the dual-number derivative of
// P_b = v_b sum_o v_o (G cos th_bo + B sin th_bo) + v_b^2 G_bb and of Q_b
// (R1) along that seed, minus the Pg seed for g[P_b] (R2), lands in
// JS[row][c] with rows in the natural x order.
__global__ void k_jvp_colored(int n_bus, int ref, int C, const int *__restrict__ bl_ptr,
                              const int *__restrict__ bl_line, const int *__restrict__ bl_other,
                              const int *__restrict__ bl_end, const double2 *__restrict__ cs,
                              const double *__restrict__ G_ft, const double *__restrict__ B_ft,
                              const double *__restrict__ G_tf, const double *__restrict__ B_tf,
                              const double *__restrict__ G_ii, const double *__restrict__ B_ii,
                              const double *__restrict__ v, const int *__restrict__ th_x, const int *__restrict__ v_x,
                              const int *__restrict__ col_th, const int *__restrict__ col_v,
                              const int *__restrict__ col_pg, double *JS) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)n_bus * C) return;
  const int b = (int)(t / C), c = (int)(t % C);
  if (b == ref) return;
  const double vb = v[b];
  const double sth_b = col_th[b] == c ? 1.0 : 0.0, sv_b = col_v[b] == c ? 1.0 : 0.0;
  double dP = 0.0, dQ = 0.0;
  for (int s = bl_ptr[b]; s < bl_ptr[b + 1]; ++s) {
    const int l = bl_line[s], o = bl_other[s];
    const double2 q = cs[l];
    const bool from = bl_end[s] == 0;
    const double G = from ? G_ft[l] : G_tf[l];
    const double B = from ? B_ft[l] : B_tf[l];
    const double co = q.x, sn = from ? q.y : -q.y;   // cos/sin(th_b - th_o)
    const double vo = v[o];
    const double sth_o = col_th[o] == c ? 1.0 : 0.0, sv_o = col_v[o] == c ? 1.0 : 0.0;
    const double gcbs = G * co + B * sn, gsbc = G * sn - B * co;
    const double dvv = sv_b * vo + vb * sv_o, vv = vb * vo, dth = sth_b - sth_o;
    dP += dvv * gcbs - vv * gsbc * dth;   // d[v_b v_o (G c + B s)]
    dQ += dvv * gsbc + vv * gcbs * dth;   // d[v_b v_o (G s - B c)]
  }
  dP += 2.0 * vb * G_ii[b] * sv_b;
  dQ -= 2.0 * vb * B_ii[b] * sv_b;
  if (col_pg[b] == c) dP -= 1.0;
  JS[(long long)th_x[b] * C + c] = dP;
  if (v_x[b] >= 0) JS[(long long)v_x[b] * C + c] = dQ;
}

// decompression: entry (pos, row, color) of J / G_p reads JS[row][color]
__global__ void k_decompress(int nj, const int *__restrict__ jpos, const int *__restrict__ jrow,
                             const int *__restrict__ jcol, double *F_val, int ng, const int *__restrict__ gpos,
                             const int *__restrict__ grow, const int *__restrict__ gcol, double *gp_val, int C,
                             const double *__restrict__ JS) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nj) F_val[jpos[t]] = JS[(long long)jrow[t] * C + jcol[t]];
  else if (t - nj < ng) {
    const int u = t - nj;
    gp_val[gpos[u]] = JS[(long long)grow[u] * C + gcol[u]];
  }
}

// The state's independent prologue in ONE launch (grid-stride segments): x, p
// into the context; zero the assembled values, the REF gradient and the pivot
// flag; bus state (theta, v, Pg per bus) and line trig (cos, sin of
// theta_f - theta_t), both read from the caller's x, p directly.
__global__ void k_state_prep(int nx, int np_, const double *__restrict__ x, const double *__restrict__ p, double *cx,
                             double *cp, long long nF, double *F_val, long long nG, double *gp_val, int nb,
                             double *refg_th, double *refg_v, int *status, const int *__restrict__ x_bus,
                             const int *__restrict__ x_kind, const int *__restrict__ p_bus,
                             const int *__restrict__ p_kind, double *th, double *v, double *pgb, int ref,
                             double theta_ref, int m, const int *__restrict__ lf, const int *__restrict__ lt,
                             const int *__restrict__ th_x, double2 *cs) {
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x, step = (long long)gridDim.x * blockDim.x;
  for (long long i = t0; i < nx; i += step) {
    const double xv = x[i];
    cx[i] = xv;
    if (x_kind[i] == RH_KIND_THETA) th[x_bus[i]] = xv;
    else v[x_bus[i]] = xv;
  }
  for (long long i = t0; i < np_; i += step) {
    const double pv = p[i];
    cp[i] = pv;
    if (p_kind[i] == RH_KIND_PG) pgb[p_bus[i]] = pv;
    else v[p_bus[i]] = pv;
  }
  for (long long l = t0; l < m; l += step) {
    const int f = lf[l], t = lt[l];
    const double tf = f == ref ? theta_ref : x[th_x[f]], tt = t == ref ? theta_ref : x[th_x[t]];
    double s, c;
    sincos(tf - tt, &s, &c);
    cs[l] = make_double2(c, s);
  }
  for (long long i = t0; i < nF; i += step) F_val[i] = 0.0;
  for (long long i = t0; i < nG; i += step) gp_val[i] = 0.0;
  for (long long i = t0; i < nb; i += step) {
    refg_th[i] = 0.0;
    refg_v[i] = 0.0;
  }
  if (t0 == 0) {
    *status = 0;
    th[ref] = theta_ref;
  }
}

__global__ void k_objective(int n_bus, int ref, const int *has_gen, const double *c2b, const double *c1b,
                            const double *c0b, const double *pgb, const double *P, const double *Pd,
                            double *scal) {
  __shared__ double red[1024];
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
// PAPER.md:764-767), static diagonal pivots (R15), three phases over the
// elimination-tree segments:
//   R_A  one CTA per block: the block's F rows staged in shared memory,
//        up-looking Doolittle row by row in local level order (warp per row);
//   R_B1 one warp per separator row: the updates from block columns;
//   R_B2 one CTA: right-looking elimination of the separator x separator
//        submatrix in shared memory (one barrier pair per pivot).
// Every entry receives its updates in a fixed order: deterministic.
// ============================================================================

// R_A: one CTA (16 warps) per block.  The block's F rows, its k-step records
// and target offsets are staged in shared memory; rows follow the block's
// forward subtree-to-warp schedule (the same one as the L / U^T sweeps: row i
// depends on Lrow(i), its descendants), so a warp eliminates its subtrees
// without CTA barriers (warp lanes split every row update; __syncwarp orders
// the rows of one warp).
constexpr int kMaxTopsFact = 64;   // tops rows of a block (analysis kMaxTops <= this)
constexpr int kFactLvl = 20;       // forward split bounds of a block (16 warps + 1, tops 2, pad)
// byte offset of k_fact_blocks' per-row metadata: after F rows + dinv (doubles),
// k-step records (int4 + int) and target offsets (uint16)
__host__ __device__ inline size_t fact_meta_offset(int fo_end, int nr, int nks, int ntg) {
  const size_t d_end = (size_t)((fo_end + nr + 1) & ~1) * 8;
  return d_end + (size_t)nks * 20 + (size_t)ntg * 2;
}
constexpr int kMaxRowsFact = 1024; // rows of a block (Rmax <= this)
__global__ void __launch_bounds__(2 * kSegThreads, 1) k_fact_blocks(FactParams f) {
  extern __shared__ double sm[];
  const int s = blockIdx.x;
  const int r0 = f.seg_row_off[s], nr = f.seg_row_off[s + 1] - r0;
  const int fb = f.blk_fo_off[s];
  const int kb = f.ks_ptr[r0], nks = f.ks_ptr[r0 + nr] - kb;
  const int tb = nks > 0 ? f.ks4[4 * kb + 3] : 0;
  const int ntg = nks > 0 ? f.ks4[4 * (kb + nks - 1) + 3] + f.ks4[4 * (kb + nks - 1) + 2] - tb : 0;
  double *SF = sm;                                   // [fo end]
  double *sdinv = SF + f.fo[fb + nr];                // [nr]
  const int d_end = (f.fo[fb + nr] + nr + 1) & ~1;   // 16-byte boundary for the int4 records
  int4 *sks = reinterpret_cast<int4 *>(SF + d_end);
  int *skk = reinterpret_cast<int *>(sks + nks);
  unsigned short *stg = reinterpret_cast<unsigned short *>(skk + nks);
  // per-row metadata (off, len, k-steps [begin, end)), (pivot offset in the row, F row), row order, levels
  int4 *s_rm = reinterpret_cast<int4 *>(reinterpret_cast<char *>(sm) + ((fact_meta_offset(f.fo[fb + nr], nr, nks, ntg) + 15) & ~15));
  int2 *s_rd = reinterpret_cast<int2 *>(s_rm + nr);
  const int *lvg = f.fwd_lvl_ptr + f.fwd_seg_lvl[s];
  int *s_lv = reinterpret_cast<int *>(s_rd + nr);
  int *s_ord = s_lv + kFactLvl;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  long long *prof = (f.dbg && threadIdx.x == 0) ? f.dbg + 8 * s : nullptr;
  if (prof) prof[0] = clock64();
  // stage the block's F rows: thread per row, 8-byte cp.async copies all in flight
  for (int a = threadIdx.x; a < nr; a += blockDim.x) {
    const int i = f.row_global[r0 + a];
    const int off = f.fo[fb + a], len = f.fo[fb + a + 1] - off, rb = f.F_rowptr[i];
    for (int t = 0; t < len; ++t) {
      const unsigned d = (unsigned)__cvta_generic_to_shared(SF + off + t);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(f.F_val + rb + t) : "memory");
    }
  }
  const int4 *gks = reinterpret_cast<const int4 *>(f.ks4);
  for (int t = threadIdx.x; t < nks; t += blockDim.x) {
    int4 v = gks[kb + t];
    v.w -= tb;
    sks[t] = v;
    skk[t] = f.ks_k[kb + t];
  }
  for (int t = threadIdx.x; t < ntg; t += blockDim.x) stg[t] = f.tgt16[tb + t];
  for (int a = threadIdx.x; a < nr; a += blockDim.x) {
    const int i = f.row_global[r0 + a];
    const int off = f.fo[fb + a];
    s_rm[a] = make_int4(off, f.fo[fb + a + 1] - off, f.ks_ptr[r0 + a] - kb, f.ks_ptr[r0 + a + 1] - kb);
    s_rd[a] = make_int2(f.F_diag[i] - f.F_rowptr[i], i);
  }
  if (threadIdx.x < kFactLvl) s_lv[threadIdx.x] = lvg[threadIdx.x] - lvg[0];
  const int q0b = lvg[0];
  for (int t = threadIdx.x; t < nr; t += blockDim.x) s_ord[t] = f.fwd_order[q0b + t];
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (prof) prof[1] = clock64();
  // forward split of the block: lvl[0..nw] = each warp's piece rows, lvl[nw+1..nw+2] = tops
  // (block-relative row positions; s_ord maps a position to the block-local row)
  const int *lv = s_lv;
  // up-looking elimination of one row: every k-step's record, pivot reciprocal
  // and target offsets are prefetched one step ahead, so the chain per k-step is
  // the row's own values (load, scale, update, store)
  auto eliminate = [&](int q) {
    const int a = s_ord[q];
    const int4 rm = s_rm[a];
    const int2 rd = s_rd[a];
    double *w = SF + rm.x;
    double amax = 0.0;
    for (int t = lane; t < rm.y; t += 32) amax = fmax(amax, fabs(w[t]));
    amax = warp_max(amax);
    const int k1 = rm.w;
    int ks = rm.z;
    int4 m = ks < k1 ? sks[ks] : make_int4(0, 0, 0, 0);
    double dk = ks < k1 ? sdinv[skk[ks]] : 0.0;
    for (; ks < k1; ++ks) {
      const int4 mn = ks + 1 < k1 ? sks[ks + 1] : m;
      const double dkn = ks + 1 < k1 ? sdinv[skk[ks + 1]] : 0.0;
      const int tgl = lane < m.z ? stg[m.w + lane] : 0;
      const double ukl = lane < m.z ? SF[m.y + 1 + lane] : 0.0;
      const double lik = w[m.x] * dk;
      __syncwarp();
      if (lane == 0) w[m.x] = lik;
      if (lane < m.z) w[tgl] -= lik * ukl;
      for (int t = lane + 32; t < m.z; t += 32) w[stg[m.w + t]] -= lik * SF[m.y + 1 + t];
      __syncwarp();
      m = mn;
      dk = dkn;
    }
    const double piv = w[rd.x];
    if (lane == 0) {
      const double di = fast_rcp(piv);
      sdinv[a] = di;
      f.dinv[rd.y] = di;
      if (!(fabs(piv) > f.pivtol * amax)) atomicMax(f.status, rd.y + 1);
      f.rowmax[rd.y] = amax;   // (rh_pivot_ratio: |u_kk| = 1 / |dinv| against it)
    }
    __syncwarp();
  };
  if (f.df) {
    // r02 (late): every row of the block in one dataflow pass - warp w takes rows
    // w, w + nw, ... in elimination order (pieces and tops alike) and applies its
    // k-steps in increasing k, each once row k is final (per-row done flags in shared
    // memory, acquire/release at CTA scope).  The static subtree-to-warp schedule left
    // the warps unbalanced (max 106k vs mean 71k cycles) and needed the two tops phases.
    __shared__ int s_rdone[kMaxRowsFact];
    for (int a = threadIdx.x; a < nr; a += blockDim.x) s_rdone[a] = 0;
    __syncthreads();
    for (int a = warp; a < nr; a += nw) {
      const int4 rm = s_rm[a];
      const int2 rd = s_rd[a];
      double *w = SF + rm.x;
      double amax = 0.0;
      for (int t = lane; t < rm.y; t += 32) amax = fmax(amax, fabs(w[t]));
      amax = warp_max(amax);
      for (int ks = rm.z; ks < rm.w; ++ks) {
        const int4 m = sks[ks];
        const int kl = skk[ks];
        const int tgl = lane < m.z ? stg[m.w + lane] : 0;
        while (ld_acquire_cta_shared(s_rdone + kl) == 0) {
        }
        const double dk = sdinv[kl];
        const double ukl = lane < m.z ? SF[m.y + 1 + lane] : 0.0;
        const double lik = w[m.x] * dk;
        __syncwarp();
        if (lane == 0) w[m.x] = lik;
        if (lane < m.z) w[tgl] -= lik * ukl;
        for (int t = lane + 32; t < m.z; t += 32) w[stg[m.w + t]] -= lik * SF[m.y + 1 + t];
        __syncwarp();
      }
      const double piv = w[rd.x];
      if (lane == 0) {
        const double di = fast_rcp(piv);
        sdinv[a] = di;
        f.dinv[rd.y] = di;
        if (!(fabs(piv) > f.pivtol * amax)) atomicMax(f.status, rd.y + 1);
        f.rowmax[rd.y] = amax;
      }
      __threadfence_block();
      __syncwarp();
      if (lane == 0) st_release_cta_shared(s_rdone + a, 1);
    }
  } else {
  for (int q = lv[warp]; q < lv[warp + 1]; ++q) eliminate(q);
  __syncthreads();
  if (prof) prof[2] = clock64();
  // tops (rows q in [tq0, tq1), ascending): T1, warp per tops row, applies the
  // k-steps from piece rows (final now; a piece row is never an ancestor of a
  // tops row, so these steps commute with the tops' own); T2 is right-looking
  // over the tops k ascending, one barrier per k: every warp takes the now
  // final pivot of row k and applies the (i, k) steps of its tops rows i > k.
  const int tq0 = lv[nw + 1], tq1 = lv[nw + 2], ntq = tq1 - tq0;
  if (ntq > 0) {
    __shared__ int s_cur[kMaxTopsFact];     // per tops row: next k-step with k in the tops
    __shared__ double s_amax[kMaxTopsFact];
    __shared__ int s_topq[kMaxTopsFact];    // block-local row of every tops row
    __shared__ int4 s_trow[kMaxTopsFact];   // per tops row: F row (global), smem row offset, pivot offset, k-steps end
    __shared__ unsigned char s_tflag[kMaxRowsFact];   // tops index + 1 by block-local row (0: not a tops row)
    __shared__ int s_tdone[kMaxTopsFact];              // T2: tops row final (dataflow flag)
    for (int a = threadIdx.x; a < nr; a += blockDim.x) s_tflag[a] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < ntq; t += blockDim.x) {
      s_topq[t] = s_ord[tq0 + t];
      s_tflag[s_topq[t]] = (unsigned char)(t + 1);
      s_tdone[t] = 0;
    }
    __syncthreads();
    auto is_top = [&](int kloc) { return s_tflag[kloc] != 0; };
    auto kstep = [&](double *w, int ks, double dk) {
      const int4 m = sks[ks];
      const double lik = w[m.x] * dk;
      __syncwarp();
      if (lane == 0) w[m.x] = lik;
      const double *uk = SF + m.y + 1;
      const unsigned short *tg = stg + m.w;
      for (int t = lane; t < m.z; t += 32) w[tg[t]] -= lik * uk[t];
      __syncwarp();
    };
    for (int t = warp; t < ntq; t += nw) {   // T1
      const int a = s_topq[t];
      const int4 rm = s_rm[a];
      const int off = rm.x, len = rm.y;
      double *w = SF + off;
      double amax = 0.0;
      for (int u = lane; u < len; u += 32) amax = fmax(amax, fabs(w[u]));
      amax = warp_max(amax);
      const int k1 = rm.w;
      int first_top = k1;
      for (int ks = rm.z; ks < k1; ++ks) {
        if (is_top(skk[ks])) {
          first_top = min(first_top, ks);
          continue;
        }
        kstep(w, ks, sdinv[skk[ks]]);
      }
      if (lane == 0) {
        s_cur[t] = first_top;
        s_amax[t] = amax;
        s_trow[t] = make_int4(s_rd[a].y, off, off + s_rd[a].x, k1);
      }
    }
    __syncthreads();
    if (prof) prof[3] = clock64();
    // T2, up-looking with dataflow flags (r02; right-looking with one CTA barrier per
    // tops row before): warp w takes tops rows t = w, w + nw, ...; row t applies its
    // k-steps on tops rows k in increasing k, each once row k is final, then forms
    // its pivot.  Every row receives the same updates in the same order as before.
    for (int t = warp; t < ntq; t += nw) {
      const int4 rt = s_trow[t];
      double *w = SF + rt.y;
      for (int ks = s_cur[t]; ks < rt.w; ++ks) {
        const int kt = (int)s_tflag[skk[ks]] - 1;   // tops index of k (-1: a piece row, applied in T1)
        if (kt < 0) continue;
        while (ld_acquire_cta_shared(s_tdone + kt) == 0) {
        }
        kstep(w, ks, sdinv[skk[ks]]);
      }
      const double piv = SF[rt.z];
      const double dk = fast_rcp(piv);
      if (lane == 0) {
        sdinv[s_topq[t]] = dk;
        f.dinv[rt.x] = dk;
        if (!(fabs(piv) > f.pivtol * s_amax[t])) atomicMax(f.status, rt.x + 1);
        f.rowmax[rt.x] = s_amax[t];
      }
      __threadfence_block();
      __syncwarp();
      if (lane == 0) st_release_cta_shared(s_tdone + t, 1);
    }
  }
  }
  __syncthreads();
  if (prof) prof[4] = clock64();
  for (int a = threadIdx.x; a < nr; a += blockDim.x) {   // write back: thread per row
    const int i = f.row_global[r0 + a];
    const int off = f.fo[fb + a], len = f.fo[fb + a + 1] - off, rb = f.F_rowptr[i];
    for (int t = 0; t < len; ++t) f.F_val[rb + t] = SF[off + t];
  }
}

// R_B1: the separator rows' updates from block columns (rows of blocks are
// final); afterwards the separator x separator entries hold the Schur
// complement.  A warp per separator row, the row staged in shared memory (max row
// length f.sep_maxlen), its k-steps against the block columns in order; each
// step's U row values and target offsets (<= 32 of them: one per lane) are
// loaded one step ahead, so only the shared-memory multiplier stays on the
// chain (r02: the row lived in global memory, one L2 round trip per step).
// per-warp staging of k_fact_sep_rows: the row, its k-steps' U values, their targets (uint16)
__host__ __device__ inline size_t sep_warp_doubles(int maxlen, int maxu) {
  return (size_t)maxlen + (size_t)maxu + ((size_t)maxu + 3) / 4;
}
__global__ void __launch_bounds__(kThreads) k_fact_sep_rows(FactParams f) {
  extern __shared__ double fsr[];   // per warp: [sep_maxlen] row, [sep_maxu] U values, [sep_maxu] targets
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int a = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (a >= f.ns) return;
  const int q = f.seg_row_off[f.nblk] + a;
  const int i = f.row_global[q];
  const int rb = f.F_rowptr[i], re = f.F_rowptr[i + 1], len = re - rb;
  double *ws = fsr + (size_t)wl * sep_warp_doubles(f.sep_maxlen, f.sep_maxu);
  double *uv = ws + f.sep_maxlen;
  unsigned short *tg = reinterpret_cast<unsigned short *>(uv + f.sep_maxu);
  const int4 *gks = reinterpret_cast<const int4 *>(f.ks4);
  const int k0 = f.ks_ptr[q], k1 = f.ks_ptr[q + 1];
  // r02 (late): everything the row's k-steps read is staged before the chain starts -
  // the row, every step's U values (cp.async, all in flight; a step's values sit at its
  // target offset, the row's targets being contiguous) and the targets - so the chain of
  // up to 59 steps runs from shared memory (a register prefetch ring still waited on L2)
  const int tb = k0 < k1 ? gks[k0].w : 0;
  for (int c0 = k0; c0 < k1; c0 += 32) {
    const int nc = min(32, k1 - c0);
    const int4 mv = lane < nc ? gks[c0 + lane] : make_int4(0, 0, 0, 0);
    for (int st = 0; st < nc; ++st) {
      const int my = __shfl_sync(0xffffffffu, mv.y, st), mz = __shfl_sync(0xffffffffu, mv.z, st);
      const int mw = __shfl_sync(0xffffffffu, mv.w, st);
      for (int j = lane; j < mz; j += 32) {
        const unsigned d = (unsigned)__cvta_generic_to_shared(uv + (mw - tb) + j);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(f.F_val + my + 1 + j) : "memory");
      }
    }
  }
  if (k1 > k0) {
    const int4 ml = gks[k1 - 1];
    for (int e = lane; e < ml.w + ml.z - tb; e += 32) tg[e] = f.tgt16[tb + e];
  }
  double amax = 0.0;
  for (int e = lane; e < len; e += 32) {
    const double v = f.F_val[rb + e];
    ws[e] = v;
    amax = fmax(amax, fabs(v));
  }
  amax = warp_max(amax);
  if (lane == 0) f.rowmax[i] = amax;
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncwarp();
  for (int c0 = k0; c0 < k1; c0 += 32) {
    const int nc = min(32, k1 - c0);
    const int4 mv = lane < nc ? gks[c0 + lane] : make_int4(0, 0, 0, 0);
    const double dv = lane < nc ? f.dinv[f.ks_k[c0 + lane]] : 0.0;
    for (int st = 0; st < nc; ++st) {
      const int mx = __shfl_sync(0xffffffffu, mv.x, st), mz = __shfl_sync(0xffffffffu, mv.z, st);
      const int mo = __shfl_sync(0xffffffffu, mv.w, st) - tb;
      const double dk = __shfl_sync(0xffffffffu, dv, st);
      const double lik = ws[mx] * dk;
      __syncwarp();
      if (lane == 0) ws[mx] = lik;
      for (int j = lane; j < mz; j += 32) ws[tg[mo + j]] -= lik * uv[mo + j];
      __syncwarp();
    }
  }
  for (int e = lane; e < len; e += 32) f.F_val[rb + e] = ws[e];
}

// ----------------------------------------------------------------------------
// Separator block: after R_B1 the separator rows' separator-column entries hold
// the Schur complement S = A_ss - L_sb U_bs.  It is densified and inverted in
// place by blocked Gauss-Jordan elimination with static (diagonal) pivots, the
// same pivots the up-looking factorization would use (R15): the
// separator's ~100-level triangular chains then become one dense product per
// batch (k_sep_gemm).  Panel width GJB; one persistent launch (k_sep_inverse).
// ----------------------------------------------------------------------------
constexpr int GJB = 32;

__global__ void k_sep_dense(int nslots, const int *__restrict__ src, const int *__restrict__ dpos,
                            const double *__restrict__ F, double *S) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nslots) S[dpos[t]] = F[src[t]];
}



// Blocked Gauss-Jordan inverse of the dense separator block S in ONE
// persistent cooperative launch (replaces 2 launches per panel).  Per panel K
// (width GJB) every CTA inverts the panel's diagonal block D itself (warp 0,
// registers; static pivots checked against the row's original max) while its
// other warps stage C = S[tile rows, K], P = S[K, tile cols] and T = S[tile];
// then, for its 64 x 64 output tiles, R = D^-1 P (D^-1 on panel columns, with
// T := 0 there) and
//   S'[panel rows] = R,   S'[other rows] = T - C R
// which is the block GJ step [D B; C E] -> [D^-1, D^-1 B; -C D^-1, E - C D^-1 B].
// S' is written to the other buffer (ping-pong), one grid barrier per panel.
constexpr int GJT = 64;   // output tile
constexpr size_t gj_smem_bytes() { return sizeof(double) * (GJB * (GJB + 1) + (3 * GJB + GJT) * (GJT + 1)); }
__global__ void __launch_bounds__(256, 1) k_sep_inverse(double *Sa, double *Sb, int ns, const double *rowmax,
                                                     const int *sep_rows, int *status, double pivtol,
                                                     unsigned *bar, long long *dbg, double *dbuf, int gj_warps,
                                                     double *seppiv) {
  extern __shared__ double gj_sm[];   // dynamic: gj_smem_bytes()
  double(*Ds)[GJB + 1] = reinterpret_cast<double(*)[GJB + 1]>(gj_sm);
  double(*Cs)[GJT + 1] = reinterpret_cast<double(*)[GJT + 1]>(gj_sm + GJB * (GJB + 1));   // C^T: Cs[m][r] = S[i0 + r][K + m]
  double(*Rs)[GJT + 1] = Cs + GJB;                                                     // P, then R
  double(*Ts)[GJT + 1] = Rs + GJB;
  double(*R2)[GJT + 1] = Ts + GJT;   // R = D^-1 P
  const int tid = threadIdx.x;
  const int nt = (ns + GJT - 1) / GJT, ntiles = nt * nt;
  unsigned gen = 0;   // barrier phase (bar[0] zeroed by the host before the launch)
  double *Sin = Sa, *Sout = Sb;
  __shared__ double prow[2][GJB];
  const int warp = tid >> 5, lane = tid & 31;
  // stage C^T, P and T (T := 0 on the panel columns) of one output tile; `t0`,
  // `nthr`: the participating threads.  Batches of 16 loads in flight per thread.
  auto load_tile = [&](const double *Sin, int K, int b, int i0, int j0, int t0, int nthr) {
    // one pass issues a thread's C, P and T loads together (all in flight: one L2
    // round trip per pass; 256 threads: one pass)
    constexpr int NB = 8;
    for (int base = t0; base < GJT * GJB; base += NB * nthr) {
      double va[NB], vb[NB], vt[2 * NB];
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        const int t = base + q * nthr;
        const int r = t / GJB, m = t % GJB, m2 = t / GJT, c = t % GJT;
        va[q] = (t < GJT * GJB && i0 + r < ns && m < b) ? __ldcg(Sin + (long long)(i0 + r) * ns + K + m) : 0.0;
        vb[q] = (t < GJT * GJB && m2 < b && j0 + c < ns) ? __ldcg(Sin + (long long)(K + m2) * ns + j0 + c) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 2 * NB; ++q) {   // T: twice the elements, the same passes
        const int t = 2 * (base - t0) + t0 + q * nthr, r = t / GJT, c = t % GJT;
        const bool inJ = j0 + c >= K && j0 + c < K + b;
        vt[q] = (t < GJT * GJT && i0 + r < ns && j0 + c < ns && !inJ) ? __ldcg(Sin + (long long)(i0 + r) * ns + j0 + c) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        const int t = base + q * nthr;
        if (t < GJT * GJB) {
          Cs[t % GJB][t / GJB] = va[q];
          Rs[t / GJT][t % GJT] = vb[q];
        }
      }
#pragma unroll
      for (int q = 0; q < 2 * NB; ++q) {
        const int t = 2 * (base - t0) + t0 + q * nthr;
        if (t < GJT * GJT) Ts[t / GJT][t % GJT] = vt[q];
      }
    }
  };
  long long *prof = (dbg && tid == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)) ? dbg + (blockIdx.x ? 512 : 0) : nullptr;
  // Gauss-Jordan inverse of the 32 x 32 block Dsrc (smem, row stride GJB + 1)
  // into Ds by warps 0-3: thread = (rows 8w..8w+7, column lane); the pivot row
  // goes through shared memory, the pivot column by shuffles; static pivots
  // checked against the separator rows' original max (rows K0 ..)
  // (NW warps: thread = (rows (32/NW) w .., column lane), named barrier 1)
  auto invert32 = [&](const double *Dsrc, int lds, int K0, int bb, bool report, auto nwc) {
    constexpr int NW = decltype(nwc)::value, RPT = GJB / NW;
    const int j = lane;
    double v[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = RPT * warp + r;
      v[r] = (i < bb && j < bb) ? Dsrc[i * lds + j] : (i == j ? 1.0 : 0.0);
    }
    bool bad = false;
#pragma unroll
    for (int k = 0; k < GJB; ++k) {
      const int wk = k / RPT, kk = k % RPT;
      if (warp == wk) prow[k & 1][j] = v[kk];
      double f[RPT];
#pragma unroll
      for (int r = 0; r < RPT; ++r) f[r] = __shfl_sync(0xffffffffu, v[r], k);
      asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
      const double pk = prow[k & 1][k];
      const double inv = fast_rcp(pk);
      const double rk = j == k ? inv : prow[k & 1][j] * inv;
      if (warp == wk && j == k && k < bb && !(fabs(pk) > pivtol * rowmax[sep_rows[K0 + k]])) bad = true;
      if (report && warp == wk && j == k && k < bb) seppiv[K0 + k] = pk;   // (rh_pivot_ratio)
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int i = RPT * warp + r;
        v[r] = i == k ? rk : (j == k ? -f[r] * inv : fma(-f[r], rk, v[r]));
      }
    }
    if (bad && report) atomicMax(status, sep_rows[K0 + j] + 1);
    asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");   // every warp has read Dsrc before Ds is written
#pragma unroll
    for (int r = 0; r < RPT; ++r) Ds[RPT * warp + r][j] = v[r];
  };
  using W2 = std::integral_constant<int, 2>;
  using W4 = std::integral_constant<int, 4>;
  using W8 = std::integral_constant<int, 8>;
  const bool helper = blockIdx.x == gridDim.x - 1;   // lookahead CTA: the next panel's D^-1
  const int ntcta = gridDim.x - 1;                   // tile CTAs
  for (int K = 0; K < ns; K += GJB) {
    const int b = min(GJB, ns - K);
    if (prof) prof[(K / GJB) * 4] = clock64();   // timing experiment (RH_DEBUG & 16)
    if (helper) {
      // panel 0: D_0^-1 first; then D'_{K+1} = S[K1,K1] - S[K1,K] D_K^-1 S[K,K1] (S = state after
      // panel K-1, what the tiles read now), inverted into Ds and published in dbuf for panel K+1.
      // The lookahead CTA is not part of the tiles' barrier: it waits for the tiles' panel
      // K-1 (the arrival counter) and publishes D_{K+1}^-1 with a flag (bar[1]), so the
      // tiles of panel K+1 start as soon as both their panel K and D_{K+1}^-1 are done.
      if (K > 0 && tid == 0) {
        const unsigned target = (unsigned)(K / GJB) * ntcta;
        while ((int)((unsigned)ld_acquire(reinterpret_cast<const int *>(bar)) - target) < 0) {
        }
        __threadfence();
      }
      __syncthreads();
      if (K == 0) {
        for (int t = tid; t < GJB * GJB; t += blockDim.x) {
          const int i = t / GJB, c = t % GJB;
          Ts[i][c] = (i < b && c < b) ? __ldcg(Sin + (long long)i * ns + c) : 0.0;
        }
        __syncthreads();
        invert32(&Ts[0][0], GJT + 1, 0, b, false, W8{});
        __syncthreads();
      }
      const int K1 = K + GJB, b1 = min(GJB, ns - K1);
      if (b1 > 0) {
        {   // Cs = S[K1,K], Rs = S[K,K1], Ts = S[K1,K1]: all 12 loads per thread in flight
          double vc[4], vr[4], vt[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int t = tid + u * 256, i = t / GJB, c = t % GJB;
            vc[u] = (i < b1 && c < b) ? __ldcg(Sin + (long long)(K1 + i) * ns + K + c) : 0.0;
            vr[u] = (i < b && c < b1) ? __ldcg(Sin + (long long)(K + i) * ns + K1 + c) : 0.0;
            vt[u] = (i < b1 && c < b1) ? __ldcg(Sin + (long long)(K1 + i) * ns + K1 + c) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int t = tid + u * 256, i = t / GJB, c = t % GJB;
            Cs[i][c] = vc[u];
            Rs[i][c] = vr[u];
            Ts[i][c] = vt[u];
          }
        }
        __syncthreads();
        // the two 32 x 32 x 32 products: thread = column c, rows i0 + 8u; each of its
        // four outputs in four partial chains over l mod 4 (16 FMA chains of 8 in
        // flight), added in a fixed order
        constexpr int NU = GJB * GJB / 256;
        {   // R2 = D_K^-1 S[K,K1]
          const int c = tid % GJB, i0 = tid / GJB;
          double acc[NU][4];
#pragma unroll
          for (int u = 0; u < NU; ++u)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[u][q] = 0.0;
#pragma unroll
          for (int l = 0; l < GJB; ++l) {
            const double r = Rs[l][c];
#pragma unroll
            for (int u = 0; u < NU; ++u) acc[u][l & 3] = fma(Ds[i0 + 8 * u][l], r, acc[u][l & 3]);
          }
#pragma unroll
          for (int u = 0; u < NU; ++u) R2[i0 + 8 * u][c] = (acc[u][0] + acc[u][1]) + (acc[u][2] + acc[u][3]);
        }
        __syncthreads();
        {   // Ts = S[K1,K1] - S[K1,K] R2
          const int c = tid % GJB, i0 = tid / GJB;
          double acc[NU][4];
#pragma unroll
          for (int u = 0; u < NU; ++u)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[u][q] = 0.0;
#pragma unroll
          for (int l = 0; l < GJB; ++l) {
            const double r = R2[l][c];
#pragma unroll
            for (int u = 0; u < NU; ++u) acc[u][l & 3] = fma(Cs[i0 + 8 * u][l], r, acc[u][l & 3]);
          }
#pragma unroll
          for (int u = 0; u < NU; ++u)
            Ts[i0 + 8 * u][c] -= (acc[u][0] + acc[u][1]) + (acc[u][2] + acc[u][3]);
        }
        __syncthreads();
        if (prof) prof[(K / GJB) * 4 + 1] = clock64();
        {   // experiment (RH_GJW): warps of the lookahead's inverse
          const int gw = gj_warps;
          if (gw == 2) {
            if (warp < 2) invert32(&Ts[0][0], GJT + 1, K1, b1, true, W2{});
          } else if (gw == 4) {
            if (warp < 4) invert32(&Ts[0][0], GJT + 1, K1, b1, true, W4{});
          } else {
            invert32(&Ts[0][0], GJT + 1, K1, b1, true, W8{});
          }
        }
        __syncthreads();
        double *db = dbuf + ((K1 / GJB) & 1) * GJB * GJB;
        for (int t = tid; t < GJB * GJB; t += blockDim.x) __stcg(db + t, Ds[t / GJB][t % GJB]);
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          st_release(reinterpret_cast<int *>(bar + 1), K1 / GJB);   // D_{K+1}^-1 published
        }
      }
    } else {
      if (K == 0) {   // panel 0: D_0^-1 locally (warps 0-3) while warps 4-7 stage the first tile
        if (warp < 4) {
          for (int t = tid; t < GJB * GJB; t += 128) {
            const int i = t / GJB, c = t % GJB;
            Ds[i][c] = (i < b && c < b) ? __ldcg(Sin + (long long)i * ns + c) : (i == c ? 1.0 : 0.0);
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          invert32(&Ds[0][0], GJB + 1, 0, b, blockIdx.x == 0, W4{});
        } else if (blockIdx.x < ntiles) {
          load_tile(Sin, K, b, (blockIdx.x / nt) * GJT, (blockIdx.x % nt) * GJT, tid - 128, 128);
        }
      } else {        // the helper's D_K^-1 (loads in flight while the first tile's are issued)
        if (tid == 0)
          while (ld_acquire(reinterpret_cast<const int *>(bar + 1)) < K / GJB) {
          }
        __syncthreads();
        const double *db = dbuf + ((K / GJB) & 1) * GJB * GJB;
        double dv[GJB * GJB / 256];
#pragma unroll
        for (int u = 0; u < GJB * GJB / 256; ++u) dv[u] = __ldcg(db + tid + 256 * u);
        if (blockIdx.x < ntiles)
          load_tile(Sin, K, b, (blockIdx.x / nt) * GJT, (blockIdx.x % nt) * GJT, tid, blockDim.x);
#pragma unroll
        for (int u = 0; u < GJB * GJB / 256; ++u) {
          const int t = tid + 256 * u;
          Ds[t / GJB][t % GJB] = dv[u];
        }
      }
    }
    for (int tile = helper ? ntiles : (int)blockIdx.x; tile < ntiles; tile += ntcta) {
      const int i0 = (tile / nt) * GJT, j0 = (tile % nt) * GJT;
      if (tile != (int)blockIdx.x) load_tile(Sin, K, b, i0, j0, tid, blockDim.x);
      __syncthreads();   // Ds (first tile), Cs, Rs = P, Ts
      if (prof && tile == (int)blockIdx.x) prof[(K / GJB) * 4 + 1] = clock64();
      {  // R = D^-1 P (D^-1 itself on panel columns): thread = 4 rows x 2 columns
        const int cg = tid & 31, rg = tid >> 5;
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int c = cg + 32 * h2, gj = j0 + c;
          double acc[4];
          if (gj >= K && gj < K + b) {
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[v] = Ds[rg + 8 * v][gj - K];
          } else {
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[v] = 0.0;
#pragma unroll 8
            for (int l = 0; l < GJB; ++l) {
              const double r = Rs[l][c];
#pragma unroll
              for (int v = 0; v < 4; ++v) acc[v] = fma(Ds[rg + 8 * v][l], r, acc[v]);
            }
          }
#pragma unroll
          for (int v = 0; v < 4; ++v) R2[rg + 8 * v][c] = acc[v];
        }
      }
      __syncthreads();
      const int tx = tid % 16, ty = tid / 16;
      double acc[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = Ts[ty + 16 * u][tx + 16 * v];
#pragma unroll 4
      for (int m = 0; m < GJB; ++m) {
        double cv[4], rv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) cv[u] = Cs[m][ty + 16 * u];
#pragma unroll
        for (int v = 0; v < 4; ++v) rv[v] = R2[m][tx + 16 * v];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fma(-cv[u], rv[v], acc[u][v]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int gi = i0 + ty + 16 * u;
        if (gi >= ns) continue;
        const bool inI = gi >= K && gi < K + b;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int gj = j0 + tx + 16 * v;
          if (gj < ns) __stcg(Sout + (long long)gi * ns + gj, inI ? R2[gi - K][tx + 16 * v] : acc[u][v]);
        }
      }
      __syncthreads();
    }
    if (prof) prof[(K / GJB) * 4 + 2] = clock64();
    if (!helper) grid_barrier_n(bar, gen, ntcta);   // the tile CTAs only (see the lookahead CTA)
    if (prof) prof[(K / GJB) * 4 + 3] = clock64();
    double *t = Sin;
    Sin = Sout;
    Sout = t;
  }
}

__global__ void k_transpose(const double *__restrict__ A, double *AT, int n) {
  __shared__ double tile[32][33];
  const int x = blockIdx.x * 32 + threadIdx.x, y0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y)
    if (x < n && y0 + r < n) tile[r][threadIdx.x] = A[(long long)(y0 + r) * n + x];
  __syncthreads();
  const int xo = blockIdx.y * 32 + threadIdx.x, yo0 = blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y)
    if (xo < n && yo0 + r < n) AT[(long long)(yo0 + r) * n + xo] = tile[threadIdx.x][r];
}

// Dense inverses of every block's top diagonal block T x T (once per state):
// M_L = (L_TT)^-1 (unit lower) and M_U = (U_TT)^-1, written as dense 32 x 32
// blocks (row stride kTopLd, zero beyond T) for the tops' DMMA product in
// k_blk: L gets M_L, U^T M_U^T, U M_U, L^T M_L^T.  One CTA per block, thread per
// entry (a, b) of each inverse: column-oriented (right-looking) substitution,
// one barrier per step:
//   M_L: for k ascending, M[a][b] -= T[a][k] M[k][b] for a > k (M starts at I);
//   M_U: for k descending, M[k][b] /= T[k][k], then M[a][b] -= T[a][k] M[k][b] for a < k.
constexpr int kMaxTops = 32;
constexpr int kTopLd = 36;   // row stride (doubles) of a block's dense tops inverse: conflict-free DMMA A fragments
__global__ void __launch_bounds__(kMaxTops * kMaxTops) k_tops_inverse(const int *top_ptr, const int *top_fpos_ptr,
                                                                     const int *top_fpos, const double *F, double *dL,
                                                                     double *dUt, double *dU, double *dLt) {
  __shared__ double T[kMaxTops][kMaxTops + 1];   // L_TT below the diagonal, U_TT on/above
  __shared__ double ML[kMaxTops][kMaxTops + 1], MU[kMaxTops][kMaxTops + 1];
  const int s = blockIdx.x;
  const int t0 = top_ptr[s], nt = top_ptr[s + 1] - t0;
  const int a = threadIdx.x / kMaxTops, b = threadIdx.x % kMaxTops;
  const bool in = a < nt && b < nt;
  ML[a][b] = MU[a][b] = a == b && a < nt ? 1.0 : 0.0;
  if (in) {
    const int pos = top_fpos[top_fpos_ptr[s] + a * nt + b];
    T[a][b] = pos >= 0 ? F[pos] : 0.0;
  }
  __syncthreads();
  for (int k = 0; k < nt; ++k) {   // M_L (unit lower); M_L[a][b] is final for a <= k
    if (in && a > k) ML[a][b] -= T[a][k] * ML[k][b];
    __syncthreads();
  }
  for (int k = nt - 1; k >= 0; --k) {   // M_U (upper): row k is final after its division
    if (in && a == k) MU[k][b] /= T[k][k];
    __syncthreads();
    if (in && a < k) MU[a][b] -= T[a][k] * MU[k][b];
    __syncthreads();
  }
  const size_t o = (size_t)s * 32 * kTopLd + a * kTopLd + b;
  dL[o] = ML[a][b];
  dUt[o] = MU[b][a];
  dU[o] = MU[a][b];
  dLt[o] = ML[b][a];
}

// G_p entry records of the L sweep's right-hand side (per state): value, then
// the tile-row byte offset and the p column packed into the second double
__global__ void k_gather_gpe(int n, const int *__restrict__ src, const int *__restrict__ row,
                             const int *__restrict__ pcol, const double *__restrict__ gp_val, double2 *rec) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n)
    rec[i] = make_double2(gp_val[src[i]],
                          __longlong_as_double((long long)(unsigned)row[i] | ((long long)pcol[i] << 32)));
}

// copy factor values into the sweep value arrays (entry order of the sweeps)
// entry slots of the per-block epilogue run records: (coefficient, tile byte offset)
__global__ void k_sr_fill(int n, const int *__restrict__ slot, const int *__restrict__ src,
                          const int *__restrict__ trow, const double *__restrict__ val, double2 *rec) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) rec[slot[k]] = make_double2(val[src[k]], __longlong_as_double((long long)trow[k]));
}

__global__ void k_gather_vals(int n, const int *__restrict__ src, const double *__restrict__ F, double *dst) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) dst[e] = src[e] >= 0 ? F[src[e]] : 0.0;   // src < 0: padding entry
}
// unit-sweep record values: src >= 0: F[src]; -1: 0; <= -2: 1 / F[-src - 2]
__global__ void k_gather_code(int n, const int *__restrict__ src, const double *__restrict__ F, double *dst) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int c = src[e];
  dst[e] = c >= 0 ? F[c] : c == -1 ? 0.0 : 1.0 / F[-c - 2];
}

// ============================================================================
// batched triangular sweeps over elimination-tree segments (SURVEY.md
// 8(a)-6, 8(a)-8).  One CTA = (segment, chunk of C columns).  The segment's
// rows x C columns live in shared memory for the whole sweep; dependencies
// outside the segment (separator rows for a block's backward sweep, block
// rows for the separator's forward sweep) are read from HBM/L2.  Each level
// of the segment is one CTA barrier; each row is C lanes (one per column),
// so the coefficient and index loads are warp-uniform broadcasts and the
// shared-memory gathers are contiguous.
// ============================================================================

__device__ __forceinline__ double load_W(const SegParams &h, int row, int col) {
  if (col >= h.N) return 0.0;
  if (h.icol) return row == __ldg(h.icol + col) ? 1.0 : 0.0;
  return h.W[(long long)row * h.ldw + col];
}

__device__ __forceinline__ long long hw_index(const SegParams &h, int row, int col) {
  const int c = h.icol ? __ldg(h.icol + col) - h.icol_base : col;
  return h.transposed ? (long long)c * h.ldhw + row : (long long)row * h.ldhw + c;
}

// chunk ci (32 columns) of block s has a nonzero right-hand side -G_p W
__device__ __forceinline__ bool tile_live(const SegParams &h, int s, int ci) {
  return !h.tmask || ((__ldg(h.tmask + s * h.tmask_words + (ci >> 5)) >> (ci & 31)) & 1u);
}

// Cartesian batch plan (full Hessian).  For W = I[:, lo:hi],
// B = G_p W is very sparse: column j touches only the blocks
// holding rows of G_p's column j (bus j's rows and, for a voltage parameter,
// its neighbours'), and a block's L sweep (which depends on nothing outside the
// block) is identically zero for every other column.  The batch's columns are
// taken in `gorder` order (all p columns sorted by their first touched block,
// then index), so each block's columns are contiguous and its nonzero L-sweep
// tiles are one or two 32-column chunks; `mask` records them.  One CTA; the
// per-column arithmetic does not depend on the order (results are bitwise
// those of the natural order).
__global__ void __launch_bounds__(1024) k_batch_plan(int n_p, int lo, int hi, const int *__restrict__ gorder,
                                                     const int *__restrict__ pcb_ptr, const int *__restrict__ pcb,
                                                     int nblk, int words, int *cols, unsigned *mask, int nch,
                                                     int *tlist) {
  __shared__ int wsum[32];
  __shared__ int base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < nblk * words; i += blockDim.x) mask[i] = 0u;
  if (tid == 0) base = 0;
  __syncthreads();
  for (int i0 = 0; i0 < n_p; i0 += blockDim.x) {
    const int i = i0 + tid;
    const int j = i < n_p ? gorder[i] : -1;
    const bool in = j >= lo && j < hi;
    const unsigned bal = __ballot_sync(0xffffffffu, in);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      int v = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
      }
      wsum[lane] = v;
    }
    __syncthreads();
    if (in) {
      const int pos = base + (warp ? wsum[warp - 1] : 0) + __popc(bal & ((1u << lane) - 1u));
      cols[pos] = j;
      for (int e = pcb_ptr[j]; e < pcb_ptr[j + 1]; ++e)
        atomicOr(mask + pcb[e] * words + (pos >> 10), 1u << ((pos >> 5) & 31));
    }
    __syncthreads();
    if (tid == 0) base += wsum[31];
    __syncthreads();
  }
  // the live tiles as a list (count, then block << 16 | chunk): the sparse L and
  // U0 sweeps take tickets over these only
  __threadfence_block();
  if (tid == 0) base = 0;
  __syncthreads();
  for (int i0 = 0; i0 < nblk * nch; i0 += blockDim.x) {
    const int i = i0 + tid, sb = i / max(nch, 1), ci = i - sb * nch;
    const bool in = i < nblk * nch && ((__ldcg(mask + sb * words + (ci >> 5)) >> (ci & 31)) & 1u);
    const unsigned bal = __ballot_sync(0xffffffffu, in);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      int v = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
      }
      wsum[lane] = v;
    }
    __syncthreads();
    if (in) tlist[1 + base + (warp ? wsum[warp - 1] : 0) + __popc(bal & ((1u << lane) - 1u))] = sb << 16 | ci;
    __syncthreads();
    if (tid == 0) base += wsum[31];
    __syncthreads();
  }
  if (tid == 0) tlist[0] = base;
}

constexpr int kSegC = 32;   // columns of the single-RHS (lambda) path

enum : int {
  MODE_L = 0,     // blocks:    rhs = -G_p W (SpMul fused), L sweep            -> Z
  MODE_LU = 1,    // separator: rhs = -G_p W - L_sb Z_b, then S^-1             -> Z
  MODE_U = 2,     // blocks:    U sweep                                        -> Z
  MODE_UT = 3,    // blocks:    U^T sweep on -Y_x                              -> P
  MODE_UTLT = 4,  // separator: -Y_x - U_bs^T P_b, then S^-T                   -> P
  MODE_LT = 5,    // blocks:    L^T sweep                                      -> P = Psi
  MODE_LX = 6,    // blocks:    L sweep, right-hand side loaded from Z (Newton)   -> Z
  MODE_LUX = 7    // separator: rhs from Z - L_sb Z_b (Newton), then S^-1        -> Z
};

__device__ __forceinline__ double rhs_gpw(const SegParams &h, int row, int col) {
  double v = 0.0;
  for (int e = h.gp_rptr[row]; e < h.gp_rptr[row + 1]; ++e) v -= h.gp_val[e] * load_W(h, h.gp_col[e], col);
  return v;
}

// ----------------------------------------------------------------------------
// Block sweeps by bus units.
// Persistent: two CTAs per SM take tickets from a global counter, heaviest
// blocks first; a ticket is one block x two 32-column chunks, the block's unit
// schedule staged once (TMA bulk copies) and the chunks' block rows moved by 2D
// TMA boxes.  While one CTA waits on its copies the other's sweep uses the SM
// (DESIGN.md "Block sweeps").  Lanes own
// columns; a warp walks its pieces' units without synchronization; a unit is
// the 1 or 2 rows of one bus, so every dependency value read from shared
// memory feeds both rows (half the shared-memory wavefronts per FMA of a
// row-by-row sweep).  The tops (a dense chain at the top of the block) are
// applied as a dense product with their inverse (k_tops_inverse).
// ----------------------------------------------------------------------------
constexpr int kBC = UnitSweep::kCols;   // columns per tile: one per lane
constexpr int kRowB = kBC * 8;           // bytes per tile row

struct UStage {
  const int4 *meta;
  const double *topM;    // [32][kTopLd] dense tops inverse of this sweep
  const int *toprow;     // [32] tile rows of the tops
  const int *lvl;
  // 32-bit shared-window addresses of the hot loop (no generic -> shared
  // conversions per access): X + lane * 8, unit records, dependency offsets
  unsigned xs, rec, doff;
};

// shared-memory accesses of the unit sweeps by 32-bit shared addresses.  All
// are volatile asm: they keep program order among themselves, which orders a
// unit's result stores before the loads of later units that read them.
__device__ __forceinline__ double ldsd(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double2 ldsd2(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ int4 ldsi4(unsigned a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ int ldsi(unsigned a) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void stsd(unsigned a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

// Unit meta (int4, UnitSweep): x = first row's tile byte offset, y = second
// row's, z = first record's byte offset, w = dependency offsets' byte offset |
// ndeps << 16 | two rows << 30 | paired with next << 31.  Dependencies come in
// slots of two (lists padded to an even count): slot = one int4 of tile-row
// byte offsets (o0, o1 of dependency 2k, then of 2k + 1) and two (one-row unit)
// or four (two-row unit) double2 coefficient records.
__device__ __forceinline__ int unit_nd(const int4 m) { return (m.w >> 16) & 0x1fff; }
__device__ __forceinline__ int unit_ns(const int4 m) { return unit_nd(m) >> 1; }
__device__ __forceinline__ bool unit_two(const int4 m) { return (m.w >> 30) & 1; }

// sf = sum c_f x, ss = sum c_s x over ns >= 1 slots.  Chains: dependency 2k ->
// (f0, f1), 2k + 1 -> (f2, f3) (and s); slot 0 starts them (products, no zero
// fill), fixed order (deterministic).
template <bool TWO>
__device__ __forceinline__ void dep_one(const UStage &t, unsigned rc, unsigned of, double &sf, double &ss) {
  int2 o;
  asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(o.x), "=r"(o.y) : "r"(of));
  const double2 p0 = ldsd2(rc), q0 = TWO ? ldsd2(rc + 16) : p0;
  const double x00 = ldsd(t.xs + o.x), x01 = ldsd(t.xs + o.y);
  sf = fma(p0.x, x00, fma(p0.y, x01, sf));
  if (TWO) ss = fma(q0.x, x00, fma(q0.y, x01, ss));
}
// a list of nd >= 1 dependencies: slots of two, then an odd last one alone
template <bool TWO>
__device__ __forceinline__ void dep_list(const UStage &t, unsigned rc, unsigned of, int nd, double &sf, double &ss);
template <bool TWO>
__device__ __forceinline__ void dep_slots(const UStage &t, unsigned rc, unsigned of, int ns, double &sf, double &ss) {
  double f0, f1, f2, f3, s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  {
    const int4 o = ldsi4(of);
    const double2 p0 = ldsd2(rc), q0 = TWO ? ldsd2(rc + 16) : p0;
    const double2 p1 = ldsd2(rc + (TWO ? 32 : 16)), q1 = TWO ? ldsd2(rc + 48) : p1;
    const double x00 = ldsd(t.xs + o.x), x01 = ldsd(t.xs + o.y), x10 = ldsd(t.xs + o.z), x11 = ldsd(t.xs + o.w);
    f0 = p0.x * x00; f1 = p0.y * x01; f2 = p1.x * x10; f3 = p1.y * x11;
    if (TWO) { s0 = q0.x * x00; s1 = q0.y * x01; s2 = q1.x * x10; s3 = q1.y * x11; }
  }
#pragma unroll 1
  for (int k = 1; k < ns; ++k) {
    rc += TWO ? 64 : 32;
    of += 16;
    const int4 o = ldsi4(of);
    const double2 p0 = ldsd2(rc), q0 = TWO ? ldsd2(rc + 16) : p0;
    const double2 p1 = ldsd2(rc + (TWO ? 32 : 16)), q1 = TWO ? ldsd2(rc + 48) : p1;
    const double x00 = ldsd(t.xs + o.x), x01 = ldsd(t.xs + o.y), x10 = ldsd(t.xs + o.z), x11 = ldsd(t.xs + o.w);
    f0 = fma(p0.x, x00, f0); f1 = fma(p0.y, x01, f1); f2 = fma(p1.x, x10, f2); f3 = fma(p1.y, x11, f3);
    if (TWO) { s0 = fma(q0.x, x00, s0); s1 = fma(q0.y, x01, s1); s2 = fma(q1.x, x10, s2); s3 = fma(q1.y, x11, s3); }
  }
  sf = (f0 + f1) + (f2 + f3);
  ss = (s0 + s1) + (s2 + s3);
}
template <bool TWO>
__device__ __forceinline__ void dep_list(const UStage &t, unsigned rc, unsigned of, int nd, double &sf, double &ss) {
  const int ns = nd >> 1;
  sf = 0.0;
  ss = 0.0;
  if (ns) dep_slots<TWO>(t, rc, of, ns, sf, ss);
  if (nd & 1) dep_one<TWO>(t, rc + ns * (TWO ? 64 : 32), of + ns * 16, sf, ss);
}

// one piece unit: x_f = (x_f - sum) d_f ; x_s = (x_s - sum - c_sf x_f) d_s.
// A unit's own rows are written by nothing but the unit itself, so their
// right-hand sides are read first (they leave the dependency chain).  A
// forwarded dependency (meta bit 31) on the unit solved just before is taken
// from that unit's results (pf, ps) in registers, its records after the header;
// it is added after the list's sums.  Returns this unit's (x_f, x_s).
template <bool DINV>
__device__ __forceinline__ double2 unit_solve(const UStage &t, const int4 m, double pf, double ps) {
  const unsigned rc = t.rec + m.z, of = t.doff + (m.w & 0xffff);
  const int nd = unit_nd(m);
  const bool fw = m.w < 0;
  const double x0 = (m.w >> 29) & 1 ? ps : pf, x1 = (m.w >> 29) & 1 ? pf : ps;   // the forwarded pair
  const double2 hd = ldsd2(rc);
  if (unit_two(m)) {
    const double bf = ldsd(t.xs + m.x), bs = ldsd(t.xs + m.y);
    const double csf = ldsd(rc + 16);
    double sf = 0.0, ss = 0.0;
    if (nd) dep_list<true>(t, rc + (fw ? 64 : 32), of, nd, sf, ss);
    if (fw) {
      const double2 p = ldsd2(rc + 32), q = ldsd2(rc + 48);
      sf = fma(p.x, x0, fma(p.y, x1, sf));
      ss = fma(q.x, x0, fma(q.y, x1, ss));
    }
    double xf = bf - sf;
    if (DINV) xf *= hd.x;
    double xs = fma(-csf, xf, bs - ss);
    if (DINV) xs *= hd.y;
    stsd(t.xs + m.x, xf);
    stsd(t.xs + m.y, xs);
    return make_double2(xf, xs);
  } else {
    const double bf = ldsd(t.xs + m.x);
    double sf = 0.0, ss;
    if (nd) dep_list<false>(t, rc + (fw ? 32 : 16), of, nd, sf, ss);
    if (fw) {
      const double2 p = ldsd2(rc + 16);
      sf = fma(p.x, x0, fma(p.y, x1, sf));
    }
    double xf = bf - sf;
    if (DINV) xf *= hd.x;
    stsd(t.xs + m.x, xf);
    return make_double2(xf, xf);
  }
}

template <bool DINV>
__device__ __forceinline__ void unit_pieces(const UStage &t, int warp) {
  const int q0 = t.lvl[warp], q1 = t.lvl[warp + 1];
  int4 m = q0 < q1 ? t.meta[q0] : make_int4(0, 0, 0, 0);
  double2 x = make_double2(0.0, 0.0);   // the previous unit's results (forwarding)
#pragma unroll 1
  for (int u = q0; u < q1; ++u) {
    const int4 mn = u + 1 < q1 ? t.meta[u + 1] : m;
    x = unit_solve<DINV>(t, m, x.x, x.y);
    m = mn;
  }
}

// tops: t_T = X_T - (dependencies outside the tops), then X_T = M t_T with M
// the inverse of the tops' diagonal block (<= kMaxTopUnits units, two per warp).
constexpr int kBlkThreads = UnitSweep::kWarps * 32;
constexpr int kTopsLvl = UnitSweep::kWarps + 1;   // lvl[kWarps + 1], lvl[kWarps + 2]: tops units
static_assert(UnitSweep::kMaxTopUnits <= 2 * UnitSweep::kWarps, "two tops units per warp at most");
__device__ __forceinline__ void unit_tops(const UStage &t, const double *X, int warp, int lane) {
  const int u0 = t.lvl[kTopsLvl], u1 = t.lvl[kTopsLvl + 1];
  if (u0 >= u1) return;
  // the product's A fragments and B row offsets do not depend on X: loaded
  // before the gather, so the DMMA chain below waits on X loads only
  const int gid = lane >> 2, tig = lane & 3, mt = warp >> 1, nb = (warp & 1) * 2;
  double a[UnitSweep::kTopRows / 4];
  int br[UnitSweep::kTopRows / 4];
#pragma unroll
  for (int k = 0; k < UnitSweep::kTopRows / 4; ++k) {
    a[k] = t.topM[(mt * 8 + gid) * kTopLd + k * 4 + tig];
    br[k] = t.toprow[k * 4 + tig] * kBC + nb * 8 + gid;
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {   // gather: t_T = X_T - (dependencies outside the tops)
    const int u = u0 + warp + k * UnitSweep::kWarps;
    if (u < u1) {
      const int4 m = t.meta[u];
      const unsigned rc = t.rec + m.z, of = t.doff + (m.w & 0xffff);
      const int nd = unit_nd(m);
      if (!nd) continue;
      double sf, ss;
      if (unit_two(m)) {
        dep_list<true>(t, rc, of, nd, sf, ss);
        stsd(t.xs + m.x, ldsd(t.xs + m.x) - sf);
        stsd(t.xs + m.y, ldsd(t.xs + m.y) - ss);
      } else {
        dep_list<false>(t, rc, of, nd, sf, ss);
        stsd(t.xs + m.x, ldsd(t.xs + m.x) - sf);
      }
    }
  }
  __syncthreads();
  // X_T = M t_T: 32 x 32 (tops rows x tile columns) on the fp64 tensor cores;
  // warp = one 8-row tile x two 8-column tiles, k in steps of 4 (8 DMMA each)
  double b[UnitSweep::kTopRows / 4][2];
#pragma unroll
  for (int k = 0; k < UnitSweep::kTopRows / 4; ++k) {
    b[k][0] = X[br[k]];
    b[k][1] = X[br[k] + 8];
  }
  double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int k = 0; k < UnitSweep::kTopRows / 4; ++k) {
#pragma unroll
    for (int j = 0; j < 2; ++j) dmma_8x8x4(c[j][0], c[j][1], a[k], b[k][j]);
  }
  __syncthreads();
  const int nt = t.lvl[kTopsLvl + 2];   // tops rows
  if (mt * 8 + gid < nt) {
    double *xr = const_cast<double *>(X) + t.toprow[mt * 8 + gid] * kBC;
#pragma unroll
    for (int j = 0; j < 2; ++j)
      *reinterpret_cast<double2 *>(xr + (nb + j) * 8 + 2 * tig) = make_double2(c[j][0], c[j][1]);
  }
  __syncthreads();
}

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}

// right-hand side -G_p W of a block's rows (SpMul fused into the L sweep,
// PAPER.md:600) from the block's staged G_p entry records (value; tile-row
// byte offset | p column << 32), row ascending: a warp takes a range of whole
// rows and keeps a running sum, 8 W loads in flight (lane = column).  The
// same per-row order as rhs_gpw (CSR order): bitwise identical.
__device__ __forceinline__ void tile_rhs_entries(const SegParams &h, const double2 *er, int e0, int e1, int col,
                                                 double *Xl) {
  double acc = 0.0;
  int cur = -1;
  for (int e = e0; e < e1; e += 8) {
    double w[8], v[8];
    int ro[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double2 r = e + u < e1 ? er[e + u] : make_double2(0.0, 0.0);
      const long long m = __double_as_longlong(r.y);
      v[u] = r.x;
      ro[u] = e + u < e1 ? (int)(m & 0xffffffffll) : -2;
      w[u] = e + u < e1 ? load_W(h, (int)(m >> 32), col) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (ro[u] == -2) break;
      if (ro[u] != cur) {
        if (cur >= 0) Xl[cur / 8] = -acc;
        acc = 0.0;
        cur = ro[u];
      }
      acc = fma(v[u], w[u], acc);
    }
  }
  if (cur >= 0) Xl[cur / 8] = -acc;
}

// TMA bulk copies (cp.async.bulk) and their mbarrier
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(mbar))
               : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
// 2D TMA box copies of block rows of Z / P (tensor map in global memory): rows
// [r0, r0 + box) x columns [c0, c0 + 32) <-> a dense [box][32] tile in shared memory
__device__ __forceinline__ void tma2d_g2s(void *dst, const void *map, int c0, int r0, unsigned long long *mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(r0), "r"(smem_u32(mbar))
      : "memory");
}
// L2 prefetch of a box (no shared memory, no barrier): the next chunk's block rows
__device__ __forceinline__ void tma2d_prefetch_l2(const void *map, int c0, int r0) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map), "r"(c0), "r"(r0)
               : "memory");
}
__device__ __forceinline__ void tma2d_s2g(const void *map, int c0, int r0, const void *src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(c0),
               "r"(r0), "r"(smem_u32(src))
               : "memory");
}
constexpr int kTmaBig = 64, kTmaSmall = 8;   // box heights (rows) of the two maps of a pair
constexpr int kTmapBytes = 128;               // sizeof(CUtensorMap)

// Block sweeps (see above): 2 CTAs of 8 warps per SM, each sweeping one
// (block, 32-column) tile at a time taken from a global ticket counter
// (blocks in decreasing cost order); the tile and the block's unit schedule
// arrive by TMA bulk copies on one mbarrier, the result leaves by bulk stores.
// While one CTA waits on copies, barriers or a dependency chain, the other
// CTA's sweep uses the SM.
__global__ void __launch_bounds__(kBlkThreads, 2) k_blk(SegParams h, int mode) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) unsigned long long mbar;
  __shared__ int s_tk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool fwd = mode == MODE_L || mode == MODE_UT || mode == MODE_LX;
  // L^T sweep of a Cartesian batch: the schedule pruned to the Psi rows G_p^T Psi reads
  const DUnit &U = fwd ? h.uf : mode == MODE_LT && h.icol ? h.ubp : h.ub;
  const bool lsw = mode == MODE_L || mode == MODE_LX;   // L values
  const double2 *vals = lsw ? h.uL : mode == MODE_U ? h.uU : mode == MODE_UT ? h.uUt : h.uLt;
  const bool dinv = mode == MODE_U || mode == MODE_UT;
  double *G = (mode <= MODE_U || mode == MODE_LX) ? h.Z : h.P;
  int *ctr = h.blk_ctr + 2 * mode;
  const int nch = h.ld / kBC;
  // a ticket = one block x up to kblk_group consecutive column chunks: the block's
  // schedule is staged once and reused (it is ~40 % of a tile's L2 -> SM bytes)
  const int cg = max(1, min(h.kblk_group, nch)), ngrp = (nch + cg - 1) / cg;
  // sparse sweeps of a Cartesian batch (L, U0): tickets over the live tiles only
  const int *tl = h.tlist && h.tmask && (mode == MODE_L || h.spike == 1) ? h.tlist : nullptr;
  const int ntiles = tl ? __ldg(tl) : h.nblk * ngrp;
  double *X = reinterpret_cast<double *>(smraw + h.smem_x_off);
  UStage st;
  st.meta = reinterpret_cast<const int4 *>(smraw + h.smem_meta_off);
  st.topM = reinterpret_cast<const double *>(smraw + h.smem_tmeta_off);
  st.toprow = reinterpret_cast<const int *>(smraw + h.smem_tmeta_off + 32 * kTopLd * 8);
  st.lvl = reinterpret_cast<const int *>(smraw + h.smem_lvl_off);
  st.xs = smem_u32(X) + lane * 8;
  st.rec = smem_u32(smraw + h.smem_rec_off);
  st.doff = smem_u32(smraw + h.smem_doff_off);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  unsigned parity = 0;
  for (;;) {
    if (tid == 0) s_tk = atomicAdd(ctr, 1);
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // my previous stores have read X
    __syncthreads();
    const int tk = s_tk;
    if (tk >= ntiles) break;
    const int te = tl ? __ldg(tl + 1 + tk) : 0;
    const int s = tl ? te >> 16 : U.blk_order[tk / ngrp], cbeg = tl ? te & 0xffff : (tk % ngrp) * cg;
    const int cend = tl ? cbeg + 1 : min(nch, cbeg + cg);
    bool staged = false;
    for (int ci = cbeg; ci < cend; ++ci) {
    // Cartesian batch: an L tile whose right-hand side is zero stays zero (not
    // computed, not stored); the U sweep starts such a tile from zeros
    const bool live = h.spike != 2 && tile_live(h, s, ci);
    if ((mode == MODE_L || h.spike == 1) && !live) continue;   // (U0: a dead tile's Z^0 is zero, never stored)
    if (h.spike == 2 && ci * kBC >= U.ext_off[s + 1] - U.ext_off[s]) continue;   // spike columns beyond the block's
    const bool first = !staged;
    staged = true;
    if (!first) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // the previous chunk's stores have read X
      __syncthreads();
    }
    const int col0 = ci * kBC, tile = (tk / ngrp) * nch + ci;
    // timing experiment (RH_DEBUG & 8, MODE_U): per tile [8 warps' pieces | units << 48, wait, tops, t0, t1]
    long long *prof = ((h.debug & 8) && h.dbg && mode == MODE_U && tile < 8192) ? h.dbg + (long long)tile * 12 : nullptr;
    const long long c_a = prof ? clock64() : 0;
    const int r0 = h.seg_row_off[s], nr = h.seg_row_off[s + 1] - r0;
    const int x0 = U.ext_off[s], nxr = mode == MODE_L ? 0 : U.ext_off[s + 1] - x0;
    const int ub = U.unit_off[s], nu = U.unit_off[s + 1] - ub;
    const int rb = U.rec_off[s], nrec = U.rec_off[s + 1] - rb;
    const int ob = U.doff_off[s], nof = U.doff_off[s + 1] - ob;
    const int nxrows = mode == MODE_L ? 0 : nr + nxr;
    // epilogue partial runs (analysis.hpp RunRecs): U^T -> separator right-hand
    // sides, L^T -> G_p^T Psi; their records staged behind the tile's rows
    const bool ep_ut = mode == MODE_UT && h.nruns > 0, ep_lt = mode == MODE_LT && h.Mp;
    const int *roff = ep_lt ? h.ma_off : h.sr_off;
    const int nsr = ep_ut || ep_lt ? roff[s + 1] - roff[s] : 0;   // run record slots
    const int rrow = ep_lt ? nr + nxr : nr;                        // their first tile row
    // block rows by 2D TMA boxes (64, then 8 rows), the rest (< 8 block rows, staged
    // separator rows) by 16-byte cp.async
    const char *tm = reinterpret_cast<const char *>(G == h.Z ? h.tmZ : h.tmP);
    const bool zfill = mode == MODE_U && !live;   // its L result is zero (or a spike tile): no block rows to load
    const int nbig = tm && !zfill ? nr / kTmaBig : 0, nsmall = tm && !zfill ? (nr - nbig * kTmaBig) / kTmaSmall : 0;
    const int rows_tma = mode == MODE_L ? 0 : nbig * kTmaBig + nsmall * kTmaSmall;
    const int rows_zero = zfill ? nr : 0;
    if (tid == 0) {
      const double *dM = lsw ? h.tL : mode == MODE_U ? h.tU : mode == MODE_UT ? h.tUt : h.tLt;
      const unsigned tx = (first ? 16u * (nu + nrec) + 4u * nof + 4u * UnitSweep::kLvl + 32u * kTopLd * 8 + 128u +
                                       (mode == MODE_L ? 16u * (h.gpe_off[s + 1] - h.gpe_off[s]) + 48u : 0u) +
                                       16u * nsr
                                 : 0u) +
                          (unsigned)rows_tma * kRowB;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(tx)
                   : "memory");
      if (first) {
      bulk_g2s(smraw + h.smem_meta_off, U.meta + ub, 16u * nu, &mbar);
      bulk_g2s(smraw + h.smem_tmeta_off, dM + (size_t)s * 32 * kTopLd, 32u * kTopLd * 8, &mbar);
      bulk_g2s(smraw + h.smem_tmeta_off + 32 * kTopLd * 8, U.top_rows + s * 32, 128u, &mbar);
      bulk_g2s(smraw + h.smem_rec_off, vals + rb, 16u * nrec, &mbar);
      if (nof) bulk_g2s(smraw + h.smem_doff_off, U.doff + ob, 4u * nof, &mbar);
      bulk_g2s(smraw + h.smem_lvl_off, U.lvl + s * UnitSweep::kLvl, 4u * UnitSweep::kLvl, &mbar);
      if (nsr)   // the block's run records behind its rows (kept across chunks)
        bulk_g2s(X + rrow * kBC, (ep_lt ? h.ma_rec : h.sr_rec) + roff[s], 16u * nsr, &mbar);
      if (mode == MODE_L) {   // G_p entry records + warp ranges, behind the block's rows (kept across chunks)
        const int g0 = h.gpe_off[s], ng = h.gpe_off[s + 1] - g0;
        if (ng) bulk_g2s(X + nr * kBC, h.gpe_rec + g0, 16u * ng, &mbar);
        bulk_g2s(reinterpret_cast<double2 *>(X + nr * kBC) + ng, h.gpe_split + s * 12, 48u, &mbar);
      }
      }
      if (rows_tma) {
        for (int i = 0; i < nbig; ++i) tma2d_g2s(X + i * kTmaBig * kBC, tm, col0, r0 + i * kTmaBig, &mbar);
        for (int i = 0; i < nsmall; ++i) {
          const int a = nbig * kTmaBig + i * kTmaSmall;
          tma2d_g2s(X + a * kBC, tm + kTmapBytes, col0, r0 + a, &mbar);
        }
      }
      // the next chunk of this ticket: its block rows into L2 while this chunk sweeps
      if (tm && mode != MODE_L && ci + 1 < cend && !(h.debug & 4096) && !(mode == MODE_U && !tile_live(h, s, ci + 1))) {
        const int nb2 = nr / kTmaBig, ns2 = (nr - nb2 * kTmaBig) / kTmaSmall;
        for (int i = 0; i < nb2; ++i) tma2d_prefetch_l2(tm, col0 + kBC, r0 + i * kTmaBig);
        for (int i = 0; i < ns2; ++i) tma2d_prefetch_l2(tm + kTmapBytes, col0 + kBC, r0 + nb2 * kTmaBig + i * kTmaSmall);
      }
    }
    {  // X rows: 16-byte cp.async (LSU path; 256 B TMA bulk copies are rate-bound on the TMA unit)
      const int c = tid & 15;
      for (int a = rows_tma + rows_zero + (tid >> 4); a < nxrows; a += blockDim.x >> 4) {
        if (a >= nr && h.spike) {   // staged separator rows: zero (U0) or identity columns (spikes)
          const int k = a - nr - col0;
          reinterpret_cast<double2 *>(X + a * kBC)[c] =
              make_double2(h.spike == 2 && k == 2 * c ? 1.0 : 0.0, h.spike == 2 && k == 2 * c + 1 ? 1.0 : 0.0);
          continue;
        }
        const long long grow = a < nr ? r0 + a : U.ext_rows[x0 + a - nr];
        cp_async16(X + a * kBC + 2 * c, G + grow * h.ld + col0 + 2 * c);
      }
    }
    if (mode == MODE_L || zfill)   // L: right-hand side -G_p W (SpMul fused): zero, then the G_p rows below
      for (int i = tid; i < nr * (kBC / 2); i += blockDim.x) reinterpret_cast<double2 *>(X)[i] = make_double2(0.0, 0.0);
    asm volatile("cp.async.wait_all;" ::: "memory");
    {  // wait for the copies of this tile
      unsigned done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(smem_u32(&mbar)), "r"(parity)
                     : "memory");
      parity ^= 1;
    }
    __syncthreads();
    if (mode == MODE_L) {   // G_p rows of the block from the staged entry records (behind the block rows)
      const double2 *er = reinterpret_cast<const double2 *>(X + nr * kBC);
      const int *sp = reinterpret_cast<const int *>(er + (h.gpe_off[s + 1] - h.gpe_off[s]));
      tile_rhs_entries(h, er, sp[warp], sp[warp + 1], col0 + lane, X + lane);
      __syncthreads();
    }
    const long long c_b = prof ? clock64() : 0;
    if (fwd) {
      if (dinv) unit_pieces<true>(st, warp); else unit_pieces<false>(st, warp);
      __syncthreads();
      unit_tops(st, X, warp, lane);
    } else {
      unit_tops(st, X, warp, lane);
      const long long c_c = prof ? clock64() : 0;
      if (dinv) unit_pieces<true>(st, warp); else unit_pieces<false>(st, warp);
      if (prof && lane == 0) {
        prof[warp] = (clock64() - c_c) | ((long long)(st.lvl[warp + 1] - st.lvl[warp]) << 48);
        if (warp == 0) {
          prof[8] = c_b - c_a;
          prof[9] = (c_c - c_b) | ((long long)first << 48);
          prof[10] = c_a;
        }
      }
      __syncthreads();
      if (prof && tid == 0) prof[11] = clock64();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // sweep writes -> bulk store reads
    __syncthreads();
    {  // (U0: Z^0 goes to P, Z keeps the L sweep's result for the separator gather)
      const char *ts = h.spike == 1 ? reinterpret_cast<const char *>(h.tmP) : tm;
      double *Gs = h.spike == 1 ? h.P : G;
      const int nbs = ts ? nr / kTmaBig : 0, nss = ts ? (nr - nbs * kTmaBig) / kTmaSmall : 0;
      const int rows_st = nbs * kTmaBig + nss * kTmaSmall;
      if (tid == 0) {
        for (int i = 0; i < nbs; ++i) tma2d_s2g(ts, col0, r0 + i * kTmaBig, X + i * kTmaBig * kBC);
        for (int i = 0; i < nss; ++i) {
          const int a = nbs * kTmaBig + i * kTmaSmall;
          tma2d_s2g(ts + kTmapBytes, col0, r0 + a, X + a * kBC);
        }
      }
      for (int a = rows_st + tid; a < nr; a += blockDim.x)
        bulk_s2g(Gs + (long long)(r0 + a) * h.ld + col0, X + a * kBC, kRowB);
    }
    if (nsr) {
      // partials of this block's runs (U^T: separator right-hand sides, k_sep_gather
      // UTLT sums them; L^T: G_p^T Psi, k_muladd sums them; X is read while the bulk
      // stores above read it too): Part[g] = sum of coefficient x tile row over run
      // g's entries, in order (entry k -> chain k & 1), from the staged run records
      double *part = ep_lt ? h.Mp : h.Tsep + (long long)h.ns * h.ld;
      const unsigned rr = smem_u32(X + rrow * kBC);
      const int rw0 = ldsi(rr + 4 * warp), rw1 = ldsi(rr + 4 * warp + 4);   // this warp's runs (LPT)
      for (int r = rw0; r < rw1; ++r) {
        const int4 rt = ldsi4(rr + 16 * (3 + r));
        double a0 = 0.0, a1 = 0.0;
        int k = 0;
        for (; k + 4 <= rt.z; k += 4) {   // four entries' loads in flight
          const unsigned ea = rr + 16 * (rt.y + k);
          const double2 n0 = ldsd2(ea), n1 = ldsd2(ea + 16), n2 = ldsd2(ea + 32), n3 = ldsd2(ea + 48);
          const double x0 = ldsd(st.xs + (int)__double_as_longlong(n0.y));
          const double x1 = ldsd(st.xs + (int)__double_as_longlong(n1.y));
          const double x2 = ldsd(st.xs + (int)__double_as_longlong(n2.y));
          const double x3 = ldsd(st.xs + (int)__double_as_longlong(n3.y));
          a0 = fma(n0.x, x0, a0);
          a1 = fma(n1.x, x1, a1);
          a0 = fma(n2.x, x2, a0);
          a1 = fma(n3.x, x3, a1);
        }
        for (; k < rt.z; ++k) {
          const double2 en = ldsd2(rr + 16 * (rt.y + k));
          const double x = ldsd(st.xs + (int)__double_as_longlong(en.y));
          if (k & 1) a1 = fma(en.x, x, a1);
          else a0 = fma(en.x, x, a0);
        }
        part[(long long)rt.x * h.ld + col0 + lane] = a0 + a1;
      }
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }   // column chunks of the ticket
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  // the last CTA out resets the ticket counter for the next launch
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(ctr + 1, 1) == (int)gridDim.x - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
      __threadfence();
    }
  }
}

// ----------------------------------------------------------------------------
// Split U sweep of Cartesian batches (SURVEY.md
// 8(a)-6).  A block's U rows depend on the separator only through its staged
// separator rows z_ext (U_bs), so by linearity
//   z_b = U_bb^-1 (y_b - U_bs z_ext) = Z_b^0 + Msp_b z_ext,
//   Z_b^0 = U_bb^-1 y_b (k_blk MODE_U, spike = 1: needs no S^-1, runs while the
//   separator is inverted; zero for the dead tiles of a Cartesian batch),
//   Msp_b = -U_bb^-1 U_bs (k_blk MODE_U, spike = 2, once per state: the block's
//   sweep of identity columns on its staged separator rows).
// k_spike forms z_b for every (block, 32-column) tile once z_ext is known: a
// dense [rows x K] x [K x 32] product on the fp64 tensor cores (DMMA m8n8k4,
// K = the block's staged separator rows rounded up to 4), accumulated onto
// Z_b^0 (live tiles) and stored.  Per column the arithmetic does not depend on
// the batch (bitwise N- and mask-invariant).
// ----------------------------------------------------------------------------
constexpr int kSpLd = 64;       // Msp row stride (the spike sweep's output): <= 64 staged separator rows
constexpr int kSpQ = 9;         // k_spike: K <= 4 kSpQ = 36 staged separator rows per block
constexpr int kSpMt = 32;       // m-tiles (8 rows) per block: blocks of <= 256 rows
constexpr int kSpThreads = 256;
// Msp in DMMA A-fragment order (once per state, after the spike sweep): for block
// s, m-tile mt and k-step q the 32 values a warp's lanes (gid, tig) hold,
// Msp[r0 + 8 mt + gid][4 q + tig], contiguous: one coalesced 256 B load each.
__global__ void k_spike_frag(SegParams h, double *Mf) {
  const int s = blockIdx.x, mt = blockIdx.y, lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  const int r0 = h.seg_row_off[s], nr = h.seg_row_off[s + 1] - r0, r = 8 * mt + (lane >> 2);
  if (q < kSpQ)
    Mf[(((long long)s * kSpMt + mt) * kSpQ + q) * 32 + lane] =
        r < nr ? h.Msp[(long long)(r0 + r) * kSpLd + 4 * q + (lane & 3)] : 0.0;
}
// z_b = Z_b^0 + Msp_b z_ext for one (block, 32-column) tile: z_ext staged in
// shared memory, A fragments by coalesced loads, one m-tile per warp at a time.
__global__ void __launch_bounds__(kSpThreads) k_spike(SegParams h, const double *__restrict__ Mf) {
  __shared__ __align__(16) double zs[4 * kSpQ][36];   // z_ext rows x 32 columns (stride 36: conflict-free B fragments)
  const int s = blockIdx.x, ci = blockIdx.y, col0 = ci * kBC;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const DUnit &U = h.ub;
  const int r0 = h.seg_row_off[s], nr = h.seg_row_off[s + 1] - r0;
  const int x0 = U.ext_off[s], nxr = U.ext_off[s + 1] - x0, K = (nxr + 3) & ~3;
  const bool live = tile_live(h, s, ci);
  {  // stage z_ext: every load in flight, then the stores
    double v[(4 * kSpQ + kSpThreads / 32 - 1) / (kSpThreads / 32)];
#pragma unroll
    for (int u = 0; u < (int)(sizeof(v) / sizeof(double)); ++u) {
      const int k = warp + u * (kSpThreads / 32);
      v[u] = k < nxr ? h.Z[(long long)U.ext_rows[x0 + k] * h.ld + col0 + lane] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < (int)(sizeof(v) / sizeof(double)); ++u) {
      const int k = warp + u * (kSpThreads / 32);
      if (k < 4 * kSpQ) zs[k][lane] = v[u];
    }
  }
  __syncthreads();
  const int gid = lane >> 2, tig = lane & 3;
  const double *mf = Mf + (long long)s * kSpMt * kSpQ * 32 + lane;
  constexpr int NW = kSpThreads / 32;
  for (int m0 = warp; m0 * 8 < nr; m0 += 2 * NW) {   // two m-tiles (m0, m0 + NW) per pass: each B fragment feeds both
    const bool two = (m0 + NW) * 8 < nr;
    double c[2][4][2];
    long long ro[2];
    bool in[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int r = (m0 + t * NW) * 8 + gid;
      in[t] = (t == 0 || two) && r < nr;
      ro[t] = (long long)(r0 + r) * h.ld + col0 + 2 * tig;
#pragma unroll
      for (int n = 0; n < 4; ++n) {   // Z^0 (k_blk U0, in P) of a live tile, else zero
        const double2 v = in[t] && live ? *reinterpret_cast<const double2 *>(h.P + ro[t] + 8 * n) : make_double2(0.0, 0.0);
        c[t][n][0] = v.x;
        c[t][n][1] = v.y;
      }
    }
    for (int q = 0; 4 * q < K; ++q) {
      const double a0 = __ldg(mf + (m0 * kSpQ + q) * 32);   // coalesced: the fragment-order spikes
      const double a1 = two ? __ldg(mf + ((m0 + NW) * kSpQ + q) * 32) : 0.0;
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        const double bq = zs[4 * q + tig][8 * n + gid];
        dmma_8x8x4(c[0][n][0], c[0][n][1], a0, bq);
        dmma_8x8x4(c[1][n][0], c[1][n][1], a1, bq);
      }
    }
#pragma unroll
    for (int t = 0; t < 2; ++t)
      if (in[t])
#pragma unroll
        for (int n = 0; n < 4; ++n)
          *reinterpret_cast<double2 *>(h.Z + ro[t] + 8 * n) = make_double2(c[t][n][0], c[t][n][1]);
  }
}

// ----------------------------------------------------------------------------
// Separator segment: (1) k_sep_gather forms the
// right-hand side of the separator rows, rhs - (block columns) x (block rows),
// fully parallel (warp per separator row, lane per column); (2) k_sep_gemm
// applies the dense inverse S^-1 (S = L_ss U_ss, inverted once per state by
// k_sep_inverse): the separator's ~100-level dependency chain becomes one
// [ns x ns] x [ns x N] fp64 GEMM, written straight into the separator rows.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_sep_gather(SegParams h, int mode) {
  const int lane = threadIdx.x & 31;
  const int qoff = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  const int col = blockIdx.y * 32 + lane;
  const int seg = h.nblk;
  const int qb = h.fwd.lvl_ptr[h.fwd.seg_lvl[seg]], qe = h.fwd.lvl_ptr[h.fwd.seg_lvl[seg + 1] - 1];
  const int q = qb + qoff;
  if (q >= qe) return;
  const bool lu = mode == MODE_LU || mode == MODE_LUX;
  const bool masked = mode == MODE_LU && h.tmask;   // Cartesian batch: skip block rows of zero L tiles
  double *G = lu ? h.Z : h.P;
  const double *val = lu ? h.vL : h.vUt;
  const int a = h.fwd.order[q];
  const int row = h.row_global[h.sep_off + a];
  const double v0 = mode == MODE_LU ? rhs_gpw(h, row, col) : G[(long long)(h.sep_off + a) * h.ld + col];
  int e = h.fwd.rptr[q];
  const int ex = h.fwd.rext[q];
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (mode == MODE_UTLT) {
    // the U^T sweep left one partial per run (k_blk MODE_UT epilogue): sum them in run order
    const double *part = h.Tsep + (long long)h.ns * h.ld + col;
    const int g0 = h.fwd.grp_ptr[qoff], g1 = h.fwd.grp_ptr[qoff + 1];
    int g = g0;
    for (; g + 4 <= g1; g += 4) {
      const double x0 = part[(long long)g * h.ld], x1 = part[(long long)(g + 1) * h.ld];
      const double x2 = part[(long long)(g + 2) * h.ld], x3 = part[(long long)(g + 3) * h.ld];
      s0 += x0;
      s1 += x1;
      s2 += x2;
      s3 += x3;
    }
    for (; g < g1; ++g) s0 += part[(long long)g * h.ld];
    h.Tsep[(long long)a * h.ld + col] = v0 - ((s0 + s1) + (s2 + s3));
    return;
  }
  if (masked) {
    // Cartesian batch: only the block runs whose tile of this chunk is live (the
    // others are identically zero).  Every live entry goes to the chain the
    // unmasked loops below give it ((e - e0) mod 4, the last (ex - e0) mod 4
    // entries to chain 0), in the same order, so both paths are bitwise equal.
    // The row's nonzero flag for this chunk goes to nzf (k_sep_spmm).
    const int e0 = e, tail = ex - ((ex - e0) & 3);
    for (int g = h.fwd.grp_ptr[qoff], g1 = h.fwd.grp_ptr[qoff + 1]; g < g1; ++g) {
      const int ee = h.fwd.grp_end[g];
      if (!tile_live(h, h.fwd.grp_blk[g], blockIdx.y)) {
        e = ee;
        continue;
      }
      for (; e < ee; e += 4) {   // (ends past ee: the next run restarts at ee)
        double x[4], c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (e + u < ee) {
            c[u] = val[e + u];
            x[u] = G[(long long)h.fwd.dep[e + u] * h.ld + col];
          }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (e + u < ee) {
            const int k = e + u >= tail ? 0 : ((e + u - e0) & 3);
            if (k == 0) s0 = fma(c[u], x[u], s0);
            else if (k == 1) s1 = fma(c[u], x[u], s1);
            else if (k == 2) s2 = fma(c[u], x[u], s2);
            else s3 = fma(c[u], x[u], s3);
          }
      }
      e = ee;
    }
    const double t = v0 - ((s0 + s1) + (s2 + s3));
    h.Tsep[(long long)a * h.ld + col] = t;
    const unsigned nz = __ballot_sync(0xffffffffu, t != 0.0);
    if (lane == 0) h.nzf[(long long)blockIdx.y * ((h.ns + 15) & ~15) + a] = nz != 0u;   // rows of 16-byte words
    return;
  }
  for (; e + 8 <= ex; e += 8) {   // 8 row gathers in flight
    int d[8];
    double c[8], x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      d[u] = h.fwd.dep[e + u];
      c[u] = val[e + u];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      x[u] = G[(long long)d[u] * h.ld + col];
    s0 = fma(c[0], x[0], s0);
    s1 = fma(c[1], x[1], s1);
    s2 = fma(c[2], x[2], s2);
    s3 = fma(c[3], x[3], s3);
    s0 = fma(c[4], x[4], s0);
    s1 = fma(c[5], x[5], s1);
    s2 = fma(c[6], x[6], s2);
    s3 = fma(c[7], x[7], s3);
  }
  auto ld_dep = [&](int e1) { return G[(long long)h.fwd.dep[e1] * h.ld + col]; };
  for (; e + 4 <= ex; e += 4) {
    const double x0 = ld_dep(e), x1 = ld_dep(e + 1), x2 = ld_dep(e + 2), x3 = ld_dep(e + 3);
    s0 = fma(val[e], x0, s0);
    s1 = fma(val[e + 1], x1, s1);
    s2 = fma(val[e + 2], x2, s2);
    s3 = fma(val[e + 3], x3, s3);
  }
  for (; e < ex; ++e) s0 = fma(val[e], ld_dep(e), s0);
  h.Tsep[(long long)a * h.ld + col] = v0 - ((s0 + s1) + (s2 + s3));
}

// C[m][n] = sum_k M[m][k] T[k][n] written to the separator slab of Z / P
// (rows sep_off + m, contiguous in segment order): the one dense contraction
// of the path, on the fp64 tensor cores (DMMA, mma.sync m8n8k4).  64 x 64
// output tile per CTA, 8 warps of 32 x 16 (4 x 2 mma tiles) per group, k in
// tiles of 16 through a GSTAGES-deep cp.async pipeline.  Both operand tiles
// are k-major with rows padded to 72 doubles, so every fragment load (lane
// (g, t) reads row t, column g) hits 16 distinct banks per half-warp: no bank
// conflicts.  The k-major A tile is a row range of the transposed operator
// (S^-T for S^-1 and vice versa).  In-CTA split-K: GGRP groups of 8 warps take
// alternate k tiles; the partial tiles are added in fixed group order
// (deterministic).
constexpr int GBM = 64, GBN = 64, GBK = 16, GGRP = 2, GTHREADS = 256 * GGRP, GSTAGES = 3, GLD = 72;
constexpr int GTILE = GBK * GLD;   // doubles per operand tile per stage
constexpr size_t gemm_smem_bytes() { return sizeof(double) * GGRP * GSTAGES * 2 * GTILE; }
__device__ __forceinline__ void cp_async8z(void *dst, const void *src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async16z(void *dst, const void *src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__global__ void __launch_bounds__(GTHREADS) k_sep_gemm(SegParams h, int mode) {
  extern __shared__ __align__(16) double gsm[];
  const int grp = threadIdx.x >> 8;
  double *As = gsm + grp * GSTAGES * 2 * GTILE;   // [stage][k][m]
  double *Bs = As + GSTAGES * GTILE;              // [stage][k][n]
  const int ns = h.ns, ld = h.ld;
  const double *MT = mode == MODE_LU ? h.SinvT : h.Sinv;   // A[m][k] = MT[k][m]
  double *G = mode == MODE_LU ? h.Z : h.P;
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN;
  const int tid = threadIdx.x & 255, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;   // warp tile rows wm*32.., cols wn*16..
  const int gid = lane >> 2, tig = lane & 3;
  const int nkt = (ns + GBK - 1) / GBK;
  const int myt = nkt > grp ? (nkt - grp + GGRP - 1) / GGRP : 0;   // k tiles grp, grp + GGRP, ...
  auto issue = [&](int t) {
    const int st = t % GSTAGES, k0 = (grp + t * GGRP) * GBK;
    double *a = As + st * GTILE, *b = Bs + st * GTILE;
#pragma unroll
    for (int r = 0; r < 4; ++r) {   // A: 16 k x 64 m doubles, 8-byte copies (ns is odd)
      const int idx = tid + r * 256, kk = idx >> 6, mm = idx & 63;
      const int gk = k0 + kk, gm = m0 + mm;
      const bool v = gk < ns && gm < ns;
      cp_async8z(a + kk * GLD + mm, MT + (v ? (long long)gk * ns + gm : 0), v);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {   // B: 16 k x 64 n doubles, 16-byte copies (ld is a multiple of 32)
      const int idx = tid + r * 256, kk = idx >> 5, nn = (idx & 31) * 2;
      const int gk = k0 + kk, gn = n0 + nn;
      const bool v = gk < ns && gn < ld;
      cp_async16z(b + kk * GLD + nn, h.Tsep + (v ? (long long)gk * ld + gn : 0), v);
    }
  };
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  auto gsync = [&]() { asm volatile("bar.sync %0, 256;" ::"r"(1 + grp) : "memory"); };
#pragma unroll
  for (int t = 0; t < GSTAGES - 1; ++t) {
    if (t < myt) issue(t);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int t = 0; t < myt; ++t) {
    asm volatile("cp.async.wait_group %0;" ::"n"(GSTAGES - 2) : "memory");
    gsync();   // tile t landed for every thread; everyone is done with tile t - 1
    if (t + GSTAGES - 1 < myt) issue(t + GSTAGES - 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const double *a = As + (t % GSTAGES) * GTILE, *b = Bs + (t % GSTAGES) * GTILE;
#pragma unroll
    for (int q = 0; q < GBK / 4; ++q) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = a[(4 * q + tig) * GLD + wm * 32 + i * 8 + gid];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = b[(4 * q + tig) * GLD + wn * 16 + j * 8 + gid];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  // fixed-order reduction: group 1 parks its partial tile, group 0 adds and stores
  __syncthreads();
  double(*Red)[GBN + 2] = reinterpret_cast<double(*)[GBN + 2]>(gsm);
  if (grp == 1) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int r = wm * 32 + i * 8 + gid, c = wn * 16 + j * 8 + 2 * tig;
        Red[r][c] = acc[i][j][0];
        Red[r][c + 1] = acc[i][j][1];
      }
  }
  __syncthreads();
  if (grp == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int gm = m0 + wm * 32 + i * 8 + gid;
      if (gm >= ns) continue;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int r = wm * 32 + i * 8 + gid, c = wn * 16 + j * 8 + 2 * tig;
        const int gn = n0 + c;
        const double o0 = acc[i][j][0] + Red[r][c], o1 = acc[i][j][1] + Red[r][c + 1];
        double *out = G + (long long)(h.sep_off + gm) * ld + gn;
        if (gn + 1 < ld) {
          *reinterpret_cast<double2 *>(out) = make_double2(o0, o1);
        } else if (gn < ld) {
          out[0] = o0;
        }
      }
    }
  }
}


// Single right-hand side (the first-order adjoint): separator rows of P =
// S^-T t, warp per row, lanes over k (coalesced rows of S^-T), fixed order.
// Cartesian batches, separator rows of the L solve: T = (rhs - L_sb Z_b) has
// few nonzero rows per 32-column chunk (the separator rows that depend on the
// chunk's home blocks, ~10 % of them), so Z_sep = S^-1 T is formed over those
// rows only: the chunk's nonzero-row list (nzf, from k_sep_gather) is
// compacted, the rows of T and the matching columns of S^-1 (S^-1 itself, so
// this does not wait for its transpose) are staged in shared memory SPK at a
// time, and each lane (= column) accumulates in increasing k.
// A row of the list that is zero in some column adds an exact zero there, so
// every column's sum is its own nonzero terms in increasing k: the result does
// not depend on the other columns of the chunk (bitwise N- and shard-invariant).
constexpr int SPK = 48, SPM = 64;   // staged k rows, output rows per CTA
__global__ void __launch_bounds__(256) k_sep_spmm(SegParams h) {
  extern __shared__ __align__(16) double spm[];
  double(*Ts)[32] = reinterpret_cast<double(*)[32]>(spm);               // [SPK][32]
  double(*As)[SPM] = reinterpret_cast<double(*)[SPM]>(spm + SPK * 32);  // [SPK][SPM]: S^-1[m0 + m][k]
  int *klist = reinterpret_cast<int *>(spm + SPK * 32 + SPK * SPM);     // [ns]
  __shared__ int s_nk;
  const int ns = h.ns, ld = h.ld, c = blockIdx.x, m0 = blockIdx.y * SPM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp == 0) {   // compact the chunk's nonzero rows, increasing k: 16 flags per 16-byte load
    const int nsf = (ns + 15) & ~15, nw16 = nsf >> 4;   // flag row stride (bytes), 16-byte words
    const uint4 *fw = reinterpret_cast<const uint4 *>(h.nzf + (long long)c * nsf);
    int n = 0;
    for (int i = 0; 32 * i < nw16; ++i) {   // 512 rows per pass (one pass up to ns = 512)
      const uint4 wi = lane + 32 * i < nw16 ? fw[lane + 32 * i] : make_uint4(0, 0, 0, 0);
      const unsigned v[4] = {wi.x, wi.y, wi.z, wi.w};
      const int r0 = 16 * (lane + 32 * i);   // flags past ns (row padding) are stale: masked
      unsigned fl = 0u;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (r0 + j < ns && ((v[j >> 2] >> (8 * (j & 3))) & 0xffu) != 0u) fl |= 1u << j;
      const int cnt = __popc(fl);
      int pre = cnt;   // inclusive scan over the lanes
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, pre, o);
        if (lane >= o) pre += t;
      }
      int at = n + pre - cnt;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (fl & (1u << j)) klist[at++] = r0 + j;
      n += __shfl_sync(0xffffffffu, pre, 31);
    }
    if (lane == 0) s_nk = n;
  }
  __syncthreads();
  const int nk = s_nk;
  double acc[SPM / 8];
#pragma unroll
  for (int i = 0; i < SPM / 8; ++i) acc[i] = 0.0;
  for (int k0 = 0; k0 < nk; k0 += SPK) {
    const int kn = min(SPK, nk - k0);
    {   // every thread's staging loads in flight at once (18 per thread at most)
      constexpr int NT = SPK * 32 / 256, NA = SPK * SPM / 256;
      double vt[NT], va[NA];
#pragma unroll
      for (int i = 0; i < NT; ++i) {
        const int t = tid + 256 * i, kk = t >> 5, cc = t & 31;
        vt[i] = kk < kn ? h.Tsep[(long long)klist[k0 + kk] * ld + c * 32 + cc] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < NA; ++i) {
        const int t = tid + 256 * i, kk = t / SPM, mm = t % SPM;
        va[i] = kk < kn && m0 + mm < ns ? h.Sinv[(long long)(m0 + mm) * ns + klist[k0 + kk]] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < NT; ++i) {
        const int t = tid + 256 * i;
        Ts[t >> 5][t & 31] = vt[i];
      }
#pragma unroll
      for (int i = 0; i < NA; ++i) {
        const int t = tid + 256 * i;
        As[t / SPM][t % SPM] = va[i];
      }
    }
    __syncthreads();
    for (int kk = 0; kk < kn; ++kk) {
      const double tv = Ts[kk][lane];
#pragma unroll
      for (int i = 0; i < SPM / 8; ++i) acc[i] = fma(As[kk][warp + 8 * i], tv, acc[i]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < SPM / 8; ++i) {
    const int m = m0 + warp + 8 * i;
    if (m < ns) h.Z[(long long)(h.sep_off + m) * ld + c * 32 + lane] = acc[i];
  }
}
inline size_t spmm_smem_bytes(int ns) { return sizeof(double) * (SPK * 32 + SPK * SPM) + sizeof(int) * (size_t)ns; }

__global__ void __launch_bounds__(kThreads) k_sep_gemv(SegParams h, int mode) {
  const int lane = threadIdx.x & 31;
  const int m = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  if (m >= h.ns) return;
  const double *M = (mode == MODE_LU ? h.Sinv : h.SinvT) + (long long)m * h.ns;
  double *G = mode == MODE_LU ? h.Z : h.P;
  double acc = 0.0;
  for (int k = lane; k < h.ns; k += 32) acc = fma(__ldg(M + k), h.Tsep[(long long)k * h.ld], acc);
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) G[(long long)(h.sep_off + m) * h.ld] = acc;
}

// ============================================================================
// BatchTensorProjection (Eq. so_model)
// by hand-written forward-over-reverse on the line graph with a hoisted tape:
// per line (K, a_i, a_j, m) is column independent (k_coefs, once per state and
// lambda); per column it is 8 FMAs per line end.  Bus-centric gather ("edges
// then nodes") without atomics.  Thread = (bus, column).
// ============================================================================

__device__ __forceinline__ double delta_src(const SegParams &h, int src, int col) {
  if (src >= 0) return h.Z[(long long)src * h.ld + col];
  if (src == -1) return 0.0;
  return load_W(h, -(src + 2), col);
}

// Staged tiles: one CTA = (bus group, 32 columns) (analysis.hpp ForGroups).
// The delta rows (dtheta, dv) of the group's buses and of their neighbours are
// staged once in shared memory (Z rows by TMA bulk copies on an mbarrier, v
// parameters from W), so each line end's gather reads shared memory instead
// of L2; warp per output bus, lane per column.
constexpr int kForThreads = 512;   // 16 warps: two CTAs per SM (shared memory), 32 warps to hide latency
__global__ void __launch_bounds__(kForThreads, 2) k_for(SegParams h) {
  extern __shared__ __align__(128) double fsm[];   // [maxrows][32] delta rows, then the tile's tape
  __shared__ __align__(8) unsigned long long mbar;
  __shared__ double sref[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int g = blockIdx.x, col0 = blockIdx.y * 32, col = col0 + lane;
  const int l0 = h.fg_off[g], nout = h.fg_nout[g], ob = h.fg_obase[g];
  const int sb = h.fg_sbase[g], nsl = h.fg_sbase[g + 1] - sb;
  const int zlo = h.fg_zlo[g], zn = h.fg_zn[g];
  const int c0 = h.fg_cp_off[g], ncp = h.fg_cp_off[g + 1] - c0;
  const int f0 = h.fg_fill_off[g], nfill = h.fg_fill_off[g + 1] - f0;
  double4 *s_coef = reinterpret_cast<double4 *>(fsm + (size_t)h.fg_maxrows * 32);
  double4 *s_meta = s_coef + h.fg_maxslots;
  int4 *s_dst = reinterpret_cast<int4 *>(s_meta + h.fg_maxout);
  // per slot: byte offsets (theta, v) of the other end's staging rows
  const int2 *s_oe = reinterpret_cast<const int2 *>(s_dst + h.fg_maxout);
  // timing experiment (RH_DEBUG & 8192): per CTA [start, armed, row copies issued, filled,
  // copies landed, end]
  long long *prof = ((h.debug & 8192) && h.dbg && g * gridDim.y + blockIdx.y < 16384)
                        ? h.dbg + 6LL * (g * gridDim.y + blockIdx.y) : nullptr;
  if (prof && tid == 0) prof[0] = clock64();
  const char *tm = reinterpret_cast<const char *>(h.tmZ);
  const int nbig = tm ? zn / kTmaBig : 0, nsmall = tm ? (zn - nbig * kTmaBig) / kTmaSmall : 0;
  const int rows_tma = nbig * kTmaBig + nsmall * kTmaSmall;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const unsigned tx = 256u * (zn + ncp) + 40u * nsl + 48u * nout;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(tx) : "memory");
    bulk_g2s(s_coef, h.fg_scoef + sb, 32u * nsl, &mbar);
    bulk_g2s(const_cast<int2 *>(s_oe), h.fg_soe + sb, 8u * nsl, &mbar);
    bulk_g2s(s_meta, h.fg_ometa + ob, 32u * nout, &mbar);
    bulk_g2s(s_dst, h.fg_odst + ob, 16u * nout, &mbar);
    // the outputs' Z row range by 2D TMA boxes (64, then 8 rows)
    for (int i = 0; i < nbig; ++i) tma2d_g2s(fsm + i * kTmaBig * 32, tm, col0, zlo + i * kTmaBig, &mbar);
    for (int i = 0; i < nsmall; ++i) {
      const int r = nbig * kTmaBig + i * kTmaSmall;
      tma2d_g2s(fsm + r * 32, tm + kTmapBytes, col0, zlo + r, &mbar);
    }
  }
  __syncthreads();   // mbarrier initialised and armed
  if (prof && tid == 0) prof[1] = clock64();
  // the rest of the range and the other Z sources: per-row bulk copies
  for (int r = rows_tma + tid; r < zn; r += blockDim.x)
    bulk_g2s(fsm + r * 32, h.Z + (long long)(zlo + r) * h.ld + col0, 256, &mbar);
  for (int i = tid; i < ncp; i += blockDim.x) {
    const int2 e = h.fg_cp[c0 + i];
    bulk_g2s(fsm + e.x * 32, h.Z + (long long)e.y * h.ld + col0, 256, &mbar);
  }
  if (prof && tid == 0) prof[2] = clock64();
  // rows without a Z source: zero, or a v parameter from W; lane = column, 4 rows in flight per warp
  for (int f = 4 * warp; f < nfill; f += 4 * nw) {
    double v[4];
    int2 q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      q[u] = f + u < nfill ? h.fg_fill[f0 + f + u] : make_int2(-1, -1);
      v[u] = q[u].y >= 0 ? load_W(h, q[u].y, col) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (f + u < nfill) fsm[q[u].x * 32 + lane] = v[u];
  }
  if (prof && tid == 0) prof[3] = clock64();
  {
    unsigned done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(smem_u32(&mbar))
                   : "memory");
  }
  __syncthreads();
  if (prof && tid == 0) prof[4] = clock64();
  const int r0 = h.fg_ref[g], r1 = h.fg_ref[g + 1];
  if (r0 < r1) {   // REF objective rank-1 term f''(Pg_ref) (grad P_ref . delta) (R22), once per tile
    if (warp == 0) {
      double sr = 0.0;
      for (int q = r0; q < r1; ++q) {
        const int4 e = h.fg_loc[l0 + h.fg_ref_loc[q]];
        sr += h.refg_th[e.z] * fsm[(e.w & 0xffff) * 32 + lane] + h.refg_v[e.z] * fsm[(e.w >> 16) * 32 + lane];
      }
      sref[lane] = sr * h.f2ref;
    }
    __syncthreads();
  }
  // warp per output bus, lane per column, all from shared memory; two buses at a
  // time (independent FMA chains, same per-bus order as one at a time)
  const char *fl = reinterpret_cast<const char *>(fsm + lane);   // this lane's column of staging row 0
  auto slot = [&](int q, double dth_b, double dv_b, double &yth, double &yv) {
    // canonical slot coefficients (k_for_tape): D = dth_b - dth_o,
    // yth += K D + c2 dv_b + c3 dv_o,  yv += c2 D + m dv_o
    const double4 k = s_coef[q];
    const int2 o = s_oe[q];
    const double D = dth_b - *reinterpret_cast<const double *>(fl + o.x);
    const double dv_o = *reinterpret_cast<const double *>(fl + o.y);
    yth = fma(k.x, D, fma(k.y, dv_b, fma(k.z, dv_o, yth)));
    yv = fma(k.y, D, fma(k.w, dv_o, yv));
  };
  auto finish = [&](const int4 d, const double4 mt, double yth, double yv) {
    if (mt.y != 0.0 || mt.z != 0.0) {
      yth += sref[lane] * mt.y;
      yv += sref[lane] * mt.z;
    }
    if (d.x >= 0) h.P[(long long)d.x * h.ld + col] = -yth;
    if (d.y >= 0) {
      h.P[(long long)d.y * h.ld + col] = -yv;
    } else if (d.y <= -2) {
      h.Yp[(long long)(-(d.y + 2)) * h.ld + col] = yv;
    }
  };
  for (int i = warp; i < nout; i += 2 * nw) {
    const int i2 = i + nw;
    const bool two = i2 < nout;
    const int4 d = s_dst[i], d2 = two ? s_dst[i2] : make_int4(-1, -1, 0, 0);
    const double4 mt = s_meta[i], mt2 = two ? s_meta[i2] : make_double4(0.0, 0.0, 0.0, 0.0);
    const int o1 = d.w, o2 = d2.w;   // own staging rows
    const double dth_b = fsm[(o1 & 0xffff) * 32 + lane], dv_b = fsm[(o1 >> 16) * 32 + lane];
    const double dth_b2 = two ? fsm[(o2 & 0xffff) * 32 + lane] : 0.0, dv_b2 = two ? fsm[(o2 >> 16) * 32 + lane] : 0.0;
    double yth = 0.0, yv = mt.x * dv_b, yth2 = 0.0, yv2 = mt2.x * dv_b2;
    const int q1 = d.z & 0xffff, q2 = d2.z & 0xffff, n1 = d.z >> 16, n2 = d2.z >> 16, nmin = min(n1, n2);
    int t = 0;
    for (; t < nmin; ++t) {
      slot(q1 + t, dth_b, dv_b, yth, yv);
      slot(q2 + t, dth_b2, dv_b2, yth2, yv2);
    }
    for (; t < n1; ++t) slot(q1 + t, dth_b, dv_b, yth, yv);
    for (; t < n2; ++t) slot(q2 + t, dth_b2, dv_b2, yth2, yv2);
    finish(d, mt, yth, yv);
    if (two) finish(d2, mt2, yth2, yv2);
  }
  if (prof) {
    __syncthreads();
    if (tid == 0) prof[5] = clock64();
  }
}

// The FoR tape in tile order (once per state and lambda, after k_coefs): the
// line coefficients (K, a_i, a_j, m) of every slot in the orientation of the
// slot's bus b: from-end (K, a_i, a_j, m), to-end (K, -a_j, -a_i, m), so that
// with D = dth_b - dth_o both ends read yth += K D + c2 dv_b + c3 dv_o and
// yv += c2 D + m dv_o; and (dcoef, grad P_ref) of every output.
__global__ void k_for_tape(int nslots, int nout, const int2 *slots, const int *out_bus, const double4 *coef,
                           const double *dcoef, const double *refg_th, const double *refg_v, double4 *scoef,
                           double4 *ometa) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nslots) {
    const int2 sl = slots[t];
    double4 k = sl.x >= 0 ? coef[sl.x] : make_double4(0.0, 0.0, 0.0, 0.0);
    if (sl.y & 1) k = make_double4(k.x, -k.z, -k.y, k.w);   // b is the to-end
    scoef[t] = k;
  } else if (t - nslots < nout) {
    const int o = t - nslots, b = out_bus[o];
    ometa[o] = make_double4(dcoef[b], refg_th[b], refg_v[b], 0.0);
  }
}

// SpMulAdd HW = Y_p + G_p^T Psi: a CTA = 32 p rows x 32 columns,
// warp per p row (4 each), lane per column, the G_p entries' Psi loads four at a
// time in flight; the tile then leaves through shared memory so that the
// transposed layout (H^T rows, the multi-GPU slabs) is written 256 B per warp
// store instead of one 8-byte sector per lane.
__global__ void __launch_bounds__(kThreads) k_muladd(SegParams h) {
  // HW = Y_p + G_p^T Psi (SpMulAdd).  Warp w takes four
  // consecutive p rows (cp0 + 4w ..).  G_p^T Psi: the L^T sweep left one partial
  // row per (p column, block) run (Mp, k_blk MODE_LT epilogue; runs numbered by
  // p column, so the four rows' runs are contiguous): the partials are added in
  // run order, then the entries on separator rows (Psi rows, CSC order).
  // Without partials (h.Mp null) every G_p entry is taken from Psi (CSC order).
  // Lane = batch column; up to 8 row loads in flight.
  __shared__ double T[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // blockIdx.x = column chunk (fastest: the CTAs of one p group read whole
  // rows together), blockIdx.y = p group
  const int cp0 = blockIdx.y * 32, col = blockIdx.x * 32 + lane;
  const int rb = cp0 + 4 * warp;   // this warp's first p row
  // the group's items (static, upload): target row j, source (Y_p row, the Pg
  // diagonal 2 c2 w, an L^T partial row, a Psi row with its G_p value), in the
  // order each row adds them; one coalesced record load, then up to 8 row loads
  // in flight (r02: the CSC / run pointer chains were 3-4 dependent round trips)
  const int g = rb >> 2;
  const int i0 = g < h.ma_ngrp ? h.ma_gptr[g] : 0, i1 = g < h.ma_ngrp ? h.ma_gptr[g + 1] : 0;
  // this warp's 4 rows accumulate in T[4 warp + j][lane] (shared memory, conflict-free):
  // one load-FMA-store per item and no per-item branch on its target row; every row
  // adds its items in list order (the same order as with register accumulators)
  double *tw = &T[4 * warp][lane];
#pragma unroll
  for (int j = 0; j < 4; ++j) tw[33 * j] = 0.0;
  for (int base = i0; base < i1; base += 32) {
    const int n = min(32, i1 - base);
    int code = 0;
    double coef = 1.0;
    if (lane < n) {
      const int2 it = h.ma_items[base + lane];
      code = it.x;
      const int kind = (code >> 28) & 3;
      coef = kind == 3 ? h.gpc_val[it.y] : kind == 1 ? h.pdiag[code & 0x0fffffff] : 1.0;
    }
    for (int k0 = 0; k0 < n; k0 += 8) {
      double x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int cd = __shfl_sync(0xffffffffu, code, (k0 + k) & 31);
        const int kind = (cd >> 28) & 3, row = cd & 0x0fffffff;
        const double *src = kind == 0 ? h.Yp : kind == 2 ? h.Mp : h.P;
        x[k] = k0 + k >= n ? 0.0 : kind == 1 ? load_W(h, row, col) : src[(long long)row * h.ld + col];
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int cd = __shfl_sync(0xffffffffu, code, (k0 + k) & 31);
        const double v = __shfl_sync(0xffffffffu, coef, (k0 + k) & 31);
        if (k0 + k >= n) break;
        double *t = tw + 33 * ((unsigned)cd >> 30);
        *t = fma(v, x[k], *t);
      }
    }
  }
  if (!h.transposed) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cp = rb + j;
      if (cp < h.n_p && col < h.N) h.HW[hw_index(h, cp, col)] = tw[33 * j];
    }
  }
  if (!h.transposed) return;
  __syncthreads();
#pragma unroll 1
  for (int c = warp; c < 32; c += kThreads / 32) {   // H^T row of column c, p rows cp0 .. cp0 + 31
    const int cc = blockIdx.x * 32 + c;
    if (cc < h.N && cp0 + lane < h.n_p) h.HW[hw_index(h, cp0 + lane, cc)] = T[lane][c];
  }
}

// natural-order copy of an internal block: out[k][col] = sgn * X[zmap[k]][col]
__global__ void k_unpermute(int n_x, int N, int ld, const int *pinv, const double *X, double sgn, double *out,
                            long long ldo) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)n_x * N) return;
  const int k = (int)(idx / N), col = (int)(idx % N);
  out[(long long)k * ldo + col] = sgn * X[(long long)pinv[k] * ld + col];
}

// ============================================================================
// Newton-Raphson projection x(p):
// the right-hand side g in Z-row order (column 0 of the one-column block), and
// the update x <- x - dx with max|dx|
// ============================================================================
__global__ void k_newton_rhs(int n_x, const int *__restrict__ zmap, const double *__restrict__ g, double *X) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n_x) X[(long long)zmap[k] * kSegC] = g[k];
}

__device__ __forceinline__ void atomic_max_nonneg(double *addr, double v) {   // v >= 0: bit order = value order
  atomicMax(reinterpret_cast<unsigned long long *>(addr), (unsigned long long)__double_as_longlong(v));
}

__global__ void k_newton_update(int n_x, const int *__restrict__ zmap, const double *__restrict__ X, double *x,
                                double *dmax) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  double m = 0.0;
  if (k < n_x) {
    const double dx = X[(long long)zmap[k] * kSegC];
    x[k] -= dx;
    m = fabs(dx);
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(dmax, m);
}

__global__ void k_absmax(int n, const double *__restrict__ v, double *out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  double m = k < n ? fabs(v[k]) : 0.0;
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, m);
}

// ============================================================================
// first-order adjoint + reduced gradient, single column
// ============================================================================

__global__ void k_grad_rhs(int n_x, const int *x_bus, const int *x_kind, const int *pinv, const double *refg_th,
                           const double *refg_v, const double *scal, double *X) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_x) return;
  const int b = x_bus[k];
  const double g = x_kind[k] == RH_KIND_THETA ? refg_th[b] : refg_v[b];
  X[(long long)pinv[k] * 32] = -scal[2] * g;
}
__global__ void k_grad_out(int n_x, int n_p, const int *pinv, const int *p_bus, const int *p_kind,
                           const double *c2b, const double *c1b, const double *p, const double *refg_v,
                           const double *scal, const int *gpc_ptr, const int *gpc_row, const double *gpc_val,
                           const double *X, double *lam, double *grad) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n_x) lam[k] = X[(long long)pinv[k] * 32];
  if (k < n_p) {
    const int b = p_bus[k];
    double acc = p_kind[k] == RH_KIND_PG ? 2.0 * c2b[b] * p[k] + c1b[b] : scal[2] * refg_v[b];
    for (int q = gpc_ptr[k]; q < gpc_ptr[k + 1]; ++q) acc += gpc_val[q] * X[(long long)gpc_row[q] * 32];
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

constexpr int kSmemMax = 227 * 1024;   // sm_100 opt-in maximum of dynamic shared memory per block
constexpr int kSmemSM = 228 * 1024;    // shared memory per SM

}  // namespace

constexpr int kNumWs = 3;   // batch workspaces / streams of a full Hessian

struct rh_ctx {
  int device = -1;
  bool host_only = true;
  bool loaded = false, has_state = false, has_mult = false;
  std::string err;
  Analysis A;
  std::vector<void *> pool;   // grid-lifetime device buffers
  long long launches = 0;
  bool timing = false;
  float stage_ms[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};

  // device grid + analysis
  int *bus_type, *lf, *lt, *bl_ptr, *bl_line, *bl_other, *bl_end, *has_gen;
  double *G_ii, *B_ii, *Pd, *Qd, *G_ft, *B_ft, *G_tf, *B_tf, *c2b, *c1b, *c0b;
  int *x_bus, *x_kind, *p_bus, *p_kind, *th_x, *v_x, *pinv;
  int *F_rowptr, *F_diag;
  double *F_val;
  int *status;
  int *diag_pos, *slot_pos, *gp_rptr, *gp_col, *gp_self_pos, *gp_pg_pos, *gp_slot_pos;
  // NEXT-4: Jacobians by column coloring + forward mode (rh_set_jacobian_mode)
  int *col_th, *col_v, *col_pg, *jd_pos, *jd_row, *jd_col, *gd_pos, *gd_row, *gd_col;
  double *JS = nullptr;   // [n_x][ncolors] compressed [J | G_p] S
  int *bl_bus = nullptr;
  double *asm_tP = nullptr, *asm_tQ = nullptr;
  int jac_mode = 0;       // 0 analytic assembly, 1 colored forward mode
  double *gp_val;
  int *gpc_ptr, *gpc_pos, *gpc_row;
  double *gpc_val;
  int *dth_src, *dv_src, *yth_dst, *yv_dst, *o_dth_src, *o_dv_src, *pg_p, *near_ref;
  // segments
  int *seg_row_off, *row_global;
  DSeg dfwd, dbwd;
  int *fwd_src_a, *fwd_src_b, *bwd_src_a, *bwd_src_b, *fwd_dsrc, *bwd_dsrc;
  double *vL, *vUt;   // separator rows' L / U^T entries (k_sep_gather)
  int nnz_fwd = 0, nnz_bwd = 0;
  // refactorization schedule
  int *blk_fo_off, *fo, *ks_ptr, *ks4, *ks_k;
  unsigned short *tgt16;
  int *sb_src, *sb_dense;
  double *Sbuf = nullptr;   // ping-pong partner of Sinv in k_sep_inverse
  double *gj_dbuf = nullptr;
  double *sep_piv = nullptr;   // the separator's Gauss-Jordan pivots (rh_pivot_ratio)   // [2][32][32] next panel's diagonal inverse (lookahead CTA)
  double *nwt = nullptr;       // Newton: max|dx|, max|g| (device scalars)
  unsigned *grid_bar = nullptr;
  int coop_blocks = 1;
  double *dinv_rows, *rowmax;
  double *Sinv = nullptr, *SinvT = nullptr;
  size_t smem_fact_blk = 0, smem_fact_sep = 0;
  // state
  double *x, *p, *th, *v, *pgb, *P, *Q, *g, *refg_th, *refg_v, *scal;
  double2 *cs;
  double *lam, *muP, *muQ, *dcoef, *X1col;
  double4 *coef;
  // workspace
  // batch workspaces: [0] on the caller's stream, [1..] on internal streams so
  // that consecutive batches of a full Hessian overlap (hessian_batches)
  struct Workspace {
    double *Z = nullptr, *P = nullptr, *Tsep = nullptr;
    size_t elems = 0, tsep_elems = 0;
    double *Yp = nullptr;        // [n_p][ld] Y_p of the voltage parameters
    size_t yp_elems = 0;
    double *Mp = nullptr;        // [ma runs][ld] L^T sweep partials of G_p^T Psi (k_muladd adds them)
    size_t mp_elems = 0;
    int *pcols = nullptr;        // Cartesian batch plan: the batch's columns, home-block order
    unsigned *pmask = nullptr;   // and its nonzero L-tile mask [nblk][words]
    int *plist = nullptr;        // and its live tiles: count, then block << 16 | chunk
    int plan_ld = 0;
    int plan_lo = -1, plan_hi = -1;   // the Cartesian batch the plan buffers hold (static per range: reused)
    int *ctr = nullptr;   // k_blk ticket counters of this workspace
  } ws[kNumWs];
  cudaStream_t sti[kNumWs] = {};                        // internal streams of workspaces 1..
  cudaEvent_t ev_fork = nullptr, ev_join[kNumWs] = {};
  cudaEvent_t ev_sa = nullptr, ev_sb = nullptr;          // state_impl fork / join
  double *e2e_buf = nullptr;     // rh_reduced_hessian_host staging (x, p, grad, H)
  cudaStream_t e2e_st = nullptr;
  int *blk_gp_ptr, *blk_gp_loc;
  int *fact_seg_lvl, *fact_lvl_ptr, *fact_order;
  int *top_ptr, *top_fpos_ptr, *top_fpos, *top_fwd_base, *top_bwd_base;
  // bus-unit block sweeps
  DUnit duf{}, dub{}, dubp{};   // dubp: dub pruned for the L^T sweep of Cartesian batches
  double2 *uL = nullptr, *uUt = nullptr, *uU = nullptr, *uLt = nullptr;
  int nrec_f = 0, nrec_b = 0;
  int *uf_src_a, *uf_src_b, *ub_src_a, *ub_src_b;
  double *tL = nullptr, *tUt = nullptr, *tU = nullptr, *tLt = nullptr;   // dense tops inverses
  int maxrx = 0, nsm = 148;
  int smem_x_off = 0, smem_meta_off = 0, smem_tmeta_off = 0, smem_rec_off = 0, smem_doff_off = 0, smem_lvl_off = 0;
  int smem_stride = 0;
  int *blk_ctr = nullptr;
  size_t smem_blk = 0, smem_for = 0;
  int *fg_off, *fg_nout, *fg_obase, *fg_sbase, *fg_ref, *fg_ref_loc, *fg_out_bus;
  int2 *fg_soe;
  int *fg_zlo, *fg_zn, *fg_cp_off, *fg_fill_off;
  int2 *fg_cp, *fg_fill;
  int fg_maxrows = 1;
  int4 *fg_loc, *fg_odst;
  int2 *fg_slots;
  double4 *fg_scoef, *fg_ometa;
  double *pdiag;   // [n_p] 2 c2 of a Pg parameter's generator, else 0 (grid data)
  int *gpe_off, *gpe_row, *gpe_col, *gpe_src, *gpe_split;
  int *gorder = nullptr, *pcb_ptr = nullptr, *pcb = nullptr;   // Cartesian batch plans (k_batch_plan)
  double2 *gpe_rec;
  DenseWs dws;                 // tracking Step 2 (dense.cu)
  // CUDA graph of the fused call (rh_reduced_hessian): captured on the second
  // identical call, replayed afterwards; dropped when any workspace moves
  struct GraphKey {
    const void *x, *p, *grad, *H, *st;
    long long ldh;
    int j0, j1, N, transposed, jac_mode;
    bool operator==(const GraphKey &o) const {
      return x == o.x && p == o.p && grad == o.grad && H == o.H && st == o.st && ldh == o.ldh && j0 == o.j0 &&
             j1 == o.j1 && N == o.N && transposed == o.transposed && jac_mode == o.jac_mode;
    }
  };
  struct GraphSlot {   // [0] rh_reduced_hessian, [1] rh_reduced_hessian_host, [2] a Newton step
    GraphKey seen{}, key{};
    bool valid = false, disabled = false;
    cudaGraphExec_t exec = nullptr;
    long long launches = 0;
  } gslot[3];
  cudaStream_t g_st = nullptr;           // capture / replay stream when the caller's is the legacy one
  cudaEvent_t g_ev[2] = {nullptr, nullptr};
  void drop_graph() {
    for (auto &g : gslot) {
      if (g.exec) cudaGraphExecDestroy(g.exec);
      g.exec = nullptr;
      g.valid = false;
      g.seen = GraphKey{};
    }
  }
  cudaStream_t cp_st = nullptr;   // host copies of finished column blocks (rh_reduced_hessian_host)
  // the fused call's gradient runs on its own stream with its own separator
  // workspace and ticket counters; batches wait for the tape before k_for
  cudaStream_t grad_st = nullptr;
  cudaEvent_t ev_state = nullptr, ev_tape = nullptr;
  cudaEvent_t ev_vl = nullptr;   // separator rows' L / U^T values ready (after R_B1)
  cudaEvent_t ev_ult = nullptr;   // fused call: L^T records (side stream)
  bool tr_pending = false;       // fused call: S^-T not yet launched (reduced_hessian_impl does it)
  bool early_gathered = false;   // the fused call's early batches also formed their separator rhs
  double *grad_tsep = nullptr;
  int sep_maxlen = 1;                          // longest separator row of F (k_fact_sep_rows staging)
  int sep_maxu = 1;                            // most U entries of one separator row's k-steps (staged too)
  // epilogue partial runs of k_blk (analysis.hpp RunRecs): U^T -> separator
  // right-hand sides (sr), L^T -> G_p^T Psi of SpMulAdd (ma)
  struct DRunRecs {
    int nruns = 0, n_ent = 0;
    int *off = nullptr, *slot = nullptr, *src = nullptr, *trow = nullptr;
    double2 *rec = nullptr;   // per-block record regions (run slots static, entries per state)
  } dsr, dma;
  int *ma_run_ptr = nullptr, *ma_sep_ptr = nullptr, *ma_sep_q = nullptr;
  int *ma_gptr = nullptr;        // k_muladd: items of each group of 4 p rows
  int2 *ma_items = nullptr;
  int ma_ngrp = 0;
  int *grad_ctr = nullptr;
  cudaEvent_t tape_wait = nullptr;   // set while a fused call enqueues its batches
  // side stream of the fused call: block-only derived values done; each early L sweep done
  cudaEvent_t ev_derived = nullptr, ev_early[kNumWs] = {};
  // split U sweep of Cartesian batches (k_spike): per-block spikes, recomputed per state
  double *Msp = nullptr, *Mfrag = nullptr;   // spikes: sweep output [n_x][kSpLd], A-fragment order
  bool spike_ok = false, spike_pending = false;
  cudaEvent_t ev_spike = nullptr;
  cudaStream_t spk_st = nullptr;
  struct TMapEntry {
    const double *base;
    int ld;
    void *dev;   // [2] CUtensorMap in device memory: boxes of 64 and 8 rows
  };
  std::vector<TMapEntry> tmaps;   // k_blk 2D TMA maps per (buffer, ld)
  cudaEvent_t ev_cp = nullptr;
  cudaEvent_t ev_trk[3] = {nullptr, nullptr, nullptr};

  void free_all() {
    drop_graph();
    if (g_st) cudaStreamDestroy(g_st), g_st = nullptr;
    for (auto &e : g_ev)
      if (e) cudaEventDestroy(e), e = nullptr;
    dense_ws_free(dws);
    for (auto &e : tmaps) cudaFree(e.dev);
    tmaps.clear();
    if (cp_st) cudaStreamDestroy(cp_st), cp_st = nullptr;
    if (grad_st) cudaStreamDestroy(grad_st), grad_st = nullptr;
    if (ev_state) cudaEventDestroy(ev_state), ev_state = nullptr;
    if (ev_tape) cudaEventDestroy(ev_tape), ev_tape = nullptr;
    if (ev_vl) cudaEventDestroy(ev_vl), ev_vl = nullptr;
    if (ev_ult) cudaEventDestroy(ev_ult), ev_ult = nullptr;
    if (grad_tsep) cudaFree(grad_tsep), grad_tsep = nullptr;
    if (grad_ctr) cudaFree(grad_ctr), grad_ctr = nullptr;
    tape_wait = nullptr;
    if (ev_derived) cudaEventDestroy(ev_derived), ev_derived = nullptr;
    if (ev_spike) cudaEventDestroy(ev_spike), ev_spike = nullptr;
    if (spk_st) cudaStreamDestroy(spk_st), spk_st = nullptr;
    for (auto &e : ev_early)
      if (e) cudaEventDestroy(e), e = nullptr;
    if (ev_cp) cudaEventDestroy(ev_cp), ev_cp = nullptr;
    for (auto &e : ev_trk)
      if (e) cudaEventDestroy(e), e = nullptr;
    for (void *q : pool) cudaFree(q);
    pool.clear();
    for (auto &w : ws) {
      if (w.Z) cudaFree(w.Z);
      if (w.P) cudaFree(w.P);
      if (w.Tsep) cudaFree(w.Tsep);
      if (w.pcols) cudaFree(w.pcols);
      if (w.pmask) cudaFree(w.pmask);
      if (w.plist) cudaFree(w.plist);
      if (w.Yp) cudaFree(w.Yp);
      if (w.Mp) cudaFree(w.Mp);
      w = Workspace();
    }
    dsr = DRunRecs();   // device arrays were in the pool
    dma = DRunRecs();
    ma_run_ptr = ma_sep_ptr = ma_sep_q = nullptr;
    ma_gptr = nullptr;
    ma_items = nullptr;
    ma_ngrp = 0;
    if (e2e_buf) cudaFree(e2e_buf);
    if (e2e_st) cudaStreamDestroy(e2e_st);
    for (int k = 0; k < kNumWs; ++k) {
      if (sti[k]) cudaStreamDestroy(sti[k]);
      if (ev_join[k]) cudaEventDestroy(ev_join[k]);
      sti[k] = nullptr;
      ev_join[k] = nullptr;
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_sa) cudaEventDestroy(ev_sa);
    if (ev_sb) cudaEventDestroy(ev_sb);
    ev_sa = ev_sb = nullptr;
    e2e_buf = nullptr;
    e2e_st = nullptr;
    ev_fork = nullptr;
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

size_t fact_smem_bytes(const Analysis &A) {
  return (size_t)(A.max_blk_fnnz + A.rmax + 2) * 8 + (size_t)A.max_blk_ks * 20 + (size_t)A.max_blk_tgt * 2 + 64 +
         16 + (size_t)A.rmax * (16 + 8 + 4) + kFactLvl * 4 + 64;   // per-row metadata
}

size_t blk_smem_layout(const Analysis &A, int *off7);
bool blk_smem_fits(const Analysis &A, size_t lim) {
  int o[7];
  return 2 * (blk_smem_layout(A, o) + 1024) <= lim;   // two CTAs per SM, + static shared memory
}


// shared-memory carve-up of k_blk (2 CTAs per SM): the X tile, then one
// block's unit schedule.  Returns the total bytes.
int blk_max_rows(const Analysis &A) {   // tile rows, incl. the L sweep's G_p entry records behind the block rows
  int m = std::max(A.ufwd.max_rows, A.ubwd.max_rows);
  for (int s = 0; s < A.nblk; ++s) {
    const int nr = A.seg_row_off[s + 1] - A.seg_row_off[s], ne = A.gpe_off[s + 1] - A.gpe_off[s];
    m = std::max(m, nr + (16 * ne + 48 + kRowB - 1) / kRowB);
    m = std::max(m, nr + (16 * (A.sr.off[s + 1] - A.sr.off[s]) + kRowB - 1) / kRowB);   // U^T: separator run records
    m = std::max(m, nr + (A.bwd.ext_off[s + 1] - A.bwd.ext_off[s]) +                     // L^T: staged separator rows,
                        (16 * (A.ma.off[s + 1] - A.ma.off[s]) + kRowB - 1) / kRowB);      // then G_p run records
  }
  return m;
}

size_t blk_smem_layout(const Analysis &A, int *off7) {
  auto al = [](size_t x) { return (x + 127) & ~(size_t)127; };
  const int maxrx = blk_max_rows(A);
  size_t off = 0;
  off7[0] = (int)off;
  off += al((size_t)maxrx * kBC * 8);
  off7[1] = (int)off;
  off += al((size_t)std::max(A.ufwd.max_units, A.ubwd.max_units) * 16);
  off7[2] = (int)off;
  off += al((size_t)32 * kTopLd * 8 + 128);   // dense tops inverse + tops rows
  off7[3] = (int)off;
  off += al((size_t)std::max(A.ufwd.max_rec, A.ubwd.max_rec) * 16);
  off7[4] = (int)off;
  off += al((size_t)std::max(A.ufwd.max_doff, A.ubwd.max_doff) * 4);
  off7[5] = (int)off;
  off += al(UnitSweep::kLvl * 4);
  off7[6] = (int)off;
  return off;
}

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
  // Z and P rows are stored in SEGMENT order (blocks, then the separator, each
  // contiguous): zrow[factor row] = segment position; zmap[natural x] = Z row.
  std::vector<int32_t> zrow(A.n_x), zmap(A.n_x);
  for (int q = 0; q < A.n_x; ++q) zrow[A.row_global[q]] = q;
  for (int k = 0; k < A.n_x; ++k) zmap[k] = zrow[A.pinv[k]];
  auto zr = [&](std::vector<int32_t> v) {  // >= 0 entries are factor rows -> Z rows
    for (auto &x : v)
      if (x >= 0) x = zrow[x];
    return v;
  };
  UP(th_x, A.th_x); UP(v_x, A.v_x); UP(pinv, zmap);
  UP(F_rowptr, A.F_rowptr); UP(F_diag, A.F_diag);
  UP(diag_pos, A.diag_pos); UP(slot_pos, A.slot_pos); UP(gp_rptr, A.gp_rptr); UP(gp_col, A.gp_col);
  UP(gp_self_pos, A.gp_self_pos); UP(gp_pg_pos, A.gp_pg_pos); UP(gp_slot_pos, A.gp_slot_pos);
  UP(col_th, A.col_th); UP(col_v, A.col_v); UP(col_pg, A.col_pg);
  UP(jd_pos, A.jd_pos); UP(jd_row, A.jd_row); UP(jd_col, A.jd_col);
  UP(gd_pos, A.gd_pos); UP(gd_row, A.gd_row); UP(gd_col, A.gd_col);
  chk(c->JS = dalloc<double>((size_t)A.n_x * std::max(1, A.ncolors), P));
  UP(bl_bus, A.bl_bus);
  chk(c->asm_tP = dalloc<double>((size_t)std::max(1, 2 * A.n_line), P));
  chk(c->asm_tQ = dalloc<double>((size_t)std::max(1, 2 * A.n_line), P));
  UP(gpc_ptr, A.gpc_ptr); UP(gpc_pos, A.gpc_pos); UP(gpc_row, zr(A.gpc_row));
  UP(dth_src, zr(A.dth_src)); UP(dv_src, zr(A.dv_src)); UP(yth_dst, zr(A.yth_dst)); UP(yv_dst, zr(A.yv_dst));
  UP(pg_p, A.pg_p); UP(near_ref, A.near_ref);
  UP(seg_row_off, A.seg_row_off); UP(row_global, A.row_global);
  UP(fact_seg_lvl, A.fact_seg_lvl); UP(fact_lvl_ptr, A.fact_lvl_ptr); UP(fact_order, A.fact_order);
  UP(top_ptr, A.top_ptr); UP(top_fpos_ptr, A.top_fpos_ptr); UP(top_fpos, A.top_fpos);
  UP(top_fwd_base, A.top_fwd_base); UP(top_bwd_base, A.top_bwd_base);
  UP(blk_gp_ptr, A.blk_gp_ptr); UP(blk_gp_loc, A.blk_gp_loc);
  UP(fwd_src_a, A.fwd.src_a); UP(fwd_src_b, A.fwd.src_b); UP(bwd_src_a, A.bwd.src_a); UP(bwd_src_b, A.bwd.src_b);
  UP(fwd_dsrc, A.fwd.dsrc); UP(bwd_dsrc, A.bwd.dsrc);
  UP(blk_fo_off, A.blk_fo_off); UP(fo, A.fo); UP(ks_ptr, A.ks_ptr); UP(ks4, A.ks4); UP(ks_k, A.ks_k);
  chk(c->tgt16 = reinterpret_cast<unsigned short *>(dalloc_copy(A.tgt16, P)));
  UP(sb_src, A.sb_src); UP(sb_dense, A.sb_dense);
#undef UP
  auto mkseg = [&](DSeg &D, const SegSweep &S0) {
    SegSweep S = S0;
    for (auto &x : S.ext_rows) x = zrow[x];
    {  // separator external entries: factor rows -> Z rows
      const int qb = S.lvl_ptr[S.seg_lvl[A.nblk]], qe = S.lvl_ptr[S.seg_lvl[A.nblk + 1] - 1];
      for (int q = qb; q < qe; ++q)
        for (int e = S.rptr[q]; e < S.rext[q]; ++e) S.dep[e] = zrow[S.dep[e]];
    }
    int *a, *b, *o, *r, *x, *d, *eo, *er;
    chk(eo = dalloc_copy(S.ext_off, P));
    chk(er = dalloc_copy(S.ext_rows, P));
    D.ext_off = eo;
    D.ext_rows = er;
    chk(a = dalloc_copy(S.seg_lvl, P));
    chk(b = dalloc_copy(S.lvl_ptr, P));
    chk(o = dalloc_copy(S.order, P));
    chk(r = dalloc_copy(S.rptr, P));
    chk(x = dalloc_copy(S.rext, P));
    chk(d = dalloc_copy(S.dep, P));
    D.seg_lvl = a;
    D.lvl_ptr = b;
    D.order = o;
    D.rptr = r;
    D.rext = x;
    D.dep = d;
  };
  mkseg(c->dfwd, A.fwd);
  {  // runs of one block in the separator rows' external dependencies (fwd), for the Cartesian batch mask
    std::vector<int32_t> ds(std::max<size_t>(1, A.fwd.dep.size()), -1);
    const int qb = A.fwd.lvl_ptr[A.fwd.seg_lvl[A.nblk]], qe = A.fwd.lvl_ptr[A.fwd.seg_lvl[A.nblk + 1] - 1];
    for (int q = qb; q < qe; ++q)
      for (int e = A.fwd.rptr[q]; e < A.fwd.rext[q]; ++e) ds[e] = A.seg_of[A.fwd.dep[e]];
    // runs of one block in every separator row's external entries
    std::vector<int32_t> gp(1, 0), gb, ge;
    for (int q = qb; q < qe; ++q) {
      for (int e = A.fwd.rptr[q]; e < A.fwd.rext[q]; ++e)
        if (e == A.fwd.rptr[q] || ds[e] != ds[e - 1]) {
          gb.push_back(ds[e]);
          ge.push_back(e + 1);
        } else {
          ge.back() = e + 1;
        }
      gp.push_back((int)gb.size());
    }
    // k_blk epilogue partials: per-block record regions (analysis.hpp RunRecs)
    auto up_runs = [&](const Analysis::RunRecs &R, rh_ctx::DRunRecs &D) {
      D.nruns = R.nruns;
      D.n_ent = (int)R.ent_src.size();
      std::vector<int32_t> init(R.init);
      if (init.empty()) init.assign(4, 0);
      chk(D.off = dalloc_copy(R.off, P));
      chk(D.rec = reinterpret_cast<double2 *>(dalloc_copy(init, P)));
      if (D.n_ent) {
        chk(D.slot = dalloc_copy(R.ent_slot, P));
        chk(D.src = dalloc_copy(R.ent_src, P));
        chk(D.trow = dalloc_copy(R.ent_trow, P));
      }
    };
    up_runs(A.sr, c->dsr);
    up_runs(A.ma, c->dma);
    {
      std::vector<int32_t> sq(A.ma_sep_q);
      if (sq.empty()) sq.push_back(0);
      chk(c->ma_run_ptr = dalloc_copy(A.ma_run_ptr, P));
      chk(c->ma_sep_ptr = dalloc_copy(A.ma_sep_ptr, P));
      chk(c->ma_sep_q = dalloc_copy(sq, P));
      // k_muladd items per group of 4 p rows: (target j << 30 | kind << 28 | row, CSC position);
      // kind 0 Y_p row, 1 Pg diagonal (2 c2 w), 2 L^T partial row (run), 3 Psi row x G_p value
      const std::vector<int32_t> zgr = zr(A.gpc_row);
      const bool part = A.ma.nruns > 0;
      std::vector<int32_t> items, gptr(1, 0);
      const int ng = (A.n_p + 3) / 4;
      for (int gi = 0; gi < ng; ++gi) {
        for (int j = 0; j < 4 && 4 * gi + j < A.n_p; ++j) {
          const int cp = 4 * gi + j;
          auto push = [&](int kind, int row, int q) {
            items.push_back((int32_t)((unsigned)j << 30 | (unsigned)kind << 28 | (unsigned)row));
            items.push_back(q);
          };
          push(A.p_kind[cp] == RH_KIND_PG ? 1 : 0, cp, 0);
          if (part) {
            for (int r = A.ma_run_ptr[cp]; r < A.ma_run_ptr[cp + 1]; ++r) push(2, r, 0);
            for (int e = A.ma_sep_ptr[cp]; e < A.ma_sep_ptr[cp + 1]; ++e) push(3, zgr[A.ma_sep_q[e]], A.ma_sep_q[e]);
          } else {
            for (int q = A.gpc_ptr[cp]; q < A.gpc_ptr[cp + 1]; ++q) push(3, zgr[q], q);
          }
        }
        gptr.push_back((int)items.size() / 2);
      }
      if (items.empty()) items.assign(2, 0);
      c->ma_ngrp = ng;
      chk(c->ma_gptr = dalloc_copy(gptr, P));
      c->ma_items = reinterpret_cast<int2 *>(dalloc_copy(items, P));
      chk(c->ma_items);
    }
    if (gb.empty()) gb.push_back(0), ge.push_back(0);
    int *g1, *g2, *g3;
    chk(g1 = dalloc_copy(gp, P));
    chk(g2 = dalloc_copy(gb, P));
    chk(g3 = dalloc_copy(ge, P));
    c->dfwd.grp_ptr = g1;
    c->dfwd.grp_blk = g2;
    c->dfwd.grp_end = g3;
  }
  {  // Cartesian batch plans: blocks touched by each p column (rows of G_p's column
     // in a block), and all p columns ordered by their first touched block, then index
    const int np_ = A.n_p;
    std::vector<int32_t> ptr(np_ + 1, 0), blk, key(np_), ord(np_);
    for (int j = 0; j < np_; ++j) {
      std::vector<int32_t> t;
      for (int q = A.gpc_ptr[j]; q < A.gpc_ptr[j + 1]; ++q) {
        const int sg = A.seg_of[A.gpc_row[q]];
        if (sg < A.nblk) t.push_back(sg);
      }
      std::sort(t.begin(), t.end());
      t.erase(std::unique(t.begin(), t.end()), t.end());
      key[j] = t.empty() ? A.nblk : t[0];
      blk.insert(blk.end(), t.begin(), t.end());
      ptr[j + 1] = (int)blk.size();
      ord[j] = j;
    }
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return key[a] < key[b]; });
    if (blk.empty()) blk.push_back(0);
    if (ord.empty()) ord.push_back(0);
    chk(c->gorder = dalloc_copy(ord, P));
    chk(c->pcb_ptr = dalloc_copy(ptr, P));
    chk(c->pcb = dalloc_copy(blk, P));
  }
  mkseg(c->dbwd, A.bwd);
  auto mkunit = [&](DUnit &D, const UnitSweep &U, const DSeg &S) {
    D.meta = reinterpret_cast<const int4 *>(dalloc_copy(U.meta, P));
    chk(D.meta);
    chk(D.top_rows = dalloc_copy(U.top_rows, P));
    chk(D.unit_off = dalloc_copy(U.unit_off, P));
    chk(D.tmeta_off = dalloc_copy(U.tmeta_off, P));
    chk(D.lvl = dalloc_copy(U.lvl, P));
    chk(D.rec_off = dalloc_copy(U.rec_off, P));
    chk(D.doff_off = dalloc_copy(U.doff_off, P));
    chk(D.doff = dalloc_copy(U.doff, P));
    std::vector<int32_t> ord(A.nblk);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return U.cost[x] > U.cost[y]; });
    chk(D.blk_order = dalloc_copy(ord, P));
    D.ext_off = S.ext_off;
    D.ext_rows = S.ext_rows;
  };
  {  // staged tensor projection tiles; delta sources and outputs -> Z rows
    const ForGroups &F = A.fg;
    std::vector<int32_t> loc = F.loc, dst = F.out_dst, soe(F.slots.size());
    for (size_t i = 0; i < loc.size(); i += 4) {
      if (loc[i] >= 0) loc[i] = zrow[loc[i]];
      if (loc[i + 1] >= 0) loc[i + 1] = zrow[loc[i + 1]];
    }
    for (size_t i = 0; i < dst.size(); i += 4) {
      if (dst[i] >= 0) dst[i] = zrow[dst[i]];
      if (dst[i + 1] >= 0) dst[i + 1] = zrow[dst[i + 1]];
    }
    // staging rows of every group: the outputs' Z row range [zlo, zlo + zn) first
    // (rows of halo buses inside it are shared), then per-row copies and fills
    const int ng = (int)F.grp_nout.size();
    std::vector<int32_t> zlo(ng, 0), zn(ng, 0), cpo(1, 0), fio(1, 0), cp, fi;
    int maxrows = 1;
    for (int gi = 0; gi < ng; ++gi) {
      const int lb = F.grp_off[gi], nl = F.grp_off[gi + 1] - lb, no = F.grp_nout[gi];
      int lo = INT32_MAX, hi = -1;
      for (int i = 0; i < no; ++i)
        for (int k = 0; k < 2; ++k) {
          const int z = loc[4 * (lb + i) + k];
          if (z >= 0) lo = std::min(lo, z), hi = std::max(hi, z);
        }
      int n_a = hi >= lo ? hi - lo + 1 : 0;
      if (n_a > 3 * no + 16 || getenv("RH_FOR_NO_RANGE")) n_a = 0;   // too sparse: per-row copies only
      zlo[gi] = n_a ? lo : 0;
      zn[gi] = n_a;
      int next = n_a;
      for (int l = 0; l < nl; ++l) {
        int rows[2];
        for (int k = 0; k < 2; ++k) {
          const int src = loc[4 * (lb + l) + k];
          if (src >= 0 && n_a && src >= lo && src < lo + n_a) {
            rows[k] = src - lo;
          } else if (src >= 0) {
            rows[k] = next++;
            cp.push_back(rows[k]);
            cp.push_back(src);
          } else {
            rows[k] = next++;
            fi.push_back(rows[k]);
            fi.push_back(src == -1 ? -1 : -(src + 2));
          }
        }
        loc[4 * (lb + l) + 3] = rows[0] | (rows[1] << 16);
      }
      cpo.push_back((int)cp.size() / 2);
      fio.push_back((int)fi.size() / 2);
      maxrows = std::max(maxrows, next);
      for (int q = F.grp_sbase[gi]; q < F.grp_sbase[gi + 1]; ++q) {   // byte offsets of the other end's rows
        const int r = loc[4 * (lb + (F.slots[2 * q + 1] >> 1)) + 3];
        soe[2 * q] = (r & 0xffff) * 256;
        soe[2 * q + 1] = (r >> 16) * 256;
      }
      for (int i = 0; i < no; ++i) {   // per output: (theta row, v row, first slot | slots << 16, own staging rows)
        const int o = F.grp_obase[gi] + i;
        dst[4 * o + 2] = dst[4 * o + 2] | (dst[4 * o + 3] << 16);
        dst[4 * o + 3] = loc[4 * (lb + i) + 3];
      }
    }
    if (cp.empty()) cp.assign(2, 0);
    if (fi.empty()) fi.assign(2, 0);
    chk(c->fg_zlo = dalloc_copy(zlo, P));
    chk(c->fg_zn = dalloc_copy(zn, P));
    chk(c->fg_cp_off = dalloc_copy(cpo, P));
    chk(c->fg_fill_off = dalloc_copy(fio, P));
    c->fg_cp = reinterpret_cast<int2 *>(dalloc_copy(cp, P));
    c->fg_fill = reinterpret_cast<int2 *>(dalloc_copy(fi, P));
    chk(c->fg_cp);
    chk(c->fg_fill);
    c->fg_maxrows = maxrows;
    c->fg_loc = reinterpret_cast<int4 *>(dalloc_copy(loc, P));
    c->fg_odst = reinterpret_cast<int4 *>(dalloc_copy(dst, P));
    c->fg_slots = reinterpret_cast<int2 *>(dalloc_copy(F.slots, P));
    chk(c->fg_loc);
    chk(c->fg_odst);
    chk(c->fg_slots);
    chk(c->fg_soe = reinterpret_cast<int2 *>(dalloc_copy(soe, P)));
    chk(c->fg_out_bus = dalloc_copy(F.out_bus, P));
    chk(c->fg_off = dalloc_copy(F.grp_off, P));
    chk(c->fg_nout = dalloc_copy(F.grp_nout, P));
    chk(c->fg_obase = dalloc_copy(F.grp_obase, P));
    chk(c->fg_sbase = dalloc_copy(F.grp_sbase, P));
    chk(c->fg_ref = dalloc_copy(F.grp_ref, P));
    chk(c->fg_ref_loc = dalloc_copy(F.ref_loc, P));
    chk(c->fg_scoef = dalloc<double4>(soe.size() / 2, P));
    std::vector<double> pdiag(A.n_p, 0.0);
    for (int q = 0; q < A.n_p; ++q)
      if (A.p_kind[q] == RH_KIND_PG) pdiag[q] = 2.0 * A.c2b[A.p_bus[q]];
    chk(c->pdiag = dalloc_copy(pdiag, P));
    chk(c->fg_ometa = dalloc<double4>(F.out_bus.size(), P));
    c->smem_for = (size_t)c->fg_maxrows * 32 * sizeof(double) + (size_t)F.max_slots * 40 + (size_t)F.max_nout * 48;
  }
  mkunit(c->duf, A.ufwd, c->dfwd);
  mkunit(c->dub, A.ubwd, c->dbwd);
  {  // L^T sweep of Cartesian batches (the full Hessian): only Psi rows in the support
     // of G_p and the rows they depend on are ever read (HW = Y_p + G_p^T Psi); the
     // closure runs upward through the L pattern (psi_i needs psi_j for L[j][i] != 0),
     // the other units are dropped from the bwd schedule (dubp; needed rows bitwise
     // unchanged, the dropped rows are never read)
    std::vector<char> need(A.n_x, 0);
    for (int q = 0; q < A.n_x; ++q) {
      bool n = A.gp_rptr[q + 1] > A.gp_rptr[q];
      for (int e = A.F_rowptr[q]; e < A.F_diag[q] && !n; ++e) n = need[A.F_col[e]] != 0;
      need[q] = n;
    }
    const UnitSweep &U = A.ubwd;
    std::vector<int32_t> meta, uoff(1, 0), lvl(U.lvl);
    for (int sb = 0; sb < A.nblk; ++sb) {
      const int ub = U.unit_off[sb], nu = U.unit_off[sb + 1] - ub, r0 = A.seg_row_off[sb];
      const int *lv = U.lvl.data() + (size_t)sb * UnitSweep::kLvl;
      std::vector<int> keep_before(nu + 1, 0);
      for (int u = 0; u < nu; ++u) {
        const int *m = U.meta.data() + 4 * (size_t)(ub + u);
        const bool tops = u >= lv[UnitSweep::kWarps + 1] && u < lv[UnitSweep::kWarps + 2];
        const bool two = (m[3] >> 30) & 1;
        const bool k = tops || need[A.row_global[r0 + m[0] / kRowB]] || (two && need[A.row_global[r0 + m[1] / kRowB]]);
        keep_before[u + 1] = keep_before[u] + (k ? 1 : 0);
        if (k) meta.insert(meta.end(), m, m + 4);
      }
      uoff.push_back(uoff.back() + keep_before[nu]);
      for (int w = 0; w <= UnitSweep::kWarps + 2; ++w) lvl[(size_t)sb * UnitSweep::kLvl + w] = keep_before[lv[w]];
    }
    if (meta.empty()) meta.assign(4, 0);
    c->dubp = c->dub;
    c->dubp.meta = reinterpret_cast<const int4 *>(dalloc_copy(meta, P));
    chk(c->dubp.meta);
    chk(c->dubp.unit_off = dalloc_copy(uoff, P));
    chk(c->dubp.lvl = dalloc_copy(lvl, P));
    if (getenv("RH_NO_LT_PRUNE")) c->dubp = c->dub;
  }
  c->nrec_f = (int)A.ufwd.src_a.size() / 2;
  c->nrec_b = (int)A.ubwd.src_a.size() / 2;
  chk(c->uf_src_a = dalloc_copy(A.ufwd.src_a, P));
  chk(c->uf_src_b = dalloc_copy(A.ufwd.src_b, P));
  chk(c->ub_src_a = dalloc_copy(A.ubwd.src_a, P));
  chk(c->ub_src_b = dalloc_copy(A.ubwd.src_b, P));
  for (double **t : {&c->tL, &c->tUt, &c->tU, &c->tLt}) chk(*t = dalloc<double>((size_t)A.nblk * 32 * kTopLd, P));
  chk(c->blk_ctr = dalloc<int>(16 * (kNumWs + 1), P));   // + the spike sweep's own tickets
  for (int k = 0; k < kNumWs; ++k) c->ws[k].ctr = c->blk_ctr + 16 * k;
  chk(c->gpe_off = dalloc_copy(A.gpe_off, P));
  chk(c->gpe_row = dalloc_copy(A.gpe_row, P));
  chk(c->gpe_col = dalloc_copy(A.gpe_col, P));
  chk(c->gpe_src = dalloc_copy(A.gpe_src, P));
  chk(c->gpe_split = dalloc_copy(A.gpe_split, P));
  chk(c->gpe_rec = dalloc<double2>(std::max<size_t>(1, A.gpe_src.size()), P));
  chk(c->uL = dalloc<double2>(c->nrec_f, P));
  chk(c->uUt = dalloc<double2>(c->nrec_f, P));
  chk(c->uU = dalloc<double2>(c->nrec_b, P));
  chk(c->uLt = dalloc<double2>(c->nrec_b, P));
  {
    int o[7];
    c->maxrx = blk_max_rows(A);
    c->smem_blk = blk_smem_layout(A, o);
    c->smem_stride = o[6];
    c->smem_x_off = o[0];
    c->smem_meta_off = o[1];
    c->smem_tmeta_off = o[2];
    c->smem_rec_off = o[3];
    c->smem_doff_off = o[4];
    c->smem_lvl_off = o[5];
  }
  c->nnz_fwd = (int)A.fwd.dep.size();
  c->nnz_bwd = (int)A.bwd.dep.size();
  std::vector<int32_t> odth(2 * A.n_line), odv(2 * A.n_line);
  const std::vector<int32_t> zdth = zr(A.dth_src), zdv = zr(A.dv_src);
  for (int s = 0; s < 2 * A.n_line; ++s) {
    odth[s] = zdth[A.bl_other[s]];
    odv[s] = zdv[A.bl_other[s]];
  }
  chk(c->o_dth_src = dalloc_copy(odth, P));
  chk(c->o_dv_src = dalloc_copy(odv, P));
  const int nx = A.n_x, np_ = A.n_p, nb = A.n_bus, m = A.n_line;
  chk(c->F_val = dalloc<double>(A.F_col.size(), P));
  chk(c->status = dalloc<int>(1, P));
  chk(c->gp_val = dalloc<double>(A.gp_col.size(), P));
  chk(c->gpc_val = dalloc<double>(A.gp_col.size(), P));
  chk(c->vL = dalloc<double>(c->nnz_fwd, P));
  chk(c->vUt = dalloc<double>(c->nnz_fwd, P));
  chk(c->dinv_rows = dalloc<double>(nx, P));
  chk(c->rowmax = dalloc<double>(nx, P));
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
  chk(c->X1col = dalloc<double>((size_t)nx * kSegC, P));
  chk(c->coef = dalloc<double4>(m, P));
  const size_t ns2 = (size_t)A.sep_rows * A.sep_rows;
  chk(c->Sinv = dalloc<double>(ns2, P));
  chk(c->SinvT = dalloc<double>(ns2, P));
  chk(c->Sbuf = dalloc<double>(std::max<size_t>(ns2, 1), P));
  chk(c->grid_bar = dalloc<unsigned>(2, P));
  chk(c->gj_dbuf = dalloc<double>(2 * 32 * 32, P));
  chk(c->sep_piv = dalloc<double>(std::max(1, A.sep_rows), P));
  chk(c->nwt = dalloc<double>(4, P));
  {  // split U sweep (k_spike): every block's staged separator rows fit the spike stride
    int mx = 0;
    for (int s = 0; s < A.nblk; ++s) mx = std::max(mx, A.bwd.ext_off[s + 1] - A.bwd.ext_off[s]);
    // (small grids are launch-latency-bound: the split adds three launches per state and
    // batch and measured slower on case1354 (0.28 -> 0.31 ms), neutral on case2869)
    c->spike_ok = A.sep_rows > 0 && A.nblk > 0 && mx <= 4 * kSpQ && A.max_seg_rows <= 8 * kSpMt &&
                  (A.n_x >= 8192 || getenv("RH_SPIKE")) && !getenv("RH_NO_SPIKE");
    if (c->spike_ok) {
      chk(c->Msp = dalloc<double>((size_t)nx * kSpLd, P));
      chk(c->Mfrag = dalloc<double>((size_t)A.nblk * kSpMt * kSpQ * 32, P));
    }
  }
  if (!ok) return fail(c, RH_E_NOMEM, "device allocation failed while loading the grid");
  // shared-memory footprints
  c->smem_fact_blk = fact_smem_bytes(A);
  {  // opt-in dynamic shared memory: the device maximum minus each kernel's static shared memory
    int optin = kSmemMax;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
    auto allow = [&](const void *fn) {
      cudaFuncAttributes fa;
      if (cudaFuncGetAttributes(&fa, fn) == cudaSuccess)
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
    };
    allow((const void *)k_fact_blocks);
    allow((const void *)k_blk);
    allow((const void *)k_sep_inverse);
    allow((const void *)k_for);
    allow((const void *)k_sep_gemm);
    cudaGetLastError();
  }
  cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, c->device);
  cudaError_t e = cudaMemset(c->X1col, 0, (size_t)nx * kSegC * sizeof(double));
  if (e == cudaSuccess) e = cudaMemset(c->blk_ctr, 0, 16 * (kNumWs + 1) * sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(c->grid_bar, 0, 2 * sizeof(unsigned));
  {  // R_B1 stages each separator row in shared memory (k_fact_sep_rows)
    int ml = 1;
    for (int q = A.seg_row_off[A.nblk]; q < A.seg_row_off[A.nblk + 1]; ++q) {
      const int r = A.row_global[q];
      ml = std::max(ml, A.F_rowptr[r + 1] - A.F_rowptr[r]);
    }
    c->sep_maxlen = ml;
    int mu = 1;   // the most U entries a separator row's k-steps read (their targets are contiguous)
    for (int q = A.seg_row_off[A.nblk]; q < A.seg_row_off[A.nblk + 1]; ++q) {
      const int k0 = A.ks_ptr[q], k1 = A.ks_ptr[q + 1];
      if (k1 > k0) mu = std::max(mu, A.ks4[4 * (k1 - 1) + 3] + A.ks4[4 * (k1 - 1) + 2] - A.ks4[4 * k0 + 3]);
    }
    c->sep_maxu = mu;
    const size_t sm = sizeof(double) * (kThreads / 32) * sep_warp_doubles(ml, mu);
    if (sm > 48 * 1024 && e == cudaSuccess)
      e = cudaFuncSetAttribute(k_fact_sep_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  }
  {  // co-resident CTAs of k_sep_inverse (cooperative launch)
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sep_inverse, 256, gj_smem_bytes());
    c->coop_blocks = std::max(1, per_sm) * c->nsm;
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return fail(c, RH_E_CUDA, std::string("upload: ") + cudaGetErrorString(e));
  return RH_OK;
}

int ensure_tsep(rh_ctx *c, int ld, int k = 0) {
  auto &w = c->ws[k];
  // Tsep + run partials + the Cartesian nonzero-row flags ([ld / 32][ns] bytes)
  const size_t need = (size_t)ld * (size_t)(std::max(1, c->A.sep_rows) + c->dsr.nruns) +
                      ((size_t)(ld / 32) * ((std::max(1, c->A.sep_rows) + 15) & ~15) + 7) / 8;
  if (need <= w.tsep_elems) return RH_OK;
  c->drop_graph();   // the captured fused call points at the old buffer
  if (w.Tsep) cudaFree(w.Tsep);
  w.Tsep = nullptr;
  w.tsep_elems = 0;
  if (cudaMalloc(&w.Tsep, need * sizeof(double)) != cudaSuccess || cudaMemset(w.Tsep, 0, need * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    return fail(c, RH_E_NOMEM, "workspace allocation failed");
  }
  w.tsep_elems = need;
  return RH_OK;
}

int ensure_ws(rh_ctx *c, int ld, int k = 0) {
  auto &w = c->ws[k];
  const size_t need = (size_t)ld * (size_t)c->A.n_x;
  if (int rc = ensure_tsep(c, ld, k)) return rc;
  const size_t nyp = (size_t)ld * (size_t)std::max(1, c->A.n_p);
  if (nyp > w.yp_elems) {
    c->drop_graph();
    if (w.Yp) cudaFree(w.Yp);
    w.Yp = nullptr;
    w.yp_elems = 0;
    if (cudaMalloc(&w.Yp, nyp * sizeof(double)) != cudaSuccess || cudaMemset(w.Yp, 0, nyp * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return fail(c, RH_E_NOMEM, "workspace allocation failed");
    }
    w.yp_elems = nyp;
  }
  const size_t nmp = (size_t)ld * (size_t)std::max(1, c->dma.nruns);
  if (nmp > w.mp_elems) {
    c->drop_graph();
    if (w.Mp) cudaFree(w.Mp);
    w.Mp = nullptr;
    w.mp_elems = 0;
    if (cudaMalloc(&w.Mp, nmp * sizeof(double)) != cudaSuccess || cudaMemset(w.Mp, 0, nmp * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return fail(c, RH_E_NOMEM, "workspace allocation failed");
    }
    w.mp_elems = nmp;
  }
  if (need <= w.elems) return RH_OK;
  c->drop_graph();
  if (w.Z) cudaFree(w.Z);
  if (w.P) cudaFree(w.P);
  w.Z = w.P = nullptr;
  w.elems = 0;
  if (cudaMalloc(&w.Z, need * sizeof(double)) != cudaSuccess || cudaMalloc(&w.P, need * sizeof(double)) != cudaSuccess ||
      cudaMemset(w.Z, 0, need * sizeof(double)) != cudaSuccess || cudaMemset(w.P, 0, need * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    return fail(c, RH_E_NOMEM, "workspace allocation failed");
  }
  w.elems = need;
  return RH_OK;
}

// Cartesian batch plan buffers of workspace k for batches of width <= ld
int ensure_plan(rh_ctx *c, int ld, int k) {
  auto &w = c->ws[k];
  if (ld <= w.plan_ld) return RH_OK;
  c->drop_graph();
  if (w.pcols) cudaFree(w.pcols);
  if (w.pmask) cudaFree(w.pmask);
  if (w.plist) cudaFree(w.plist);
  w.pcols = nullptr;
  w.pmask = nullptr;
  w.plist = nullptr;
  w.plan_ld = 0;
  const size_t words = (size_t)(ld / 32 + 31) / 32;
  if (cudaMalloc(&w.pcols, (size_t)ld * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&w.pmask, (size_t)std::max(1, c->A.nblk) * words * sizeof(unsigned)) != cudaSuccess ||
      cudaMalloc(&w.plist, ((size_t)std::max(1, c->A.nblk) * (ld / 32) + 1) * sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    return fail(c, RH_E_NOMEM, "plan allocation failed");
  }
  w.plan_ld = ld;
  w.plan_lo = w.plan_hi = -1;
  return RH_OK;
}

// 2D tensor maps of a [n_x][ld] fp64 buffer for k_blk's block-row boxes
// (cuTensorMapEncodeTiled through the runtime's driver entry point, no -lcuda);
// cached per (buffer, ld).  Returns nullptr if unavailable (k_blk then copies rows).
const void *tmap_pair(rh_ctx *c, const double *G, int ld) {
  for (auto &e : c->tmaps)
    if (e.base == G && e.ld == ld) return e.dev;
  using Encode = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<Encode>(fn);
    cudaGetLastError();
  }
  if (!encode || getenv("RH_NO_TMA2D")) return nullptr;
  static_assert(sizeof(CUtensorMap) == kTmapBytes, "tensor map size");
  CUtensorMap m[2];
  const cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)c->A.n_x};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  const cuuint32_t estr[2] = {1, 1};
  const cuuint32_t rows[2] = {(cuuint32_t)kTmaBig, (cuuint32_t)kTmaSmall};
  for (int i = 0; i < 2; ++i) {
    const cuuint32_t box[2] = {(cuuint32_t)kBC, rows[i]};
    if (encode(&m[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(G), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return nullptr;
  }
  void *dev = nullptr;
  if (cudaMalloc(&dev, sizeof m) != cudaSuccess || cudaMemcpy(dev, m, sizeof m, cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaGetLastError();
    if (dev) cudaFree(dev);
    return nullptr;
  }
  c->tmaps.push_back({G, ld, dev});
  return dev;
}

SegParams make_params(rh_ctx *c, int k = 0) {
  SegParams h{};
  const Analysis &A = c->A;
  h.n_x = A.n_x;
  h.n_p = A.n_p;
  h.n_bus = A.n_bus;
  h.nblk = A.nblk;
  h.seg_row_off = c->seg_row_off;
  h.row_global = c->row_global;
  h.fwd = c->dfwd;
  h.bwd = c->dbwd;
  h.vL = c->vL;
  h.vUt = c->vUt;
  h.Z = c->ws[k].Z;
  h.P = c->ws[k].P;
  h.Yp = c->ws[k].Yp;
  h.kblk_group = 4;   // (r02: 4 chunks per ticket, fused step 1.453 -> 1.436 ms; 1: 1.49, 6: 1.47, 8: 1.46)
  if (const char *env = getenv("RH_KBLK_GROUP")) h.kblk_group = std::max(1, atoi(env));   // tuning override
  h.spike = 0;
  h.Msp = c->Msp;
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
  h.ns = A.sep_rows;
  h.sep_off = A.seg_row_off[A.nblk];
  h.Sinv = c->Sinv;
  h.Tsep = c->ws[k].Tsep;
  h.nruns = c->dsr.nruns;
  h.sr_off = c->dsr.off;
  h.sr_rec = c->dsr.rec;
  h.ma_off = c->dma.off;
  h.ma_rec = c->dma.rec;
  h.Mp = c->dma.nruns > 0 ? c->ws[k].Mp : nullptr;
  h.ma_run_ptr = c->ma_run_ptr;
  h.ma_sep_ptr = c->ma_sep_ptr;
  h.ma_sep_q = c->ma_sep_q;
  h.ma_gptr = c->ma_gptr;
  h.ma_items = c->ma_items;
  h.ma_ngrp = c->ma_ngrp;
  h.blk_gp_ptr = c->blk_gp_ptr;
  h.blk_gp_loc = c->blk_gp_loc;
  if (const char *env = getenv("RH_DEBUG")) h.debug = atoi(env);  // timing experiments only
  if (h.debug & (8 | 8192)) {
    static long long *dbg = nullptr;
    if (!dbg) cudaMalloc(&dbg, sizeof(long long) * 26 * 65536);
    h.dbg = dbg;
  }
  h.SinvT = c->SinvT;
  h.uf = c->duf;
  h.ub = c->dub;
  h.ubp = c->dubp;
  h.uL = c->uL;
  h.uUt = c->uUt;
  h.uU = c->uU;
  h.uLt = c->uLt;
  h.tL = c->tL;
  h.tUt = c->tUt;
  h.tU = c->tU;
  h.tLt = c->tLt;
  h.gpe_off = c->gpe_off;
  h.gpe_split = c->gpe_split;
  h.gpe_rec = c->gpe_rec;
  h.maxrx = c->maxrx;
  h.fg_off = c->fg_off;
  h.fg_maxrows = c->fg_maxrows;
  h.fg_zlo = c->fg_zlo;
  h.fg_zn = c->fg_zn;
  h.fg_cp_off = c->fg_cp_off;
  h.fg_fill_off = c->fg_fill_off;
  h.fg_cp = c->fg_cp;
  h.fg_fill = c->fg_fill;
  h.fg_maxout = A.fg.max_nout;
  h.fg_maxslots = A.fg.max_slots;
  h.fg_nout = c->fg_nout;
  h.fg_obase = c->fg_obase;
  h.fg_sbase = c->fg_sbase;
  h.fg_ref = c->fg_ref;
  h.fg_ref_loc = c->fg_ref_loc;
  h.fg_loc = c->fg_loc;
  h.fg_odst = c->fg_odst;
  h.fg_soe = c->fg_soe;
  h.fg_scoef = c->fg_scoef;
  h.fg_ometa = c->fg_ometa;
  h.p_kind = c->p_kind;
  h.pdiag = c->pdiag;
  h.smem_stride = c->smem_stride;
  h.blk_ctr = c->ws[k].ctr;
  h.smem_x_off = c->smem_x_off;
  h.smem_meta_off = c->smem_meta_off;
  h.smem_tmeta_off = c->smem_tmeta_off;
  h.smem_rec_off = c->smem_rec_off;
  h.smem_doff_off = c->smem_doff_off;
  h.smem_lvl_off = c->smem_lvl_off;
  return h;
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
  const int nsl = (int)A.fg.slots.size() / 2, nout = (int)A.fg.out_bus.size();
  k_for_tape<<<nblk(nsl + nout), kThreads, 0, st>>>(nsl, nout, c->fg_slots, c->fg_out_bus, c->coef, c->dcoef,
                                                   c->refg_th, c->refg_v, c->fg_scoef, c->fg_ometa);
  RH_LAUNCHED(c);
  c->has_mult = true;
  return RH_OK;
}


// one Alg. 2 batch: eight stream-ordered kernels, no host
// synchronization (cf. the two explicit syncs of PAPER.md:798-805).
// W == nullptr with ident_j0 >= 0 selects the Cartesian block e_{j0..j0+N-1}.
// phase: 0 = the whole batch, 1 = only the first block sweep (L, which needs
// nothing of the separator), 2 = the rest (after a phase-1 launch on workspace wsi),
// 3 = only the separator right-hand sides (needs the separator rows' L values, not
// S^-1; after phase 1), 4 = the rest after phases 1 and 3
void dbg_mark(cudaStream_t st, const char *label);
// The blocks' spikes Msp_b = -U_bb^-1 U_bs of the split U sweep (k_spike), once
// per state before the first Cartesian batch: k_blk MODE_U (spike = 2) on
// identity columns of each block's staged separator rows (one or two 32-column
// chunks per block), written in Z's row order with row stride kSpLd.
int ensure_spikes(rh_ctx *c, cudaStream_t st) {
  if (!c->spike_ok || !c->spike_pending) return RH_OK;
  SegParams h = make_params(c, 0);
  h.N = kSpLd;
  h.ld = kSpLd;
  h.Z = const_cast<double *>(c->Msp);
  h.tmZ = tmap_pair(c, c->Msp, kSpLd);
  h.tmP = nullptr;
  h.spike = 2;
  // its own ticket counters: in the fused call it runs on its own stream, concurrently
  // with the early batches' L and Z^0 sweeps (which use the workspaces' counters)
  h.blk_ctr = c->blk_ctr + 16 * kNumWs;
  const int g = (int)std::min<long long>(2LL * c->nsm, (long long)c->A.nblk * (kSpLd / kBC));
  k_blk<<<g, kBlkThreads, c->smem_blk, st>>>(h, MODE_U);
  RH_LAUNCHED(c);
  k_spike_frag<<<dim3(c->A.nblk, kSpMt), kSpQ * 32, 0, st>>>(h, c->Mfrag);
  RH_LAUNCHED(c);
  c->spike_pending = false;
  return RH_OK;
}

int hvp_impl(rh_ctx *c, const double *W, long long ldw, int ident_lo, double *HW, long long ldhw,
             int transposed, int N, cudaStream_t st, double *Zo = nullptr, double *Yxo = nullptr,
             double *Psio = nullptr, long long ldz = 0, int wsi = 0, int phase = 0) {
  if (N <= 0) return RH_OK;
  const Analysis &A = c->A;
  const int ld = (N + kBC - 1) / kBC * kBC;
  int rc = ensure_ws(c, ld, wsi);
  if (rc) return rc;
  if (ident_lo >= 0 && (rc = ensure_plan(c, ld, wsi))) return rc;
  SegParams h = make_params(c, wsi);
  const bool timing = c->timing && phase == 0;
  h.N = N;
  h.ld = ld;
  h.nzf = reinterpret_cast<unsigned char *>(h.Tsep + (long long)ld * (std::max(1, A.sep_rows) + c->dsr.nruns));
  h.tmZ = tmap_pair(c, h.Z, ld);
  h.tmP = tmap_pair(c, h.P, ld);
  h.W = W;
  h.ldw = ldw;
  if (ident_lo >= 0) {   // Cartesian batch e_{ident_lo .. ident_lo + N - 1}: columns in home-block order
    h.icol = c->ws[wsi].pcols;
    h.icol_base = ident_lo;
    h.tmask = c->ws[wsi].pmask;
    h.tlist = c->ws[wsi].plist;
    h.tmask_words = (ld / 32 + 31) / 32;
    auto &wp = c->ws[wsi];
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cst);
    const bool capturing = cst != cudaStreamCaptureStatusNone;
    if ((phase == 0 || phase == 1) && (capturing || !(wp.plan_lo == ident_lo && wp.plan_hi == ident_lo + N))) {
      // the plan of a column range is static (gorder and the G_p blocks): an eager call
      // reuses the workspace's plan of the same range; a captured graph always carries
      // its own plans (graph launches invalidate the cache: graph_run)
      wp.plan_lo = capturing ? -1 : ident_lo;
      wp.plan_hi = capturing ? -1 : ident_lo + N;
      k_batch_plan<<<1, 1024, 0, st>>>(A.n_p, ident_lo, ident_lo + N, c->gorder, c->pcb_ptr, c->pcb, A.nblk,
                                       h.tmask_words, c->ws[wsi].pcols, c->ws[wsi].pmask, ld / kBC,
                                       c->ws[wsi].plist);
      RH_LAUNCHED(c);
    }
    if (getenv("RH_NO_MASK")) h.tmask = nullptr;   // experiment: dense L sweep on the same column order
  }
  h.HW = HW;
  h.ldhw = ldhw;
  h.transposed = transposed;
  const int nb = A.nblk;
  const bool has_sep = A.sep_rows > 0;
  const int gA = (int)std::min<long long>(((h.debug & 64) ? 1LL : 2LL) * c->nsm, (long long)nb * (ld / kBC));   // debug 64: 1 CTA/SM (experiment)
  // column chunks per k_blk ticket: up to 4 (the schedule staged once per ticket), but
  // never fewer tickets than CTAs (small grids keep one chunk per ticket)
  if (!getenv("RH_KBLK_GROUP"))
    h.kblk_group = (int)std::max(1LL, std::min(4LL, (long long)nb * (ld / kBC) / std::max(1, gA)));
  const dim3 gSg(nblk(A.sep_rows, kThreads / 32), ld / 32),
      gSm((ld + GBN - 1) / GBN, (A.sep_rows + GBM - 1) / GBM);
  const dim3 gF((int)A.fg.grp_nout.size(), ld / 32), gM(ld / 32, (A.n_p + 31) / 32);   // k_muladd: column chunks fastest
  const int nx = A.n_x;
  const long long tot = (long long)nx * N;
  cudaEvent_t ev[9];
  if (timing)
    for (auto &e : ev) cudaEventCreate(&e);
  static const char *kMarkNames[kNumWs][9] = {
      {"w0 start", "w0 A_L done", "w0 B_LU done", "w0 A_U done", "w0 FoR done", "w0 A_Ut done", "w0 B_UtLt done",
       "w0 A_Lt done", "w0 MulAdd done"},
      {"w1 start", "w1 A_L done", "w1 B_LU done", "w1 A_U done", "w1 FoR done", "w1 A_Ut done", "w1 B_UtLt done",
       "w1 A_Lt done", "w1 MulAdd done"},
      {"w2 start", "w2 A_L done", "w2 B_LU done", "w2 A_U done", "w2 FoR done", "w2 A_Ut done", "w2 B_UtLt done",
       "w2 A_Lt done", "w2 MulAdd done"}};
  auto mark = [&](int i) {
    if (timing) cudaEventRecord(ev[i], st);
    if (wsi < kNumWs && (phase != 1 || i <= 1) && (phase < 2 || i >= 1)) dbg_mark(st, kMarkNames[wsi][i]);
  };
  // Cartesian batches: split U sweep (k_spike) - Z^0 (into P) right after the L
  // sweep (it needs neither R_B1 nor S^-1: in the fused call it runs while the
  // separator is factored and inverted), the spikes' product once z_ext is known
  const bool split = h.icol && c->spike_ok && has_sep;
  if (phase <= 1) {
    mark(0);
    k_blk<<<gA, kBlkThreads, c->smem_blk, st>>>(h, MODE_L);
    RH_LAUNCHED(c);
    if (split) {
      SegParams hu = h;
      hu.spike = 1;
      k_blk<<<gA, kBlkThreads, c->smem_blk, st>>>(hu, MODE_U);
      RH_LAUNCHED(c);
    }
  }
  if (phase == 1) return RH_OK;
  if (phase != 3) mark(1);
  if (has_sep) {
    if (phase != 4) {
      k_sep_gather<<<gSg, kThreads, 0, st>>>(h, MODE_LU);
      RH_LAUNCHED(c);
    }
    if (phase == 3) return RH_OK;
    if (h.tmask && !getenv("RH_NO_SPMM")) {   // Cartesian batch: S^-1 over T's nonzero rows only
      k_sep_spmm<<<dim3(ld / 32, (A.sep_rows + SPM - 1) / SPM), 256, spmm_smem_bytes(A.sep_rows), st>>>(h);
    } else {
      // reads S^-T: formed on the state's stream (rh_set_state) or, in the fused
      // call, on the gradient stream that the call joins before it returns
      k_sep_gemm<<<gSm, GTHREADS, gemm_smem_bytes(), st>>>(h, MODE_LU);
    }
    RH_LAUNCHED(c);
  }
  if (phase == 3) return RH_OK;
  mark(2);
  if (split)
    k_spike<<<dim3(nb, ld / kBC), kSpThreads, 0, st>>>(h, c->Mfrag);
  else
    k_blk<<<gA, kBlkThreads, c->smem_blk, st>>>(h, MODE_U);
  RH_LAUNCHED(c);
  if ((h.debug & 8) && h.dbg && !split) {  // timing experiment: per-tile cycles of this launch (tools/kblk_prof.py)
    std::vector<long long> hb((size_t)12 * std::min(8192, nb * (ld / kBC)));
    cudaMemcpyAsync(hb.data(), h.dbg, hb.size() * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (FILE *fp = fopen("gpurun_out/kblk_prof.bin", "wb")) {
      fwrite(hb.data(), 8, hb.size(), fp);
      fclose(fp);
    }
  }
  if (Zo) {
    k_unpermute<<<nblk(tot), kThreads, 0, st>>>(nx, N, ld, c->pinv, h.Z, 1.0, Zo, ldz);
    RH_LAUNCHED(c);
  }
  mark(3);
  if (c->tape_wait) RH_CUDA(c, cudaStreamWaitEvent(st, c->tape_wait, 0));   // FoR needs the gradient's tape
  k_for<<<gF, kForThreads, c->smem_for, st>>>(h);
  RH_LAUNCHED(c);
  if ((h.debug & 8192) && h.dbg) {  // timing experiment: per-CTA phase cycles of k_for (tools/kfor_prof.py)
    std::vector<long long> hb((size_t)6 * std::min<long long>(16384, (long long)gF.x * gF.y));
    cudaMemcpyAsync(hb.data(), h.dbg, hb.size() * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (FILE *fp = fopen("gpurun_out/kfor_prof.bin", "wb")) {
      fwrite(hb.data(), 8, hb.size(), fp);
      fclose(fp);
    }
  }
  if (Yxo) {
    k_unpermute<<<nblk(tot), kThreads, 0, st>>>(nx, N, ld, c->pinv, h.P, -1.0, Yxo, ldz);
    RH_LAUNCHED(c);
  }
  mark(4);
  k_blk<<<gA, kBlkThreads, c->smem_blk, st>>>(h, MODE_UT);
  RH_LAUNCHED(c);
  mark(5);
  if (has_sep) {
    k_sep_gather<<<gSg, kThreads, 0, st>>>(h, MODE_UTLT);
    RH_LAUNCHED(c);
    k_sep_gemm<<<gSm, GTHREADS, gemm_smem_bytes(), st>>>(h, MODE_UTLT);
    RH_LAUNCHED(c);
  }
  mark(6);
  k_blk<<<gA, kBlkThreads, c->smem_blk, st>>>(h, MODE_LT);
  RH_LAUNCHED(c);
  if (Psio) {
    k_unpermute<<<nblk(tot), kThreads, 0, st>>>(nx, N, ld, c->pinv, h.P, 1.0, Psio, ldz);
    RH_LAUNCHED(c);
  }
  mark(7);
  k_muladd<<<gM, kThreads, 0, st>>>(h);
  RH_LAUNCHED(c);
  mark(8);
  if (timing) {
    cudaEventSynchronize(ev[8]);
    float tot_ms = 0.f;
    for (int s = 0; s < 8; ++s) {
      cudaEventElapsedTime(&c->stage_ms[s], ev[s], ev[s + 1]);
      tot_ms += c->stage_ms[s];
    }
    c->stage_ms[8] = tot_ms;
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
  // block size: the largest whose shared-memory stages fit
  // Prefer the largest block size that fits AND leaves at least kMinBlocks
  // blocks (few blocks serialize the refactorization and the sweeps on few
  // CTAs: case118 0.46 -> 0.32 ms, case1354 0.42-0.51 -> 0.41 ms; case2869 and
  // case9241 keep 256); otherwise the fitting size with the most blocks.
  constexpr int kMinBlocks = 16;
  std::string msg;
  bool fits = false;
  std::vector<int> cands = {256, 128, 64, 512};
  const bool forced = getenv("RH_RMAX") != nullptr;
  if (forced) cands.insert(cands.begin(), atoi(getenv("RH_RMAX")));  // tuning override
  int fallback = -1, fallback_blocks = 0;
  for (int rmax : cands) {
    msg = analyze(*g, c->A, rmax);
    if (!msg.empty()) return fail(c, RH_E_GRID, msg);
    const Analysis &A = c->A;
    const size_t lim = (size_t)kSmemMax;
    fits =
           (size_t)8 * A.sep_rows * sizeof(double) <= lim &&
           fact_smem_bytes(A) <= lim && blk_smem_fits(A, kSmemSM) && A.max_seg_rows <= kMaxRowsFact &&
           A.ufwd.max_tunits <= UnitSweep::kMaxTopUnits && A.ubwd.max_tunits <= UnitSweep::kMaxTopUnits;
    if (fits && A.nblk > fallback_blocks) {
      fallback = rmax;
      fallback_blocks = A.nblk;
    }
    if (fits && (forced || A.nblk >= kMinBlocks)) break;
    fits = false;
  }
  if (!fits && fallback >= 0) {
    msg = analyze(*g, c->A, fallback);
    if (!msg.empty()) return fail(c, RH_E_GRID, msg);
    fits = true;
  }
  if (!fits) return fail(c, RH_E_GRID, "grid too large for the shared-memory segment kernels");
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
  info->n_blocks = A.nblk;
  info->sep_rows = A.sep_rows;
  info->seg_levels = std::max(A.fwd.max_levels, A.bwd.max_levels);
  int64_t wse = 0;
  for (const auto &w : c->ws) wse += (int64_t)w.elems;
  info->workspace_bytes = wse * 2 * (int64_t)sizeof(double);
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

int rh_segments(const rh_ctx *c, int32_t *segment_of_row) {
  if (!c) return RH_E_ARG;
  if (!c->loaded) return RH_E_ORDER;
  if (segment_of_row) std::copy(c->A.seg_of.begin(), c->A.seg_of.end(), segment_of_row);
  return RH_OK;
}

}  // extern "C"

namespace {
// rh_set_state's work.  With a side stream, the block-only derived values
// (unit-sweep records, tops inverses, G_p records) and `early` (e.g. the first
// block sweeps of Hessian batches) run on `side` as soon as the block factors
// exist, concurrently with the separator's elimination and inversion on `st`;
// `st` joins `side` before the pivot flag is read.
// timing experiment (RH_DEBUG & 1024): events on the caller's stream at stage
// boundaries of the fused call, printed by dbg_report
struct DbgMark {
  const char *label;
  cudaEvent_t ev;
};
std::vector<DbgMark> g_marks;
bool dbg_on() {
  static int v = -1;
  if (v < 0) v = getenv("RH_DEBUG") && (atoi(getenv("RH_DEBUG")) & 1024) ? 1 : 0;
  return v == 1;
}
void dbg_mark(cudaStream_t st, const char *label) {
  if (!dbg_on()) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, st);
  g_marks.push_back({label, e});
}
void dbg_report(cudaStream_t st) {
  if (!dbg_on() || g_marks.empty()) return;
  cudaStreamSynchronize(st);
  cudaDeviceSynchronize();
  std::vector<std::pair<float, const char *>> tl;
  for (auto &m : g_marks) {
    float t = 0.f;
    cudaEventElapsedTime(&t, g_marks[0].ev, m.ev);
    tl.push_back({t, m.label});
  }
  std::stable_sort(tl.begin(), tl.end(), [](const std::pair<float, const char *> &a,
                                            const std::pair<float, const char *> &b) { return a.first < b.first; });
  float prev = 0.f;
  for (auto &m : tl) {
    fprintf(stderr, "  %-28s %8.3f ms  (+%.3f)\n", m.second, m.first, m.first - prev);
    prev = m.first;
  }
  for (auto &m : g_marks) cudaEventDestroy(m.ev);
  g_marks.clear();
}

// NEXT-4: JS = [J | G_p] S by forward-mode tangents (needs line trig and bus
// state of the current point); decompress = overwrite J's and G_p's values
int colored_jacobian(rh_ctx *c, cudaStream_t st, bool decompress) {
  const Analysis &A = c->A;
  const int C = std::max(1, A.ncolors);
  const long long nt = (long long)A.n_bus * C;
  k_jvp_colored<<<(unsigned)((nt + kThreads - 1) / kThreads), kThreads, 0, st>>>(
      A.n_bus, A.ref, C, c->bl_ptr, c->bl_line, c->bl_other, c->bl_end, c->cs, c->G_ft, c->B_ft, c->G_tf, c->B_tf,
      c->G_ii, c->B_ii, c->v, c->th_x, c->v_x, c->col_th, c->col_v, c->col_pg, c->JS);
  RH_LAUNCHED(c);
  if (decompress) {
    const int nj = (int)A.jd_pos.size(), ng = (int)A.gd_pos.size();
    k_decompress<<<nblk(nj + ng), kThreads, 0, st>>>(nj, c->jd_pos, c->jd_row, c->jd_col, c->F_val, ng, c->gd_pos,
                                                     c->gd_row, c->gd_col, c->gp_val, C, c->JS);
    RH_LAUNCHED(c);
  }
  return RH_OK;
}

int check_pivots(rh_ctx *c, cudaStream_t st) {   // reads the refactorization's pivot flag (one sync)
  int status = 0;
  RH_CUDA(c, cudaMemcpyAsync(&status, c->status, sizeof(int), cudaMemcpyDeviceToHost, st));
  RH_CUDA(c, cudaStreamSynchronize(st));
  if (status != 0) {
    c->has_state = c->has_mult = false;
    char buf[160];
    snprintf(buf, sizeof buf, "refactorization: pivot of permuted row %d below 1e-14 * row max", status - 1);
    return fail(c, RH_E_SINGULAR, buf);
  }
  return RH_OK;
}

// CUDA graph of a fused call: `enqueue(cs)`
// enqueues the whole call on cs without the final pivot check.  Captured on the
// second identical call (same key), replayed afterwards; the pivot flag is read
// after each run.  Returns false when the caller should run uncaptured (first
// call, graphs disabled, capture unsupported); else rc holds the result.
template <typename F>
bool graph_run(rh_ctx *c, int slot, const rh_ctx::GraphKey &key, cudaStream_t st, int &rc, F &&enqueue,
               bool mult = true) {
  auto &g = c->gslot[slot];
  if (g.disabled || getenv("RH_NO_GRAPH") || dbg_on()) return false;
  const bool replay = g.valid && key == g.key, capture = !replay && key == g.seen;
  if (!replay && !capture) {
    g.seen = key;
    return false;
  }
  auto cuda = [&](cudaError_t e) {
    if (e == cudaSuccess) return true;
    rc = fail(c, RH_E_CUDA, cudaGetErrorString(e));
    return false;
  };
  if (!cuda(cudaSetDevice(c->device))) return true;
  // the legacy default stream cannot be captured: run on an internal stream
  // ordered after / before the caller's
  cudaStream_t cs = st;
  if (!st) {
    if (!c->g_st && !cuda(cudaStreamCreateWithFlags(&c->g_st, cudaStreamNonBlocking))) return true;
    for (auto &e : c->g_ev)
      if (!e && !cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming))) return true;
    if (!cuda(cudaEventRecord(c->g_ev[0], st)) || !cuda(cudaStreamWaitEvent(c->g_st, c->g_ev[0], 0))) return true;
    cs = c->g_st;
  }
  auto join = [&]() {
    if (!st) {
      cudaEventRecord(c->g_ev[1], cs);
      cudaStreamWaitEvent(st, c->g_ev[1], 0);
    }
  };
  auto finish = [&]() {
    c->has_state = true;
    c->has_mult = mult;   // a state-only replay (Newton) leaves no valid multipliers
    join();
    rc = check_pivots(c, cs);
    return true;
  };
  for (auto &w : c->ws) w.plan_lo = w.plan_hi = -1;   // graphs rebuild their batches' plans
  if (replay) {
    if (!cuda(cudaGraphLaunch(g.exec, cs))) return true;
    c->launches += g.launches;
    return finish();
  }
  if (g.exec) cudaGraphExecDestroy(g.exec);   // this slot only: the others stay valid
  g.exec = nullptr;
  g.valid = false;
  const long long l0 = c->launches;
  cudaGraph_t gr = nullptr;
  if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
    const int rc2 = enqueue(cs);
    const cudaError_t e = cudaStreamEndCapture(cs, &gr);
    cudaGraphExec_t ex = nullptr;
    if (rc2 == RH_OK && e == cudaSuccess && gr && cudaGraphInstantiate(&ex, gr, 0) == cudaSuccess) {
      cudaGraphDestroy(gr);
      g.exec = ex;
      g.key = key;
      g.valid = true;
      g.launches = c->launches - l0;
      c->launches = l0;
      c->err.clear();
      if (!cuda(cudaGraphLaunch(ex, cs))) return true;
      c->launches += g.launches;
      return finish();
    }
    if (gr) cudaGraphDestroy(gr);
  }
  // capture unsupported for this call: run uncaptured from now on
  cudaGetLastError();
  join();
  g.disabled = true;
  c->launches = l0;
  c->err.clear();
  return false;
}

// defer_check: do not read the pivot flag (the caller does, after enqueuing more work)
int state_impl(rh_ctx *c, const double *x, const double *p, cudaStream_t st, cudaStream_t side,
               const std::function<int(cudaStream_t, int)> &early, bool defer_check = false) {
  if (!c || !x || !p) return fail(c, RH_E_ARG, "null argument");
  if (c->host_only) return fail(c, RH_E_NODEV, "host-only context (device = -1)");
  if (!c->loaded) return fail(c, RH_E_ORDER, "no grid loaded");
  RH_CUDA(c, cudaSetDevice(c->device));
  const Analysis &A = c->A;
  const int nx = A.n_x, np_ = A.n_p, nb = A.n_bus, m = A.n_line;
  c->has_state = c->has_mult = false;
  c->spike_pending = true;
  dbg_mark(st, "state start");
  // x, p into the context, zeroed accumulators, bus state and line trig (one launch)
  k_state_prep<<<2 * c->nsm, kThreads, 0, st>>>(nx, np_, x, p, c->x, c->p, (long long)A.F_col.size(), c->F_val,
                                                (long long)A.gp_col.size(), c->gp_val, nb, c->refg_th, c->refg_v,
                                                c->status, c->x_bus, c->x_kind, c->p_bus, c->p_kind, c->th, c->v,
                                                c->pgb, A.ref, A.theta_ref, m, c->lf, c->lt, c->th_x, c->cs);
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
  a.bl_bus = c->bl_bus;
  a.tP = c->asm_tP;
  a.tQ = c->asm_tQ;
  a.n_inc = 2 * m;
  dbg_mark(st, "bus state + line trig");
  if (A.asm_unique && !getenv("RH_ASM_SERIAL")) {
    k_asm_lines<<<nblk(2 * m), kThreads, 0, st>>>(a);
    RH_LAUNCHED(c);
    k_asm_buses<<<nblk(nb), kThreads, 0, st>>>(a);
    RH_LAUNCHED(c);
  } else {
    k_assemble<<<nblk(nb, 128), 128, 0, st>>>(a);
    RH_LAUNCHED(c);
  }
  dbg_mark(st, "k_assemble");
  if (c->jac_mode == 1)
    if (int rc = colored_jacobian(c, st, true)) return rc;
  // numeric refactorization: blocks, separator rows (block updates), separator
  FactParams f{};
  f.nblk = A.nblk;
  f.ns = A.sep_rows;
  f.seg_row_off = c->seg_row_off;
  f.row_global = c->row_global;
  f.fwd_seg_lvl = c->dfwd.seg_lvl;   // blocks: forward subtree-to-warp schedule
  f.fwd_lvl_ptr = c->dfwd.lvl_ptr;
  f.fwd_order = c->dfwd.order;
  f.blk_fo_off = c->blk_fo_off;
  f.fo = c->fo;
  f.F_rowptr = c->F_rowptr;
  f.F_diag = c->F_diag;
  f.F_val = c->F_val;
  f.ks_ptr = c->ks_ptr;
  f.ks_k = c->ks_k;
  f.ks4 = c->ks4;
  f.tgt16 = c->tgt16;
  f.dinv = c->dinv_rows;
  f.rowmax = c->rowmax;
  f.status = c->status;
  f.pivtol = 1e-14;
  f.df = !getenv("RH_FACT_STATIC");   // (RH_FACT_STATIC: the static pieces + tops phases, experiment)
  static long long *fdbg = nullptr;
  const bool fprof = getenv("RH_DEBUG") && (atoi(getenv("RH_DEBUG")) & 128);
  if (fprof) {
    if (!fdbg) cudaMalloc(&fdbg, 8 * 4096 * sizeof(long long));
    f.dbg = fdbg;
  }
  dbg_mark(st, "assembled");
  // dataflow pass: 32 warps (any count works); the static schedule needs its 16
  int fthreads = f.df ? 2 * kSegThreads : kSegThreads;
  if (const char *env = getenv("RH_FACT_THREADS")) fthreads = f.df ? atoi(env) : kSegThreads;   // experiment
  k_fact_blocks<<<A.nblk, fthreads, c->smem_fact_blk, st>>>(f);
  RH_LAUNCHED(c);
  dbg_mark(st, "k_fact_blocks");
  if (fprof) {  // timing experiment: per-block phase stamps (tools/fact_prof.py)
    std::vector<long long> hb((size_t)8 * A.nblk);
    cudaMemcpyAsync(hb.data(), fdbg, hb.size() * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (FILE *fp = fopen("gpurun_out/fact_prof.bin", "wb")) {
      fwrite(hb.data(), 8, hb.size(), fp);
      fclose(fp);
    }
  }
  // block-only values (and `early`) on the side stream while the separator is eliminated on st
  cudaStream_t sb = side ? side : st;
  if (side) {
    if (!c->ev_sa) RH_CUDA(c, cudaEventCreateWithFlags(&c->ev_sa, cudaEventDisableTiming));
    if (!c->ev_sb) RH_CUDA(c, cudaEventCreateWithFlags(&c->ev_sb, cudaEventDisableTiming));
    RH_CUDA(c, cudaEventRecord(c->ev_sa, st));
    RH_CUDA(c, cudaStreamWaitEvent(side, c->ev_sa, 0));
  }
  // the objective and its REF terms (needed by the gradient, not by the factorization)
  k_objective<<<1, 1024, 0, sb>>>(nb, A.ref, c->has_gen, c->c2b, c->c1b, c->c0b, c->pgb, c->P, c->Pd, c->scal);
  RH_LAUNCHED(c);
  if (!A.gpe_src.empty()) {
    const int ne = (int)A.gpe_src.size();
    k_gather_gpe<<<nblk(ne), kThreads, 0, sb>>>(ne, c->gpe_src, c->gpe_row, c->gpe_col, c->gp_val, c->gpe_rec);
    RH_LAUNCHED(c);
  }
  const int ngp = (int)A.gp_col.size();
  if (ngp > 0) {
    k_gather_vals<<<nblk(ngp), kThreads, 0, sb>>>(ngp, c->gpc_pos, c->gp_val, c->gpc_val);
    RH_LAUNCHED(c);
    if (c->dma.n_ent) {   // G_p values into the per-block run record regions (k_blk MODE_LT epilogue)
      k_sr_fill<<<nblk(c->dma.n_ent), kThreads, 0, sb>>>(c->dma.n_ent, c->dma.slot, c->dma.src, c->dma.trow,
                                                          c->gpc_val, c->dma.rec);
      RH_LAUNCHED(c);
    }
  }
  struct GU {
    int n;
    const int *src;
    double2 *dst;
  } gu[] = {{c->nrec_f, c->uf_src_a, c->uL}, {c->nrec_f, c->uf_src_b, c->uUt}, {c->nrec_b, c->ub_src_a, c->uU}};
  for (const GU &q : gu) {
    if (q.n <= 0) continue;
    k_gather_code<<<nblk(2LL * q.n), kThreads, 0, sb>>>(2 * q.n, q.src, c->F_val, reinterpret_cast<double *>(q.dst));
    RH_LAUNCHED(c);
  }
  if (A.max_tops > 0) {
    k_tops_inverse<<<A.nblk, kMaxTops * kMaxTops, 0, sb>>>(c->top_ptr, c->top_fpos_ptr, c->top_fpos, c->F_val,
                                                           c->tL, c->tUt, c->tU, c->tLt);
    RH_LAUNCHED(c);
  }
  if (early) {
    if (!c->ev_derived) RH_CUDA(c, cudaEventCreateWithFlags(&c->ev_derived, cudaEventDisableTiming));
    RH_CUDA(c, cudaEventRecord(c->ev_derived, sb));   // what st needs from the side stream
    if (side && c->spike_ok && A.sep_rows > 0) {   // the split U sweep's spikes on a stream of their own
      if (!c->spk_st) RH_CUDA(c, cudaStreamCreateWithFlags(&c->spk_st, cudaStreamNonBlocking));
      if (!c->ev_spike) RH_CUDA(c, cudaEventCreateWithFlags(&c->ev_spike, cudaEventDisableTiming));
      RH_CUDA(c, cudaStreamWaitEvent(c->spk_st, c->ev_derived, 0));
      if (int rc = ensure_spikes(c, c->spk_st)) return rc;
      RH_CUDA(c, cudaEventRecord(c->ev_spike, c->spk_st));
    }
    const int rc = early(sb, 1);
    if (rc) return rc;
  }
  if (A.sep_rows > 0) {
    dbg_mark(st, "side stream forked");
    f.sep_maxlen = c->sep_maxlen;
    f.sep_maxu = c->sep_maxu;
    k_fact_sep_rows<<<nblk((long long)A.sep_rows * 32), kThreads,
                      sizeof(double) * (kThreads / 32) * sep_warp_doubles(f.sep_maxlen, f.sep_maxu), st>>>(f);
    RH_LAUNCHED(c);
    {  // separator rows' entries of the forward pattern (k_sep_gather): L and U^T values
       // (final after R_B1; the Gauss-Jordan inverse below does not touch F)
      const int qb = A.fwd.lvl_ptr[A.fwd.seg_lvl[A.nblk]], qe = A.fwd.lvl_ptr[A.fwd.seg_lvl[A.nblk + 1] - 1];
      const int e0 = A.fwd.rptr[qb], ne = A.fwd.rptr[qe] - e0;
      if (ne > 0) {
        k_gather_vals<<<nblk(ne), kThreads, 0, st>>>(ne, c->fwd_src_a + e0, c->F_val, c->vL + e0);
        RH_LAUNCHED(c);
        k_gather_vals<<<nblk(ne), kThreads, 0, st>>>(ne, c->fwd_src_b + e0, c->F_val, c->vUt + e0);
        RH_LAUNCHED(c);
        if (c->dsr.n_ent) {   // U^T values into the per-block run record regions (k_blk MODE_UT epilogue)
          k_sr_fill<<<nblk(c->dsr.n_ent), kThreads, 0, st>>>(c->dsr.n_ent, c->dsr.slot, c->dsr.src, c->dsr.trow,
                                                              c->vUt, c->dsr.rec);
          RH_LAUNCHED(c);
        }
      }
    }
    if (early && side) {   // the early batches' separator right-hand sides need these values, not S^-1
      if (!c->ev_vl) RH_CUDA(c, cudaEventCreateWithFlags(&c->ev_vl, cudaEventDisableTiming));
      RH_CUDA(c, cudaEventRecord(c->ev_vl, st));
      RH_CUDA(c, cudaStreamWaitEvent(sb, c->ev_vl, 0));
      if (c->nrec_b > 0) {   // L^T records need R_B1's values, not S^-1: off the critical path too
        k_gather_code<<<nblk(2LL * c->nrec_b), kThreads, 0, sb>>>(2 * c->nrec_b, c->ub_src_b, c->F_val,
                                                                   reinterpret_cast<double *>(c->uLt));
        RH_LAUNCHED(c);
      }
      if (!c->ev_ult) RH_CUDA(c, cudaEventCreateWithFlags(&c->ev_ult, cudaEventDisableTiming));
      RH_CUDA(c, cudaEventRecord(c->ev_ult, sb));
      if (int rc = early(sb, 2)) return rc;
    }
    // dense Schur complement of the separator, inverted by blocked Gauss-Jordan
    const int ns = A.sep_rows;
    RH_CUDA(c, cudaMemsetAsync(c->Sinv, 0, sizeof(double) * (size_t)ns * ns, st));
    const int nsl = (int)A.sb_src.size();
    k_sep_dense<<<nblk(nsl), kThreads, 0, st>>>(nsl, c->sb_src, c->sb_dense, c->F_val, c->Sinv);
    RH_LAUNCHED(c);
    // blocked Gauss-Jordan, one cooperative launch; the result lands in Sinv
    const int npanel = (ns + GJB - 1) / GJB;
    double *Sa = (npanel & 1) ? c->Sbuf : c->Sinv, *Sb = (npanel & 1) ? c->Sinv : c->Sbuf;
    if (Sa != c->Sinv) RH_CUDA(c, cudaMemcpyAsync(Sa, c->Sinv, sizeof(double) * (size_t)ns * ns, cudaMemcpyDeviceToDevice, st));
    const int *sep_rows = c->row_global + A.seg_row_off[A.nblk];
    int nsv = ns;
    double pivtol = 1e-14;
    const double *rowmax = c->rowmax;
    int *status = c->status;
    unsigned *bar = c->grid_bar;
    long long *gdbg = nullptr;
    if (const char *env = getenv("RH_DEBUG"))   // timing experiment: per-panel stamps
      if (atoi(env) & 16) {
        static long long *buf = nullptr;
        if (!buf) cudaMalloc(&buf, 1024 * sizeof(long long));
        gdbg = buf;
      }
    double *dbuf = c->gj_dbuf;
    int gj_warps = 8;
    if (const char *env = getenv("RH_GJW")) gj_warps = atoi(env);   // experiment
    double *seppiv = c->sep_piv;
    void *args[] = {&Sa, &Sb, &nsv, &rowmax, &sep_rows, &status, &pivtol, &bar, &gdbg, &dbuf, &gj_warps, &seppiv};
    const int ntl = ((ns + GJT - 1) / GJT) * ((ns + GJT - 1) / GJT);
    const int grid = std::max(1, std::min(ntl, c->coop_blocks - 1)) + 1;   // tile CTAs + the lookahead CTA
    RH_CUDA(c, cudaMemsetAsync(c->grid_bar, 0, 2 * sizeof(unsigned), st));   // tiles' arrivals, D^-1 flag
    RH_CUDA(c, cudaLaunchCooperativeKernel((const void *)k_sep_inverse, dim3(grid), dim3(256), args, gj_smem_bytes(), st));
    RH_LAUNCHED(c);
    if (gdbg) {
      std::vector<long long> hb(1024);
      cudaMemcpyAsync(hb.data(), gdbg, 1024 * 8, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      if (FILE *fp = fopen("gpurun_out/gj_prof.bin", "wb")) {
        fwrite(hb.data(), 8, hb.size(), fp);
        fclose(fp);
      }
    }
    dbg_mark(st, "k_sep_inverse");
    // S^-T (the dense L-side product of random-W batches, the gradient's transposed
    // GEMV): in the fused call on the gradient stream (which the call joins before
    // it returns), so the Cartesian batches (their L-side product reads S^-1) do
    // not wait for it
    if (early && side) {
      c->tr_pending = true;   // the fused call runs it first on the gradient stream
    } else {
      k_transpose<<<dim3((ns + 31) / 32, (ns + 31) / 32), dim3(32, 8), 0, st>>>(c->Sinv, c->SinvT, ns);
      RH_LAUNCHED(c);
    }
  }
  if (c->nrec_b > 0 && !(early && side && A.sep_rows > 0)) {   // L^T records: block rows' L entries include L_sb (R_B1)
    k_gather_code<<<nblk(2LL * c->nrec_b), kThreads, 0, st>>>(2 * c->nrec_b, c->ub_src_b, c->F_val,
                                                               reinterpret_cast<double *>(c->uLt));
    RH_LAUNCHED(c);
  }
  if (early && side && A.sep_rows > 0) RH_CUDA(c, cudaStreamWaitEvent(st, c->ev_ult, 0));   // (done during the inverse)
  if (side && early) {   // the early sweeps are joined batch by batch (hessian_batches)
    RH_CUDA(c, cudaStreamWaitEvent(st, c->ev_derived, 0));
    if (c->spike_ok && !c->spike_pending) RH_CUDA(c, cudaStreamWaitEvent(st, c->ev_spike, 0));
  } else if (side) {
    RH_CUDA(c, cudaEventRecord(c->ev_sb, side));
    RH_CUDA(c, cudaStreamWaitEvent(st, c->ev_sb, 0));
  }
  c->has_state = true;
  return defer_check ? RH_OK : check_pivots(c, st);
}
}  // namespace

extern "C" {

int rh_set_state(rh_ctx *c, const double *x, const double *p, void *stream) {
  // block-only derived values on a side stream, concurrent with the separator's elimination
  if (c && !c->host_only && c->loaded && !c->sti[1]) {
    RH_CUDA(c, cudaSetDevice(c->device));
    RH_CUDA(c, cudaStreamCreateWithFlags(&c->sti[1], cudaStreamNonBlocking));
  }
  return state_impl(c, x, p, (cudaStream_t)stream, c ? c->sti[1] : nullptr, nullptr);
}

int rh_residual(rh_ctx *c, double *g, double *f, void *stream) {
  int rc = check_ready(c, false);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (g) RH_CUDA(c, cudaMemcpyAsync(g, c->g, sizeof(double) * c->A.n_x, cudaMemcpyDeviceToDevice, st));
  if (f) RH_CUDA(c, cudaMemcpyAsync(f, c->scal + 3, sizeof(double), cudaMemcpyDeviceToDevice, st));
  return RH_OK;
}

}  // extern "C"

namespace {
// first-order adjoint + reduced gradient + FoR tape on `st`; own_ws: use the
// gradient's private separator workspace and ticket counters (concurrent with
// Hessian batches in the fused call)
int gradient_impl(rh_ctx *c, double *grad_p, double *lambda_out, cudaStream_t st, bool own_ws) {
  int rc = check_ready(c, false);
  if (rc) return rc;
  if (!grad_p) return fail(c, RH_E_ARG, "grad_p is null");
  const Analysis &A = c->A;
  k_grad_rhs<<<nblk(A.n_x), kThreads, 0, st>>>(A.n_x, c->x_bus, c->x_kind, c->pinv, c->refg_th, c->refg_v,
                                                c->scal, c->X1col);
  RH_LAUNCHED(c);
  // J^T lambda = -grad_x f: U^T then L^T sweeps, one column
  if (int rc2 = ensure_tsep(c, kSegC)) return rc2;
  SegParams h = make_params(c);
  if (const char *env = getenv("RH_DEBUG")) h.debug = atoi(env);
  h.N = 1;
  h.ld = kSegC;   // column 0 carries the right-hand side, columns 1..31 stay zero
  h.P = c->X1col;
  h.Mp = nullptr;   // no SpMulAdd partials (k_grad_out forms G_p^T lambda itself)
  if (own_ws) {
    if (!c->grad_tsep) {
      if (cudaMalloc(&c->grad_tsep, sizeof(double) * kSegC * (std::max(1, A.sep_rows) + c->dsr.nruns)) != cudaSuccess ||
          cudaMalloc(&c->grad_ctr, 16 * sizeof(int)) != cudaSuccess || cudaMemset(c->grad_ctr, 0, 16 * sizeof(int)) != cudaSuccess) {
        cudaGetLastError();
        return fail(c, RH_E_NOMEM, "gradient workspace allocation failed");
      }
    }
    h.Tsep = c->grad_tsep;
    h.blk_ctr = c->grad_ctr;
  }
  const int g1 = std::min(2 * c->nsm, A.nblk);
  k_blk<<<g1, kBlkThreads, c->smem_blk, st>>>(h, MODE_UT);
  RH_LAUNCHED(c);
  if (A.sep_rows > 0) {
    k_sep_gather<<<dim3(nblk(A.sep_rows, kThreads / 32), 1), kThreads, 0, st>>>(h, MODE_UTLT);
    RH_LAUNCHED(c);
    k_sep_gemv<<<nblk(A.sep_rows, kThreads / 32), kThreads, 0, st>>>(h, MODE_UTLT);
    RH_LAUNCHED(c);
  }
  k_blk<<<g1, kBlkThreads, c->smem_blk, st>>>(h, MODE_LT);
  RH_LAUNCHED(c);
  k_grad_out<<<nblk(std::max(A.n_x, A.n_p)), kThreads, 0, st>>>(
      A.n_x, A.n_p, c->pinv, c->p_bus, c->p_kind, c->c2b, c->c1b, c->p, c->refg_v, c->scal, c->gpc_ptr, c->gpc_row,
      c->gpc_val, c->X1col, c->lam, grad_p);
  RH_LAUNCHED(c);
  if (lambda_out)
    RH_CUDA(c, cudaMemcpyAsync(lambda_out, c->lam, sizeof(double) * A.n_x, cudaMemcpyDeviceToDevice, st));
  return build_tape(c, st);
}
}  // namespace

extern "C" {

int rh_reduced_gradient(rh_ctx *c, double *grad_p, double *lambda_out, void *stream) {
  return gradient_impl(c, grad_p, lambda_out, (cudaStream_t)stream, false);
}

int rh_set_multipliers(rh_ctx *c, const double *lambda, void *stream) {
  int rc = check_ready(c, false);
  if (rc) return rc;
  if (!lambda) return fail(c, RH_E_ARG, "lambda is null");
  cudaStream_t st = (cudaStream_t)stream;
  RH_CUDA(c, cudaMemcpyAsync(c->lam, lambda, sizeof(double) * c->A.n_x, cudaMemcpyDeviceToDevice, st));
  return build_tape(c, st);
}

}  // extern "C"

namespace {
// Newton projection; final_state: leave state + factors at the final x (else the
// caller recomputes them, e.g. the tracking step's fused Hessian call)
int newton_impl(rh_ctx *c, double *x, const double *p, double tol, int extra, int maxit, int *iters, double *resid,
                cudaStream_t st, bool final_state) {
  if (!c || !x || !p || maxit <= 0 || extra < 0 || !(tol >= 0.0)) return fail(c, RH_E_ARG, "bad argument");
  if (c->host_only) return fail(c, RH_E_NODEV, "host-only context (device = -1)");
  if (!c->loaded) return fail(c, RH_E_ORDER, "no grid loaded");
  RH_CUDA(c, cudaSetDevice(c->device));
  const Analysis &A = c->A;
  if (int rc = ensure_tsep(c, kSegC)) return rc;
  int left = -1, it = 0;
  bool done = false;
  // block-only derived values on a side stream, concurrent with the separator's elimination
  if (!c->sti[1]) RH_CUDA(c, cudaStreamCreateWithFlags(&c->sti[1], cudaStreamNonBlocking));
  // one Newton step, enqueued without host syncs: state, assembly and
  // refactorization at x_k (g_k in c->g, factors of J_k); J_k dx = g_k by the
  // block L sweep, the separator (S^-1), the U sweep; x_{k+1} = x_k - dx
  // and max|dx|.  Replayed as a CUDA graph from the third step.
  auto step = [&](cudaStream_t cs) -> int {
    if (int rc = state_impl(c, x, p, cs, c->sti[1], nullptr, true)) return rc;
    k_newton_rhs<<<nblk(A.n_x), kThreads, 0, cs>>>(A.n_x, c->pinv, c->g, c->X1col);
    RH_LAUNCHED(c);
    SegParams h = make_params(c);
    h.N = 1;
    h.ld = kSegC;
    h.Z = c->X1col;
    const int g1 = std::min(2 * c->nsm, A.nblk);
    k_blk<<<g1, kBlkThreads, c->smem_blk, cs>>>(h, MODE_LX);
    RH_LAUNCHED(c);
    if (A.sep_rows > 0) {
      k_sep_gather<<<dim3(nblk(A.sep_rows, kThreads / 32), 1), kThreads, 0, cs>>>(h, MODE_LUX);
      RH_LAUNCHED(c);
      k_sep_gemv<<<nblk(A.sep_rows, kThreads / 32), kThreads, 0, cs>>>(h, MODE_LU);
      RH_LAUNCHED(c);
    }
    k_blk<<<g1, kBlkThreads, c->smem_blk, cs>>>(h, MODE_U);
    RH_LAUNCHED(c);
    RH_CUDA(c, cudaMemsetAsync(c->nwt, 0, sizeof(double), cs));
    k_newton_update<<<nblk(A.n_x), kThreads, 0, cs>>>(A.n_x, c->pinv, c->X1col, x, c->nwt);
    RH_LAUNCHED(c);
    return RH_OK;
  };
  const rh_ctx::GraphKey key{x, p, nullptr, nullptr, (const void *)st, 0, -2, 0, 0, 0, c->jac_mode};
  for (; it < maxit && !done; ++it) {
    int rc = -1;
    if (!graph_run(c, 2, key, st, rc, step, false)) {
      rc = step(st);
      if (!rc) rc = check_pivots(c, st);
    }
    if (rc) return rc;
    double dmax = 0.0;
    RH_CUDA(c, cudaMemcpyAsync(&dmax, c->nwt, sizeof(double), cudaMemcpyDeviceToHost, st));
    RH_CUDA(c, cudaStreamSynchronize(st));
    if (getenv("RH_DEBUG") && (atoi(getenv("RH_DEBUG")) & 256)) fprintf(stderr, "newton step %d: max|dx| %.3e\n", it, dmax);
    // the oracle's stopping rule: `extra` more steps after max|dx| <= tol
    if (left < 0 && dmax <= tol) left = extra;
    if (left >= 0) {
      if (left == 0) done = true;
      else --left;
    }
  }
  if (iters) *iters = it;
  if (!done) return fail(c, RH_E_NOCONV, "Newton did not converge within maxit steps");
  if (!final_state) return RH_OK;
  // leave the state (g, factors) at the final x
  if (int rc = state_impl(c, x, p, st, c->sti[1], nullptr)) return rc;
  if (resid) {
    RH_CUDA(c, cudaMemsetAsync(c->nwt + 1, 0, sizeof(double), st));
    k_absmax<<<nblk(A.n_x), kThreads, 0, st>>>(A.n_x, c->g, c->nwt + 1);
    RH_LAUNCHED(c);
    RH_CUDA(c, cudaMemcpyAsync(resid, c->nwt + 1, sizeof(double), cudaMemcpyDeviceToHost, st));
    RH_CUDA(c, cudaStreamSynchronize(st));
  }
  return RH_OK;
}
}  // namespace

extern "C" {

int rh_newton(rh_ctx *c, double *x, const double *p, double tol, int32_t extra, int32_t maxit, int32_t *iters,
              double *resid, void *stream) {
  int it = 0;
  int rc = newton_impl(c, x, p, tol, extra, maxit, &it, resid, (cudaStream_t)stream, true);
  if (iters) *iters = it;
  return rc;
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

}  // extern "C"

namespace {
// Batches of Cartesian columns [j0, j1): balanced batches of
// width <= N go round-robin to the caller's stream (workspace 0) and internal
// streams (workspaces 1, 2), so consecutive batches overlap (tails,
// latency-bound kernels); the caller's stream joins them at the end.  With Hhost
// (non-transposed H only), every finished column block is copied to the host
// on its batch's stream while the next batches compute.
int num_ws(int nb, int cap = kNumWs) {
  int nws = cap;
  if (const char *env = getenv("RH_STREAMS")) nws = std::max(1, std::min(kNumWs, atoi(env)));   // tuning override
  return std::max(1, std::min(nws, nb));
}

// batch b of ncols columns split into nb balanced batches: [a0, a1)
inline void batch_range(int ncols, int nb, int b, int &a0, int &a1) {
  a0 = (int)((long long)ncols * b / nb);
  a1 = (int)((long long)ncols * (b + 1) / nb);
}

// batch bounds of a host-copy call: full batches of N first, then the remainder
// split into pieces of <= tail columns (the last batch's copy is the tail that
// nothing overlaps, so it should be small)
// Host copies of H are the e2e bound when H is large (case9241: 66.8 MB = 1.2 ms
// of D2H against a 1.6 ms step): then batches run one after another on one
// stream, each copied while the next computes, and the remainder is split so the
// last copy is small (e2e probe: 2.58 -> 2.35 ms).  Smaller H (case2869: 8.3 MB,
// 0.15 ms) is compute-bound: two concurrent streams, remainder in one batch.
bool host_copy_bound(int n_p) { return (double)n_p * n_p * 8.0 >= 32.0 * (1 << 20); }

std::vector<int> host_cuts(int ncols, int N, bool copy_bound) {
  std::vector<int> cuts(1, 0);
  if (ncols <= 0) return cuts;
  int tail = copy_bound ? std::max(32, N / 2) : N, first = N;
  if (const char *env = getenv("RH_E2E_TAIL")) tail = std::max(32, atoi(env));     // tuning override
  if (const char *env = getenv("RH_E2E_FIRST")) first = std::max(32, atoi(env));   // tuning override
  int a = 0;
  if (ncols > first && first < N) cuts.push_back(a = first);   // an early first block for the copy stream
  while (ncols - a > N) cuts.push_back(a += N);
  const int r = ncols - a, np = (r + tail - 1) / tail;
  for (int q = 1; q <= np; ++q) cuts.push_back(a + (int)((long long)r * q / np));
  return cuts;
}

// `early`: the first `early` batches already ran their first block sweep (phase 1,
// workspace b) and now run the rest (phase 2)
int hessian_batches(rh_ctx *c, int j0, int j1, int N, double *H, long long ldh, int transposed, cudaStream_t st,
                    double *Hhost, int early = 0) {
  const int ncols = j1 - j0;
  if (int rc = ensure_spikes(c, st)) return rc;   // (before the batches fork to other streams)
  int nb = (ncols + N - 1) / N;
  std::vector<int> cuts;   // batch bounds (host copies only)
  if (Hhost) {
    cuts = host_cuts(ncols, N, host_copy_bound(c->A.n_p));
    nb = (int)cuts.size() - 1;
  }
  // with host copies each finished column block travels on a copy stream while
  // later batches compute; copy-bound calls (host_copy_bound) run their batches
  // one after the other so the copies start as early as possible
  int host_streams = host_copy_bound(c->A.n_p) ? 1 : 2;   // host copies (host_copy_bound)
  if (const char *env = getenv("RH_E2E_STREAMS")) host_streams = std::max(1, atoi(env));   // tuning override
  const int nws = num_ws(nb, Hhost ? host_streams : kNumWs);
  if (Hhost) {
    if (!c->cp_st) RH_CUDA(c, cudaStreamCreateWithFlags(&c->cp_st, cudaStreamNonBlocking));
    if (!c->ev_cp) RH_CUDA(c, cudaEventCreateWithFlags(&c->ev_cp, cudaEventDisableTiming));
  }
  if (nws > 1) {
    if (!c->ev_fork) RH_CUDA(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    RH_CUDA(c, cudaEventRecord(c->ev_fork, st));
    for (int k = 1; k < nws; ++k) {
      if (!c->sti[k]) RH_CUDA(c, cudaStreamCreateWithFlags(&c->sti[k], cudaStreamNonBlocking));
      if (!c->ev_join[k]) RH_CUDA(c, cudaEventCreateWithFlags(&c->ev_join[k], cudaEventDisableTiming));
      RH_CUDA(c, cudaStreamWaitEvent(c->sti[k], c->ev_fork, 0));
    }
  }
  auto range = [&](int b, int &a0, int &a1) {
    if (Hhost) {
      a0 = cuts[b];
      a1 = cuts[b + 1];
    } else {
      batch_range(ncols, nb, b, a0, a1);
    }
  };
  for (int b = 0; b < nb; ++b) {
    int a0, a1;
    range(b, a0, a1);
    double *out = transposed ? H + (long long)a0 * ldh : H + a0;
    const int k = b % nws;
    cudaStream_t sb = k ? c->sti[k] : st;
    if (b < early) RH_CUDA(c, cudaStreamWaitEvent(sb, c->ev_early[b], 0));   // its L sweep (side stream)
    int rc = hvp_impl(c, nullptr, 0, j0 + a0, out, ldh, transposed, a1 - a0, sb, nullptr, nullptr, nullptr, 0, k,
                      b < early ? (c->early_gathered ? 4 : 2) : 0);
    if (rc) return rc;
    if (Hhost) {
      RH_CUDA(c, cudaEventRecord(c->ev_cp, sb));
      RH_CUDA(c, cudaStreamWaitEvent(c->cp_st, c->ev_cp, 0));
      RH_CUDA(c, cudaMemcpy2DAsync(Hhost + a0, ldh * sizeof(double), out, ldh * sizeof(double),
                                   (size_t)(a1 - a0) * sizeof(double), (size_t)c->A.n_p, cudaMemcpyDeviceToHost,
                                   c->cp_st));
    }
  }
  for (int k = 1; k < nws; ++k) {
    RH_CUDA(c, cudaEventRecord(c->ev_join[k], c->sti[k]));
    RH_CUDA(c, cudaStreamWaitEvent(st, c->ev_join[k], 0));
  }
  if (Hhost) {
    RH_CUDA(c, cudaEventRecord(c->ev_cp, c->cp_st));
    RH_CUDA(c, cudaStreamWaitEvent(st, c->ev_cp, 0));
  }
  return RH_OK;
}
}  // namespace

extern "C" {

int rh_hessian_columns(rh_ctx *c, int32_t j0, int32_t j1, int32_t N, double *H, int64_t ldh, int32_t transposed,
                       void *stream) {
  int rc = check_ready(c, true);
  if (rc) return rc;
  const int np_ = c->A.n_p;
  if (j0 < 0 || j1 > np_ || j0 > j1 || N <= 0 || !H) return fail(c, RH_E_ARG, "bad column range / N / H");
  if ((!transposed && ldh < j1 - j0) || (transposed && ldh < np_)) return fail(c, RH_E_ARG, "ldh too small");
  return hessian_batches(c, j0, j1, N, H, ldh, transposed, (cudaStream_t)stream, nullptr);
}

int rh_full_hessian(rh_ctx *c, int32_t N, double *H, void *stream) {
  int rc = check_ready(c, true);
  if (rc) return rc;
  return rh_hessian_columns(c, 0, c->A.n_p, N, H, c->A.n_p, 0, stream);
}

}  // extern "C"

namespace {
// state + reduced gradient + Hessian columns [j0, j1), with the first block
// sweep of the first batches overlapping the separator's refactorization
int reduced_hessian_impl(rh_ctx *c, const double *x, const double *p, int j0, int j1, int N, double *grad_p,
                         double *H, long long ldh, int transposed, cudaStream_t st, double *Hhost,
                         bool defer_pivots = false) {
  if (!c || !x || !p || !grad_p || (j1 > j0 && !H)) return fail(c, RH_E_ARG, "null argument");
  if (c->host_only) return fail(c, RH_E_NODEV, "host-only context (device = -1)");
  if (!c->loaded) return fail(c, RH_E_ORDER, "no grid loaded");
  const int np_ = c->A.n_p;
  if (j0 < 0 || j1 > np_ || j0 > j1 || N <= 0) return fail(c, RH_E_ARG, "bad column range / N");
  if ((!transposed && ldh < j1 - j0) || (transposed && ldh < np_)) return fail(c, RH_E_ARG, "ldh too small");
  RH_CUDA(c, cudaSetDevice(c->device));
  const int ncols = j1 - j0;
  const std::vector<int> cuts = Hhost ? host_cuts(ncols, N, host_copy_bound(c->A.n_p)) : std::vector<int>();
  const int nb = Hhost ? (int)cuts.size() - 1 : ncols > 0 ? (ncols + N - 1) / N : 0;
  int host_streams = host_copy_bound(c->A.n_p) ? 1 : 2;   // as hessian_batches
  if (const char *env = getenv("RH_E2E_STREAMS")) host_streams = std::max(1, atoi(env));   // tuning override
  const int early = nb > 0 ? std::min(nb, num_ws(nb, Hhost ? host_streams : kNumWs)) : 0;
  // the widest batch actually run (front-loaded batches of N for host copies,
  // else ceil(ncols / nb)), not the caller's N: a shard or N > n_p must not
  // allocate workspaces no batch uses
  int wmax = 0;
  if (Hhost)
    for (int b = 0; b < nb; ++b) wmax = std::max(wmax, cuts[b + 1] - cuts[b]);
  else if (nb > 0)
    wmax = (ncols + nb - 1) / nb;
  const int ld = (wmax + kBC - 1) / kBC * kBC;
  for (int k = 0; k < early; ++k)   // allocate before anything is enqueued
    if (int rc = ensure_ws(c, ld, k)) return rc;
  if (!c->sti[1]) RH_CUDA(c, cudaStreamCreateWithFlags(&c->sti[1], cudaStreamNonBlocking));
  // stage 1 (as soon as the block factors exist): plan + L sweep of the first
  // batches; stage 2 (as soon as the separator rows' L values exist, while S^-1 is
  // still being computed): their separator right-hand sides
  c->early_gathered = false;
  auto first_sweeps = [&](cudaStream_t sb, int stage) -> int {
    if (stage == 2 && getenv("RH_NO_EARLY_GATHER")) return RH_OK;
    for (int b = 0; b < early; ++b) {
      int a0, a1;
      if (Hhost) {
        a0 = cuts[b];
        a1 = cuts[b + 1];
      } else {
        batch_range(ncols, nb, b, a0, a1);
      }
      double *out = transposed ? H + (long long)a0 * ldh : H + a0;
      if (int rc = hvp_impl(c, nullptr, 0, j0 + a0, out, ldh, transposed, a1 - a0, sb, nullptr, nullptr, nullptr, 0,
                            b, stage == 1 ? 1 : 3))
        return rc;
      if (!c->ev_early[b]) RH_CUDA(c, cudaEventCreateWithFlags(&c->ev_early[b], cudaEventDisableTiming));
      RH_CUDA(c, cudaEventRecord(c->ev_early[b], sb));
    }
    if (stage == 2) c->early_gathered = true;
    return RH_OK;
  };
  // everything is enqueued before the one host sync (the pivot flag, read last)
  int rc = state_impl(c, x, p, st, c->sti[1], first_sweeps, true);
  dbg_mark(st, "state done (joined side)");
  // the gradient (and the tape) on its own stream; the batches' separator and U
  // sweeps run meanwhile, each batch waits for the tape right before k_for
  if (!rc) {
    if (!c->grad_st) {   // high priority: its small latency-bound kernels go first when SMs free up
      int lo = 0, hi = 0;
      RH_CUDA(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
      RH_CUDA(c, cudaStreamCreateWithPriority(&c->grad_st, cudaStreamNonBlocking, getenv("RH_NO_PRIO") ? lo : hi));
    }
    if (!c->ev_state) RH_CUDA(c, cudaEventCreateWithFlags(&c->ev_state, cudaEventDisableTiming));
    if (!c->ev_tape) RH_CUDA(c, cudaEventCreateWithFlags(&c->ev_tape, cudaEventDisableTiming));
    RH_CUDA(c, cudaEventRecord(c->ev_state, st));
    RH_CUDA(c, cudaStreamWaitEvent(c->grad_st, c->ev_state, 0));
    if (c->tr_pending) {   // S^-T off the batches' critical path: the gradient's GEMV reads it
      const int ns = c->A.sep_rows;
      k_transpose<<<dim3((ns + 31) / 32, (ns + 31) / 32), dim3(32, 8), 0, c->grad_st>>>(c->Sinv, c->SinvT, ns);
      RH_LAUNCHED(c);
      c->tr_pending = false;
    }
    rc = gradient_impl(c, grad_p, nullptr, c->grad_st, true);
    if (!rc) RH_CUDA(c, cudaEventRecord(c->ev_tape, c->grad_st));
  }
  if (!rc && nb > 0) {
    c->tape_wait = c->ev_tape;
    rc = hessian_batches(c, j0, j1, N, H, ldh, transposed, st, Hhost, early);
    c->tape_wait = nullptr;
  }
  if (!rc) RH_CUDA(c, cudaStreamWaitEvent(st, c->ev_tape, 0));
  dbg_mark(st, "gradient + batches joined");
  dbg_report(st);
  if (!rc && !defer_pivots) rc = check_pivots(c, st);
  return rc;
}
}  // namespace

extern "C" {

int rh_reduced_hessian(rh_ctx *c, const double *x, const double *p, int32_t j0, int32_t j1, int32_t N,
                       double *grad_p, double *H, int64_t ldh, int32_t transposed, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (c && c->loaded && !c->host_only && x && p && grad_p && (j1 <= j0 || H)) {
    rh_ctx::GraphKey key{x, p, grad_p, H, (const void *)st, (long long)ldh, j0, j1, N, transposed, c->jac_mode};
    int rc = -1;
    if (graph_run(c, 0, key, st, rc, [&](cudaStream_t cs) {
          return reduced_hessian_impl(c, x, p, j0, j1, N, grad_p, H, ldh, transposed, cs, nullptr, true);
        }))
      return rc;
  }
  return reduced_hessian_impl(c, x, p, j0, j1, N, grad_p, H, ldh, transposed, st, nullptr);
}

int rh_reduced_hessian_host(rh_ctx *c, const double *x, const double *p, int32_t N, double *grad_p, double *H) {
  if (!c || !x || !p || !H) return fail(c, RH_E_ARG, "null argument");
  if (c->host_only) return fail(c, RH_E_NODEV, "host-only context (device = -1)");
  if (!c->loaded) return fail(c, RH_E_ORDER, "no grid loaded");
  RH_CUDA(c, cudaSetDevice(c->device));
  const Analysis &A = c->A;
  const size_t nx = A.n_x, np_ = A.n_p;
  // context-owned staging buffers and stream (allocated once per grid)
  if (!c->e2e_st) RH_CUDA(c, cudaStreamCreateWithFlags(&c->e2e_st, cudaStreamNonBlocking));
  if (!c->e2e_buf) {
    if (cudaMalloc(&c->e2e_buf, (nx + 2 * np_ + np_ * np_) * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return fail(c, RH_E_NOMEM, "allocation failed");
    }
  }
  cudaStream_t st = c->e2e_st;
  double *dx = c->e2e_buf, *dp = dx + nx, *dg = dp + np_, *dH = dg + np_;
  // H2D inputs; state, gradient and Hessian batches (first sweeps overlapping the
  // separator's refactorization); column blocks leave for the host as their
  // batches finish; the gradient last.  Repeated calls replay a CUDA graph
  // (pinned host buffers; pageable ones fall back to plain enqueues).
  auto enqueue = [&](cudaStream_t cs, bool defer) -> int {
    RH_CUDA(c, cudaMemcpyAsync(dx, x, nx * 8, cudaMemcpyHostToDevice, cs));
    RH_CUDA(c, cudaMemcpyAsync(dp, p, np_ * 8, cudaMemcpyHostToDevice, cs));
    int rc = reduced_hessian_impl(c, dx, dp, 0, (int)np_, N, dg, dH, (long long)np_, 0, cs, H, true);
    if (rc) return rc;
    if (grad_p) RH_CUDA(c, cudaMemcpyAsync(grad_p, dg, np_ * 8, cudaMemcpyDeviceToHost, cs));
    return defer ? RH_OK : check_pivots(c, cs);
  };
  rh_ctx::GraphKey key{x, p, grad_p, H, (const void *)st, (long long)np_, 0, (int)np_, N, 0, c->jac_mode};
  int rc = -1;
  if (!graph_run(c, 1, key, st, rc, [&](cudaStream_t cs) { return enqueue(cs, true); })) rc = enqueue(st, false);
  if (rc) return rc;
  RH_CUDA(c, cudaStreamSynchronize(st));
  return RH_OK;
}

int64_t rh_launch_count(const rh_ctx *c) { return c ? c->launches : 0; }

}  // extern "C"

namespace {
constexpr int kMaxShifts = 64;

// tracking Step 2 (dense.cu): tau = 0, then 1e-6 doubling (R-T4); one sync per attempt
int dense_solve_impl(rh_ctx *c, int n, const double *H, long long ldh, const double *g, double *d, double *p,
                     double alpha, double *tau_out, int *attempts_out, cudaStream_t st) {
  double tau = 0.0;
  int att = 0;
  if (n > 0) {
    cudaError_t e = dense_ws_ensure(c->dws, n, c->device);
    if (e != cudaSuccess) return fail(c, RH_E_CUDA, std::string("dense workspace: ") + cudaGetErrorString(e));
    bool ok = false;
    for (att = 1; att <= kMaxShifts; ++att) {
      int nl = 0;
      e = dense_spd_attempt(c->dws, n, H, ldh, g, tau, p, alpha, st, &nl);
      c->launches += nl;
      if (e != cudaSuccess) return fail(c, RH_E_CUDA, std::string("dense Cholesky: ") + cudaGetErrorString(e));
      int fl = 0;
      RH_CUDA(c, cudaMemcpyAsync(&fl, c->dws.fail, sizeof(int), cudaMemcpyDeviceToHost, st));
      RH_CUDA(c, cudaStreamSynchronize(st));
      if (fl == 0) {
        ok = true;
        break;
      }
      tau = (tau == 0.0) ? 1e-6 : 2.0 * tau;
    }
    if (!ok) return fail(c, RH_E_NOTPD, "dense Cholesky: not positive definite after 64 diagonal shifts");
    if (d) RH_CUDA(c, cudaMemcpyAsync(d, c->dws.dbuf, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  }
  if (tau_out) *tau_out = tau;
  if (attempts_out) *attempts_out = att;
  return RH_OK;
}
}  // namespace

extern "C" {

int rh_set_loads(rh_ctx *c, const double *Pd, const double *Qd, void *stream) {
  if (!c) return RH_E_ARG;
  if (c->host_only) return fail(c, RH_E_NODEV, "host-only context (device = -1)");
  if (!c->loaded) return fail(c, RH_E_ORDER, "no grid loaded");
  RH_CUDA(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t bytes = sizeof(double) * c->A.n_bus;
  if (Pd) RH_CUDA(c, cudaMemcpyAsync(c->Pd, Pd, bytes, cudaMemcpyDeviceToDevice, st));
  if (Qd) RH_CUDA(c, cudaMemcpyAsync(c->Qd, Qd, bytes, cudaMemcpyDeviceToDevice, st));
  c->has_state = c->has_mult = false;
  return RH_OK;
}

int rh_dense_spd_solve(rh_ctx *c, int32_t n, const double *H, int64_t ldh, const double *g, double *d, double *p,
                       double alpha, double *tau, int32_t *attempts, void *stream) {
  if (!c) return RH_E_ARG;
  if (c->host_only) return fail(c, RH_E_NODEV, "host-only context (device = -1)");
  if (n < 0 || ldh < n || (n > 0 && (!H || !g))) return fail(c, RH_E_ARG, "bad n / ldh / H / g");
  RH_CUDA(c, cudaSetDevice(c->device));
  int att = 0;
  const int rc = dense_solve_impl(c, n, H, ldh, g, d, p, alpha, tau, &att, (cudaStream_t)stream);
  if (attempts) *attempts = att;
  return rc;
}

int rh_tracking_step(rh_ctx *c, double *x, double *p, const double *Pd, const double *Qd, int32_t j0, int32_t j1,
                     int32_t N, double alpha, double *grad_p, double *H, int64_t ldh, double *d, double *info,
                     void *stream) {
  if (!c || !x || !p || !grad_p || !H) return fail(c, RH_E_ARG, "null argument");
  if (c->host_only) return fail(c, RH_E_NODEV, "host-only context (device = -1)");
  if (!c->loaded) return fail(c, RH_E_ORDER, "no grid loaded");
  const int np_ = c->A.n_p;
  if (j0 < 0 || j1 > np_ || j0 >= j1 || N <= 0 || ldh < np_) return fail(c, RH_E_ARG, "bad j0/j1/N/ldh");
  RH_CUDA(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  for (auto &e : c->ev_trk)
    if (!e) RH_CUDA(c, cudaEventCreate(&e));
  RH_CUDA(c, cudaEventRecord(c->ev_trk[0], st));
  if (Pd || Qd)
    if (int rc = rh_set_loads(c, Pd, Qd, stream)) return rc;
  int it = 0;
  // x(p_t; w_t); the fused call below recomputes state and factors at the final x
  if (int rc = newton_impl(c, x, p, 1e-11, 2, 40, &it, nullptr, st, false)) return rc;
  // Step 1: g_t and the free columns of H_t (Alg. 2), transposed
  if (int rc = reduced_hessian_impl(c, x, p, j0, j1, N, grad_p, H, ldh, 1, st, nullptr)) return rc;
  RH_CUDA(c, cudaEventRecord(c->ev_trk[1], st));
  double hv[2] = {0.0, 0.0};   // max|g|, F
  RH_CUDA(c, cudaMemsetAsync(c->nwt + 1, 0, sizeof(double), st));
  k_absmax<<<nblk(c->A.n_x), kThreads, 0, st>>>(c->A.n_x, c->g, c->nwt + 1);
  RH_LAUNCHED(c);
  RH_CUDA(c, cudaMemcpyAsync(&hv[0], c->nwt + 1, sizeof(double), cudaMemcpyDeviceToHost, st));
  RH_CUDA(c, cudaMemcpyAsync(&hv[1], c->scal + 3, sizeof(double), cudaMemcpyDeviceToHost, st));
  // Step 2 on the [j0, j1) block: M[k][a] = H_t[j0 + a][j0 + k] (symmetrized inside)
  double tau = 0.0;
  int att = 0;
  if (int rc = dense_solve_impl(c, j1 - j0, H + j0, ldh, grad_p + j0, d, p + j0, alpha, &tau, &att, st)) return rc;
  RH_CUDA(c, cudaEventRecord(c->ev_trk[2], st));
  RH_CUDA(c, cudaEventSynchronize(c->ev_trk[2]));
  if (info) {
    float m1 = 0.f, m2 = 0.f;
    cudaEventElapsedTime(&m1, c->ev_trk[0], c->ev_trk[1]);
    cudaEventElapsedTime(&m2, c->ev_trk[1], c->ev_trk[2]);
    info[0] = it;
    info[1] = hv[0];
    info[2] = hv[1];
    info[3] = tau;
    info[4] = att;
    info[5] = m1;
    info[6] = m2;
  }
  return RH_OK;
}

int rh_set_jacobian_mode(rh_ctx *c, int32_t mode) {
  if (!c) return RH_E_ARG;
  if (mode != RH_JAC_ANALYTIC && mode != RH_JAC_COLORED) return fail(c, RH_E_ARG, "unknown Jacobian mode");
  c->jac_mode = mode;
  c->has_state = c->has_mult = false;
  return RH_OK;
}

int rh_coloring(const rh_ctx *c, int32_t *colors, int32_t *ncolors) {
  if (!c) return RH_E_ARG;
  if (!c->loaded) return RH_E_ORDER;
  if (colors) std::copy(c->A.colors.begin(), c->A.colors.end(), colors);
  if (ncolors) *ncolors = c->A.ncolors;
  return RH_OK;
}

int rh_compressed_jacobian(rh_ctx *c, double *JS, void *stream) {
  int rc = check_ready(c, false);
  if (rc) return rc;
  if (!JS) return fail(c, RH_E_ARG, "JS is null");
  cudaStream_t st = (cudaStream_t)stream;
  if ((rc = colored_jacobian(c, st, false))) return rc;
  RH_CUDA(c, cudaMemcpyAsync(JS, c->JS, sizeof(double) * c->A.n_x * std::max(1, c->A.ncolors),
                             cudaMemcpyDeviceToDevice, st));
  return RH_OK;
}

int rh_set_timing(rh_ctx *c, int enable) {
  if (!c) return RH_E_ARG;
  c->timing = enable != 0;
  return RH_OK;
}

int rh_pivot_ratio(const rh_ctx *c, double *min_ratio) {
  if (!c || !min_ratio) return RH_E_ARG;
  if (c->host_only) return RH_E_NODEV;
  if (!c->has_state) return RH_E_ORDER;
  const Analysis &A = c->A;
  const int nx = A.n_x, ns = A.sep_rows;
  std::vector<double> dinv(nx), rmax(nx), sp(std::max(1, ns));
  if (cudaSetDevice(c->device) != cudaSuccess ||
      cudaMemcpy(dinv.data(), c->dinv_rows, nx * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(rmax.data(), c->rowmax, nx * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(sp.data(), c->sep_piv, sp.size() * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
    return RH_E_CUDA;
  double r = INFINITY;
  for (int q = 0; q < nx; ++q) {   // segment position -> permuted row
    const int i = A.row_global[q];
    const bool sep = q >= A.seg_row_off[A.nblk];
    const double piv = sep ? std::fabs(sp[q - A.seg_row_off[A.nblk]]) : 1.0 / std::fabs(dinv[i]);
    if (rmax[i] > 0.0) r = std::min(r, piv / rmax[i]);
  }
  *min_ratio = r;
  return RH_OK;
}

int rh_stage_times(const rh_ctx *c, float *ms_out) {
  if (!c || !ms_out) return RH_E_ARG;
  for (int i = 0; i < 9; ++i) ms_out[i] = c->stage_ms[i];
  return RH_OK;
}

}  // extern "C"
