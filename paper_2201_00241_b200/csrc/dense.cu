// Dense SPD solve of the real-time tracking step, Step 2 (PAPER.md:970-977,
// Eq. qp_rto: H_t d_t = -g_t by a dense Cholesky factorization).  See dense.hpp.
//
// Layout: the bordered matrix
//     M = [ Hs + tau I    0 ]      Hs = (H + H^T) / 2   (R-T1)
//         [ -g^T          1 ]      padded with identity rows to nt 32
// lives row-major in A (only the lower 32 x 32 tiles are touched).  Its
// Cholesky factor has y = L^-1 (-g) as the bordered row, so the forward
// substitution costs nothing extra; k_chol_bwd then solves L^T d = y.
//
// k_chol (one cooperative launch, 8 warps per CTA, one warp per 32 x 32 tile task):
//   fill the lower tiles of M; grid barrier; for k = -1 .. nt-2:
//     every trailing tile (i, j), k < j <= i:  A_ij -= L_ik L_jk^T   (DMMA m8n8k4)
//     tiles of column k+1 then finish it: the diagonal tile is factored and its
//     inverse published by warp 0 of CTA 0 (flag = epoch); the others wait for
//     the flag and form L_i,k+1 = A_i,k+1 Linv^T (DMMA); grid barrier.
// All global reads of A / Linv go through L2 (__ldcg): tiles change owners
// between iterations and L1 is not coherent.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>

#include "dense.hpp"
#include "devutil.cuh"

namespace rh {
namespace {

constexpr int kCholWarps = 8;
constexpr int kSLd = 33;   // smem tile row stride (doubles)

struct CholArgs {
  const double *H;
  long long ldh;
  const double *g;
  double tau;
  int n, nt;
  double *A;
  long long lda;
  double *Linv;
  unsigned *bar;
  int *flags, *fail;
  int epoch;
  long long *dbg;   // timing experiment (RH_DEBUG & 512): per-iteration globaltimer stamps
};

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// u -> (r, c), 0 <= c <= r: row-major enumeration of a lower triangle
__device__ __forceinline__ void tri_decode(long long u, int &r, int &c) {
  int rr = (int)((sqrt(8.0 * (double)u + 1.0) - 1.0) * 0.5);
  while ((long long)(rr + 1) * (rr + 2) / 2 <= u) ++rr;
  while ((long long)rr * (rr + 1) / 2 > u) --rr;
  r = rr;
  c = (int)(u - (long long)rr * (rr + 1) / 2);
}

__device__ __forceinline__ double2 ldcg2(const double *p) { return __ldcg(reinterpret_cast<const double2 *>(p)); }

// 32 x 32 tile <-> D-fragment registers: acc[rb][cb] = T[rb 8 + gid][cb 8 + 2 tig + {0,1}]
__device__ __forceinline__ void tile_load(double (&acc)[4][4][2], const double *T, long long ld, int gid, int tig) {
#pragma unroll
  for (int rb = 0; rb < 4; ++rb)
#pragma unroll
    for (int cb = 0; cb < 4; ++cb) {
      const double2 v = ldcg2(T + (long long)(rb * 8 + gid) * ld + cb * 8 + 2 * tig);
      acc[rb][cb][0] = v.x;
      acc[rb][cb][1] = v.y;
    }
}
__device__ __forceinline__ void tile_store(const double (&acc)[4][4][2], double *T, long long ld, int gid, int tig) {
#pragma unroll
  for (int rb = 0; rb < 4; ++rb)
#pragma unroll
    for (int cb = 0; cb < 4; ++cb)
      __stcg(reinterpret_cast<double2 *>(T + (long long)(rb * 8 + gid) * ld + cb * 8 + 2 * tig),
             make_double2(acc[rb][cb][0], acc[rb][cb][1]));
}

// acc -= Li Lj^T over the 32 columns of the panel.  The k index is permuted
// per thread (thread tig owns k = 8 tig + 4 h + q) so that each thread's
// operands are contiguous: both operands use the same permutation, so every
// k is summed exactly once.
__device__ __forceinline__ void tile_syrk(double (&acc)[4][4][2], const double *Li, const double *Lj, long long ld,
                                          int gid, int tig) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    double a[4][4], b[4][4];
#pragma unroll
    for (int rb = 0; rb < 4; ++rb) {
      const double *pa = Li + (long long)(rb * 8 + gid) * ld + tig * 8 + h * 4;
      const double2 v0 = ldcg2(pa), v1 = ldcg2(pa + 2);
      a[rb][0] = -v0.x;
      a[rb][1] = -v0.y;
      a[rb][2] = -v1.x;
      a[rb][3] = -v1.y;
      const double *pb = Lj + (long long)(rb * 8 + gid) * ld + tig * 8 + h * 4;
      const double2 w0 = ldcg2(pb), w1 = ldcg2(pb + 2);
      b[rb][0] = w0.x;
      b[rb][1] = w0.y;
      b[rb][2] = w1.x;
      b[rb][3] = w1.y;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int rb = 0; rb < 4; ++rb)
#pragma unroll
        for (int cb = 0; cb < 4; ++cb) dmma_8x8x4(acc[rb][cb][0], acc[rb][cb][1], a[rb][q], b[cb][q]);
  }
}

// Fill tile (i, j) of the bordered, symmetrized, shifted matrix M (one warp).
__device__ void fill_tile(const CholArgs &a, int i, int j, double (*s)[kSLd], int lane) {
  const int n = a.n;
  // mirrored tile H[j 32 + r][i 32 + lane] -> s[r][lane]
  for (int r = 0; r < 32; ++r) {
    const int R = j * 32 + r, C = i * 32 + lane;
    s[r][lane] = (R < n && C < n) ? __ldg(a.H + (long long)R * a.ldh + C) : 0.0;
  }
  __syncwarp();
  for (int r = 0; r < 32; ++r) {
    const int R = i * 32 + r, C = j * 32 + lane;
    double v;
    if (R < n && C < n)
      v = 0.5 * (__ldg(a.H + (long long)R * a.ldh + C) + s[lane][r]) + (R == C ? a.tau : 0.0);
    else if (R == n && C < n)
      v = -__ldg(a.g + C);
    else
      v = (R == C) ? 1.0 : 0.0;
    __stcg(a.A + (long long)R * a.lda + C, v);
  }
  __syncwarp();
}

// 1/sqrt(x): hardware approximation + three Newton steps (full fp64 accuracy)
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
#pragma unroll
  for (int it = 0; it < 3; ++it) y = y * fma(-h * y, y, 1.5);
  return y;
}

// Factor the diagonal tile in s (one warp; lane r owns row r in registers,
// fully unrolled so every register index is static; the pivot and the step's
// column are broadcast through shared memory), write L back to s and the
// inverse of L to Linv.  Pivots of rows >= n (padding and the bordered
// right-hand-side row) are taken as 1.  (tools/micro/diagf2.cu: 2.6x faster
// than a rolled loop with rotated registers, 2.4x faster than shuffles.)
__device__ __forceinline__ void diag_factor(const CholArgs &a, int kt, double (*s)[kSLd], double *dv, double *col,
                                            int lane) {
  const int base = kt * 32;
  double q[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) q[m] = s[lane][m];
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    if (lane == c) col[c] = q[c];
    __syncwarp();
    double piv = col[c];
    if (base + c >= a.n) {
      piv = 1.0;
    } else if (!(piv > 0.0)) {   // not positive definite (NaN included)
      if (lane == 0) atomicCAS(a.fail, 0, base + c + 1);
      piv = 1.0;
    }
    const double rs = rsqrt_nr(piv);
    const double l = q[c] * rs;   // L[lane][c] for lane > c
    q[c] = (lane == c) ? piv * rs : (lane > c ? l : 0.0);
    if (lane == 0) dv[c] = rs;
    __syncwarp();
    col[lane] = l;
    __syncwarp();
#pragma unroll
    for (int m = c + 1; m < 32; ++m)
      if (m <= lane) q[m] = fma(-l, col[m], q[m]);
    __syncwarp();   // every lane has read col before the next step overwrites it
  }
#pragma unroll
  for (int m = 0; m < 32; ++m) s[lane][m] = (m <= lane) ? q[m] : 0.0;
  __syncwarp();
  // X = L^-1, lane j owns column j: X[r][j] = -(sum_{m < r} L[r][m] X[m][j]) / L[r][r]
  // (X[m][j] = 0 for m < j), X[j][j] = 1 / L[j][j]; four partial sums per row
  double *Li = a.Linv + (long long)kt * 1024;
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    double t[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int m = 0; m < r; ++m) t[m & 3] = fma(s[r][m], q[m], t[m & 3]);
    const double dr = dv[r];
    q[r] = (r < lane) ? 0.0 : (r == lane ? dr : -((t[0] + t[1]) + (t[2] + t[3])) * dr);
    __stcg(Li + r * 32 + lane, q[r]);
  }
}

__global__ void __launch_bounds__(kCholWarps * 32, 1) k_chol(CholArgs a) {
  extern __shared__ double csm[];

  __shared__ double s_dv[32], s_col[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  double(*s)[kSLd] = reinterpret_cast<double(*)[kSLd]>(csm + warp * 32 * kSLd);
  unsigned gen = 0;   // barrier phase (a.bar[0] zeroed by the host before the launch)
  const int nt = a.nt;
  const long long W = (long long)gridDim.x * kCholWarps, gw = (long long)blockIdx.x * kCholWarps + warp;
  const long long nfill = (long long)nt * (nt + 1) / 2;
  for (long long u = gw; u < nfill; u += W) {
    int i, j;
    tri_decode(u, i, j);
    fill_tile(a, i, j, s, lane);
  }
  grid_barrier_count(a.bar, gen);
  for (int k = -1; k <= nt - 2; ++k) {
    const int c1 = k + 1, m = nt - c1;
    if (a.dbg && blockIdx.x == 0 && threadIdx.x == 0 && k + 1 < 256) a.dbg[(k + 1) * 4 + 0] = gtimer();
    const long long ntask = k < 0 ? m : m + (long long)m * (m - 1) / 2;
    for (long long t = gw; t < ntask; t += W) {
      int i, j;
      if (t < m) {
        i = c1 + (int)t;
        j = c1;
      } else {
        int rr, cc;
        tri_decode(t - m, rr, cc);
        i = c1 + 1 + rr;
        j = c1 + 1 + cc;
      }
      double acc[4][4][2];
      double *T = a.A + (long long)i * 32 * a.lda + j * 32;
      tile_load(acc, T, a.lda, gid, tig);
      if (k >= 0)
        tile_syrk(acc, a.A + (long long)i * 32 * a.lda + k * 32, a.A + (long long)j * 32 * a.lda + k * 32, a.lda,
                  gid, tig);
      if (j != c1) {
        tile_store(acc, T, a.lda, gid, tig);
        continue;
      }
      // column k+1: park the updated tile in shared memory
#pragma unroll
      for (int rb = 0; rb < 4; ++rb)
#pragma unroll
        for (int cb = 0; cb < 4; ++cb) {
          s[rb * 8 + gid][cb * 8 + 2 * tig] = acc[rb][cb][0];
          s[rb * 8 + gid][cb * 8 + 2 * tig + 1] = acc[rb][cb][1];
        }
      __syncwarp();
      if (i == c1) {
        if (a.dbg && lane == 0 && c1 < 256) a.dbg[c1 * 4 + 1] = gtimer();
        diag_factor(a, c1, s, s_dv, s_col, lane);
        if (a.dbg && lane == 0 && c1 < 256) a.dbg[c1 * 4 + 2] = gtimer();
        for (int r = 0; r < 32; ++r) __stcg(T + (long long)r * a.lda + lane, s[r][lane]);   // L (and y) of the tile
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release(a.flags + c1, a.epoch);
        __syncwarp();
      } else {
        if (lane == 0)
          while (ld_acquire(a.flags + c1) != a.epoch) {
          }
        __syncwarp();
        // L_i,c1 = A_i,c1 Linv^T: a = S[rb 8 + gid][kk], b = Linv[cb 8 + gid][kk], kk = 8 tig + q
        const double *Li = a.Linv + (long long)c1 * 1024;
        double o[4][4][2];
#pragma unroll
        for (int rb = 0; rb < 4; ++rb)
#pragma unroll
          for (int cb = 0; cb < 4; ++cb) o[rb][cb][0] = o[rb][cb][1] = 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double av[4][4], bv[4][4];
#pragma unroll
          for (int rb = 0; rb < 4; ++rb)
#pragma unroll
            for (int q = 0; q < 4; ++q) av[rb][q] = s[rb * 8 + gid][tig * 8 + h * 4 + q];
#pragma unroll
          for (int cb = 0; cb < 4; ++cb) {
            const double *pb = Li + (cb * 8 + gid) * 32 + tig * 8 + h * 4;
            const double2 w0 = ldcg2(pb), w1 = ldcg2(pb + 2);
            bv[cb][0] = w0.x;
            bv[cb][1] = w0.y;
            bv[cb][2] = w1.x;
            bv[cb][3] = w1.y;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int rb = 0; rb < 4; ++rb)
#pragma unroll
              for (int cb = 0; cb < 4; ++cb) dmma_8x8x4(o[rb][cb][0], o[rb][cb][1], av[rb][q], bv[cb][q]);
        }
        tile_store(o, T, a.lda, gid, tig);
        if (a.dbg && t == 1 && lane == 0 && c1 < 256) a.dbg[c1 * 4 + 3] = gtimer();
      }
      __syncwarp();
    }
    grid_barrier_count(a.bar, gen);
  }
}

// L^T d = y (y = the bordered row of the factor), one warp per 32-block,
// blocks taken in decreasing order by ticket; block k waits for d_j (j > k)
// in decreasing j and accumulates L_jk^T d_j as they land, then
// d_k = Linv_k^T (y_k - acc).  On success p[0..n) += alpha d.
__global__ void __launch_bounds__(32) k_chol_bwd(const double *A, long long lda, const double *Linv, int n, int nt,
                                                 double *dbuf, double *p, double alpha, int *fail, int *flags_d,
                                                 int epoch) {
  if (__ldcg(fail) != 0) return;   // factorization failed: nothing to solve
  const int lane = threadIdx.x;
  int t = 0;
  if (lane == 0) t = atomicAdd(fail + 1, 1);
  t = __shfl_sync(0xffffffffu, t, 0);
  const int k = nt - 1 - t;
  const int idx = k * 32 + lane;
  double acc = (idx < n) ? __ldcg(A + (long long)n * lda + idx) : 0.0;
  double li[32];   // column `lane` of Linv_k (final before this launch)
  const double *Li = Linv + (long long)k * 1024;
#pragma unroll
  for (int r = 0; r < 32; ++r) li[r] = __ldcg(Li + r * 32 + lane);
  for (int j = nt - 1; j > k; --j) {
    double lt[32];   // column k 32 + lane of tile row j (final): fetched before waiting for d_j
    const double *Lt = A + (long long)j * 32 * lda + k * 32 + lane;
#pragma unroll
    for (int r = 0; r < 32; ++r) lt[r] = __ldcg(Lt + (long long)r * lda);
    if (lane == 0)
      while (ld_acquire(flags_d + j) != epoch) {
      }
    __syncwarp();
    const double dj = __ldcg(dbuf + j * 32 + lane);
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int r = 0; r < 32; r += 2) {
      s0 = fma(lt[r], __shfl_sync(0xffffffffu, dj, r), s0);
      s1 = fma(lt[r + 1], __shfl_sync(0xffffffffu, dj, r + 1), s1);
    }
    acc -= s0 + s1;
  }
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int r = 0; r < 32; r += 2) {
    s0 = fma(li[r], __shfl_sync(0xffffffffu, acc, r), s0);
    s1 = fma(li[r + 1], __shfl_sync(0xffffffffu, acc, r + 1), s1);
  }
  const double dk = (idx < n) ? s0 + s1 : 0.0;
  __stcg(dbuf + idx, dk);
  if (p && idx < n) p[idx] += alpha * dk;
  __threadfence();
  __syncwarp();
  if (lane == 0) st_release(flags_d + k, epoch);
}

constexpr size_t chol_smem() { return sizeof(double) * kCholWarps * 32 * kSLd; }

}  // namespace

cudaError_t dense_ws_ensure(DenseWs &w, int n, int device) {
  const int nt = (n + 1 + 31) / 32;   // + the bordered row
  if (!w.nsm) {
    cudaDeviceGetAttribute(&w.nsm, cudaDevAttrMultiProcessorCount, device);
    cudaError_t e = cudaFuncSetAttribute(k_chol, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chol_smem());
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&w.coop_per_sm, k_chol, kCholWarps * 32, chol_smem());
    if (e != cudaSuccess) return e;
    if (w.coop_per_sm < 1) return cudaErrorLaunchOutOfResources;
    e = cudaMalloc(&w.fail, 2 * sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&w.bar, 2 * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(w.bar, 0, 2 * sizeof(unsigned));
    if (e != cudaSuccess) return e;
  }
  if (nt <= w.cap) return cudaSuccess;
  cudaFree(w.A);
  cudaFree(w.Linv);
  cudaFree(w.dbuf);
  cudaFree(w.flags);
  cudaFree(w.flags_d);
  w.A = w.Linv = w.dbuf = nullptr;
  w.flags = w.flags_d = nullptr;
  w.cap = 0;
  const size_t ld = (size_t)nt * 32;
  cudaError_t e = cudaMalloc(&w.A, sizeof(double) * ld * ld);
  if (e == cudaSuccess) e = cudaMalloc(&w.Linv, sizeof(double) * 1024 * nt);
  if (e == cudaSuccess) e = cudaMalloc(&w.dbuf, sizeof(double) * ld);
  if (e == cudaSuccess) e = cudaMalloc(&w.flags, sizeof(int) * nt);
  if (e == cudaSuccess) e = cudaMalloc(&w.flags_d, sizeof(int) * nt);
  if (e == cudaSuccess) e = cudaMemset(w.flags, 0, sizeof(int) * nt);
  if (e == cudaSuccess) e = cudaMemset(w.flags_d, 0, sizeof(int) * nt);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return e;
  w.cap = nt;
  w.epoch = 0;
  return cudaSuccess;
}

void dense_ws_free(DenseWs &w) {
  cudaFree(w.A);
  cudaFree(w.Linv);
  cudaFree(w.dbuf);
  cudaFree(w.flags);
  cudaFree(w.flags_d);
  cudaFree(w.fail);
  cudaFree(w.bar);
  w = DenseWs{};
}

cudaError_t dense_spd_attempt(DenseWs &w, int n, const double *H, long long ldh, const double *g, double tau,
                              double *p, double alpha, cudaStream_t st, int *launches) {
  const int nt = (n + 1 + 31) / 32;
  if (nt > w.cap) return cudaErrorInvalidValue;
  if (++w.epoch <= 0) w.epoch = 1;   // flags compare against the epoch: never reset
  cudaError_t e = cudaMemsetAsync(w.fail, 0, 2 * sizeof(int), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(w.bar, 0, sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  CholArgs a;
  a.H = H;
  a.ldh = ldh;
  a.g = g;
  a.tau = tau;
  a.n = n;
  a.nt = nt;
  a.A = w.A;
  a.lda = (long long)nt * 32;
  a.Linv = w.Linv;
  a.bar = w.bar;
  a.flags = w.flags;
  a.fail = w.fail;
  a.epoch = w.epoch;
  a.dbg = nullptr;
  static long long *dbg = nullptr;
  if (const char *env = getenv("RH_DEBUG"))
    if (atoi(env) & 512) {
      if (!dbg) cudaMalloc(&dbg, 1024 * sizeof(long long));
      cudaMemsetAsync(dbg, 0, 1024 * sizeof(long long), st);
      a.dbg = dbg;
    }
  const long long tasks = (long long)nt * (nt + 1) / 2;
  const int grid = (int)std::min<long long>((long long)w.coop_per_sm * w.nsm, (tasks + kCholWarps - 1) / kCholWarps);
  void *args[] = {&a};
  e = cudaLaunchCooperativeKernel((const void *)k_chol, dim3(std::max(grid, 1)), dim3(kCholWarps * 32), args,
                                  chol_smem(), st);
  if (e != cudaSuccess) return e;
  k_chol_bwd<<<nt, 32, 0, st>>>(w.A, (long long)nt * 32, w.Linv, n, nt, w.dbuf, p, alpha, w.fail, w.flags_d,
                                w.epoch);
  if (launches) *launches += 2;
  if (a.dbg) {
    long long h[1024];
    cudaMemcpyAsync(h, a.dbg, sizeof h, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const int K = std::min(nt, 256);
    double sd = 0, sf = 0, sp = 0, sit = 0;
    for (int k = 1; k + 1 < K; ++k) {
      sd += h[k * 4 + 1] - h[k * 4 + 0];
      sf += h[k * 4 + 2] - h[k * 4 + 1];
      sp += h[k * 4 + 3] - h[k * 4 + 2];
      sit += h[(k + 1) * 4 + 0] - h[k * 4 + 0];
    }
    const double c = K > 2 ? 1.0 / (K - 2) : 0.0;
    fprintf(stderr, "k_chol n=%d grid=%d: per iteration (ns) update-to-diag %.0f factor %.0f panel-after %.0f total %.0f\n",
            n, grid, sd * c, sf * c, sp * c, sit * c);
  }
  return cudaGetLastError();
}

}  // namespace rh
