// Device helpers shared by the library's translation units (redhess.cu, dense.cu).
#pragma once

#include <cuda_runtime.h>

namespace rh {

__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// 1/x to ~1 ulp: hardware approximation + two Newton steps (pivot reciprocals
// on the Gauss-Jordan critical path; static pivots, R15)
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}


// Grid-wide barrier of a cooperative launch (all CTAs co-resident) on a
// monotonic arrival counter zeroed by the host before the launch: barrier
// number `phase` (1, 2, ...) completes when the counter reaches
// phase * gridDim.x.  One atomic per CTA, no reset on the critical path.
__device__ __forceinline__ void grid_barrier_count(unsigned *cnt, unsigned &phase) {
  __syncthreads();
  ++phase;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(cnt, 1u);
    const unsigned target = phase * gridDim.x;
    while ((int)((unsigned)ld_acquire(reinterpret_cast<const int *>(cnt)) - target) < 0) {
    }
    __threadfence();
  }
  __syncthreads();
}

// The same on a subset of the grid: the first `n` CTAs (phase * n arrivals).
__device__ __forceinline__ void grid_barrier_n(unsigned *cnt, unsigned &phase, int n) {
  __syncthreads();
  ++phase;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(cnt, 1u);
    const unsigned target = phase * (unsigned)n;
    while ((int)((unsigned)ld_acquire(reinterpret_cast<const int *>(cnt)) - target) < 0) {
    }
    __threadfence();
  }
  __syncthreads();
}

// D(8x8) += A(8x4) B(4x8) on the fp64 tensor cores: a = A[gid][tig], b = B[tig][gid],
// (c0, c1) = D[gid][2 tig], D[gid][2 tig + 1] (gid = lane / 4, tig = lane % 4)
__device__ __forceinline__ void dmma_8x8x4(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

}  // namespace rh
