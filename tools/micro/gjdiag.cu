#include <cstdio>
#include <cuda_runtime.h>
constexpr int GJB = 32;
__global__ void k(const double *S, double *Dinv, long long *clk, int variant) {
  const int j = threadIdx.x & 31;
  double d[GJB];
#pragma unroll
  for (int i = 0; i < GJB; ++i) d[i] = S[i * 32 + j];
  long long t0 = clock64();
  if (variant == 0) {
#pragma unroll 1
    for (int k = 0; k < GJB; ++k) {
      double dk = 0.0;
#pragma unroll
      for (int i = 0; i < GJB; ++i) if (i == k) dk = d[i];
      const double piv = __shfl_sync(0xffffffffu, dk, k);
      const double inv = 1.0 / piv;
      const double rk = j == k ? inv : dk * inv;
#pragma unroll
      for (int i = 0; i < GJB; ++i) {
        const double f = __shfl_sync(0xffffffffu, d[i], k);
        d[i] = i == k ? rk : (j == k ? -f * inv : fma(-f, rk, d[i]));
      }
    }
  } else {
    // fully unrolled k (large code)
#pragma unroll
    for (int k = 0; k < GJB; ++k) {
      const double piv = __shfl_sync(0xffffffffu, d[k], k);
      const double inv = 1.0 / piv;
      const double rk = j == k ? inv : d[k] * inv;
      double f[GJB];
#pragma unroll
      for (int i = 0; i < GJB; ++i) f[i] = __shfl_sync(0xffffffffu, d[i], k);
#pragma unroll
      for (int i = 0; i < GJB; ++i) if (i != k) d[i] = j == k ? -f[i] * inv : fma(-f[i], rk, d[i]);
      d[k] = rk;
    }
  }
  long long t1 = clock64();
#pragma unroll
  for (int i = 0; i < GJB; ++i) Dinv[i * 32 + j] = d[i];
  if (j == 0) *clk = t1 - t0;
}
int main() {
  double h[1024];
  for (int i = 0; i < 32; ++i) for (int j = 0; j < 32; ++j) h[i * 32 + j] = (i == j ? 40.0 : 0.0) + 0.01 * ((i * 7 + j * 13) % 17);
  double *S, *D; long long *c; cudaMalloc(&S, 8192); cudaMalloc(&D, 8192); cudaMalloc(&c, 8);
  cudaMemcpy(S, h, 8192, cudaMemcpyHostToDevice);
  for (int v = 0; v < 2; ++v) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<<<1, 32>>>(S, D, c, v);
    cudaEventRecord(e0); k<<<1, 32>>>(S, D, c, v); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); long long hc; cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("variant %d: loop %lld cycles, kernel %.1f us\n", v, hc, ms * 1e3);
  }
}
