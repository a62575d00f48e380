// Microbenchmark: one-warp 32x32 Cholesky with the pivot column broadcast by
// shuffles, the column loop unrolled by template recursion (static register
// indices), against the shared-memory broadcast version used in dense.cu (v3).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
#pragma unroll
  for (int it = 0; it < 3; ++it) y = y * fma(-h * y, y, 1.5);
  return y;
}
template <int C>
struct Step {
  __device__ __forceinline__ static void run(double (&q)[32], double (&dv)[32], int lane) {
    const double piv = __shfl_sync(0xffffffffu, q[C], C);
    const double rs = rsqrt_nr(piv);
    const double l = q[C] * rs;
    q[C] = (lane == C) ? piv * rs : (lane > C ? l : 0.0);
    dv[C] = rs;
#pragma unroll
    for (int m = C + 1; m < 32; ++m) {
      const double lm = __shfl_sync(0xffffffffu, l, m);
      if (m <= lane) q[m] = fma(-l, lm, q[m]);
    }
    Step<C + 1>::run(q, dv, lane);
  }
};
template <>
struct Step<32> {
  __device__ __forceinline__ static void run(double (&)[32], double (&)[32], int) {}
};
__global__ void v7(const double *A, double *out, long long *cyc) {
  const int lane = threadIdx.x;
  double q[32], dv[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) q[m] = A[lane * 32 + m];
  __syncwarp();
  long long t0 = clock64();
  Step<0>::run(q, dv, lane);
  __syncwarp();
  long long t1 = clock64();
#pragma unroll
  for (int m = 0; m < 32; ++m) out[lane * 32 + m] = q[m] + dv[m];
  if (lane == 0) { cyc[0] = t1 - t0; }
}
int main() {
  double h[1024];
  for (int i = 0; i < 32; ++i) for (int j = 0; j < 32; ++j) h[i * 32 + j] = (i == j) ? 40.0 : 1.0 / (1 + i + j);
  double *A, *o; long long *c; cudaMalloc(&A, 8192); cudaMalloc(&o, 8192); cudaMalloc(&c, 16);
  cudaMemcpy(A, h, 8192, cudaMemcpyHostToDevice);
  long long hc[2];
  for (int rep = 0; rep < 3; ++rep) {
    v7<<<1, 32>>>(A, o, c); cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost); printf("v7 shuffle, template-unrolled: factor %lld cycles\n", hc[0]);
  }
  return 0;
}
