// Microbenchmark: one warp factors + inverts a 32x32 SPD tile (k_chol's diagonal step).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kSLd = 33;
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
#pragma unroll
  for (int it = 0; it < 3; ++it) y = y * fma(-h * y, y, 1.5);
  return y;
}
template <int VAR>
__global__ void kf(const double *A, double *out, long long *cyc) {
  __shared__ double s[32][kSLd];
  __shared__ double dv[32];
  const int lane = threadIdx.x;
  for (int r = 0; r < 32; ++r) s[r][lane] = A[r * 32 + lane];
  __syncwarp();
  long long t0 = clock64();
  double q[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) q[m] = s[lane][m];
#pragma unroll 1
  for (int c = 0; c < 32; ++c) {
    double piv = __shfl_sync(0xffffffffu, q[0], c);
    const double rs = VAR == 2 ? 1.0 / piv : rsqrt_nr(piv);
    const double l = q[0] * rs;
    if (lane == c) { s[c][c] = piv * rs; dv[c] = rs; } else if (lane > c) s[lane][c] = l;
#pragma unroll
    for (int m = 1; m < 32; ++m) {
      const double lm = __shfl_sync(0xffffffffu, l, (c + m) & 31);
      if (c + m <= lane) q[m] = fma(-l, lm, q[m]);
    }
#pragma unroll
    for (int m = 0; m < 31; ++m) q[m] = q[m + 1];
  }
  __syncwarp();
  long long t1 = clock64();
  if (VAR != 1) {
#pragma unroll
    for (int i = 0; i < 32; ++i) q[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll 1
    for (int m = 0; m < 32; ++m) {
      const double xm = q[0] * dv[m];
      out[m * 32 + lane] = xm;
#pragma unroll
      for (int i = 1; i < 32; ++i) {
        const int r = m + i;
        if (r < 32) q[i] = fma(-s[r][m], xm, q[i]);
      }
#pragma unroll
      for (int i = 0; i < 31; ++i) q[i] = q[i + 1];
    }
  }
  __syncwarp();
  long long t2 = clock64();
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}
int main() {
  double h[1024];
  for (int i = 0; i < 32; ++i) for (int j = 0; j < 32; ++j) h[i * 32 + j] = (i == j) ? 40.0 : 1.0 / (1 + i + j);
  double *A, *o; long long *c; cudaMalloc(&A, 8192); cudaMalloc(&o, 8192); cudaMalloc(&c, 16);
  cudaMemcpy(A, h, 8192, cudaMemcpyHostToDevice);
  long long hc[2];
  for (int rep = 0; rep < 3; ++rep) {
    kf<0><<<1, 32>>>(A, o, c); cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost); printf("full: factor %lld inverse %lld cycles\n", hc[0], hc[1]);
    kf<1><<<1, 32>>>(A, o, c); cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost); printf("no inverse: factor %lld\n", hc[0]);
    kf<2><<<1, 32>>>(A, o, c); cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost); printf("div instead of rsqrt: factor %lld inverse %lld\n", hc[0], hc[1]);
  }
  return 0;
}
