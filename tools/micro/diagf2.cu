// Microbenchmark: variants of the one-warp 32x32 Cholesky + triangular inverse.
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
// V3: fully unrolled, row per lane, column broadcast through shared memory
__global__ void v3(const double *A, double *out, long long *cyc) {
  __shared__ double s[32][kSLd];
  __shared__ double col[32];
  __shared__ double dv[32];
  const int lane = threadIdx.x;
  for (int r = 0; r < 32; ++r) s[r][lane] = A[r * 32 + lane];
  __syncwarp();
  long long t0 = clock64();
  double q[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) q[m] = s[lane][m];
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    if (lane == c) col[c] = q[c];
    __syncwarp();
    const double piv = col[c];
    const double rs = rsqrt_nr(piv);
    const double l = q[c] * rs;
    q[c] = (lane == c) ? piv * rs : l;
    if (lane == 0) dv[c] = rs;
    col[lane] = l;
    __syncwarp();
#pragma unroll
    for (int m = c + 1; m < 32; ++m)
      if (m <= lane) q[m] = fma(-l, col[m], q[m]);
    __syncwarp();
  }
#pragma unroll
  for (int m = 0; m < 32; ++m) s[lane][m] = q[m];
  __syncwarp();
  long long t1 = clock64();
  // inverse, lane j = column j, fully unrolled, L from shared memory (broadcast)
  double x[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int m = 0; m < r; ++m) {
      if (m & 1) s1 = fma(s[r][m], x[m], s1);
      else s0 = fma(s[r][m], x[m], s0);
    }
    x[r] = (r < lane) ? 0.0 : (r == lane ? dv[r] : -(s0 + s1) * dv[r]);
  }
#pragma unroll
  for (int r = 0; r < 32; ++r) out[r * 32 + lane] = x[r];
  __syncwarp();
  long long t2 = clock64();
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}
// V4: fully unrolled factor with shuffles
__global__ void v4(const double *A, double *out, long long *cyc) {
  __shared__ double s[32][kSLd];
  const int lane = threadIdx.x;
  for (int r = 0; r < 32; ++r) s[r][lane] = A[r * 32 + lane];
  __syncwarp();
  long long t0 = clock64();
  double q[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) q[m] = s[lane][m];
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const double piv = __shfl_sync(0xffffffffu, q[c], c);
    const double rs = rsqrt_nr(piv);
    const double l = q[c] * rs;
    q[c] = (lane == c) ? piv * rs : l;
#pragma unroll
    for (int m = c + 1; m < 32; ++m) {
      const double lm = __shfl_sync(0xffffffffu, l, m);
      if (m <= lane) q[m] = fma(-l, lm, q[m]);
    }
  }
  long long t1 = clock64();
#pragma unroll
  for (int m = 0; m < 32; ++m) out[lane * 32 + m] = q[m];
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = 0; }
}
// V5: 8 warps cooperate: warp w owns rows 4w..4w+3 of the trailing update (smem)
__global__ void v5(const double *A, double *out, long long *cyc) {
  __shared__ double s[32][kSLd];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 1024; i += blockDim.x) s[i / 32][i % 32] = A[i];
  __syncthreads();
  long long t0 = clock64();
  // right-looking; each step: thread (r, m) pairs update the trailing lower triangle
  for (int c = 0; c < 32; ++c) {
    const double piv = s[c][c];
    const double rs = rsqrt_nr(piv);
    __syncthreads();
    if (tid < 32) {
      if (tid > c) s[tid][c] *= rs;
      else if (tid == c) s[c][c] = piv * rs;
    }
    __syncthreads();
    for (int i = tid; i < 1024; i += blockDim.x) {
      const int r = i >> 5, m = i & 31;
      if (m > c && m <= r) s[r][m] = fma(-s[r][c], s[m][c], s[r][m]);
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid < 32) for (int m = 0; m < 32; ++m) out[lane * 32 + m] = s[lane][m];
  if (tid == 0) { cyc[0] = t1 - t0; cyc[1] = 0; }
}
int main() {
  double h[1024];
  for (int i = 0; i < 32; ++i) for (int j = 0; j < 32; ++j) h[i * 32 + j] = (i == j) ? 40.0 : 1.0 / (1 + i + j);
  double *A, *o; long long *c; cudaMalloc(&A, 8192); cudaMalloc(&o, 8192); cudaMalloc(&c, 16);
  cudaMemcpy(A, h, 8192, cudaMemcpyHostToDevice);
  long long hc[2];
  for (int rep = 0; rep < 2; ++rep) {
    v3<<<1, 32>>>(A, o, c); cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost); printf("v3 smem-broadcast unrolled: factor %lld inverse %lld\n", hc[0], hc[1]);
    v4<<<1, 32>>>(A, o, c); cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost); printf("v4 shuffle unrolled: factor %lld\n", hc[0]);
    v5<<<1, 256>>>(A, o, c); cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost); printf("v5 8 warps smem: factor %lld\n", hc[0]);
  }
  return 0;
}
