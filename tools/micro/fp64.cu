#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, int n) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 1.0000001, c = 1e-9;
  for (int i = 0; i < n; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void lat(double *out, int n, long long *t) {
  double a = threadIdx.x; const double b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  out[threadIdx.x] = a; if (threadIdx.x == 0) *t = t1 - t0;
}
int main() {
  double *d; cudaMalloc(&d, 1 << 26); long long *t; cudaMalloc(&t, 8);
  int n = 20000;
  lat<<<1, 32>>>(d, n, t); lat<<<1, 32>>>(d, n, t); long long h; cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
  printf("DFMA latency %.2f cycles\n", (double)h / n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<148 * 8, 256>>>(d, n);
  cudaEventRecord(e0); k<<<148 * 8, 256>>>(d, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 8 * n * 148.0 * 8 * 256;
  printf("DFMA throughput %.2f TFLOP/s\n", flops / ms / 1e9);
  return 0;
}
