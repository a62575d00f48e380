// fp64 tensor-core throughput probe: mma.sync.aligned.m8n8k4.row.col.f64 on sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, int n) {
  double a = 1.0 + threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-3;
  double c0[8], c1[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c0[i] = 0.0; c1[i] = 0.0; }
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c0[i]), "+d"(c1[i]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += c0[i] + c1[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double *d; cudaMalloc(&d, 148 * 8 * 256 * 8);
  int n = 4000;
  k<<<148 * 4, 256>>>(d, n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<<<148 * 4, 256>>>(d, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 8 * 8 * 4 * 8.0 * n * (148 * 4 * 256 / 32);
  printf("DMMA m8n8k4 throughput %.2f TFLOP/s (%s)\n", flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
