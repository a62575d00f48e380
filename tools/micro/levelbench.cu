// Micro-benchmark: cost of a CTA-wide level step (barrier + one warp's dependent chain).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int nlev, int chain, int useDouble, long long *out, int threads) {
  extern __shared__ double sm[];
  int *si = reinterpret_cast<int *>(sm + 4096);
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) { sm[i] = 1.0 + i * 1e-9; si[i] = (i * 7 + 3) & 4095; }
  __syncthreads();
  long long t0 = clock64();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc = 0; int idx = lane;
  for (int l = 0; l < nlev; ++l) {
    if (warp == (l % (threads / 32))) {
      for (int c = 0; c < chain; ++c) {
        idx = si[idx];                       // dependent LDS chain
        if (useDouble) acc = fma(sm[idx], 1.0000001, acc);
      }
      sm[lane] = acc + idx;                 // store
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
int main() {
  long long *d; cudaMalloc(&d, 8 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int cfg[][3] = {{512, 0, 0}, {512, 1, 0}, {512, 4, 0}, {512, 4, 1}, {512, 16, 1}, {128, 0, 0}, {128, 4, 1}, {1024, 4, 1}};
  for (auto &c : cfg) {
    int threads = c[0], chain = c[1], dbl = c[2];
    int nlev = 1000;
    k<<<1, threads, 64 * 1024>>>(nlev, chain, dbl, d, threads);
    k<<<1, threads, 64 * 1024>>>(nlev, chain, dbl, d, threads);
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("threads %4d chain %2d double %d : %.1f cycles/level\n", threads, chain, dbl, (double)h / nlev);
    // many CTAs concurrently: 148 SMs x 1
    k<<<148, threads, 64 * 1024>>>(nlev, chain, dbl, d, threads);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("   (148 CTAs) %.1f cycles/level\n", (double)h / nlev);
  }
  return 0;
}
