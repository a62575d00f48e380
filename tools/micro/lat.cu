// latency microbenchmarks: dependent DFMA, DADD, LDS chain, STS->LDS round trip, int->LDS
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int n, long long *out, double *dout) {
  __shared__ double sm[1024];
  __shared__ int si[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = 1.0 + 1e-9 * i; si[i] = (i + 1) & 1023; }
  __syncthreads();
  double a = sm[threadIdx.x], b = 1.0000001, c = 1e-7;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) a = a + c;
  long long t2 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < n; ++i) idx = si[idx];
  long long t3 = clock64();
  double v = 0;
  for (int i = 0; i < n; ++i) { sm[threadIdx.x] = v + 1.0; v = sm[threadIdx.x]; }
  long long t4 = clock64();
  float f = a; float g = 1.0001f;
  for (int i = 0; i < n; ++i) f = fmaf(f, g, 1e-7f);
  long long t5 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4; }
  dout[threadIdx.x] = a + idx + v + f;
}
int main() {
  long long *d; double *dd; cudaMalloc(&d, 64); cudaMalloc(&dd, 8192);
  int n = 10000;
  k<<<1, 32>>>(n, d, dd); k<<<1, 32>>>(n, d, dd);
  long long h[5]; cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
  printf("DFMA dep latency %.1f cycles\nDADD dep latency %.1f\nLDS dependent chain %.1f\nSTS->LDS round trip + DADD %.1f\nFFMA dep %.1f\n",
         (double)h[0] / n, (double)h[1] / n, (double)h[2] / n, (double)h[3] / n, (double)h[4] / n);
  return 0;
}
