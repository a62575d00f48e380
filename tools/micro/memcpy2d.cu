// D2H bandwidth of one column block of H (2889 rows x w doubles, host row pitch 2889) by
// cudaMemcpy2DAsync vs a contiguous 1D copy of the same bytes (pinned host memory).
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t n = 2889;
  double *d, *h;
  cudaMalloc(&d, n * n * 8);
  cudaMallocHost(&h, n * n * 8);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (size_t w : {1024, 841, 256}) {
    float ms2 = 0, ms1 = 0;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0, st);
      cudaMemcpy2DAsync(h, n * 8, d, n * 8, w * 8, n, cudaMemcpyDeviceToHost, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms2, e0, e1);
      cudaEventRecord(e0, st);
      cudaMemcpyAsync(h, d, n * w * 8, cudaMemcpyDeviceToHost, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms1, e0, e1);
    }
    const double mb = n * w * 8 / 1e6;
    printf("w=%zu (%.1f MB): 2D %.3f ms (%.1f GB/s)  1D %.3f ms (%.1f GB/s)\n", w, mb, ms2, mb / ms2, ms1, mb / ms1);
  }
  return 0;
}
