// FP64 FMA throughput probe: 148 x 4 CTAs x 256 threads, 8 independent DFMA chains.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters) {
  double a[8];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], b, c);
  double s = 0;
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 12345.0) out[0] = s;
}
int main() {
  int sm; cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 8);
  const int iters = 20000, blocks = sm * 4, threads = 256;
  k<<<blocks, threads>>>(d, 100);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 8 * iters * (double)blocks * threads;
  printf("{\"dfma_tflops\": %.2f, \"sm\": %d}\n", flops / ms / 1e9, sm);
}
