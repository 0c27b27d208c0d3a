// Throughput probe of the affine K-loop instruction mix (per k-step, per
// thread: 8 neurons x 2 boxes).  Variant 0 = current FP32 mix:
//   2 FFMA2 (base,A1),(A2,A3) + 1 FFMA.RP (v)          per (neuron, box)
// Variant 1 = FP64 base column:
//   1 DFMA (base, W converted once per neuron) + 1 FFMA2 (A1,A2) + 1 FFMA (A3) + 1 FFMA.RP (v)
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2fma(float w, u64 x, u64 a) {
  asm("{.reg .b64 wd;\n mov.b64 wd, {%1, %1};\n fma.rn.f32x2 %0, wd, %2, %0;}" : "+l"(a) : "f"(w), "l"(x));
  return a;
}
template <int V>
__global__ void __launch_bounds__(256, 1) k(float* out, int iters) {
  __shared__ float W[32 * 256];
  __shared__ float X[64 * 24];
  for (int i = threadIdx.x; i < 32 * 256; i += 256) W[i] = 1e-3f * (i % 97);
  for (int i = threadIdx.x; i < 64 * 24; i += 256) X[i] = 1e-3f * (i % 89);
  __syncthreads();
  u64 p0[8][2], p1[8][2];
  float a3[8][2], ae[8][2];
  double b64[8][2];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 2; ++j) { p0[i][j] = p1[i][j] = 0; a3[i][j] = ae[i][j] = 0.f; b64[i][j] = 0.0; }
  const int ng = threadIdx.x % 32;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 4
    for (int kk = 0; kk < 64; ++kk) {
      const float4 wa = *reinterpret_cast<const float4*>(W + (kk & 31) * 256 + ng * 4);
      const float4 wb = *reinterpret_cast<const float4*>(W + (kk & 31) * 256 + 128 + ng * 4);
      const float w[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
      const ulonglong2 x0 = *reinterpret_cast<const ulonglong2*>(X + kk * 24);
      const ulonglong2 x1 = *reinterpret_cast<const ulonglong2*>(X + kk * 24 + 4);
      const ulonglong2 x2 = *reinterpret_cast<const ulonglong2*>(X + kk * 24 + 8);
      const u64 xs[6] = {x0.x, x0.y, x1.x, x1.y, x2.x, x2.y};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double wd = V ? (double)w[i] : 0.0;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (V == 0) {
            p0[i][j] = f2fma(w[i], xs[3 * j], p0[i][j]);
            p1[i][j] = f2fma(w[i], xs[3 * j + 1], p1[i][j]);
            ae[i][j] = __fmaf_ru(fabsf(w[i]), __uint_as_float((unsigned)(xs[3 * j + 2] >> 32)), ae[i][j]);
          } else {
            b64[i][j] = fma(wd, __longlong_as_double((long long)xs[3 * j]), b64[i][j]);
            p0[i][j] = f2fma(w[i], xs[3 * j + 1], p0[i][j]);
            a3[i][j] = __fmaf_rn(w[i], __uint_as_float((unsigned)xs[3 * j + 2]), a3[i][j]);
            ae[i][j] = __fmaf_ru(fabsf(w[i]), __uint_as_float((unsigned)(xs[3 * j + 2] >> 32)), ae[i][j]);
          }
        }
      }
    }
  }
  float s = 0.f;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 2; ++j)
      s += __uint_as_float((unsigned)p0[i][j]) + __uint_as_float((unsigned)p1[i][j]) + a3[i][j] + ae[i][j] +
           (float)b64[i][j];
  if (s == 1234.5f) out[0] = s;
}
int main() {
  int sm;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  float* d;
  cudaMalloc(&d, 8);
  const int iters = 2000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int v = 0; v < 2; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (v == 0) k<0><<<sm, 256>>>(d, iters); else k<1><<<sm, 256>>>(d, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      // useful FMAs: 5 columns per (neuron, box) per k-step
      double fmas = 5.0 * 16 * 64 * (double)iters * 256 * sm;
      if (rep) printf("{\"variant\": %d, \"ms\": %.3f, \"col_fma_tflops\": %.2f}\n", v, ms, 2 * fmas / ms / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
