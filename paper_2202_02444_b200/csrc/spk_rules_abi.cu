// Elementwise activation rules as a C-ABI entry (range_core.py:213-366):
// the device's sound affine rules (spk_rules.cuh) over arrays of per-neuron
// bounds.  Used by the single-form definitional operations of the Python
// layer (affine_nonlinear), so no copy of the rule math lives on the host.
#include <algorithm>
#include <vector>

#include "spk_abi_internal.h"

namespace spk {
namespace {

template <typename T>
__global__ void affine_rule_kernel(int act, long long n, const double* __restrict__ lo,
                                   const double* __restrict__ hi, double* alpha, double* beta, double* gamma) {
  const long long i = (long long)blockIdx.x * 256 + threadIdx.x;
  if (i >= n) return;
  // bounds enter outward-rounded in T
  const T l = Num<T>::from_d_rd(lo[i]), h = Num<T>::from_d_ru(hi[i]);
  T a, b, g;
  const int kind = affine_rule<T>(act, l, h, a, b, g);
  if (kind == 0) {
    a = T(1);
    b = T(0);
    g = T(0);
  } else if (kind == 1) {
    a = T(0);
    b = T(0);
    g = T(0);
  }
  alpha[i] = (double)a;
  beta[i] = (double)b;
  gamma[i] = (double)g;
}

}  // namespace
}  // namespace spk

using namespace spk;

extern "C" int spk_affine_rule(int act, int precision, int64_t n, const double* lo, const double* hi, double* alpha,
                               double* beta, double* gamma) {
  if (n < 0) return fail(SPK_ERR_DIMENSION, "negative size");
  if (n > 0 && (!lo || !hi || !alpha || !beta || !gamma)) return fail(SPK_ERR_INVALID_PARAMETER, "null argument");
  if (act < SPK_OP_RELU || act > SPK_OP_IDENTITY) return fail(SPK_ERR_UNSUPPORTED_ACT, "no affine rule for this op");
  if (n == 0) return SPK_OK;
  double* d = nullptr;
  cudaError_t e = cudaMalloc(&d, (size_t)n * 5 * sizeof(double));
  if (e != cudaSuccess) return cuda_fail(e, "rule alloc");
  e = cudaMemcpy(d, lo, n * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d + n, hi, n * 8, cudaMemcpyHostToDevice);
  const int blk = (int)((n + 255) / 256);
  if (e == cudaSuccess) {
    if (precision == SPK_FP64)
      affine_rule_kernel<double><<<blk, 256>>>(act, n, d, d + n, d + 2 * n, d + 3 * n, d + 4 * n);
    else
      affine_rule_kernel<float><<<blk, 256>>>(act, n, d, d + n, d + 2 * n, d + 3 * n, d + 4 * n);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(alpha, d + 2 * n, n * 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(beta, d + 3 * n, n * 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(gamma, d + 4 * n, n * 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e == cudaSuccess ? SPK_OK : cuda_fail(e, "affine rule");
}
