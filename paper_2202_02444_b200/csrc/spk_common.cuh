// Shared device helpers: directed-rounding arithmetic per scalar type,
// unit roundoff constants, activation codes.  sm_100a only.
#pragma once
#include <atomic>
#include <cstdint>
#include <cfloat>
#include <cuda_runtime.h>

#include "../../include/spelunk_b200.h"

#define SPK_DEV __device__ __forceinline__

namespace spk {

// Activation codes shared with the C-ABI (include/spelunk_b200.h).
enum Act : int {
  ACT_RELU = SPK_OP_RELU,
  ACT_ELU = SPK_OP_ELU,
  ACT_SIN = SPK_OP_SIN,
  ACT_TANH = SPK_OP_TANH,
  ACT_IDENTITY = SPK_OP_IDENTITY,
  // test hook only (spk_net_debug_corrupt_relu): ReLU whose affine remainder
  // is negated -- the reference's mutation test (test_cli.py:150-164); point
  // values and interval images stay ReLU's
  ACT_RELU_BROKEN = 1000,
};

// Directed-rounding arithmetic.  Every error-channel update is an upper
// bound computed with round-toward-+inf (FFMA.RP / DFMA.RP in SASS), so the
// FP32 enclosure stays sound without interval libraries.
template <typename T> struct Num;

template <> struct Num<float> {
  static constexpr float U = 5.9604644775390625e-8f;     // 2^-24 unit roundoff
  static constexpr float RHO = 1.1920928955078125e-7f;   // 2u, covers one RN op
  static constexpr float TINY = FLT_MIN;                 // underflow guard per op group
  SPK_DEV static float add_ru(float a, float b) { return __fadd_ru(a, b); }
  SPK_DEV static float add_rd(float a, float b) { return __fadd_rd(a, b); }
  SPK_DEV static float sub_ru(float a, float b) { return __fsub_ru(a, b); }
  SPK_DEV static float sub_rd(float a, float b) { return __fsub_rd(a, b); }
  SPK_DEV static float mul_ru(float a, float b) { return __fmul_ru(a, b); }
  SPK_DEV static float mul_rd(float a, float b) { return __fmul_rd(a, b); }
  SPK_DEV static float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
  SPK_DEV static float fma_ru(float a, float b, float c) { return __fmaf_ru(a, b, c); }
  SPK_DEV static float mul_rn(float a, float b) { return __fmul_rn(a, b); }
  SPK_DEV static float div_rn(float a, float b) { return __fdiv_rn(a, b); }
  SPK_DEV static float div_fast(float a, float b) { return __fdividef(a, b); }
  SPK_DEV static float from_d_rn(double x) { return __double2float_rn(x); }
  SPK_DEV static float from_d_ru(double x) { return __double2float_ru(x); }
  SPK_DEV static float from_d_rd(double x) { return __double2float_rd(x); }
};

template <> struct Num<double> {
  static constexpr double U = 1.1102230246251565e-16;    // 2^-53
  static constexpr double RHO = 2.220446049250313e-16;   // 2u
  static constexpr double TINY = DBL_MIN;
  SPK_DEV static double add_ru(double a, double b) { return __dadd_ru(a, b); }
  SPK_DEV static double add_rd(double a, double b) { return __dadd_rd(a, b); }
  SPK_DEV static double sub_ru(double a, double b) { return __dsub_ru(a, b); }
  SPK_DEV static double sub_rd(double a, double b) { return __dsub_rd(a, b); }
  SPK_DEV static double mul_ru(double a, double b) { return __dmul_ru(a, b); }
  SPK_DEV static double mul_rd(double a, double b) { return __dmul_rd(a, b); }
  SPK_DEV static double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
  SPK_DEV static double fma_ru(double a, double b, double c) { return __fma_ru(a, b, c); }
  SPK_DEV static double mul_rn(double a, double b) { return __dmul_rn(a, b); }
  SPK_DEV static double div_rn(double a, double b) { return __ddiv_rn(a, b); }
  SPK_DEV static double div_fast(double a, double b) { return __ddiv_rn(a, b); }
  SPK_DEV static double from_d_rn(double x) { return x; }
  SPK_DEV static double from_d_ru(double x) { return x; }
  SPK_DEV static double from_d_rd(double x) { return x; }
};

// Upper bound of |x - fl(x)| when converting an exact double to T.  FP32:
// |x - RN(x)| <= u |x| <= u/(1-u) |RN(x)| for normal results, plus 2^-150
// below the normal range -- one FFMA.RP instead of the exact residual's two
// FP64 conversions and a DADD (slow-pipe ops on every input coordinate).
template <typename T>
SPK_DEV T conv_err(double x, T xt) {
  if constexpr (sizeof(T) == 4) {
    (void)x;
    return __fmaf_ru(fabsf(xt), 0x1.000002p-24f, 0x1p-149f);
  } else {
    return Num<T>::from_d_ru(fabs(x - (double)xt));
  }
}

// gamma_n = n u / (1 - n u), rounded up: the classic bound on the rounding
// error of an n-term floating-point dot product, any summation order.
inline double gamma_n_host(int n, bool fp32) {
  const double u = fp32 ? 5.9604644775390625e-8 : 1.1102230246251565e-16;
  const double nu = n * u;
  return (nu / (1.0 - nu)) * (1.0 + 4.0 * 2.220446049250313e-16);
}

// Opt a kernel into more than 48 KB of dynamic shared memory on the CURRENT
// device.  The attribute is per (function, device): `done` (one static per
// launch site) records the devices already opted in, so later launches skip
// the call; a failure is returned and NOT cached, so a transient error is
// retried on the next launch.
inline cudaError_t smem_optin(const void* kfn, int bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = dev < 64 ? (1ull << dev) : 0ull;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
  e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_release);
  return e;
}

}  // namespace spk
