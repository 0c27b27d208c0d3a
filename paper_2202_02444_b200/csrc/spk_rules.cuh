// Sound activation linearisations and interval images.
//
// Each affine rule follows the reference's choice of slope alpha
// (range_core.py:213-317) but derives (beta, gamma) from rigorous bounds of
// the remainder g(x) = h(x) - alpha*x on [lo, hi] for the alpha that is
// actually stored in T, so the enclosure |h(x) - alpha x - beta| <= gamma
// holds in floating point, not only in exact arithmetic.
//  * ReLU runs entirely in T with directed rounding (remainder extremes at
//    lo, 0, hi).
//  * ELU / sin / tanh evaluate the remainder at the reference's candidate
//    points in FP64 and pad every candidate by a few FP64 ulps (libm error)
//    before rounding outward to T; for sin/tanh the candidate critical points
//    are only approximately located, which costs a second-order term that
//    the pad also covers.
// Interval images (range_core.py:326-349) are rounded outward the same way.
#pragma once
#include "spk_common.cuh"

namespace spk {

constexpr double kTwoPi = 6.283185307179586;
constexpr double kPi = 3.141592653589793;
constexpr double kHalfPi = 1.5707963267948966;

// Relative + absolute pad covering a few FP64 roundings / libm ulps.
SPK_DEV double pad64(double scale) { return 1.0e-15 * scale + 1e-300; }

// Turn FP64 bounds r_l <= g <= r_u into (beta, gamma) in T, soundly.
template <typename T>
SPK_DEV void finish_remainder(double r_l, double r_u, T& beta, T& gamma) {
  const T b = Num<T>::from_d_rn(0.5 * (r_l + r_u));
  const double bd = (double)b;
  const double g = fmax(__dsub_ru(r_u, bd), __dsub_ru(bd, r_l));
  gamma = Num<T>::from_d_ru(fmax(g, 0.0));
  beta = b;
}

// ----------------------------------------------------------------- ReLU
// range_core.py:213-231: alpha = hi/(hi-lo) on straddling lanes.
// Returns 0: identity (alpha 1, beta 0, gamma 0), 1: zero, 2: general.
template <typename T>
SPK_DEV int relu_affine(T lo, T hi, T& alpha, T& beta, T& gamma) {
  if (lo >= T(0)) { alpha = T(1); beta = T(0); gamma = T(0); return 0; }
  if (hi <= T(0)) { alpha = T(0); beta = T(0); gamma = T(0); return 1; }
  // any slope in [0, 1] is sound (gamma is derived for the stored slope),
  // so the FP32 path uses the fast reciprocal-multiply division
  T a = Num<T>::div_fast(hi, hi - lo);
  a = fmin(fmax(a, T(0)), T(1));  // NaN-safe clamp
  // g(x) = relu(x) - a x is >= 0 on [lo, hi] (g(0) = 0) with
  // max(g) = max(-a lo, hi - a hi).
  const T ru = fmax(Num<T>::mul_ru(-a, lo), Num<T>::fma_ru(-a, hi, hi));
  const T b = Num<T>::mul_rn(ru, T(0.5));
  alpha = a;
  beta = b;
  gamma = fmax(b, Num<T>::sub_ru(ru, b));
  return 2;
}

// ------------------------------------------------------------------ ELU
SPK_DEV double elu64(double x) { return x >= 0.0 ? x : expm1(x); }

// range_core.py:238-264.  g = elu(x) - a x is convex, so its max is at an
// endpoint and its global minimum is (a - 1) - a ln a (tangent point
// x* = ln a); with a <= 0 (secant underflow) g = elu - a x is monotone.
#define SPK_RULE __device__ __noinline__

template <typename T>
SPK_RULE int elu_affine(T lo_t, T hi_t, T& alpha, T& beta, T& gamma) {
  const double lo = (double)lo_t, hi = (double)hi_t;
  if (lo >= 0.0) { alpha = T(1); beta = T(0); gamma = T(0); return 0; }
  const double flo = elu64(lo), fhi = elu64(hi);
  double a;
  if (hi == lo) a = exp(lo);
  else a = (fhi - flo) / (hi - lo);
  T at = Num<T>::from_d_rn(a);
  if (!(at > T(0))) at = T(0);
  if (at > T(1)) at = T(1);
  const double ad = (double)at;
  const double g_lo = flo - ad * lo, g_hi = fhi - ad * hi;
  const double p_lo = pad64(fabs(flo) + fabs(ad * lo) + 1.0);
  const double p_hi = pad64(fabs(fhi) + fabs(ad * hi) + 1.0);
  double r_u = fmax(g_lo + p_lo, g_hi + p_hi);
  double r_l = fmin(g_lo - p_lo, g_hi - p_hi);
  if (ad > 0.0) {
    const double gs = (ad - 1.0) - ad * log(ad);
    r_l = fmin(r_l, gs - pad64(2.0 + fabs(ad * log(ad))));
  }
  alpha = at;
  finish_remainder<T>(r_l, r_u, beta, gamma);
  return 2;
}

// ------------------------------------------------------------------ sin
// cos range over [lo, hi] by modular extremum detection (range_core.py:267-274)
SPK_DEV void cos_range64(double lo, double hi, double& cmin, double& cmax) {
  const double clo = cos(lo), chi = cos(hi);
  cmin = fmin(clo, chi);
  cmax = fmax(clo, chi);
  if (floor(hi / kTwoPi) * kTwoPi >= lo) cmax = 1.0;
  if (floor((hi - kPi) / kTwoPi) * kTwoPi + kPi >= lo) cmin = -1.0;
}

// range_core.py:277-294: alpha = midpoint of the cos range; remainder
// extremes among lo, hi and the first two 2pi-translates (at/after lo) of
// +-arccos(alpha).
template <typename T>
SPK_RULE int sin_affine(T lo_t, T hi_t, T& alpha, T& beta, T& gamma) {
  const double lo = (double)lo_t, hi = (double)hi_t;
  double cmin, cmax;
  cos_range64(lo, hi, cmin, cmax);
  const T at = Num<T>::from_d_rn(0.5 * (cmin + cmax));
  const double ad = (double)at;
  const double e = acos(fmin(fmax(ad, -1.0), 1.0));
  double r_u = -1e300, r_l = 1e300;
  auto visit = [&](double x) {
    const double g = sin(x) - ad * x;
    const double p = pad64(4.0 + 2.0 * fabs(ad * x) + fabs(x) * 1e-3);
    r_u = fmax(r_u, g + p);
    r_l = fmin(r_l, g - p);
  };
  visit(lo);
  visit(hi);
#pragma unroll
  for (int sgn = 0; sgn < 2; ++sgn) {
    const double root = sgn ? -e : e;
    const double first = root + kTwoPi * ceil((lo - root) / kTwoPi);
    visit(fmin(fmax(first, lo), hi));
    visit(fmin(fmax(first + kTwoPi, lo), hi));
  }
  alpha = at;
  finish_remainder<T>(r_l, r_u, beta, gamma);
  return 2;
}

// ----------------------------------------------------------------- tanh
// range_core.py:297-317: secant slope; remainder extremes at lo, hi and
// +-artanh(sqrt(1 - alpha)) clamped into [lo, hi].
template <typename T>
SPK_RULE int tanh_affine(T lo_t, T hi_t, T& alpha, T& beta, T& gamma) {
  const double lo = (double)lo_t, hi = (double)hi_t;
  const double flo = tanh(lo), fhi = tanh(hi);
  const double a = (hi == lo) ? 1.0 - flo * flo : (fhi - flo) / (hi - lo);
  T at = Num<T>::from_d_rn(a);
  const double ad = (double)at;
  double r_u = -1e300, r_l = 1e300;
  auto visit = [&](double x) {
    const double g = tanh(x) - ad * x;
    const double p = pad64(4.0 + 2.0 * fabs(ad * x));
    r_u = fmax(r_u, g + p);
    r_l = fmin(r_l, g - p);
  };
  visit(lo);
  visit(hi);
  const double inner = sqrt(fmin(fmax(1.0 - ad, 0.0), 1.0));
  const double xs = inner >= 1.0 ? 1e300 : atanh(inner);
  visit(fmin(fmax(xs, lo), hi));
  visit(fmin(fmax(-xs, lo), hi));
  alpha = at;
  finish_remainder<T>(r_l, r_u, beta, gamma);
  return 2;
}

template <typename T>
SPK_DEV int affine_rule(int act, T lo, T hi, T& alpha, T& beta, T& gamma) {
  switch (act) {
    case ACT_RELU: return relu_affine<T>(lo, hi, alpha, beta, gamma);
    case ACT_RELU_BROKEN: {
      const int k = relu_affine<T>(lo, hi, alpha, beta, gamma);
      gamma = -gamma;
      return k;
    }
    case ACT_ELU: return elu_affine<T>(lo, hi, alpha, beta, gamma);
    case ACT_SIN: return sin_affine<T>(lo, hi, alpha, beta, gamma);
    case ACT_TANH: return tanh_affine<T>(lo, hi, alpha, beta, gamma);
    default: alpha = T(1); beta = T(0); gamma = T(0); return 0;
  }
}

// ------------------------------------------------------- interval images
// range_core.py:326-349, rounded outward.
template <typename T>
SPK_RULE void interval_image_slow(int act, T lo, T hi, T& out_lo, T& out_hi);

// FP32 sin image for |lo|, |hi| <= 2048 (range_core.py:338-345).  sinf is
// within 2 ulp (<= 2^-23 absolute on [-1, 1]).  The FP32 modular test can
// only misplace an extremum by the rounding of (x - pi/2)/2pi, k*2pi and the
// adds: <= 6e-4 for |x| <= 2048.  A peak wrongly detected yields +-1 (safe);
// a peak wrongly missed lies within 6e-4 of an endpoint, where sin is within
// (6e-4)^2/2 < 2e-7 of +-1, so the 2^-18 pad keeps the image sound.  Larger
// arguments take the FP64 path.
SPK_DEV bool sin_image_f32(float lo, float hi, float& out_lo, float& out_hi) {
  if (!(fabsf(lo) <= 2048.f && fabsf(hi) <= 2048.f)) return false;
  constexpr float kTwoPiF = 6.2831855f, kHalfPiF = 1.5707964f, pad = 3.814697265625e-06f;  // 2^-18
  const float sl = sinf(lo), sh = sinf(hi);
  float mn = __fsub_rd(fminf(sl, sh), pad), mx = __fadd_ru(fmaxf(sl, sh), pad);
  if (floorf((hi - kHalfPiF) / kTwoPiF) * kTwoPiF + kHalfPiF >= lo) mx = 1.f;
  if (floorf((hi + kHalfPiF) / kTwoPiF) * kTwoPiF - kHalfPiF >= lo) mn = -1.f;
  out_lo = fmaxf(mn, -1.f);
  out_hi = fminf(mx, 1.f);
  return true;
}

template <typename T>
SPK_DEV void interval_image(int act, T lo, T hi, T& out_lo, T& out_hi) {
  if (act == ACT_RELU || act == ACT_RELU_BROKEN) {
    out_lo = fmax(lo, T(0));
    out_hi = fmax(hi, T(0));
    return;
  }
  if constexpr (sizeof(T) == 4) {
    if (act == ACT_SIN && sin_image_f32(lo, hi, out_lo, out_hi)) return;
  }
  interval_image_slow<T>(act, lo, hi, out_lo, out_hi);
}

template <typename T>
SPK_RULE void interval_image_slow(int act, T lo, T hi, T& out_lo, T& out_hi) {
  switch (act) {
    case ACT_ELU: {
      const double a = elu64((double)lo), b = elu64((double)hi);
      out_lo = lo >= T(0) ? lo : Num<T>::from_d_rd(a - pad64(fabs(a)));
      out_hi = hi >= T(0) ? hi : Num<T>::from_d_ru(b + pad64(fabs(b)));
      return;
    }
    case ACT_SIN: {
      const double l = (double)lo, h = (double)hi;
      const double sl = sin(l), sh = sin(h);
      double mn = fmin(sl, sh) - pad64(1.0), mx = fmax(sl, sh) + pad64(1.0);
      if (floor((h - kHalfPi) / kTwoPi) * kTwoPi + kHalfPi >= l) mx = 1.0;
      if (floor((h + kHalfPi) / kTwoPi) * kTwoPi - kHalfPi >= l) mn = -1.0;
      out_lo = Num<T>::from_d_rd(fmax(mn, -1.0));
      out_hi = Num<T>::from_d_ru(fmin(mx, 1.0));
      return;
    }
    case ACT_TANH: {
      const double a = tanh((double)lo), b = tanh((double)hi);
      out_lo = Num<T>::from_d_rd(a - pad64(1.0));
      out_hi = Num<T>::from_d_ru(b + pad64(1.0));
      return;
    }
    default:
      out_lo = lo;
      out_hi = hi;
      return;
  }
}

// Pointwise value (network.py:149-160), used by point evaluation.  ReLU is
// inline; the other activations live out of line so the unrolled epilogue
// stays small (instruction-cache pressure).
// FP32 ELU value (point evaluation): expm1 on [-1, 0) as its degree-10 Taylor
// polynomial (<= 1.7e-7 relative), exp(x) - 1 below -1 (no cancellation,
// <= 2.1e-7 relative with the MUFU exponential) -- within 3 ulp like the FP32
// dot products around it, and ~3x cheaper than expm1f, which dominated the
// ELU nets' point passes (C4 corner evaluation).  Bounds never use it: the
// ELU affine and interval rules evaluate in FP64 (elu_affine, elu64).
SPK_DEV float elu_f32(float x) {
  float p = 2.7557319e-07f;        // 1/10!
  p = fmaf(p, x, 2.7557319e-06f);  // 1/9!
  p = fmaf(p, x, 2.4801587e-05f);  // 1/8!
  p = fmaf(p, x, 1.9841270e-04f);  // 1/7!
  p = fmaf(p, x, 1.3888889e-03f);  // 1/6!
  p = fmaf(p, x, 8.3333333e-03f);  // 1/5!
  p = fmaf(p, x, 4.1666667e-02f);  // 1/4!
  p = fmaf(p, x, 1.6666667e-01f);  // 1/3!
  p = fmaf(p, x, 0.5f);
  p = fmaf(p, x, 1.0f);
  p *= x;
  const float q = __expf(x) - 1.0f;
  return x >= 0.0f ? x : (x >= -1.0f ? p : q);
}

template <typename T>
SPK_DEV T elu_value(T x) {
  if constexpr (sizeof(T) == 4) {
    return elu_f32(x);
  } else {
    return x >= T(0) ? x : expm1(x);
  }
}

template <typename T>
SPK_RULE T act_value_slow(int act, T x) {  // float / double overloads of the CUDA math library
  switch (act) {
    case ACT_RELU_BROKEN: return fmax(x, T(0));
    case ACT_ELU: return elu_value<T>(x);
    case ACT_SIN: return sin(x);
    case ACT_TANH: return tanh(x);
    default: return x;
  }
}
// Inline twin of act_value_slow for rolled loops (no call, no ABI spills).
template <typename T>
SPK_DEV T act_value_inline(int act, T x) {
  switch (act) {
    case ACT_RELU_BROKEN: return fmax(x, T(0));
    case ACT_ELU: return elu_value<T>(x);
    case ACT_SIN: return sin(x);
    case ACT_TANH: return tanh(x);
    default: return x;
  }
}
template <typename T>
SPK_DEV T act_value(int act, T x) {
  if (act == ACT_RELU || act == ACT_RELU_BROKEN) return fmax(x, T(0));
  return act_value_slow<T>(act, x);
}

}  // namespace spk
