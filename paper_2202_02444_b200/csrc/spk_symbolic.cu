// Host side of the symbol-carrying policies (affine-truncate, affine-full):
#include <algorithm>
#include <string>
// capacity planning (range_core.py:530-544) and dispatch to sym_bound_kernel.
#include "spk_symbolic.cuh"
#include "spk_abi_internal.h"

namespace spk {

template <typename T>
static cudaError_t sym_any(int mmax, int kc, const NetDev<T>& nd, const BoxInput& in, const BoundOutput& out,
                           long long n, const SymParams& P, int sm, cudaStream_t st) {
  switch (mmax) {
    case 32: return dispatch_sym<T, 32>(kc, nd, in, out, n, P, sm, st);
    case 64: return dispatch_sym<T, 64>(kc, nd, in, out, n, P, sm, st);
    case 128: return dispatch_sym<T, 128>(kc, nd, in, out, n, P, sm, st);
    case 256: return dispatch_sym<T, 256>(kc, nd, in, out, n, P, sm, st);
    default: return dispatch_sym<T, 512>(kc, nd, in, out, n, P, sm, st);
  }
}

// Symbol capacity (range_core.py:530-544): truncate keeps <= n_keep (and the
// input symbols); full keeps s + every hidden activation's width.  The final
// layer's activations fold into the error channel (identical lo/hi).
static int plan_capacity(const spk_net* net, int policy, int n_keep, int s, int* kc, SymParams* P) {
  if (!net->pre_acts.empty())
    return fail(SPK_ERR_UNSUPPORTED_SHAPE, "symbolic policies: activation before the first dense layer");
  int need;
  int big = 0;  // large-capacity (K3F) symbol count if the register tile is too small
  if (policy == SPK_POLICY_AFFINE_TRUNCATE) {
    need = std::max(n_keep, s);
    // K3F capacity: max over layers of min(prev, n_keep) + m (range_core.py:530-544)
    int cur = s;
    big = s;
    for (size_t l = 0; l + 1 < net->layers.size(); ++l)
      for (int a : net->layers[l].acts)
        if (a != SPK_OP_IDENTITY) {
          cur += net->layers[l].m_out;
          big = std::max(big, cur);
          cur = std::min(cur, n_keep);
        }
  } else {
    need = s;
    for (size_t l = 0; l + 1 < net->layers.size(); ++l)
      for (int a : net->layers[l].acts)
        if (a != SPK_OP_IDENTITY) need += net->layers[l].m_out;
  }
  const int kcmax = net->mmax <= 64 ? 32 : 16;
  if (need > kcmax) {
    // beyond the register-tiled kernel: the large-capacity path (spk_full.cu)
    *kc = -(policy == SPK_POLICY_AFFINE_FULL ? need : big);
    P->n_keep = policy == SPK_POLICY_AFFINE_TRUNCATE ? n_keep : 0;
    return SPK_OK;
  }
  *kc = need <= 8 ? 8 : (need <= 16 ? 16 : 32);
  P->n_keep = policy == SPK_POLICY_AFFINE_TRUNCATE ? n_keep : *kc;
  P->full = policy == SPK_POLICY_AFFINE_FULL;
  P->s0 = s;
  return SPK_OK;
}

static int run_sym(const spk_net* cnet, int policy, int n_keep, int precision, const BoxInput& in,
                   const BoundOutput& out, long long n, int s, cudaStream_t st) {
  spk_net* net = const_cast<spk_net*>(cnet);
  if (precision == SPK_FP32_REFINE) {
    // FP32 symbolic pass, then the near-certifiable UNKNOWN boxes in FP64
    if (int rc = run_sym(cnet, policy, n_keep, SPK_FP32, in, out, n, s, st)) return rc;
    if (out.lo == nullptr || out.hi == nullptr || n <= 0) return SPK_OK;
    return refine_rebound(net, MODE_AFFINE, in, out, n, st, [&](const BoxInput& in2) {
      return run_sym(cnet, policy, n_keep, SPK_FP64, in2, out, n, s, st);
    });
  }
  int kc;
  SymParams P;
  if (int rc = plan_capacity(net, policy, n_keep, s, &kc, &P)) return rc;
  if (kc < 0) return launch_full(net, precision, in, out, n, s, -kc, P.n_keep, st);
  DeviceGuard g(net->device);
  const int sm = sm_count_for(net->device);
  if (sm <= 0) return fail(SPK_ERR_CUDA, "no CUDA device");
  cudaError_t e;
  if (precision == SPK_FP64) {
    NetDev<double> nd_copy;
    const NetDev<double>* nd = &nd_copy;
    if (int rc = get_dev<double>(net, &nd_copy)) return rc;
    e = sym_any<double>(net->mmax, kc, *nd, in, out, n, P, sm, st);
  } else {
    NetDev<float> nd_copy;
    const NetDev<float>* nd = &nd_copy;
    if (int rc = get_dev<float>(net, &nd_copy)) return rc;
    e = sym_any<float>(net->mmax, kc, *nd, in, out, n, P, sm, st);
  }
  if (e != cudaSuccess) return cuda_fail(e, "symbolic kernel launch");
  return SPK_OK;
}

int launch_symbolic(const spk_net* net, int policy, int n_keep, int precision, long long n, int s,
                    const double* centers, const double* axes, double* lo, double* hi, int8_t* cls,
                    cudaStream_t st) {
  if (s > MAX_AXES) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "more than 8 box axes");
  BoxInput in{IN_BOXES, s, centers, axes, 0, 0, 0.0, nullptr};
  BoundOutput o{lo, hi, cls};
  return run_sym(net, policy, n_keep, precision, in, o, n, s, st);
}

int launch_symbolic_in(const spk_net* net, int policy, int n_keep, int precision, const BoxInput& in,
                       const BoundOutput& o, long long n_cap, int s, cudaStream_t st) {
  return run_sym(net, policy, n_keep, precision, in, o, n_cap, s, st);
}

}  // namespace spk
