// Internal host-side types shared by the C-ABI translation units.
#pragma once
#include <cstdint>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include "spk_pass.cuh"

namespace spk {

struct HostLayer {
  int m_in = 0, m_out = 0;
  std::vector<double> W;  // m_out x m_in row-major
  std::vector<double> b;
  std::vector<int> acts;  // activations after this dense layer
};

template <typename T>
struct DevNet {
  bool ready = false;
  NetDev<T> nd;
  T* tiles = nullptr;
  T* small = nullptr;
};

struct BoxInput;
struct BoundOutput;

int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
// RayCastParams.__post_init__ (reference rays.py:56-71) for callers that bind
// the C-ABI directly: params6 = t_max, sigma0, eta_plus, eta_minus, delta,
// safety.  Written as negated comparisons so NaNs are rejected too.
inline int check_ray_params(const double* p) {
  if (!(p[0] > 0.0)) return fail(SPK_ERR_INVALID_PARAMETER, "t_max must be positive");
  if (!(p[1] > 0.0)) return fail(SPK_ERR_INVALID_PARAMETER, "sigma0 must be positive");
  if (!(p[2] > 1.0)) return fail(SPK_ERR_INVALID_PARAMETER, "eta_plus must exceed 1");
  if (!(p[3] > 0.0 && p[3] < 1.0)) return fail(SPK_ERR_INVALID_PARAMETER, "eta_minus must lie in (0, 1)");
  if (!(p[4] > 0.0)) return fail(SPK_ERR_INVALID_PARAMETER, "delta must be positive");
  if (!(p[5] > 0.0 && p[5] <= 1.0)) return fail(SPK_ERR_INVALID_PARAMETER, "safety must lie in (0, 1]");
  return SPK_OK;
}
int sm_count_for(int device);

class DeviceGuard {
 public:
  explicit DeviceGuard(int dev);
  ~DeviceGuard();
 private:
  int prev_ = 0, dev_ = 0;
};

int run_pass(const struct ::spk_net* net, int mode, int S, int precision, const BoxInput& in,
             const BoundOutput& out, long long n, cudaStream_t st);

// SPK_FP32_REFINE's FP64 half (spk_abi.cu): after an FP32 pass wrote `out`,
// re-bound the near-certifiable UNKNOWN boxes with fp64_pass(in with perm /
// n_dev set to the candidate list)
int refine_rebound(::spk_net* net, int mode, const BoxInput& in, const BoundOutput& out, long long n,
                   cudaStream_t st, const std::function<int(const BoxInput&)>& fp64_pass);

// affine-truncate / affine-full (symbol-carrying policies), spk_symbolic.cu
int launch_symbolic(const struct ::spk_net* net, int policy, int n_keep, int precision, long long n, int s,
                    const double* centers, const double* axes, double* lo, double* hi, int8_t* cls,
                    cudaStream_t st);
int launch_symbolic_in(const struct ::spk_net* net, int policy, int n_keep, int precision, const BoxInput& in,
                       const BoundOutput& o, long long n_cap, int s, cudaStream_t st);
// affine-full (n_keep = 0) or affine-truncate:n_keep beyond the register-tiled
// capacity (spk_full.cu); need = the planned symbol capacity
int launch_full(const struct ::spk_net* net, int precision, const BoxInput& in, const BoundOutput& out,
                long long n, int s0, int need, int n_keep, cudaStream_t st);
int bound_aabb_internal(const struct ::spk_net* net, int policy, int n_keep, int precision, long long n_cap,
                        const long long* n_dev, const double* box_lo, const double* box_hi, double* lo, double* hi,
                        int8_t* cls, cudaStream_t st, int pair_order = 0);
// Morton processing order of a large batch (spk_order.cu); *perm lives in
// *scratch, released by the caller with cudaFreeAsync after the kernel.
int spatial_order(const BoxInput& in, int d, long long n, int sm, cudaStream_t st, int** perm, void** scratch);
int eval_internal(const struct ::spk_net* net, int precision, long long n_cap, const long long* n_dev,
                  const double* xs, double* out, cudaStream_t st);

// host-pointer pipeline, spk_host.cu
int host_pipeline(const struct ::spk_net* net, int policy, int n_keep, int precision, long long n, int s,
                  const double* centers, const double* axes, double* lo, double* hi, int8_t* cls);

}  // namespace spk

struct spk_net {
  int input_dim = 0;
  int device = 0;
  int mmax = 0;
  int max_width = 0;
  int64_t macs = 0;
  int corrupt_relu = 0;  // test hook (spk_net_debug_corrupt_relu)
  int flags = 0;         // SPK_NET_* (spk_net_create_ex)
  std::vector<int> pre_acts;
  std::vector<spk::HostLayer> layers;
  std::mutex mu;
  // SPK_FP32_REFINE: per-mode calibrated band (interval, affine-fixed; < 0 =
  // not yet calibrated), spk_abi.cu refine_tau_for
  std::mutex calib_mu;
  double refine_tau[2] = {-1.0, -1.0};
  spk::DevNet<float> f32;
  spk::DevNet<double> f64;
  template <typename T> spk::DevNet<T>& dev();
};
template <> inline spk::DevNet<float>& spk_net::dev<float>() { return f32; }
template <> inline spk::DevNet<double>& spk_net::dev<double>() { return f64; }

namespace spk {
template <typename T>
int get_dev(::spk_net* net, NetDev<T>* out);  // copies the program under net->mu
}
