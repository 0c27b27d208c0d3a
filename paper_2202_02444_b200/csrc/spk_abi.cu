// C-ABI implementation (include/spelunk_b200.h): network upload, argument
// validation mirroring the reference's exceptions, dispatch to the fused
// kernels, and the host-pointer pipelined path.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "spk_kernels.cuh"
#include "spk_abi_internal.h"

#ifndef SPK_SMALL_TILE
#define SPK_SMALL_TILE 1  // few-hundred-box FP32 batches on width-256 nets: the SM = 1 tile
#endif
#ifndef SPK_SPREAD_SMALL
#define SPK_SPREAD_SMALL 1  // small FP32 batches on wide nets: one box group per SM sub-partition
#endif
#ifndef SPK_SPATIAL_ORDER
#define SPK_SPATIAL_ORDER 1  // Morton order for large batches (spk_order.cu)
#endif
#ifndef SPK_ORDER_MIN_MMAX
#define SPK_ORDER_MIN_MMAX 256  // narrowest net width that Morton-orders large batches
#endif

namespace spk {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(SPK_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

int sm_count_for(int device) {
  static std::mutex mu;
  static std::vector<int> cache;
  std::lock_guard<std::mutex> lk(mu);
  if ((int)cache.size() <= device) cache.resize(device + 1, 0);
  if (cache[device] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
    cache[device] = v;
  }
  return cache[device];
}

DeviceGuard::DeviceGuard(int dev) {
  cudaGetDevice(&prev_);
  if (prev_ != dev) cudaSetDevice(dev);
  dev_ = dev;
}
DeviceGuard::~DeviceGuard() {
  if (prev_ != dev_) cudaSetDevice(prev_);
}

static const int kMmaxChoices[] = {32, 64, 128, 256, 512};

template <typename T>
static int kt_for(int mmax) {
  switch (mmax) {
    case 32: return KTOf<T, 32>::KT;
    case 64: return KTOf<T, 64>::KT;
    case 128: return KTOf<T, 128>::KT;
    case 256: return KTOf<T, 256>::KT;
    default: return KTOf<T, 512>::KT;
  }
}

template <typename T>
static int pad_for(int mmax) {
  switch (mmax) {
    case 32: return KTOf<T, 32>::PAD;
    case 64: return KTOf<T, 64>::PAD;
    case 128: return KTOf<T, 128>::PAD;
    case 256: return KTOf<T, 256>::PAD;
    default: return KTOf<T, 512>::PAD;
  }
}

// W tiles of a dense layer in host (KT-row) units: the layer's rows padded to
// a multiple of PAD, the largest tile any kernel of this width reads
// (Cfg::KT_PAD), so kernels with PAD-row tiles see whole pairs of host tiles.
static int layer_tiles(int m_in, int kt, int pad) { return ((m_in + pad - 1) / pad) * (pad / kt); }

template <typename T>
static int sub_for(int mmax) {
  switch (mmax) {
    case 32: return KTOf<T, 32>::SUB;
    case 64: return KTOf<T, 64>::SUB;
    case 128: return KTOf<T, 128>::SUB;
    case 256: return KTOf<T, 256>::SUB;
    default: return KTOf<T, 512>::SUB;
  }
}

template <typename T>
static T round_up_to(double x) {
  T t = (T)x;
  if ((double)t < x) t = std::nextafter(t, (T)INFINITY);
  return t;
}

// Activation code as the kernels see it (the test hook swaps ReLU for the
// rule with a negated remainder).
static int act_code(const spk_net* net, int act) {
  return (net->corrupt_relu && act == ACT_RELU) ? (int)ACT_RELU_BROKEN : act;
}

// ReLU-specialised kernels apply (every dense layer's activations are exactly
// [] or [ReLU], none before the first layer, the test hook off)
// (2: the same with ELU, for the ELU-specialised FP32 point passes)
static int relu_net_of(const spk_net* net) {
  if (net->corrupt_relu || !net->pre_acts.empty()) return 0;
  for (int kind : {SPK_OP_RELU, SPK_OP_ELU}) {
    bool all = true;
    for (const auto& L : net->layers) {
      if (L.acts.size() > 1 || (L.acts.size() == 1 && L.acts[0] != kind)) all = false;
    }
    if (all) return kind == SPK_OP_RELU ? 1 : 2;
  }
  return 0;
}

template <typename T>
static void recode_acts(spk_net* net, DevNet<T>& dn) {
  if (!dn.ready) return;
  dn.nd.relu_net = relu_net_of(net);
  for (int i = 0; i < dn.nd.n_pre; ++i) dn.nd.pre_act[i] = act_code(net, net->pre_acts[i]);
  for (size_t l = 0; l < net->layers.size(); ++l)
    for (int a = 0; a < dn.nd.L[l].n_act; ++a) dn.nd.L[l].act[a] = act_code(net, net->layers[l].acts[a]);
}

#ifndef SPK_RUNERR_LAYERS
#define SPK_RUNERR_LAYERS 1  // leading wide layers on the running-error K loop (FP32)
#endif

// Build the device program for one precision (lazily, once per net).
template <typename T>
int build_device_net(spk_net* net, DevNet<T>& dn) {
  const bool fp32 = sizeof(T) == 4;
  const int mmax = net->mmax;
  const int KT = kt_for<T>(mmax);
  const int PADR = pad_for<T>(mmax);
  const int tile = KT * mmax;
  NetDev<T> nd;
  std::memset(&nd, 0, sizeof(nd));
  nd.d = net->input_dim;
  nd.n_pre = (int)net->pre_acts.size();
  for (int i = 0; i < nd.n_pre; ++i) nd.pre_act[i] = act_code(net, net->pre_acts[i]);
  nd.n_layers = (int)net->layers.size();

  std::vector<T> tiles;
  std::vector<T> small;   // narrow W, biases, bias errors (offsets patched later)
  struct Offs { size_t w = 0, b = 0, be = 0; };
  std::vector<Offs> offs(net->layers.size());
  std::vector<double> gam(net->layers.size());
  // weight rounding budget u_w per layer: 0 when every weight and bias of the
  // layer is exactly representable in T (e.g. nets trained in FP32 and
  // exported): the device then holds the reference's FP64 network exactly
  std::vector<double> uw(net->layers.size(), 0.0);
  for (size_t l = 0; l < net->layers.size() && fp32; ++l) {
    const HostLayer& L = net->layers[l];
    bool exact = true;
    for (double w : L.W) exact = exact && ((double)(float)w == w);
    for (double b : L.b) exact = exact && ((double)(float)b == b);
    uw[l] = exact ? 0.0 : 5.9604644775390625e-8 * (1.0 + 1e-6);
  }
  for (size_t l = 0; l < net->layers.size(); ++l) {
    const HostLayer& L = net->layers[l];
    // only the final (width-1) layer takes the warp-reduction path; every
    // hidden layer streams through the W tile ring
    const bool narrow = (l + 1 == net->layers.size()) && L.m_out <= NARROW_MAX;
    int n_eff;
    if (narrow) {
      // warp butterfly (32 lanes; K3F) or 4-lane groups (nets of width <= 64)
      const int lp = mmax <= 64 ? 4 : 32;
      n_eff = std::max((L.m_in + 31) / 32 + 6, (L.m_in + lp - 1) / lp + 3);
      // the fused output layer of the ReLU-specialised passes (spk_pass.cuh
      // generic_layer FF, nets of width <= 64): a TI-term chain per thread,
      // log2(NG) butterfly levels, the bias -- TI = 8 neurons per thread,
      // NG = mmax / 8
      if (mmax <= 64) {
        int lg = 0;
        while ((8 << lg) < mmax) ++lg;
        n_eff = std::max(n_eff, 8 + lg + 1);
      }
    } else {
      const int nt = layer_tiles(L.m_in, KT, PADR);
      const int sub = sub_for<T>(mmax);
      n_eff = std::min(sub, L.m_in) + (L.m_in + sub - 1) / sub + 1;
      for (int t = 0; t < nt; ++t) {
        for (int kk = 0; kk < KT; ++kk) {
          const int k = t * KT + kk;
          for (int i = 0; i < mmax; ++i) {
            T v = T(0);
            if (k < L.m_in && i < L.m_out) v = (T)L.W[(size_t)i * L.m_in + k];
            tiles.push_back(v);
          }
        }
      }
    }
    // + u for FP32: W and b are rounded from FP64 to T, |dW| <= u|W|, so the
    // certified function is the reference's FP64 network (0 for FP32-exact layers)
    gam[l] = gamma_n_host(n_eff, fp32) + uw[l];
    // SPK_NET_FP64_UNPADDED: the reference's own FP64 arithmetic (no a-priori
    // dot-product budget), for callers that compare at 1e-15 (integration shim)
    if (!fp32 && (net->flags & SPK_NET_FP64_UNPADDED)) gam[l] = 0.0;
#ifdef SPK_DEBUG_GAMMA_KEEP_MASK
    // measurement-only builds (tools/build_variant.py): UNSOUND, attributes the
    // FP32 enclosure excess to the rounding budgets of individual layers
    if (fp32 && !((SPK_DEBUG_GAMMA_KEEP_MASK >> l) & 1)) gam[l] = 0.0;
#endif
    if (narrow) {
      offs[l].w = small.size();
      for (size_t q = 0; q < L.W.size(); ++q) small.push_back((T)L.W[q]);
    }
    // bias and bias-budget arrays start 16-byte aligned and are zero-padded to
    // a multiple of 4 entries: the K loops read them as one vector per group
    // of G consecutive neurons (spk_pass.cuh load_group)
    while (small.size() % 4) small.push_back(T(0));
    offs[l].b = small.size();
    for (int i = 0; i < L.m_out; ++i) small.push_back((T)L.b[i]);
    while (small.size() % 4) small.push_back(T(0));
    offs[l].be = small.size();
    for (int i = 0; i < L.m_out; ++i) {
      // |b_i| enters the FMA chain exactly once; its share of the rounding
      // budget plus an underflow guard, rounded up.
      const double be = (!fp32 && (net->flags & SPK_NET_FP64_UNPADDED))
                            ? 0.0
                            : gam[l] * std::fabs((double)(T)L.b[i]) * (1.0 + 1e-6) +
                                  (fp32 ? 1e-37 : 1e-300) * (L.m_in + 2);
      small.push_back(round_up_to<T>(be));
    }
    while (small.size() % 4) small.push_back(T(0));
  }
  T* d_tiles = nullptr;
  T* d_small = nullptr;
  cudaError_t e;
  if (!tiles.empty()) {
    e = cudaMalloc(&d_tiles, tiles.size() * sizeof(T));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(tiles)");
    e = cudaMemcpy(d_tiles, tiles.data(), tiles.size() * sizeof(T), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(tiles)");
  }
  e = cudaMalloc(&d_small, std::max<size_t>(small.size(), 4) * sizeof(T));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(small)");
  e = cudaMemcpy(d_small, small.data(), small.size() * sizeof(T), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(small)");

  nd.wtiles = d_tiles;
  nd.tiles_per_pass = (int)(tiles.size() / (size_t)tile);
  nd.gamma_first = round_up_to<T>(gam.empty() ? 0.0 : gam[0]);
  nd.relu_net = relu_net_of(net);
  // which generic layers run the running-error K loop (FP32 affine passes)
  std::vector<int> runerr(net->layers.size(), 0);
  for (size_t l = 0, k = 0; l < net->layers.size() && (int)k < SPK_RUNERR_LAYERS; ++l) {
    const bool narrow = (l + 1 == net->layers.size()) && net->layers[l].m_out <= NARROW_MAX;
    if (!narrow && net->layers[l].m_in >= 64) {
      runerr[l] = 1;
      ++k;
    }
  }
  auto run_layer = [&](size_t l) { return SPK_RUNERR && runerr[l] != 0; };
  for (size_t l = 0; l < net->layers.size(); ++l) {
    const HostLayer& L = net->layers[l];
    LayerDev<T>& D = nd.L[l];
    D.m_in = L.m_in;
    D.m_out = L.m_out;
    D.narrow = (l + 1 == net->layers.size()) && L.m_out <= NARROW_MAX;
    D.ntiles = D.narrow ? 0 : layer_tiles(L.m_in, KT, PADR);
    D.n_act = (int)L.acts.size();
    for (int a = 0; a < D.n_act; ++a) D.act[a] = act_code(net, L.acts[a]);
    D.w = D.narrow ? d_small + offs[l].w : nullptr;
    D.bias = d_small + offs[l].b;
    D.berr = d_small + offs[l].be;
    D.gamma_next = (l + 1 < net->layers.size()) ? round_up_to<T>(gam[l + 1]) : T(0);
    // running-error K loops (FP32, spk_pass.cuh dense_kloop_f32): the first
    // SPK_RUNERR_LAYERS generic layers with >= 64 inputs bound their base
    // column's FMA rounding a posteriori, so the pack feeding them charges only
    // the weights' FP64 -> T rounding (u |W| |base|) a priori
    D.runerr = fp32 && run_layer(l) ? 1 : 0;
    D.gamma_base_next = (fp32 && l + 1 < net->layers.size() && run_layer(l + 1))
                            ? round_up_to<T>(uw[l + 1] + (SPK_F64_BASE ? 1e-13 : 0.0))  // + gamma_n of FP64 (n <= 513)
                            : D.gamma_next;
  }
  dn.nd = nd;
  dn.tiles = d_tiles;
  dn.small = d_small;
  dn.ready = true;
  return SPK_OK;
}

template <typename T>
int get_dev(spk_net* net, NetDev<T>* out) {
  // the kernel-parameter copy is taken under the net's lock, so a concurrent
  // spk_net_debug_corrupt_relu (which recodes the cached program) never
  // tears a launch's activation list
  DevNet<T>& dn = net->dev<T>();
  std::lock_guard<std::mutex> lk(net->mu);
  if (!dn.ready) {
    DeviceGuard g(net->device);
    int rc = build_device_net<T>(net, dn);
    if (rc != SPK_OK) return rc;
  }
  *out = dn.nd;
  return SPK_OK;
}
template int get_dev<float>(spk_net*, NetDev<float>*);
template int get_dev<double>(spk_net*, NetDev<double>*);

template <typename T>
cudaError_t dispatch_any(int mmax, int mode, int S, const NetDev<T>& nd, const BoxInput& in,
                         const BoundOutput& out, long long n, int sm, cudaStream_t st) {
  switch (mmax) {
    case 32: return dispatch_bound<T, 32>(mode, S, nd, in, out, n, sm, st);
    case 64: return dispatch_bound<T, 64>(mode, S, nd, in, out, n, sm, st);
    case 128: return dispatch_bound<T, 128>(mode, S, nd, in, out, n, sm, st);
    case 256: return dispatch_bound<T, 256>(mode, S, nd, in, out, n, sm, st);
    default: return dispatch_bound<T, 512>(mode, S, nd, in, out, n, sm, st);
  }
}

// ------------------------------------------------- FP64 certification refinement
// SPK_FP32_REFINE: the FP32 pass bounds every box; boxes it leaves UNKNOWN but
// whose enclosure reaches within tau * (S + w) of certification (-lo or hi <=
// tau (S + w), S = max(1, |lo|, |hi|), w = hi - lo) are re-bounded by the FP64
// pass, which reads them through a processing order (BoxInput::perm) and a
// device-side count, and overwrites their lo / hi / class in place.  FP32 and
// FP64 bounds are both sound, so every box's result stays sound; the FP64
// pass (the reference's precision) decides the boxes where the FP32 rounding
// budget could have cost a certification.  Per-box results do not depend on
// which other boxes are refined or in which order (each box's bound is
// independent of its batch).
// process-wide override of the per-net band (< 0: calibrate per net)
static std::atomic<double> g_refine_tau{-1.0};

__global__ void refine_select_kernel(const double* __restrict__ lo, const double* __restrict__ hi,
                                     long long n_cap, const long long* __restrict__ n_dev, double tau,
                                     int* __restrict__ idx, long long* __restrict__ cnt) {
  const long long n = n_dev ? *n_dev : n_cap;
  const int lane = threadIdx.x & 31;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < n; base += (long long)gridDim.x * blockDim.x) {
    const long long i = base + threadIdx.x;
    bool c = false;
    if (i < n) {
      const double l = lo[i], h = hi[i];
      if (!(l > 0.0) && !(h < 0.0)) {  // UNKNOWN (NaN bounds never qualify below)
        const double s = fmax(1.0, fmax(fabs(l), fabs(h)));
        const double band = tau * (s + (h - l));
        c = (-l <= band) || (h <= band);
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, c);
    if (m == 0u) continue;
    long long b0 = 0;
    if (lane == 0) b0 = (long long)atomicAdd(reinterpret_cast<unsigned long long*>(cnt), (unsigned long long)__popc(m));
    b0 = __shfl_sync(0xffffffffu, b0, 0);
    if (c) idx[b0 + __popc(m & ((1u << lane) - 1u))] = (int)i;
  }
}

static int run_pass_once(const spk_net* cnet, int mode, int S, int precision, const BoxInput& in,
                         const BoundOutput& out, long long n, cudaStream_t st);

// max over boxes of the FP32 excess over the FP64 enclosure in units of
// S + w (finite bounds only); non-negative doubles order like their bits
__global__ void refine_excess_kernel(const double* __restrict__ b32, const double* __restrict__ b64, int n,
                                     unsigned long long* __restrict__ out) {
  double m = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double l3 = b32[i], h3 = b32[n + i], l6 = b64[i], h6 = b64[n + i];
    const double s = fmax(1.0, fmax(fabs(l6), fabs(h6)));
    const double r = fmax(l6 - l3, h3 - h6) / (s + (h6 - l6));
    if (isfinite(r) && r > m) m = r;
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// The refine band of a net and mode: the FP32 excess over FP64 depends on the
// network (measured max / (S + w): 1e-5 on the 7x32 golden nets, 1.1e-3 on
// C5_64, 5.4e-2 on the 8x256 / 8x512 configs; tools/excess_dist.py), so a
// fixed band either misses certifications (wide deep nets) or re-bounds most
// boxes (narrow nets).  Calibrated once per (net, mode), on first use: 4096
// random cubes over [-1, 1]^d at each of two half-extents (2^-6 and 2^-14:
// the ratio grows as boxes shrink, towards the point budget), bounded in
// both precisions; band = 3 x the largest ratio seen.  One host sync per net
// and mode.  The band only selects which boxes the FP64 pass re-bounds:
// every result stays sound whatever it is.
static int refine_tau_for(spk_net* net, int mode, cudaStream_t st, double* tau) {
  const double forced = g_refine_tau.load();
  if (forced >= 0.0) {
    *tau = forced;
    return SPK_OK;
  }
  const int slot = mode == MODE_INTERVAL ? 0 : 1;
  std::lock_guard<std::mutex> lk(net->calib_mu);
  if (net->refine_tau[slot] >= 0.0) {
    *tau = net->refine_tau[slot];
    return SPK_OK;
  }
  constexpr int NC = 4096;
  const double halves[2] = {0.015625, 6.103515625e-05};
  void* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, 8 * NC * sizeof(double) + 16, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(refine calibration)");
  double* b32 = static_cast<double*>(scratch);   // [lo(2NC), hi(2NC)]
  double* b64 = b32 + 4 * NC;
  unsigned long long* mx = reinterpret_cast<unsigned long long*>(b64 + 4 * NC);
  int rc = SPK_OK;
  for (int h = 0; h < 2 && rc == SPK_OK; ++h) {
    BoxInput in{IN_RANDOM, net->input_dim, nullptr, nullptr, (long long)h * NC, 0x5EEDull, halves[h], nullptr};
    BoundOutput o32{b32 + h * NC, b32 + 2 * NC + h * NC, nullptr};
    BoundOutput o64{b64 + h * NC, b64 + 2 * NC + h * NC, nullptr};
    rc = run_pass_once(net, mode, net->input_dim, SPK_FP32, in, o32, NC, st);
    if (rc == SPK_OK) rc = run_pass_once(net, mode, net->input_dim, SPK_FP64, in, o64, NC, st);
  }
  unsigned long long bits = 0;
  if (rc == SPK_OK) {
    e = cudaMemsetAsync(mx, 0, sizeof(unsigned long long), st);
    if (e == cudaSuccess) {
      refine_excess_kernel<<<16, 256, 0, st>>>(b32, b64, 2 * NC, mx);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(&bits, mx, sizeof(bits), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_fail(e, "refine calibration");
  }
  const cudaError_t ef = cudaFreeAsync(scratch, st);
  if (rc == SPK_OK && ef != cudaSuccess) rc = cuda_fail(ef, "cudaFreeAsync(refine calibration)");
  if (rc != SPK_OK) return rc;
  double ratio;
  std::memcpy(&ratio, &bits, sizeof(ratio));
  net->refine_tau[slot] = std::min(0.25, 3.0 * ratio);
  *tau = net->refine_tau[slot];
  return SPK_OK;
}

int run_pass(const spk_net* cnet, int mode, int S, int precision, const BoxInput& in,
             const BoundOutput& out, long long n, cudaStream_t st) {
  if (precision != SPK_FP32_REFINE) return run_pass_once(cnet, mode, S, precision, in, out, n, st);
  // point values and missing outputs: plain FP32
  if (mode == MODE_POINT || out.lo == nullptr || out.hi == nullptr || n <= 0)
    return run_pass_once(cnet, mode, S, SPK_FP32, in, out, n, st);
  if (int rc = run_pass_once(cnet, mode, S, SPK_FP32, in, out, n, st)) return rc;
  return refine_rebound(const_cast<spk_net*>(cnet), mode, in, out, n, st,
                        [&](const BoxInput& in2) { return run_pass_once(cnet, mode, S, SPK_FP64, in2, out, n, st); });
}

// The FP64 half of SPK_FP32_REFINE, after an FP32 pass wrote out: list the
// near-certifiable UNKNOWN boxes (band of the net's `mode`; the symbol-carrying
// policies use the affine-fixed band) and let `fp64_pass` re-bound them in
// place through a processing order and a device-side count.
int refine_rebound(spk_net* net, int mode, const BoxInput& in, const BoundOutput& out, long long n,
                   cudaStream_t st, const std::function<int(const BoxInput&)>& fp64_pass) {
  DeviceGuard g(net->device);
  const int sm = sm_count_for(net->device);
  double tau = 0.0;
  if (int rc = refine_tau_for(net, mode == MODE_INTERVAL ? MODE_INTERVAL : MODE_AFFINE, st, &tau)) return rc;
  // candidates: n_cap indices + the device count (16-byte aligned)
  void* scratch = nullptr;
  const size_t idx_bytes = (((size_t)n * sizeof(int)) + 15) & ~(size_t)15;
  cudaError_t e = cudaMallocAsync(&scratch, idx_bytes + 16, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(refine)");
  int* idx = static_cast<int*>(scratch);
  long long* cnt = reinterpret_cast<long long*>(static_cast<char*>(scratch) + idx_bytes);
  e = cudaMemsetAsync(cnt, 0, sizeof(long long), st);
  if (e == cudaSuccess) {
    const long long blocks = std::min<long long>((n + 255) / 256, (long long)sm * 8);
    refine_select_kernel<<<(int)blocks, 256, 0, st>>>(out.lo, out.hi, n, in.n_dev, tau, idx, cnt);
    e = cudaGetLastError();
  }
  int rc = SPK_OK;
  if (e != cudaSuccess) {
    rc = cuda_fail(e, "refine select");
  } else {
    BoxInput in2 = in;
    in2.perm = idx;
    in2.n_dev = cnt;
    in2.pair_order = 0;
    in2.spread = 0;
    in2.small = 0;
    rc = fp64_pass(in2);
  }
  const cudaError_t ef = cudaFreeAsync(scratch, st);
  if (rc == SPK_OK && ef != cudaSuccess) rc = cuda_fail(ef, "cudaFreeAsync(refine)");
  return rc;
}

static int run_pass_once(const spk_net* cnet, int mode, int S, int precision, const BoxInput& in,
                         const BoundOutput& out, long long n, cudaStream_t st) {
  spk_net* net = const_cast<spk_net*>(cnet);
  DeviceGuard g(net->device);
  const int sm = sm_count_for(net->device);
  if (sm <= 0) return fail(SPK_ERR_CUDA, "no CUDA device");
  cudaError_t e;
  if (precision == SPK_FP64) {
    NetDev<double> nd_copy;
    const NetDev<double>* nd = &nd_copy;
    int rc = get_dev<double>(net, &nd_copy);
    if (rc) return rc;
    e = dispatch_any<double>(net->mmax, mode, S, *nd, in, out, n, sm, st);
  } else {
    NetDev<float> nd_copy;
    const NetDev<float>* nd = &nd_copy;
    int rc = get_dev<float>(net, &nd_copy);
    if (rc) return rc;
    // large batches of independent boxes on wide nets: Morton processing
    // order, so box groups hold neighbouring boxes and the live-row masks
    // skip more ReLU-inactive rows (identical results; spk_order.cu)
    // (tree levels keep their sibling-pair order: Morton-sorting them as well
    // measured 0.6% slower -- the sort costs more than the extra coherence)
    const bool order = SPK_SPATIAL_ORDER && (mode == MODE_AFFINE || mode == MODE_INTERVAL) &&
                       net->mmax >= SPK_ORDER_MIN_MMAX && n >= (1ll << 16) && in.n_dev == nullptr && !in.pair_order && in.perm == nullptr &&
                       (in.kind == IN_RANDOM || in.kind == IN_BOXES || in.kind == IN_AABB);
    // small batches (fewer boxes than 8 per SM, e.g. the top tree levels) are
    // spread over every SM, one box group per SM sub-partition first
    // (spread_node); empty groups skip their K loops through the live-row masks
    const bool spread = SPK_SPREAD_SMALL && (mode == MODE_AFFINE || mode == MODE_INTERVAL) && net->mmax >= 256 &&
                        n <= (long long)sm * 8 && in.perm == nullptr;
    // a few hundred boxes on a width-256 net (the top tree levels): the
    // small tile, one neuron per thread, a box pair per CTA, 2 CTAs per SM
    const bool small = SPK_SMALL_TILE && (mode == MODE_INTERVAL || (mode == MODE_AFFINE && S == 3)) &&
                       net->mmax == 256 && n <= (long long)sm * 4 && in.perm == nullptr && !in.spread;
    if (small) {
      BoxInput in2 = in;
      in2.small = 1;
      e = dispatch_any<float>(net->mmax, mode, S, *nd, in2, out, n, sm, st);
    } else if (spread) {
      BoxInput in2 = in;
      in2.spread = 1;
      in2.spread_n = n;
      e = dispatch_any<float>(net->mmax, mode, S, *nd, in2, out, n, sm, st);
    } else if (order) {
      int* perm = nullptr;
      void* scratch = nullptr;
      rc = spatial_order(in, net->input_dim, n, sm, st, &perm, &scratch);
      if (rc) return rc;
      BoxInput in2 = in;
      in2.perm = perm;
      in2.pair_order = 0;
      e = dispatch_any<float>(net->mmax, mode, S, *nd, in2, out, n, sm, st);
      if (scratch) {
        const cudaError_t ef = cudaFreeAsync(scratch, st);
        if (e == cudaSuccess) e = ef;
      }
    } else {
      e = dispatch_any<float>(net->mmax, mode, S, *nd, in, out, n, sm, st);
    }
  }
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return SPK_OK;
}

static int check_policy(int policy, int n_keep, int* mode);

// Internal entry points with an optional device-side count: n_cap sizes the
// launch, *n_dev (when given) is the live count the kernels read.
int bound_aabb_internal(const spk_net* net, int policy, int n_keep, int precision, long long n_cap,
                        const long long* n_dev, const double* box_lo, const double* box_hi, double* lo, double* hi,
                        int8_t* cls, cudaStream_t st, int pair_order) {
  int mode;
  if (int rc = check_policy(policy, n_keep, &mode)) return rc;
  if (net->input_dim > MAX_AXES) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "AABB path supports d <= 8");
  if (n_cap <= 0) return n_cap < 0 ? fail(SPK_ERR_DIMENSION, "negative batch") : SPK_OK;
  BoxInput in{IN_AABB, net->input_dim, box_lo, box_hi, 0, 0, 0.0, n_dev};
  // sibling-pair processing order: fused pass only (K3F reads its own inputs)
  in.pair_order = (pair_order && mode >= 0) ? 1 : 0;
  BoundOutput o{lo, hi, cls};
  if (mode < 0) return launch_symbolic_in(net, -mode, n_keep, precision, in, o, n_cap, net->input_dim, st);
  return run_pass(net, mode, net->input_dim, precision, in, o, n_cap, st);
}

int eval_internal(const spk_net* net, int precision, long long n_cap, const long long* n_dev, const double* xs,
                  double* out, cudaStream_t st) {
  if (n_cap <= 0) return n_cap < 0 ? fail(SPK_ERR_DIMENSION, "negative batch") : SPK_OK;
  BoxInput in{IN_POINTS, 0, xs, nullptr, 0, 0, 0.0, n_dev};
  BoundOutput o{out, nullptr, nullptr};
  return run_pass(net, MODE_POINT, 0, precision, in, o, n_cap, st);
}

static int check_policy(int policy, int n_keep, int* mode) {
  switch (policy) {
    case SPK_POLICY_INTERVAL: *mode = MODE_INTERVAL; return SPK_OK;
    case SPK_POLICY_AFFINE_FIXED: *mode = MODE_AFFINE; return SPK_OK;
    case SPK_POLICY_AFFINE_TRUNCATE:
      if (n_keep < 1) return fail(SPK_ERR_INVALID_PARAMETER, "affine-truncate requires n_keep >= 1");
      *mode = -SPK_POLICY_AFFINE_TRUNCATE;
      return SPK_OK;
    case SPK_POLICY_AFFINE_FULL: *mode = -SPK_POLICY_AFFINE_FULL; return SPK_OK;
    default: return fail(SPK_ERR_INVALID_PARAMETER, "unknown policy");
  }
}

}  // namespace spk

using namespace spk;

extern "C" {

const char* spk_last_error(void) { return g_last_error.c_str(); }
int spk_version(void) { return 100; }

int spk_net_refine_band(const spk_net* net, int policy, void* stream, double* tau) {
  if (!net || !tau) return fail(SPK_ERR_INVALID_PARAMETER, "null argument");
  int mode;
  if (int rc = check_policy(policy, 1, &mode)) return rc;
  if (mode < 0) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "refinement covers interval / affine-fixed");
  if (net->input_dim > MAX_AXES) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "refinement supports d <= 8");
  spk_net* n = const_cast<spk_net*>(net);
  DeviceGuard g(n->device);
  return refine_tau_for(n, mode, (cudaStream_t)stream, tau);
}

int spk_refine_band(double tau, double* previous) {
  if (std::isnan(tau) || std::isinf(tau)) return fail(SPK_ERR_INVALID_PARAMETER, "refine band must be finite");
  // tau >= 0: fixed band; -1: query only; -2: back to per-net calibration
  const double old = tau == -2.0 ? g_refine_tau.exchange(-1.0) : (tau < 0.0 ? g_refine_tau.load() : g_refine_tau.exchange(tau));
  if (previous) *previous = old;
  return SPK_OK;
}

int spk_device_sm_count(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  return sm_count_for(dev);
}

int spk_net_create(int input_dim, int n_ops, const int* op_kind, const int* op_out_dim,
                   const double* params, int64_t n_params, int device, spk_net** out) {
  return spk_net_create_ex(input_dim, n_ops, op_kind, op_out_dim, params, n_params, device, 0, out);
}

int spk_net_create_ex(int input_dim, int n_ops, const int* op_kind, const int* op_out_dim,
                      const double* params, int64_t n_params, int device, int flags, spk_net** out) {
  if (!out) return fail(SPK_ERR_INVALID_PARAMETER, "null output handle");
  *out = nullptr;
  if (input_dim < 1) return fail(SPK_ERR_DIMENSION, "input_dim must be >= 1");
  if (flags & ~SPK_NET_FP64_UNPADDED) return fail(SPK_ERR_INVALID_PARAMETER, "unknown net flags");
  auto net = std::make_unique<spk_net>();
  net->input_dim = input_dim;
  net->device = device;
  net->flags = flags;
  int dim = input_dim;
  int64_t off = 0;
  int max_w = input_dim;
  for (int i = 0; i < n_ops; ++i) {
    const int k = op_kind[i];
    if (k == SPK_OP_DENSE) {
      HostLayer L;
      L.m_in = dim;
      L.m_out = op_out_dim[i];
      if (L.m_out < 1) return fail(SPK_ERR_DIMENSION, "dense layer needs >= 1 output");
      const int64_t nw = (int64_t)L.m_in * L.m_out;
      if (off + nw + L.m_out > n_params) return fail(SPK_ERR_DIMENSION, "params shorter than layer shapes");
      L.W.assign(params + off, params + off + nw);
      off += nw;
      L.b.assign(params + off, params + off + L.m_out);
      off += L.m_out;
      for (double v : L.W) if (!std::isfinite(v)) return fail(SPK_ERR_INVALID_PARAMETER, "non-finite weight");
      for (double v : L.b) if (!std::isfinite(v)) return fail(SPK_ERR_INVALID_PARAMETER, "non-finite bias");
      dim = L.m_out;
      max_w = std::max(max_w, std::max(L.m_in, L.m_out));
      net->layers.push_back(std::move(L));
    } else if (k >= SPK_OP_RELU && k <= SPK_OP_IDENTITY) {
      auto& acts = net->layers.empty() ? net->pre_acts : net->layers.back().acts;
      if ((int)acts.size() >= MAX_ACTS) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "too many consecutive activations");
      acts.push_back(k);
    } else {
      return fail(SPK_ERR_UNSUPPORTED_ACT, "unknown op kind");
    }
  }
  if (net->layers.empty()) return fail(SPK_ERR_DIMENSION, "network has no dense layers");
  if (dim != 1) return fail(SPK_ERR_DIMENSION, "final layer must output 1 value");
  if ((int)net->layers.size() > MAX_LAYERS) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "too many dense layers");
  if (off != n_params) return fail(SPK_ERR_DIMENSION, "params longer than layer shapes");
  net->mmax = 0;
  for (int m : kMmaxChoices) {
    if (m >= max_w) { net->mmax = m; break; }
  }
  if (net->mmax == 0) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "layer width above 512");
  net->max_width = max_w;
  for (auto& L : net->layers) net->macs += (int64_t)L.m_in * L.m_out;
  *out = net.release();
  return SPK_OK;
}

int spk_net_destroy(spk_net* net) {
  if (!net) return SPK_OK;
  {
    DeviceGuard g(net->device);
    if (net->f32.ready) { cudaFree(net->f32.tiles); cudaFree(net->f32.small); }
    if (net->f64.ready) { cudaFree(net->f64.tiles); cudaFree(net->f64.small); }
  }
  delete net;
  return SPK_OK;
}

int spk_net_debug_corrupt_relu(spk_net* net, int on) {
  if (!net) return fail(SPK_ERR_INVALID_PARAMETER, "null net");
  std::lock_guard<std::mutex> lk(net->mu);
  net->corrupt_relu = on ? 1 : 0;
  recode_acts<float>(net, net->f32);
  recode_acts<double>(net, net->f64);
  return SPK_OK;
}

int spk_net_info(const spk_net* net, int* max_width, int* n_dense, int64_t* macs) {
  if (!net) return fail(SPK_ERR_INVALID_PARAMETER, "null net");
  if (max_width) *max_width = net->max_width;
  if (n_dense) *n_dense = (int)net->layers.size();
  if (macs) *macs = net->macs;
  return SPK_OK;
}

int spk_bound_batch(const spk_net* net, int policy, int n_keep, int precision, int64_t n, int s,
                    const double* centers, const double* axes, double* lo, double* hi, int8_t* cls,
                    void* stream) {
  if (!net) return fail(SPK_ERR_INVALID_PARAMETER, "null net");
  int mode;
  if (int rc = check_policy(policy, n_keep, &mode)) return rc;
  if (s < 0) return fail(SPK_ERR_DIMENSION, "axes must be (n, s, d)");
  if (n < 0) return fail(SPK_ERR_DIMENSION, "negative batch");
  if (n == 0) return SPK_OK;
  if (mode < 0) return launch_symbolic(net, -mode, n_keep, precision, n, s, centers, axes, lo, hi, cls,
                                       (cudaStream_t)stream);
  if (s > MAX_AXES) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "more than 8 box axes");
  BoxInput in{IN_BOXES, s, centers, axes, 0, 0, 0.0, nullptr};
  BoundOutput o{lo, hi, cls};
  if (mode == MODE_INTERVAL) {
    // interval only needs the hull: pass all s axes through the radius sum
    in.s = s;
  }
  return run_pass(net, mode, s, precision, in, o, n, (cudaStream_t)stream);
}

int spk_bound_aabb(const spk_net* net, int policy, int n_keep, int precision, int64_t n,
                   const double* box_lo, const double* box_hi, double* lo, double* hi, int8_t* cls,
                   void* stream) {
  if (!net) return fail(SPK_ERR_INVALID_PARAMETER, "null net");
  int mode;
  if (int rc = check_policy(policy, n_keep, &mode)) return rc;
  if (net->input_dim > MAX_AXES) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "AABB path supports d <= 8");
  if (n <= 0) return n < 0 ? fail(SPK_ERR_DIMENSION, "negative batch") : SPK_OK;
  return bound_aabb_internal(net, policy, n_keep, precision, n, nullptr, box_lo, box_hi, lo, hi, cls,
                             (cudaStream_t)stream);
}

int spk_bound_random_cubes(const spk_net* net, int policy, int n_keep, int precision, int64_t n,
                           int64_t first_index, uint64_t seed, double half, double* lo, double* hi,
                           int8_t* cls, void* stream) {
  if (!net) return fail(SPK_ERR_INVALID_PARAMETER, "null net");
  int mode;
  if (int rc = check_policy(policy, n_keep, &mode)) return rc;
  if (mode < 0) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "random cubes: interval / affine-fixed only");
  if (net->input_dim > MAX_AXES) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "random cubes support d <= 8");
  if (!(half >= 0.0)) return fail(SPK_ERR_INVALID_PARAMETER, "half-extent must be >= 0");
  if (n <= 0) return SPK_OK;
  BoxInput in{IN_RANDOM, net->input_dim, nullptr, nullptr, (long long)first_index, seed, half, nullptr};
  BoundOutput o{lo, hi, cls};
  return run_pass(net, mode, net->input_dim, precision, in, o, n, (cudaStream_t)stream);
}

int spk_eval_batch(const spk_net* net, int precision, int64_t n, const double* xs, double* out,
                   void* stream) {
  if (!net) return fail(SPK_ERR_INVALID_PARAMETER, "null net");
  if (n <= 0) return n < 0 ? fail(SPK_ERR_DIMENSION, "negative batch") : SPK_OK;
  return eval_internal(net, precision, n, nullptr, xs, out, (cudaStream_t)stream);
}

int spk_bound_batch_host(const spk_net* net, int policy, int n_keep, int precision, int64_t n, int s,
                         const double* centers, const double* axes, double* lo, double* hi,
                         int8_t* cls) {
  if (!net) return fail(SPK_ERR_INVALID_PARAMETER, "null net");
  if (n <= 0) return n < 0 ? fail(SPK_ERR_DIMENSION, "negative batch") : SPK_OK;
  return host_pipeline(net, policy, n_keep, precision, n, s, centers, axes, lo, hi, cls);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// FP32 FFMA throughput probe: the roofline denominator for the FFMA-bound
// bound kernels, measured on the box at its current clocks (bench.py).
namespace spk {
__global__ void __launch_bounds__(256) ffma_probe_kernel(float* out, int iters, float seed, float mp, float cp) {
  // 16 independent FFMA chains per thread with register operands (a = a*b + c);
  // b and c are the same registers for every chain, the classic peak probe.
  float a[16], b, c;
  asm volatile("mov.f32 %0, %1;" : "=f"(b) : "f"(mp));
  asm volatile("mov.f32 %0, %1;" : "=f"(c) : "f"(cp));
#pragma unroll
  for (int j = 0; j < 16; ++j) a[j] = seed + j * 1e-3f + threadIdx.x * 1e-7f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = fmaf(a[j], b, c);
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += a[j];
  if (s == 12345.678f) out[0] = s;  // keep the chains alive
}
}  // namespace spk

extern "C" int spk_ffma_peak(int iters, double* flops_per_s, void* stream) {
  using namespace spk;
  int dev = 0;
  cudaGetDevice(&dev);
  const int sm = sm_count_for(dev);
  if (sm <= 0) return fail(SPK_ERR_CUDA, "no CUDA device");
  float* out = nullptr;
  if (cudaMalloc(&out, sizeof(float)) != cudaSuccess) return fail(SPK_ERR_OUT_OF_MEMORY, "probe");
  cudaStream_t st = (cudaStream_t)stream;
  const int blocks = sm * 8, threads = 256;
  ffma_probe_kernel<<<blocks, threads, 0, st>>>(out, 64, 1.0f, 0.9999f, 1e-6f);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  ffma_probe_kernel<<<blocks, threads, 0, st>>>(out, iters, 1.0f, 0.9999f, 1e-6f);
  cudaEventRecord(e1, st);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (e != cudaSuccess) return cuda_fail(e, "ffma probe");
  *flops_per_s = 2.0 * 16.0 * (double)iters * blocks * threads / (ms * 1e-3);
  return SPK_OK;
}
