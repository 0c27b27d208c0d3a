// K6: adaptive range-marching ray caster (_march_arrays, rays.py:88-138;
// Alg. 2 of the paper) with device-resident ray state.
//
// Every ray keeps t and sigma in FP64 (the reference never floors sigma, so
// an FP32 sigma would underflow after ~126 failures and the step sequence
// would diverge).  Each lock-step round over the compacted active set:
//   1. gen: probe point p + (t+delta) r, segment box centre p + (t+sigma/2) r,
//      axis (sigma/2) r -- FP64, exactly the reference's expressions;
//   2. one point-evaluation pass and one bound pass (any policy) through the
//      fused network kernels;
//   3. update: sign flip against f(origin) -> hit at t; else sigma *= eta+ /
//      eta- and t += max(safety*sigma*, delta) (rays.py:133-136); survivors
//      with t < t_max are re-compacted (warp ballot + block prefix) for the
//      next round.
// With the certification decisions equal, t is bit-identical to the
// reference's (same FP64 operations in the same order).  For interval and
// affine-fixed the probe evaluation and the segment bound run as ONE fused
// network pass per round (spk_march_pass.cuh); truncate / full use the
// point kernel + symbolic bound kernel.
// Camera rays (Camera.pixel_dirs, camera.py:74-92) are generated on the
// device with round-to-nearest FP64 ops in numpy's evaluation order, so they
// match the reference bit for bit.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <vector>

#include "spk_march_pass.cuh"
#include "spk_abi_internal.h"

namespace spk {

constexpr int MT = 256;

__global__ void camera_dirs_kernel(int W, int H, double fx, double fy, double fz, double rx, double ry, double rz,
                                   double ux, double uy, double uz, double half_w, double half_h,
                                   double* __restrict__ dirs) {
  const long long q = (long long)blockIdx.x * MT + threadIdx.x;
  if (q >= (long long)W * H) return;
  const int j = (int)(q / W), i = (int)(q % W);
  // u = ((i + 0.5) / W * 2 - 1) * half_w ; v = (1 - (j + 0.5) / H * 2) * half_h
  const double u = __dmul_rn(__dsub_rn(__dmul_rn(__ddiv_rn(__dadd_rn((double)i, 0.5), (double)W), 2.0), 1.0), half_w);
  const double v = __dmul_rn(__dsub_rn(1.0, __dmul_rn(__ddiv_rn(__dadd_rn((double)j, 0.5), (double)H), 2.0)), half_h);
  // d = (fwd + u * right) + v * up   (numpy broadcast order)
  const double dx = __dadd_rn(__dadd_rn(fx, __dmul_rn(u, rx)), __dmul_rn(v, ux));
  const double dy = __dadd_rn(__dadd_rn(fy, __dmul_rn(u, ry)), __dmul_rn(v, uy));
  const double dz = __dadd_rn(__dadd_rn(fz, __dmul_rn(u, rz)), __dmul_rn(v, uz));
  const double nrm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
  dirs[q * 3 + 0] = __ddiv_rn(dx, nrm);
  dirs[q * 3 + 1] = __ddiv_rn(dy, nrm);
  dirs[q * 3 + 2] = __ddiv_rn(dz, nrm);
}

__global__ void broadcast_kernel(long long n, double* __restrict__ v) {
  const long long i = (long long)blockIdx.x * MT + threadIdx.x;
  const double x = v[0];
  __syncthreads();
  if (i > 0 && i < n) v[i] = x;
}

SPK_DEV const double* origin_of(const double* origins, long long stride, long long i) { return origins + i * stride; }

// initial state: f0 at the origin decides on-surface hits and the inside flag
__global__ void march_init_kernel(long long n, const double* __restrict__ f0, const double* __restrict__ t_init,
                                  const double* __restrict__ s_init, MarchParamsDev P, double* __restrict__ t,
                                  double* __restrict__ sig, double* __restrict__ steps, uint8_t* __restrict__ hit,
                                  double* __restrict__ t_out, uint8_t* __restrict__ neg0, uint8_t* __restrict__ live) {
  const long long i = (long long)blockIdx.x * MT + threadIdx.x;
  if (i >= n) return;
  const double ti = t_init ? t_init[i] : 0.0;
  t[i] = ti;
  sig[i] = s_init ? s_init[i] : P.sigma0;
  steps[i] = 0.0;
  const bool surf = f0[i] == 0.0;
  hit[i] = surf ? 1 : 0;
  t_out[i] = surf ? 0.0 : INFINITY;
  neg0[i] = f0[i] < 0.0 ? 1 : 0;
  live[i] = (!surf && ti < P.t_max) ? 1 : 0;
}

// compaction of the live flags into an index list (ballot + block prefix)
__global__ void count_kernel(long long n, const uint8_t* __restrict__ live, const int* __restrict__ idx_in,
                             int* __restrict__ block_cnt) {
  const long long q = (long long)blockIdx.x * MT + threadIdx.x;
  bool f = false;
  if (q < n) f = live[idx_in ? idx_in[q] : q] != 0;
  __shared__ int wc[MT / 32];
  const unsigned m = __ballot_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0) wc[threadIdx.x >> 5] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < MT / 32; ++w) s += wc[w];
    block_cnt[blockIdx.x] = s;
  }
}

__global__ void compact_kernel(long long n, const uint8_t* __restrict__ live, const int* __restrict__ idx_in,
                               const int* __restrict__ block_cnt, int* __restrict__ idx_out) {
  const long long q = (long long)blockIdx.x * MT + threadIdx.x;
  long long off = 0;
  {
    long long s = 0;
    for (int b = threadIdx.x; b < (int)blockIdx.x; b += MT) s += block_cnt[b];
    __shared__ long long red[MT / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    for (int w = 0; w < MT / 32; ++w) off += red[w];
  }
  int ray = -1;
  bool f = false;
  if (q < n) {
    ray = idx_in ? idx_in[q] : (int)q;
    f = live[ray] != 0;
  }
  __shared__ int wc[MT / 32];
  const unsigned m = __ballot_sync(0xffffffffu, f);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) wc[w] = __popc(m);
  __syncthreads();
  int before = 0;
  for (int v = 0; v < w; ++v) before += wc[v];
  if (f) idx_out[off + before + __popc(m & ((1u << lane) - 1u))] = ray;
}

__global__ void march_gen_kernel(long long na, const int* __restrict__ idx, const double* __restrict__ origins,
                                 long long ostride, const double* __restrict__ dirs, const double* __restrict__ t,
                                 const double* __restrict__ sig, MarchParamsDev P, double* __restrict__ probe,
                                 double* __restrict__ centre, double* __restrict__ axis) {
  const long long j = (long long)blockIdx.x * MT + threadIdx.x;
  if (j >= na) return;
  const int i = idx[j];
  const double* p = origin_of(origins, ostride, i);
  const double* r = dirs + (long long)i * 3;
  const double ti = t[i], si = sig[i];
  const double tp = __dadd_rn(ti, P.delta);                  // t + delta
  const double tc = __dadd_rn(ti, __ddiv_rn(si, 2.0));       // t + sigma/2
  const double hs = __ddiv_rn(si, 2.0);                      // sigma/2
  for (int k = 0; k < 3; ++k) {
    probe[j * 3 + k] = __dadd_rn(p[k], __dmul_rn(tp, r[k]));
    centre[j * 3 + k] = __dadd_rn(p[k], __dmul_rn(tc, r[k]));
    axis[j * 3 + k] = __dmul_rn(hs, r[k]);
  }
}

__global__ void march_update_kernel(long long na, const int* __restrict__ idx, const double* __restrict__ fp,
                                    const double* __restrict__ blo, const double* __restrict__ bhi, MarchParamsDev P,
                                    double* __restrict__ t, double* __restrict__ sig, double* __restrict__ steps,
                                    uint8_t* __restrict__ hit, double* __restrict__ t_out,
                                    const uint8_t* __restrict__ neg0, uint8_t* __restrict__ live,
                                    unsigned long long* __restrict__ certified) {
  const long long j = (long long)blockIdx.x * MT + threadIdx.x;
  if (j >= na) return;
  const int i = idx[j];
  steps[i] = __dadd_rn(steps[i], 1.0);
  const bool flip = (fp[j] < 0.0) != (neg0[i] != 0);
  if (flip) {
    hit[i] = 1;
    t_out[i] = t[i];
    live[i] = 0;
    return;
  }
  const double sa = sig[i];
  const bool known = (blo[j] > 0.0) || (bhi[j] < 0.0);
  const double star = known ? sa : 0.0;
  sig[i] = known ? __dmul_rn(sa, P.eta_plus) : __dmul_rn(sa, P.eta_minus);
  const double nt = __dadd_rn(t[i], fmax(__dmul_rn(P.safety, star), P.delta));
  t[i] = nt;
  live[i] = nt < P.t_max ? 1 : 0;
  if (known) atomicAdd(certified, 1ull);
}

// the calling thread's record of its last spk_march: (active rays, ms) per round
static std::vector<std::pair<long long, double>>& round_log() {
  thread_local std::vector<std::pair<long long, double>> log;
  return log;
}

}  // namespace spk

using namespace spk;

extern "C" {

int spk_camera_dirs(const double* frame9, double half_w, double half_h, int width, int height, double* dirs,
                    void* stream) {
  if (!frame9 || width < 1 || height < 1) return fail(SPK_ERR_INVALID_PARAMETER, "bad camera");
  const long long n = (long long)width * height;
  camera_dirs_kernel<<<(int)((n + MT - 1) / MT), MT, 0, (cudaStream_t)stream>>>(
      width, height, frame9[0], frame9[1], frame9[2], frame9[3], frame9[4], frame9[5], frame9[6], frame9[7],
      frame9[8], half_w, half_h, dirs);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SPK_OK : cuda_fail(e, "camera dirs");
}

int spk_march_round_log(int64_t* active, double* ms, int cap) {
  const auto& log = round_log();
  const int n = (int)log.size();
  for (int i = 0; i < n && i < cap; ++i) {
    if (active) active[i] = log[i].first;
    if (ms) ms[i] = log[i].second;
  }
  return n;
}

int spk_march(const spk_net* net, int policy, int n_keep, int precision, int64_t n, const double* origins,
              int64_t origin_stride, const double* dirs, const double* t_init, const double* sigma_init,
              const double* params6, uint8_t* hit, double* t_out, double* steps, int64_t* stats, void* stream) {
  if (!net || !params6) return fail(SPK_ERR_INVALID_PARAMETER, "null argument");
  if (net->input_dim != 3) return fail(SPK_ERR_DIMENSION, "ray casting needs a 3-d network");
  if (int rc = check_ray_params(params6)) return rc;
  if (origin_stride != 0 && origin_stride != 3)
    return fail(SPK_ERR_INVALID_PARAMETER, "origin_stride must be 0 (shared origin) or 3");
  if (n <= 0) return n < 0 ? fail(SPK_ERR_DIMENSION, "negative ray count") : SPK_OK;
  if (n > (int64_t)INT32_MAX) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "too many rays in one call");
  MarchParamsDev P{params6[0], params6[1], params6[2], params6[3], params6[4], params6[5]};
  DeviceGuard g(net->device);
  cudaStream_t st = (cudaStream_t)stream;
  // scratch from the stream-ordered pool
  double *t = nullptr, *sig = nullptr, *f0 = nullptr, *probe = nullptr, *cen = nullptr, *ax = nullptr, *fp = nullptr,
         *blo = nullptr, *bhi = nullptr;
  uint8_t *neg0 = nullptr, *live = nullptr;
  int *idx_a = nullptr, *idx_b = nullptr, *bcnt = nullptr;
  unsigned long long* cert = nullptr;
  const int nblk = (int)((n + MT - 1) / MT);
  cudaError_t e = cudaSuccess;
  auto A = [&](void** p, size_t bytes) {
    if (e == cudaSuccess) e = cudaMallocAsync(p, std::max<size_t>(bytes, 16), st);
  };
  A((void**)&t, n * 8); A((void**)&sig, n * 8); A((void**)&f0, n * 8); A((void**)&probe, n * 24);
  A((void**)&cen, n * 24); A((void**)&ax, n * 24); A((void**)&fp, n * 8); A((void**)&blo, n * 8);
  A((void**)&bhi, n * 8); A((void**)&neg0, n); A((void**)&live, n); A((void**)&idx_a, n * 4);
  A((void**)&idx_b, n * 4); A((void**)&bcnt, (size_t)nblk * 4); A((void**)&cert, 8);
  int rc = SPK_OK;
  std::vector<int> hcnt(nblk);
  long long rounds = 0, evals = 0;
  // per-round record of this call (spk_march_round_log): active rays and the
  // host wall time of the round (kernel + count + the one synchronisation)
  round_log().clear();
  auto t_round = std::chrono::steady_clock::now();
  if (e != cudaSuccess) {
    rc = cuda_fail(e, "march alloc");
  } else {
    cudaMemsetAsync(cert, 0, 8, st);
    // f0: origins (a stride-0 origin is evaluated once and broadcast)
    rc = spk_eval_batch(net, precision, origin_stride == 0 ? 1 : n, origins, f0, st);
    if (rc == SPK_OK && origin_stride == 0) broadcast_kernel<<<nblk, MT, 0, st>>>(n, f0);
  }
  evals += origin_stride == 0 ? 1 : n;
  long long na = 0;
  int* cur = idx_a;
  int* nxt = idx_b;
  if (rc == SPK_OK) {
    march_init_kernel<<<nblk, MT, 0, st>>>(n, f0, t_init, sigma_init, P, t, sig, steps, hit, t_out, neg0, live);
    count_kernel<<<nblk, MT, 0, st>>>(n, live, nullptr, bcnt);
    e = cudaMemcpyAsync(hcnt.data(), bcnt, nblk * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_fail(e, "march init");
    for (int b = 0; b < nblk; ++b) na += hcnt[b];
    if (rc == SPK_OK) compact_kernel<<<nblk, MT, 0, st>>>(n, live, nullptr, bcnt, cur);
  }
  const bool fused = policy == SPK_POLICY_INTERVAL || policy == SPK_POLICY_AFFINE_FIXED;
  const int sm = sm_count_for(net->device);
  while (rc == SPK_OK && na > 0) {
    const int ab = (int)((na + MT - 1) / MT);
    if (fused) {
      MarchState M{cur, origins, origin_stride, dirs, t, sig, steps, hit, t_out, neg0, live, cert};
      cudaError_t ke;
      if (precision == SPK_FP64) {
        NetDev<double> nd_copy;
        const NetDev<double>* nd = &nd_copy;
        if ((rc = get_dev<double>(const_cast<spk_net*>(net), &nd_copy)) != SPK_OK) break;
        ke = dispatch_march_round<double>(net->mmax, policy == SPK_POLICY_AFFINE_FIXED, *nd, M, P, na, sm, st);
      } else {
        NetDev<float> nd_copy;
        const NetDev<float>* nd = &nd_copy;
        if ((rc = get_dev<float>(const_cast<spk_net*>(net), &nd_copy)) != SPK_OK) break;
        ke = dispatch_march_round<float>(net->mmax, policy == SPK_POLICY_AFFINE_FIXED, *nd, M, P, na, sm, st);
      }
      if (ke != cudaSuccess) { rc = cuda_fail(ke, "march round"); break; }
    } else {
      march_gen_kernel<<<ab, MT, 0, st>>>(na, cur, origins, origin_stride, dirs, t, sig, P, probe, cen, ax);
      rc = spk_eval_batch(net, precision, na, probe, fp, st);
      if (rc != SPK_OK) break;
      rc = spk_bound_batch(net, policy, n_keep, precision, na, 1, cen, ax, blo, bhi, nullptr, st);
      if (rc != SPK_OK) break;
      march_update_kernel<<<ab, MT, 0, st>>>(na, cur, fp, blo, bhi, P, t, sig, steps, hit, t_out, neg0, live, cert);
    }
    evals += na;
    ++rounds;
    count_kernel<<<ab, MT, 0, st>>>(na, live, cur, bcnt);
    e = cudaMemcpyAsync(hcnt.data(), bcnt, ab * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { rc = cuda_fail(e, "march round"); break; }
    long long nn = 0;
    for (int b = 0; b < ab; ++b) nn += hcnt[b];
    {
      const auto now = std::chrono::steady_clock::now();
      round_log().push_back({na, std::chrono::duration<double, std::milli>(now - t_round).count()});
      t_round = now;
    }
    if (nn > 0) compact_kernel<<<ab, MT, 0, st>>>(na, live, cur, bcnt, nxt);
    std::swap(cur, nxt);
    na = nn;
  }
  if (rc == SPK_OK) {
    e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_fail(e, "march kernels");
  }
  unsigned long long hc = 0;
  if (rc == SPK_OK && stats) {
    cudaMemcpyAsync(&hc, cert, 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    stats[0] = rounds;
    stats[1] = evals - (origin_stride == 0 ? 1 : n);  // ray-steps (one probe + one bound each)
    stats[2] = (int64_t)hc;                            // certified steps
  }
  void* bufs[] = {t, sig, f0, probe, cen, ax, fp, blo, bhi, neg0, live, idx_a, idx_b, bcnt, cert};
  for (void* b : bufs)
    if (b) cudaFreeAsync(b, st);
  return rc;
}

}  // extern "C"
