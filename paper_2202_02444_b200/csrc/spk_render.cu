// §8(f2): render post-processing on the device (render.py:36-141).
//
//   spk_render_shade      _refine_hits (48 bisections of [t, t + delta]),
//                         _normals (central differences, h = delta / 10)
//                         and Lambert shading of every hit pixel; misses get
//                         the background colour.
//   spk_fixed_step_march  _fixed_step_march: the uniform-marching baseline
//                         (sample at t = step, 2 step, ...; first sign flip).
//
// Both are point-evaluation work (K4): every network pass goes through the
// fused point kernel with a DEVICE-side count, so the 48-step bisection and
// the normal pass run without a host round trip; the hit set is compacted
// once (ballot + block prefix + one atomic per block).  Per-point scalar
// arithmetic is FP64 round-to-nearest in numpy's operation order.
#include <algorithm>
#include <cmath>
#include <vector>

#include "spk_abi_internal.h"

namespace spk {
namespace {

constexpr int RT = 256;

struct Scratch {
  cudaStream_t st;
  std::vector<void*> bufs;
  cudaError_t err = cudaSuccess;
  explicit Scratch(cudaStream_t s) : st(s) {}
  ~Scratch() {
    for (void* p : bufs) cudaFreeAsync(p, st);
  }
  template <typename P>
  P* get(size_t bytes) {
    void* p = nullptr;
    if (err == cudaSuccess) err = cudaMallocAsync(&p, std::max<size_t>(bytes, 16), st);
    if (err == cudaSuccess) bufs.push_back(p);
    return (P*)p;
  }
};

SPK_DEV const double* ray_origin(const double* o, long long stride, long long i) { return o + i * stride; }

// indices of flagged rays, order-preserving within a block; one atomic per block
__global__ void select_kernel(long long n, const uint8_t* __restrict__ flag, int* __restrict__ out,
                              long long* __restrict__ count) {
  __shared__ int warp_tot[RT / 32];
  __shared__ long long base;
  const long long i = (long long)blockIdx.x * RT + threadIdx.x;
  const bool f = i < n && flag[i];
  const unsigned m = __ballot_sync(0xffffffffu, f);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) warp_tot[w] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int k = 0; k < RT / 32; ++k) {
      const int c = warp_tot[k];
      warp_tot[k] = tot;
      tot += c;
    }
    base = tot ? (long long)atomicAdd((unsigned long long*)count, (unsigned long long)tot) : 0;
  }
  __syncthreads();
  if (f) out[base + warp_tot[w] + __popc(m & ((1u << lane) - 1))] = (int)i;
}

// ---- _refine_hits -------------------------------------------------------------

__global__ void refine_init_kernel(long long cap, const long long* __restrict__ nh, const int* __restrict__ idx,
                                   const double* __restrict__ t, double delta, double* lo, double* hi) {
  const long long q = (long long)blockIdx.x * RT + threadIdx.x;
  if (q >= *nh || q >= cap) return;
  const double tq = t[idx[q]];
  lo[q] = tq;
  hi[q] = __dadd_rn(tq, delta);
}

// mid = 0.5 * (lo + hi); point = origin + mid * dir
__global__ void refine_mid_kernel(long long cap, const long long* __restrict__ nh, const int* __restrict__ idx,
                                  const double* __restrict__ origins, long long ostride,
                                  const double* __restrict__ dirs, const double* __restrict__ lo,
                                  const double* __restrict__ hi, double* mid, double* pts) {
  const long long q = (long long)blockIdx.x * RT + threadIdx.x;
  if (q >= *nh || q >= cap) return;
  const long long r = idx[q];
  const double m = __dmul_rn(0.5, __dadd_rn(lo[q], hi[q]));
  mid[q] = m;
  const double* o = ray_origin(origins, ostride, r);
#pragma unroll
  for (int k = 0; k < 3; ++k) pts[q * 3 + k] = __dadd_rn(o[k], __dmul_rn(m, dirs[r * 3 + k]));
}

__global__ void refine_update_kernel(long long cap, const long long* __restrict__ nh, const double* __restrict__ f0,
                                     const double* __restrict__ fm, const double* __restrict__ mid, double* lo,
                                     double* hi) {
  const long long q = (long long)blockIdx.x * RT + threadIdx.x;
  if (q >= *nh || q >= cap) return;
  const bool flip = (fm[q] < 0.0) != (f0[0] < 0.0);
  if (flip)
    hi[q] = mid[q];
  else
    lo[q] = mid[q];
}

// ---- _normals + shading ----------------------------------------------------------

// pts = origin + t_ref * dir; 6 probes p + h e_k, p - h e_k (k = 0, 1, 2)
__global__ void normal_probe_kernel(long long cap, const long long* __restrict__ nh, const int* __restrict__ idx,
                                    const double* __restrict__ origins, long long ostride,
                                    const double* __restrict__ dirs, const double* __restrict__ tref, double h,
                                    double* probes) {
  const long long q = (long long)blockIdx.x * RT + threadIdx.x;
  if (q >= *nh || q >= cap) return;
  const long long r = idx[q];
  const double* o = ray_origin(origins, ostride, r);
  double p[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) p[k] = __dadd_rn(o[k], __dmul_rn(tref[q], dirs[r * 3 + k]));
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double* plus = probes + (q * 6 + 2 * k) * 3;
    double* minus = plus + 3;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      plus[c] = c == k ? __dadd_rn(p[c], h) : __dadd_rn(p[c], 0.0);
      minus[c] = c == k ? __dsub_rn(p[c], h) : __dsub_rn(p[c], 0.0);
    }
  }
}

__global__ void shade_kernel(long long cap, const long long* __restrict__ nh, const int* __restrict__ idx,
                             const double* __restrict__ fprobe, double lx, double ly, double lz, uint8_t* pixels) {
  const long long q = (long long)blockIdx.x * RT + threadIdx.x;
  if (q >= *nh || q >= cap) return;
  double g[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) g[k] = __dsub_rn(fprobe[q * 6 + 2 * k], fprobe[q * 6 + 2 * k + 1]);
  // np.linalg.norm(g, axis=1): sqrt((g0^2 + g1^2) + g2^2); zero norm -> 1
  double nrm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(g[0], g[0]), __dmul_rn(g[1], g[1])), __dmul_rn(g[2], g[2])));
  if (nrm == 0.0) nrm = 1.0;
  const double n0 = __ddiv_rn(g[0], nrm), n1 = __ddiv_rn(g[1], nrm), n2 = __ddiv_rn(g[2], nrm);
  // n @ LIGHT_DIR, clip to [0, 1], rint(* 255)
  double lam = __fma_rn(n2, lz, __fma_rn(n1, ly, __dmul_rn(n0, lx)));
  lam = fmin(fmax(lam, 0.0), 1.0);
  const uint8_t gray = (uint8_t)rint(__dmul_rn(lam, 255.0));
  const long long p = idx[q];
  pixels[p * 3 + 0] = gray;
  pixels[p * 3 + 1] = gray;
  pixels[p * 3 + 2] = gray;
}

__global__ void scale_count_kernel(const long long* __restrict__ n, int k, long long* out) { *out = *n * k; }

__global__ void background_kernel(long long n, uint8_t r, uint8_t g, uint8_t b, uint8_t* pixels) {
  const long long i = (long long)blockIdx.x * RT + threadIdx.x;
  if (i >= n) return;
  pixels[i * 3 + 0] = r;
  pixels[i * 3 + 1] = g;
  pixels[i * 3 + 2] = b;
}

// ---- _fixed_step_march -------------------------------------------------------------

__global__ void fixed_init_kernel(long long n, const double* __restrict__ f0, long long f0_stride, uint8_t* hit,
                                  double* t_out, uint8_t* neg0, uint8_t* alive) {
  const long long i = (long long)blockIdx.x * RT + threadIdx.x;
  if (i >= n) return;
  const double f = f0[i * f0_stride];
  const bool surf = f == 0.0;
  hit[i] = surf;
  t_out[i] = surf ? 0.0 : INFINITY;
  neg0[i] = f < 0.0;
  alive[i] = !surf;
}

__global__ void fixed_probe_kernel(long long cap, const long long* __restrict__ na, const int* __restrict__ idx,
                                   const double* __restrict__ origins, long long ostride,
                                   const double* __restrict__ dirs, double t, double* pts) {
  const long long q = (long long)blockIdx.x * RT + threadIdx.x;
  if (q >= *na || q >= cap) return;
  const long long r = idx[q];
  const double* o = ray_origin(origins, ostride, r);
#pragma unroll
  for (int k = 0; k < 3; ++k) pts[q * 3 + k] = __dadd_rn(o[k], __dmul_rn(t, dirs[r * 3 + k]));
}

// sign flip -> hit at t - step; survivors re-compacted into nxt (block-ordered)
__global__ void fixed_update_kernel(long long cap, const long long* __restrict__ na, const int* __restrict__ idx,
                                    const double* __restrict__ fc, const uint8_t* __restrict__ neg0, double t_hit,
                                    uint8_t* hit, double* t_out, int* nxt, long long* n_next) {
  __shared__ int warp_tot[RT / 32];
  __shared__ long long base;
  const long long q = (long long)blockIdx.x * RT + threadIdx.x;
  const bool valid = q < *na && q < cap;
  bool keep = false;
  int r = 0;
  if (valid) {
    r = idx[q];
    const bool flip = (fc[q] < 0.0) != (bool)neg0[r];
    if (flip) {
      hit[r] = 1;
      t_out[r] = t_hit;
    }
    keep = !flip;
  }
  const unsigned m = __ballot_sync(0xffffffffu, keep);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) warp_tot[w] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int k = 0; k < RT / 32; ++k) {
      const int c = warp_tot[k];
      warp_tot[k] = tot;
      tot += c;
    }
    base = tot ? (long long)atomicAdd((unsigned long long*)n_next, (unsigned long long)tot) : 0;
  }
  __syncthreads();
  if (keep) nxt[base + warp_tot[w] + __popc(m & ((1u << lane) - 1))] = r;
}

}  // namespace
}  // namespace spk

using namespace spk;

extern "C" {

int spk_render_shade(const spk_net* net, int precision, int64_t n, const double* origins, int64_t origin_stride,
                     const double* dirs, const uint8_t* hit, const double* t, double delta, int iters,
                     const double* light3, const uint8_t* background3, uint8_t* pixels, int64_t* n_hits,
                     void* stream) {
  if (!net || !light3 || !background3 || (n > 0 && (!origins || !dirs || !hit || !t || !pixels)))
    return fail(SPK_ERR_INVALID_PARAMETER, "null argument");
  if (net->input_dim != 3) return fail(SPK_ERR_DIMENSION, "rendering needs a 3-d network");
  if (origin_stride != 0 && origin_stride != 3)
    return fail(SPK_ERR_INVALID_PARAMETER, "origin_stride must be 0 (shared origin) or 3");
  if (!(delta > 0.0)) return fail(SPK_ERR_INVALID_PARAMETER, "delta must be positive");
  if (n < 0 || iters < 0) return fail(SPK_ERR_DIMENSION, "negative size");
  if (n > (int64_t)INT32_MAX / 6) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "too many pixels in one call");
  if (n == 0) {
    if (n_hits) *n_hits = 0;
    return SPK_OK;
  }
  DeviceGuard g(net->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int blk = (int)((n + RT - 1) / RT);
  Scratch S(st);
  long long* nh = S.get<long long>(8);
  int* idx = S.get<int>(n * 4);
  double* f0 = S.get<double>(8);
  double* lo = S.get<double>(n * 8);
  double* hi = S.get<double>(n * 8);
  double* mid = S.get<double>(n * 8);
  double* fm = S.get<double>(n * 6 * 8);     // bisection values, then the 6 probe values
  double* pts = S.get<double>(n * 6 * 24);   // bisection points, then the 6 probes
  long long* nh6 = S.get<long long>(8);
  if (S.err != cudaSuccess) return cuda_fail(S.err, "render alloc");
  cudaMemsetAsync(nh, 0, 8, st);
  background_kernel<<<blk, RT, 0, st>>>(n, background3[0], background3[1], background3[2], pixels);
  select_kernel<<<blk, RT, 0, st>>>(n, hit, idx, nh);
  // f(origin of ray 0) decides the inside flag (render.py:134-135: one camera)
  int rc = spk_eval_batch(net, precision, 1, origins, f0, st);
  if (rc != SPK_OK) return rc;
  refine_init_kernel<<<blk, RT, 0, st>>>(n, nh, idx, t, delta, lo, hi);
  for (int it = 0; it < iters; ++it) {
    refine_mid_kernel<<<blk, RT, 0, st>>>(n, nh, idx, origins, origin_stride, dirs, lo, hi, mid, pts);
    if ((rc = eval_internal(net, precision, n, nh, pts, fm, st)) != SPK_OK) return rc;
    refine_update_kernel<<<blk, RT, 0, st>>>(n, nh, f0, fm, mid, lo, hi);
  }
  // the refined hit is lo; 6 central-difference probes per hit, h = delta / 10
  const double h = delta / 10.0;
  normal_probe_kernel<<<blk, RT, 0, st>>>(n, nh, idx, origins, origin_stride, dirs, lo, h, pts);
  // 6 probes per hit: one point pass over 6 * n_h points (device count)
  scale_count_kernel<<<1, 1, 0, st>>>(nh, 6, nh6);
  if ((rc = eval_internal(net, precision, 6 * n, nh6, pts, fm, st)) != SPK_OK) return rc;
  shade_kernel<<<blk, RT, 0, st>>>(n, nh, idx, fm, light3[0], light3[1], light3[2], pixels);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "render kernels");
  if (n_hits) {
    long long hn = 0;
    e = cudaMemcpyAsync(&hn, nh, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "render hits");
    *n_hits = hn;
  }
  return SPK_OK;
}

int spk_fixed_step_march(const spk_net* net, int precision, int64_t n, const double* origins, int64_t origin_stride,
                         const double* dirs, double step, double t_max, uint8_t* hit, double* t_out, int64_t* stats,
                         void* stream) {
  if (!net || (n > 0 && (!origins || !dirs || !hit || !t_out)))
    return fail(SPK_ERR_INVALID_PARAMETER, "null argument");
  if (!(step > 0.0)) return fail(SPK_ERR_INVALID_PARAMETER, "fixed_step mode needs a positive step");
  if (!(t_max > 0.0)) return fail(SPK_ERR_INVALID_PARAMETER, "t_max must be positive");
  if (origin_stride != 0 && origin_stride != 3)
    return fail(SPK_ERR_INVALID_PARAMETER, "origin_stride must be 0 (shared origin) or 3");
  if (net->input_dim != 3) return fail(SPK_ERR_DIMENSION, "ray casting needs a 3-d network");
  if (n < 0) return fail(SPK_ERR_DIMENSION, "negative ray count");
  if (n > (int64_t)INT32_MAX) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "too many rays in one call");
  if (n == 0) return SPK_OK;
  DeviceGuard g(net->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int blk = (int)((n + RT - 1) / RT);
  Scratch S(st);
  double* f0 = S.get<double>(origin_stride == 0 ? 8 : n * 8);
  uint8_t* neg0 = S.get<uint8_t>(n);
  uint8_t* alive = S.get<uint8_t>(n);
  int* ia = S.get<int>(n * 4);
  int* ib = S.get<int>(n * 4);
  long long* cnt = S.get<long long>(16);
  double* pts = S.get<double>(n * 24);
  double* fc = S.get<double>(n * 8);
  if (S.err != cudaSuccess) return cuda_fail(S.err, "fixed-step alloc");
  int rc = spk_eval_batch(net, precision, origin_stride == 0 ? 1 : n, origins, f0, st);
  if (rc != SPK_OK) return rc;
  fixed_init_kernel<<<blk, RT, 0, st>>>(n, f0, origin_stride == 0 ? 0 : 1, hit, t_out, neg0, alive);
  cudaMemsetAsync(cnt, 0, 16, st);
  select_kernel<<<blk, RT, 0, st>>>(n, alive, ia, cnt);
  long long na = 0;
  cudaError_t e = cudaMemcpyAsync(&na, cnt, 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "fixed-step init");
  // t accumulates on the host exactly like the reference's python float
  double t = step;
  int64_t rounds = 0, evals = 0;
  int* cur = ia;
  int* nxt = ib;
  long long* ncur = cnt;
  long long* nnext = cnt + 1;
  while (na > 0 && t < t_max) {
    const int ab = (int)((na + RT - 1) / RT);
    evals += na;
    fixed_probe_kernel<<<ab, RT, 0, st>>>(na, ncur, cur, origins, origin_stride, dirs, t, pts);
    if ((rc = spk_eval_batch(net, precision, na, pts, fc, st)) != SPK_OK) return rc;
    cudaMemsetAsync(nnext, 0, 8, st);
    fixed_update_kernel<<<ab, RT, 0, st>>>(na, ncur, cur, fc, neg0, t - step, hit, t_out, nxt, nnext);
    e = cudaMemcpyAsync(&na, nnext, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "fixed-step round");
    ++rounds;
    std::swap(cur, nxt);
    std::swap(ncur, nnext);
    t += step;
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "fixed-step kernels");
  if (stats) {
    stats[0] = rounds;
    stats[1] = evals;
  }
  return SPK_OK;
}

}  // extern "C"
