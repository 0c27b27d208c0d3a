// §8(f1): frustum range-marching over a camera's pixel grid
// (cast_frustum_image, rays.py:232-341; Frustum, rays.py:187-209;
// Camera.frustum_slab_box, camera.py:99-135).
//
// Rectangles of pixels march as one oriented slab box per step: while the
// frustum's front face (world width at parameter t along its longer pixel
// side) stays within 2 sigma, one bound of the slab between t and t + sigma
// certifies (or refuses) the step for every contained pixel ray at once;
// wider frusta split in half across that side.  Single-pixel frusta finish
// on the device ray march (spk_march, K6) from their (t, sigma).
//
// Everything runs on the device; the host only reads two counters a round.
// One round (the reference's outer `while frontier` iteration):
//   expand  one thread per frontier frustum replays the reference's split
//           stack for it (DFS over its rectangle; the split decision only
//           depends on the rectangle and the frustum's t, sigma) and appends
//           each marching rectangle -- with its slab box -- to the marching
//           list and each single pixel to the hand-off list (atomic slots:
//           order is irrelevant, every frustum and pixel is independent);
//   bound   the fused bound pass over the marching slab boxes (s = 3, rows
//           beyond a slab's own s zero, as in the reference's padding);
//   update  one warp per marching frustum: amortised steps += 1/n_pixels
//           over its pixels (one frustum per pixel per round, so the FP64
//           sums run in the reference's order), then t / sigma as
//           rays.py:324-330.  The marching list is the next frontier.
// All geometry is FP64 with explicit round-to-nearest intrinsics in numpy's
// operation order (the 3-vector norm as numpy's 1-D dot, an FMA chain), so
// with FP64 bounds the result is bit-identical to the reference's.
//
// Termination guard (not in the reference): an uncertified multi-pixel
// frustum whose sigma drops below delta * 2^-32 dissolves into single-pixel
// hand-offs.  At t = 0 a frustum's front width is 0, so it can never split;
// when the bound's rounding slack exceeds |f| at the camera the reference
// loops forever there.  The per-ray march always advances by >= delta.
#include <algorithm>
#include <cmath>
#include <vector>

#include "spk_abi_internal.h"

namespace spk {
namespace {

constexpr int FT = 256;
constexpr int MAX_DFS = 64;  // 2 * log2(max side) + 2 suffices (sides <= 2^31)

struct CamDev {
  double pos[3], fwd[3], right[3], up[3];
  double half_w, half_h;
  int W, H;
};

struct FrustumParams {
  double t_max, eta_plus, eta_minus, delta, safety, sigma_floor;
};

// ---- camera geometry, numpy's operation order (camera.py:68-135) ----------

SPK_DEV double u_of(const CamDev& c, int i) {
  return __dmul_rn(__dsub_rn(__dmul_rn(__ddiv_rn(__dadd_rn((double)i, 0.5), (double)c.W), 2.0), 1.0), c.half_w);
}
SPK_DEV double v_of(const CamDev& c, int j) {
  return __dmul_rn(__dsub_rn(1.0, __dmul_rn(__ddiv_rn(__dadd_rn((double)j, 0.5), (double)c.H), 2.0)), c.half_h);
}
// np.linalg.norm of a 3-vector = sqrt(x.dot(x)) = sqrt(fma(z, z, fma(y, y, x * x)))
SPK_DEV double norm_dot(double x, double y, double z) {
  return __dsqrt_rn(__fma_rn(z, z, __fma_rn(y, y, __dmul_rn(x, x))));
}
// Camera.pixel_dir: (fwd + u * right) + v * up, / norm
SPK_DEV void pixel_dir(const CamDev& c, int i, int j, double* d) {
  const double u = u_of(c, i), v = v_of(c, j);
  double g[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) g[k] = __dadd_rn(__dadd_rn(c.fwd[k], __dmul_rn(u, c.right[k])), __dmul_rn(v, c.up[k]));
  const double n = norm_dot(g[0], g[1], g[2]);
#pragma unroll
  for (int k = 0; k < 3; ++k) d[k] = __ddiv_rn(g[k], n);
}
SPK_DEV double dist(const double* a, const double* b) {
  return norm_dot(__dsub_rn(a[0], b[0]), __dsub_rn(a[1], b[1]), __dsub_rn(a[2], b[2]));
}

// Frustum.front_widths along the split side (rays.py:203-209): t * max of
// the two corner-ray separations; python max(a, b) = b if b > a else a.
SPK_DEV double front_width(const CamDev& c, int4 r, double t, bool along_x) {
  double r00[3], r10[3], r01[3], r11[3];
  pixel_dir(c, r.x, r.w - 1, r00);
  pixel_dir(c, r.y - 1, r.w - 1, r10);
  pixel_dir(c, r.x, r.z, r01);
  pixel_dir(c, r.y - 1, r.z, r11);
  double a, b;
  if (along_x) {
    a = dist(r10, r00);
    b = dist(r11, r01);
  } else {
    a = dist(r01, r00);
    b = dist(r11, r10);
  }
  return __dmul_rn(t, b > a ? b : a);
}

// Camera.frustum_slab_box: per frame axis the hull of the 9 candidate
// weights (corners + zero-clamped midlines) at both parameter ends.
SPK_DEV void slab_box(const CamDev& c, int4 r, double t0, double t1, double* centre, double* axes) {
  const double u0 = u_of(c, r.x), u1 = u_of(c, r.y - 1);
  const double v0 = v_of(c, r.w - 1), v1 = v_of(c, r.z);
  const double mu = u0 > 0.0 ? u0 : 0.0, mv = v0 > 0.0 ? v0 : 0.0;  // python max(0.0, .)
  const double us[3] = {u0, u1, u1 < mu ? u1 : mu};                  // python min(., u1)
  const double vs[3] = {v0, v1, v1 < mv ? v1 : mv};
  double wmin[3] = {INFINITY, INFINITY, INFINITY}, wmax[3] = {-INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const double uu = us[b], vv = vs[a];
      const double ell = __dsqrt_rn(__dadd_rn(__dadd_rn(1.0, __dmul_rn(uu, uu)), __dmul_rn(vv, vv)));
      const double w[3] = {__ddiv_rn(1.0, ell), __ddiv_rn(uu, ell), __ddiv_rn(vv, ell)};
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        wmin[k] = fmin(wmin[k], w[k]);
        wmax[k] = fmax(wmax[k], w[k]);
      }
    }
  double mid[3], half[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double lo = fmin(__dmul_rn(t0, wmin[k]), __dmul_rn(t1, wmin[k]));
    const double hi = fmax(__dmul_rn(t0, wmax[k]), __dmul_rn(t1, wmax[k]));
    mid[k] = __dmul_rn(__dadd_rn(lo, hi), 0.5);   // (lo + hi) / 2, exact scaling
    half[k] = __dmul_rn(__dsub_rn(hi, lo), 0.5);
  }
#pragma unroll
  for (int q = 0; q < 3; ++q)
    centre[q] = __dadd_rn(__dadd_rn(__dadd_rn(c.pos[q], __dmul_rn(mid[0], c.fwd[q])), __dmul_rn(mid[1], c.right[q])),
                          __dmul_rn(mid[2], c.up[q]));
  const double* vec[3] = {c.fwd, c.right, c.up};
  int s = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k)
    if (half[k] > 0.0) {
#pragma unroll
      for (int q = 0; q < 3; ++q) axes[s * 3 + q] = __dmul_rn(half[k], vec[k][q]);
      ++s;
    }
  for (int rr = s; rr < 3; ++rr)
#pragma unroll
    for (int q = 0; q < 3; ++q) axes[rr * 3 + q] = 0.0;
}

SPK_DEV int npix(int4 r) { return (r.y - r.x) * (r.w - r.z); }

// ---- kernels ----------------------------------------------------------------

__global__ void frustum_seed_kernel(int gw, int gh, int bw, int bh, double sigma0, int4* rect, double* t,
                                    double* sig, uint8_t* dis) {
  const int q = blockIdx.x * FT + threadIdx.x;
  if (q >= gw * gh) return;
  const int by = q / gw, bx = q % gw;
  rect[q] = make_int4(bx * bw, (bx + 1) * bw, by * bh, (by + 1) * bh);
  t[q] = 0.0;
  sig[q] = sigma0;
  dis[q] = 0;
}

__global__ void frustum_image_init_kernel(long long npx, uint8_t* hit, double* t, double* steps, int all_hit) {
  const long long q = (long long)blockIdx.x * FT + threadIdx.x;
  if (q >= npx) return;
  hit[q] = all_hit ? 1 : 0;
  t[q] = all_hit ? 0.0 : INFINITY;
  steps[q] = 0.0;
}

struct Lists {
  // marching list (= next frontier) and its slab boxes
  int4* m_rect;
  double *m_t, *m_sig, *m_cen, *m_ax;
  uint8_t* m_dis;
  // single-pixel hand-offs
  int* p_pix;
  double *p_t, *p_sig;
  int* counters;  // [0] marching this round, [1] hand-offs so far, [2] dissolved so far
};

SPK_DEV void push_pending(const Lists& L, int W, int x, int y, double t, double sig) {
  const int k = atomicAdd(&L.counters[1], 1);
  L.p_pix[k] = y * W + x;
  L.p_t[k] = t;
  L.p_sig[k] = sig;
}

__global__ void __launch_bounds__(FT) frustum_expand_kernel(CamDev cam, FrustumParams P, int n_f,
                                                            const int4* __restrict__ f_rect,
                                                            const double* __restrict__ f_t,
                                                            const double* __restrict__ f_sig,
                                                            const uint8_t* __restrict__ f_dis, Lists L) {
  const int i = blockIdx.x * FT + threadIdx.x;
  if (i >= n_f) return;
  const int4 r0 = f_rect[i];
  const double t = f_t[i], sig = f_sig[i];
  if (f_dis[i]) {  // dissolved by the guard last round: every pixel hands off
    const int n = npix(r0), w = r0.y - r0.x;
    const int base = atomicAdd(&L.counters[1], n);
    for (int k = 0; k < n; ++k) {
      L.p_pix[base + k] = (r0.z + k / w) * cam.W + r0.x + k % w;
      L.p_t[base + k] = t;
      L.p_sig[base + k] = sig;
    }
    return;
  }
  if (npix(r0) == 1) {
    push_pending(L, cam.W, r0.x, r0.z, t, sig);
    return;
  }
  if (t >= P.t_max) return;  // certified empty to t_max: every pixel misses
  const double two_sig = __dmul_rn(2.0, sig);
  int4 stack[MAX_DFS];
  int sp = 0;
  stack[sp++] = r0;
  while (sp > 0) {
    const int4 r = stack[--sp];
    const int nx = r.y - r.x, ny = r.w - r.z;
    if (nx * ny == 1) {
      push_pending(L, cam.W, r.x, r.z, t, sig);
      continue;
    }
    const bool along_x = (nx >= ny && nx > 1) || ny == 1;
    if (front_width(cam, r, t, along_x) > two_sig && sp + 2 <= MAX_DFS) {
      if (along_x) {
        const int m = r.x + nx / 2;
        stack[sp++] = make_int4(r.x, m, r.z, r.w);
        stack[sp++] = make_int4(m, r.y, r.z, r.w);
      } else {
        const int m = r.z + ny / 2;
        stack[sp++] = make_int4(r.x, r.y, r.z, m);
        stack[sp++] = make_int4(r.x, r.y, m, r.w);
      }
      continue;
    }
    const int k = atomicAdd(&L.counters[0], 1);
    L.m_rect[k] = r;
    L.m_t[k] = t;
    L.m_sig[k] = sig;
    L.m_dis[k] = 0;
    slab_box(cam, r, t, __dadd_rn(t, sig), L.m_cen + 3ll * k, L.m_ax + 9ll * k);
  }
}

// one warp per marching frustum
__global__ void __launch_bounds__(FT) frustum_update_kernel(FrustumParams P, int W, int n_m, Lists L,
                                                            const double* __restrict__ lo,
                                                            const double* __restrict__ hi, double* steps) {
  const int w = (blockIdx.x * FT + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= n_m) return;
  const int4 r = L.m_rect[w];
  const int n = npix(r), rw = r.y - r.x;
  const double share = __ddiv_rn(1.0, (double)n);
  for (int k = lane; k < n; k += 32) {
    const long long p = (long long)(r.z + k / rw) * W + r.x + k % rw;
    steps[p] = __dadd_rn(steps[p], share);
  }
  if (lane == 0) {
    double t = L.m_t[w], sig = L.m_sig[w];
    if (lo[w] > 0.0 || hi[w] < 0.0) {
      const double adv = __dmul_rn(P.safety, sig);
      t = __dadd_rn(t, P.delta > adv ? P.delta : adv);
      sig = __dmul_rn(sig, P.eta_plus);
    } else {
      sig = __dmul_rn(sig, P.eta_minus);
      if (sig < P.sigma_floor) {
        L.m_dis[w] = 1;
        atomicAdd(&L.counters[2], 1);
      }
    }
    L.m_t[w] = t;
    L.m_sig[w] = sig;
  }
}

__global__ void frustum_handoff_dirs_kernel(CamDev cam, int n, const int* __restrict__ pix, double* dirs) {
  const int q = blockIdx.x * FT + threadIdx.x;
  if (q >= n) return;
  const int p = pix[q];
  pixel_dir(cam, p % cam.W, p / cam.W, dirs + 3ll * q);
}

__global__ void frustum_scatter_kernel(int n, const int* __restrict__ pix, const uint8_t* __restrict__ ph,
                                       const double* __restrict__ pt, const double* __restrict__ ps, uint8_t* hit,
                                       double* t, double* steps) {
  const int q = blockIdx.x * FT + threadIdx.x;
  if (q >= n) return;
  const int p = pix[q];
  hit[p] = ph[q];
  t[p] = pt[q];
  steps[p] = __dadd_rn(steps[p], ps[q]);
}

// stream-ordered scratch, freed (stream-ordered) on scope exit
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

}  // namespace
}  // namespace spk

using namespace spk;

extern "C" {

int spk_frustum_cast(const spk_net* net, int policy, int n_keep, int precision, const double* position3,
                     const double* frame9, double half_w, double half_h, int width, int height, int initial_grid,
                     const double* params6, uint8_t* hit, double* t_out, double* steps_out, int64_t* stats,
                     void* stream) {
  if (!net || !position3 || !frame9 || !params6 || !hit || !t_out || !steps_out)
    return fail(SPK_ERR_INVALID_PARAMETER, "null argument");
  if (net->input_dim != 3) return fail(SPK_ERR_DIMENSION, "ray casting needs a 3-d network");
  if (int rc = check_ray_params(params6)) return rc;
  if (width < 1 || height < 1 || initial_grid < 1) return fail(SPK_ERR_INVALID_PARAMETER, "bad resolution / grid");
  if ((long long)width * height > (long long)INT32_MAX)
    return fail(SPK_ERR_UNSUPPORTED_SHAPE, "image too large for one frustum cast");
  const int gw = std::min(initial_grid, width), gh = std::min(initial_grid, height);
  if (width % gw || height % gh)
    return fail(SPK_ERR_INVALID_PARAMETER, "resolution not divisible into the frustum grid");
  FrustumParams P{params6[0], params6[2], params6[3], params6[4], params6[5], params6[4] * 0x1p-32};
  const double sigma0 = params6[1];
  CamDev cam;
  for (int k = 0; k < 3; ++k) {
    cam.pos[k] = position3[k];
    cam.fwd[k] = frame9[k];
    cam.right[k] = frame9[3 + k];
    cam.up[k] = frame9[6 + k];
  }
  cam.half_w = half_w;
  cam.half_h = half_h;
  cam.W = width;
  cam.H = height;
  DeviceGuard g(net->device);
  cudaStream_t st = (cudaStream_t)stream;
  const long long npx = (long long)width * height;
  const int pblk = (int)((npx + FT - 1) / FT);
  const long long cap_m = std::max<long long>(npx / 2, gw * gh);  // marching frusta hold >= 2 pixels

  Scratch S(st);
  double* pos_d = S.get<double>(24);
  double* f0_d = S.get<double>(8);
  int* counters = S.get<int>(16);
  // two frustum lists (frontier <-> marching), slab boxes, bounds
  int4* rect[2] = {S.get<int4>(cap_m * 16), S.get<int4>(cap_m * 16)};
  double* ft[2] = {S.get<double>(cap_m * 8), S.get<double>(cap_m * 8)};
  double* fs[2] = {S.get<double>(cap_m * 8), S.get<double>(cap_m * 8)};
  uint8_t* fd[2] = {S.get<uint8_t>(cap_m), S.get<uint8_t>(cap_m)};
  double* cen = S.get<double>(cap_m * 24);
  double* ax = S.get<double>(cap_m * 72);
  double* blo = S.get<double>(cap_m * 8);
  double* bhi = S.get<double>(cap_m * 8);
  int* p_pix = S.get<int>(npx * 4);
  double* p_t = S.get<double>(npx * 8);
  double* p_sig = S.get<double>(npx * 8);
  if (S.err != cudaSuccess) return cuda_fail(S.err, "frustum alloc");

  int hc[3] = {0, 0, 0};
  double f0 = 0.0;
  cudaError_t e = cudaMemcpyAsync(pos_d, cam.pos, 24, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "frustum upload");
  int rc = spk_eval_batch(net, precision, 1, pos_d, f0_d, st);
  if (rc != SPK_OK) return rc;
  if ((e = cudaMemcpyAsync(&f0, f0_d, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess)
    return cuda_fail(e, "frustum f0");
  frustum_image_init_kernel<<<pblk, FT, 0, st>>>(npx, hit, t_out, steps_out, f0 == 0.0 ? 1 : 0);
  if (f0 == 0.0) {  // camera on the surface: every pixel hits at t = 0
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "frustum init");
    if (stats) stats[0] = stats[1] = stats[2] = stats[3] = stats[4] = 0;
    return SPK_OK;
  }
  cudaMemsetAsync(counters, 0, 16, st);
  frustum_seed_kernel<<<(gw * gh + FT - 1) / FT, FT, 0, st>>>(gw, gh, width / gw, height / gh, sigma0, rect[0],
                                                               ft[0], fs[0], fd[0]);
  int n_f = gw * gh, cur = 0;
  int64_t rounds = 0, frustum_steps = 0;
  while (n_f > 0) {
    const int nxt = cur ^ 1;
    Lists L{rect[nxt], ft[nxt], fs[nxt], cen, ax, fd[nxt], p_pix, p_t, p_sig, counters};
    cudaMemsetAsync(counters, 0, 4, st);
    frustum_expand_kernel<<<(n_f + FT - 1) / FT, FT, 0, st>>>(cam, P, n_f, rect[cur], ft[cur], fs[cur], fd[cur], L);
    if ((e = cudaMemcpyAsync(hc, counters, 12, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess)
      return cuda_fail(e, "frustum expand");
    const int n_m = hc[0];
    if (n_m == 0) break;
    rc = spk_bound_batch(net, policy, n_keep, precision, n_m, 3, cen, ax, blo, bhi, nullptr, st);
    if (rc != SPK_OK) return rc;
    frustum_update_kernel<<<(int)(((long long)n_m * 32 + FT - 1) / FT), FT, 0, st>>>(P, width, n_m, L, blo, bhi,
                                                                                      steps_out);
    ++rounds;
    frustum_steps += n_m;
    n_f = n_m;
    cur = nxt;
  }
  if ((e = cudaMemcpyAsync(hc, counters, 12, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess)
    return cuda_fail(e, "frustum rounds");
  const int np = hc[1];
  int64_t ray_steps = 0;
  if (np > 0) {
    Scratch T(st);
    double* dirs = T.get<double>((size_t)np * 24);
    uint8_t* ph = T.get<uint8_t>(np);
    double* pt = T.get<double>((size_t)np * 8);
    double* ps = T.get<double>((size_t)np * 8);
    if (T.err != cudaSuccess) return cuda_fail(T.err, "frustum hand-off alloc");
    frustum_handoff_dirs_kernel<<<(np + FT - 1) / FT, FT, 0, st>>>(cam, np, p_pix, dirs);
    int64_t ms[3] = {0, 0, 0};
    rc = spk_march(net, policy, n_keep, precision, np, pos_d, 0, dirs, p_t, p_sig, params6, ph, pt, ps, ms, st);
    if (rc != SPK_OK) return rc;
    ray_steps = ms[1];
    frustum_scatter_kernel<<<(np + FT - 1) / FT, FT, 0, st>>>(np, p_pix, ph, pt, ps, hit, t_out, steps_out);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "frustum kernels");
  if (stats) {
    stats[0] = rounds;         // frustum rounds
    stats[1] = frustum_steps;  // frustum steps (slab bounds)
    stats[2] = np;             // single-pixel hand-offs
    stats[3] = ray_steps;      // their ray steps
    stats[4] = hc[2];          // frusta dissolved by the sigma floor
  }
  return SPK_OK;
}

}  // extern "C"
