// §8(f1): frustum range-marching over a camera's pixel grid
// (cast_frustum_image, rays.py:232-341; camera.py:99-135).
//
// Rectangles of pixels march as one oriented slab box per step: while the
// frustum's front face (world width at parameter t along its longer pixel
// side) stays within 2 sigma, one bound of the slab between t and t+sigma
// certifies (or refuses) the step for every contained pixel ray at once;
// wider frusta split in half across that side.  Single-pixel frusta are
// handed to the device ray march (spk_march, K6) with their (t, sigma).
//
// Split: the host drives the bookkeeping (it is O(frusta) integer/FP64
// scalar work and the frustum count is a few thousand at most), the GPU
// does every network pass: one batched slab-box bound per round through
// spk_bound_batch (the fused affine kernels, s <= 3) and the per-pixel
// finish through spk_march.  All scalar geometry is FP64 with
// round-to-nearest in numpy's operation order -- no contraction, and the
// 3-vector norm as numpy's dot (an FMA chain) -- so with FP64 bounds the
// frustum sequence, the hand-off (t, sigma) and the amortised step counts
// are bit-identical to the reference's.
#include <algorithm>
#include <cmath>
#include <vector>

#include "spk_abi_internal.h"

namespace spk {
namespace {

constexpr int FT = 256;

// ---- camera geometry (camera.py:68-92, 99-135) -----------------------------

struct PinholeGrid {
  double pos[3], fwd[3], right[3], up[3];
  double half_w, half_h;
  int W, H;

  double u(int i) const { return (((double)i + 0.5) / W * 2.0 - 1.0) * half_w; }
  double v(int j) const { return (1.0 - ((double)j + 0.5) / H * 2.0) * half_h; }

  // numpy 1-D dot(x, x): fma(x2, x2, fma(x1, x1, x0 * x0))
  static double norm3(const double* x) {
    const double sq = x[0] * x[0];
    return std::sqrt(std::fma(x[2], x[2], std::fma(x[1], x[1], sq)));
  }

  void dir(int i, int j, double* d) const {
    const double uu = u(i), vv = v(j);
    double g[3];
    for (int k = 0; k < 3; ++k) {
      const double a = uu * right[k];
      const double b = vv * up[k];
      const double s = fwd[k] + a;
      g[k] = s + b;
    }
    const double n = norm3(g);
    for (int k = 0; k < 3; ++k) d[k] = g[k] / n;
  }

  // oriented box holding every pixel-centre ray of [px0,px1) x [py0,py1)
  // over [t0, t1]: per frame axis, the hull of the 9 candidate weights
  // (corners + zero-clamped midlines) at both parameter ends.  Returns s.
  int slab(int px0, int px1, int py0, int py1, double t0, double t1, double* centre, double* axes) const {
    const double u0 = u(px0), u1 = u(px1 - 1);
    const double v0 = v(py1 - 1), v1 = v(py0);
    auto clamp0 = [](double a, double b) {
      const double m = a > 0.0 ? a : 0.0;  // python max(0.0, a)
      return b < m ? b : m;                // python min(m, b)
    };
    const double us[3] = {u0, u1, clamp0(u0, u1)};
    const double vs[3] = {v0, v1, clamp0(v0, v1)};
    double wmin[3] = {INFINITY, INFINITY, INFINITY}, wmax[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (double vv : vs)
      for (double uu : us) {
        const double a = 1.0 + uu * uu;
        const double ell = std::sqrt(a + vv * vv);
        const double w[3] = {1.0 / ell, uu / ell, vv / ell};
        for (int k = 0; k < 3; ++k) {
          wmin[k] = std::min(wmin[k], w[k]);
          wmax[k] = std::max(wmax[k], w[k]);
        }
      }
    double mid[3], half[3];
    for (int k = 0; k < 3; ++k) {
      const double lo = std::min(t0 * wmin[k], t1 * wmin[k]);
      const double hi = std::max(t0 * wmax[k], t1 * wmax[k]);
      mid[k] = (lo + hi) / 2.0;
      half[k] = (hi - lo) / 2.0;
    }
    for (int c = 0; c < 3; ++c) {
      const double a = mid[0] * fwd[c];
      const double b = mid[1] * right[c];
      const double d = mid[2] * up[c];
      double x = pos[c] + a;
      x = x + b;
      centre[c] = x + d;
    }
    const double* vec[3] = {fwd, right, up};
    int s = 0;
    for (int k = 0; k < 3; ++k)
      if (half[k] > 0.0) {
        for (int c = 0; c < 3; ++c) axes[s * 3 + c] = half[k] * vec[k][c];
        ++s;
      }
    for (int r = s; r < 3; ++r)
      for (int c = 0; c < 3; ++c) axes[r * 3 + c] = 0.0;
    return s;
  }
};

struct Frustum {
  int px0, px1, py0, py1;
  double t, sigma;
  int n_pixels() const { return (px1 - px0) * (py1 - py0); }
};

static double dist3(const double* a, const double* b) {
  const double d[3] = {a[0] - b[0], a[1] - b[1], a[2] - b[2]};
  return PinholeGrid::norm3(d);
}

// ---- device side: image initialisation and the single-pixel scatter -------

__global__ void frustum_init_kernel(long long npix, const double* __restrict__ steps_host_img, uint8_t* hit,
                                    double* t, double* steps, int all_hit) {
  const long long q = (long long)blockIdx.x * FT + threadIdx.x;
  if (q >= npix) return;
  hit[q] = all_hit ? 1 : 0;
  t[q] = all_hit ? 0.0 : INFINITY;
  steps[q] = steps_host_img ? steps_host_img[q] : 0.0;
}

__global__ void frustum_scatter_kernel(int n, const int* __restrict__ pix, const uint8_t* __restrict__ ph,
                                       const double* __restrict__ pt, const double* __restrict__ ps, uint8_t* hit,
                                       double* t, double* steps) {
  const int q = blockIdx.x * FT + threadIdx.x;
  if (q >= n) return;
  const int p = pix[q];
  hit[p] = ph[q];
  t[p] = pt[q];
  steps[p] += ps[q];
}

// grow-only scratch: pinned host staging + stream-ordered device buffers
struct Staging {
  cudaStream_t st;
  std::vector<void*> host, dev;
  explicit Staging(cudaStream_t s) : st(s) {}
  ~Staging() {
    for (void* p : dev) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
    for (void* p : host) cudaFreeHost(p);
  }
  cudaError_t h(void** p, size_t bytes) {
    cudaError_t e = cudaMallocHost(p, std::max<size_t>(bytes, 16));
    if (e == cudaSuccess) host.push_back(*p);
    return e;
  }
  cudaError_t d(void** p, size_t bytes) {
    cudaError_t e = cudaMallocAsync(p, std::max<size_t>(bytes, 16), st);
    if (e == cudaSuccess) dev.push_back(*p);
    return e;
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
  if (width < 1 || height < 1 || initial_grid < 1) return fail(SPK_ERR_INVALID_PARAMETER, "bad resolution / grid");
  const int gw = std::min(initial_grid, width), gh = std::min(initial_grid, height);
  if (width % gw || height % gh)
    return fail(SPK_ERR_INVALID_PARAMETER, "resolution not divisible into the frustum grid");
  const double t_max = params6[0], sigma0 = params6[1], eta_plus = params6[2], eta_minus = params6[3],
               delta = params6[4], safety = params6[5];
  DeviceGuard g(net->device);
  cudaStream_t st = (cudaStream_t)stream;
  PinholeGrid cam;
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
  const long long npix = (long long)width * height;
  const int pblk = (int)((npix + FT - 1) / FT);
  Staging S(st);
  int64_t st_rounds = 0, st_frusta = 0, st_pending = 0, st_ray_steps = 0;

  // f(camera position): exactly zero -> every pixel hits at t = 0
  double *pos_d = nullptr, *f0_d = nullptr, *f0_h = nullptr;
  cudaError_t e = S.d((void**)&pos_d, 24);
  if (e == cudaSuccess) e = S.d((void**)&f0_d, 8);
  if (e == cudaSuccess) e = S.h((void**)&f0_h, 8);
  if (e == cudaSuccess) e = cudaMemcpyAsync(pos_d, cam.pos, 24, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "frustum alloc");
  int rc = spk_eval_batch(net, precision, 1, pos_d, f0_d, st);
  if (rc != SPK_OK) return rc;
  if ((e = cudaMemcpyAsync(f0_h, f0_d, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess)
    return cuda_fail(e, "frustum f0");
  if (*f0_h == 0.0) {
    frustum_init_kernel<<<pblk, FT, 0, st>>>(npix, nullptr, hit, t_out, steps_out, 1);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "frustum init");
    if (stats) stats[0] = stats[1] = stats[2] = stats[3] = 0;
    return SPK_OK;
  }

  std::vector<double> steps_img((size_t)npix, 0.0);
  std::vector<Frustum> frontier, stack, marching, pending;
  const int bw = width / gw, bh = height / gh;
  for (int by = 0; by < gh; ++by)
    for (int bx = 0; bx < gw; ++bx)
      frontier.push_back({bx * bw, (bx + 1) * bw, by * bh, (by + 1) * bh, 0.0, sigma0});

  // per-round buffers, grown on demand
  size_t cap = 0;
  double *cen_h = nullptr, *ax_h = nullptr, *lo_h = nullptr, *hi_h = nullptr;
  double *cen_d = nullptr, *ax_d = nullptr, *lo_d = nullptr, *hi_d = nullptr;
  std::vector<double> cen_tmp, ax_tmp;
  while (!frontier.empty()) {
    marching.clear();
    stack.swap(frontier);
    frontier.clear();
    while (!stack.empty()) {
      Frustum f = stack.back();
      stack.pop_back();
      if (f.n_pixels() == 1) {
        pending.push_back(f);
        continue;
      }
      if (f.t >= t_max) continue;  // certified empty to t_max: miss
      const int nx = f.px1 - f.px0, ny = f.py1 - f.py0;
      const bool along_x = (nx >= ny && nx > 1) || ny == 1;
      double r00[3], r10[3], r01[3], r11[3];
      cam.dir(f.px0, f.py1 - 1, r00);
      cam.dir(f.px1 - 1, f.py1 - 1, r10);
      cam.dir(f.px0, f.py0, r01);
      cam.dir(f.px1 - 1, f.py0, r11);
      double a, b;
      if (along_x) {
        a = dist3(r10, r00);
        b = dist3(r11, r01);
      } else {
        a = dist3(r01, r00);
        b = dist3(r11, r10);
      }
      const double wfront = f.t * (b > a ? b : a);
      if (wfront > 2.0 * f.sigma) {
        if (along_x) {
          const int m = f.px0 + nx / 2;
          stack.push_back({f.px0, m, f.py0, f.py1, f.t, f.sigma});
          stack.push_back({m, f.px1, f.py0, f.py1, f.t, f.sigma});
        } else {
          const int m = f.py0 + ny / 2;
          stack.push_back({f.px0, f.px1, f.py0, m, f.t, f.sigma});
          stack.push_back({f.px0, f.px1, m, f.py1, f.t, f.sigma});
        }
        continue;
      }
      marching.push_back(f);
    }
    if (marching.empty()) break;
    const size_t n = marching.size();
    if (n > cap) {
      const size_t nc = std::max(n, cap * 2);
      if ((e = S.h((void**)&cen_h, nc * 24)) != cudaSuccess || (e = S.h((void**)&ax_h, nc * 72)) != cudaSuccess ||
          (e = S.h((void**)&lo_h, nc * 8)) != cudaSuccess || (e = S.h((void**)&hi_h, nc * 8)) != cudaSuccess ||
          (e = S.d((void**)&cen_d, nc * 24)) != cudaSuccess || (e = S.d((void**)&ax_d, nc * 72)) != cudaSuccess ||
          (e = S.d((void**)&lo_d, nc * 8)) != cudaSuccess || (e = S.d((void**)&hi_d, nc * 8)) != cudaSuccess)
        return cuda_fail(e, "frustum alloc");
      cap = nc;
    }
    // slab boxes; s = the batch's widest slab (rows beyond a box's own s are zero)
    int s_max = 0;
    cen_tmp.resize(n * 3);
    ax_tmp.resize(n * 9);
    for (size_t i = 0; i < n; ++i) {
      const Frustum& f = marching[i];
      const int s = cam.slab(f.px0, f.px1, f.py0, f.py1, f.t, f.t + f.sigma, &cen_tmp[i * 3], &ax_tmp[i * 9]);
      s_max = std::max(s_max, s);
    }
    const int s = std::max(s_max, 1);
    std::copy(cen_tmp.begin(), cen_tmp.end(), cen_h);
    for (size_t i = 0; i < n; ++i) std::copy(&ax_tmp[i * 9], &ax_tmp[i * 9] + s * 3, ax_h + i * s * 3);
    if ((e = cudaMemcpyAsync(cen_d, cen_h, n * 24, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(ax_d, ax_h, n * s * 24, cudaMemcpyHostToDevice, st)) != cudaSuccess)
      return cuda_fail(e, "frustum upload");
    rc = spk_bound_batch(net, policy, n_keep, precision, (int64_t)n, s, cen_d, ax_d, lo_d, hi_d, nullptr, st);
    if (rc != SPK_OK) return rc;
    if ((e = cudaMemcpyAsync(lo_h, lo_d, n * 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(hi_h, hi_d, n * 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess)
      return cuda_fail(e, "frustum bounds");
    ++st_rounds;
    st_frusta += (int64_t)n;
    for (size_t i = 0; i < n; ++i) {
      Frustum f = marching[i];
      const double share = 1.0 / f.n_pixels();
      for (int y = f.py0; y < f.py1; ++y)
        for (int x = f.px0; x < f.px1; ++x) steps_img[(size_t)y * width + x] += share;
      if (lo_h[i] > 0.0 || hi_h[i] < 0.0) {
        const double adv = safety * f.sigma;
        f.t += delta > adv ? delta : adv;
        f.sigma *= eta_plus;
      } else {
        f.sigma *= eta_minus;
      }
      frontier.push_back(f);
    }
  }

  // images: steps so far, then the single-pixel finishes scattered on top
  double* steps_img_d = nullptr;
  if ((e = S.d((void**)&steps_img_d, (size_t)npix * 8)) != cudaSuccess ||
      (e = cudaMemcpyAsync(steps_img_d, steps_img.data(), (size_t)npix * 8, cudaMemcpyHostToDevice, st)) !=
          cudaSuccess)
    return cuda_fail(e, "frustum steps");
  frustum_init_kernel<<<pblk, FT, 0, st>>>(npix, steps_img_d, hit, t_out, steps_out, 0);
  const int np = (int)pending.size();
  st_pending = np;
  if (np > 0) {
    std::vector<double> dirs((size_t)np * 3), t0(np), s0(np);
    std::vector<int> pix(np);
    for (int i = 0; i < np; ++i) {
      const Frustum& f = pending[i];
      cam.dir(f.px0, f.py0, &dirs[(size_t)i * 3]);
      t0[i] = f.t;
      s0[i] = f.sigma;
      pix[i] = f.py0 * width + f.px0;
    }
    double *dirs_d, *t0_d, *s0_d, *pt_d, *ps_d;
    uint8_t* ph_d;
    int* pix_d;
    if ((e = S.d((void**)&dirs_d, (size_t)np * 24)) != cudaSuccess || (e = S.d((void**)&t0_d, np * 8ull)) != cudaSuccess ||
        (e = S.d((void**)&s0_d, np * 8ull)) != cudaSuccess || (e = S.d((void**)&pt_d, np * 8ull)) != cudaSuccess ||
        (e = S.d((void**)&ps_d, np * 8ull)) != cudaSuccess || (e = S.d((void**)&ph_d, np)) != cudaSuccess ||
        (e = S.d((void**)&pix_d, np * 4ull)) != cudaSuccess)
      return cuda_fail(e, "frustum pending alloc");
    if ((e = cudaMemcpyAsync(dirs_d, dirs.data(), (size_t)np * 24, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(t0_d, t0.data(), np * 8ull, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(s0_d, s0.data(), np * 8ull, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(pix_d, pix.data(), np * 4ull, cudaMemcpyHostToDevice, st)) != cudaSuccess)
      return cuda_fail(e, "frustum pending upload");
    int64_t ms[3] = {0, 0, 0};
    rc = spk_march(net, policy, n_keep, precision, np, pos_d, 0, dirs_d, t0_d, s0_d, params6, ph_d, pt_d, ps_d, ms,
                   st);
    if (rc != SPK_OK) return rc;
    st_ray_steps = ms[1];
    frustum_scatter_kernel<<<(np + FT - 1) / FT, FT, 0, st>>>(np, pix_d, ph_d, pt_d, ps_d, hit, t_out, steps_out);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "frustum kernels");
  if (stats) {
    stats[0] = st_rounds;     // frustum rounds
    stats[1] = st_frusta;     // frustum steps (slab bounds)
    stats[2] = st_pending;    // single-pixel hand-offs
    stats[3] = st_ray_steps;  // their ray steps
  }
  return SPK_OK;  // Staging's destructor syncs the stream before freeing host staging
}

}  // extern "C"
