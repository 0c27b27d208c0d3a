// §8(f3): volumetric queries on the bound kernels (spatial.py:292-684).
//
//   spk_certified_radii  _certified_radii (spatial.py:318-343): for many
//                        points at once, the largest cube half-extent
//                        r_start / 2^j >= floor whose bound is sign-definite
//                        (empty_box_radius for one point, walk_on_spheres'
//                        inner query, the paper's empty-box queries).  Device
//                        loop: one fused bound pass over the undecided points'
//                        cubes per halving round, survivors compacted.
//   spk_intersect        test_intersection (spatial.py:544-588): simultaneous
//                        breadth-first subdivision under two networks.  A
//                        level = one bound pass per network, an ordered
//                        ballot/prefix classification (survive / witness /
//                        tiny / split) and the reference's child layout
//                        [low halves ; high halves].
//   spk_bisect           batched segment bisection between opposite-sign
//                        points (closest_point's surface witness,
//                        spatial.py:631-638), sync-free: iters x (midpoint,
//                        point pass, side update).
// All geometry is FP64 in the reference's operation order.
#include <algorithm>
#include <cmath>
#include <vector>

#include "spk_abi_internal.h"

namespace spk {
namespace {

constexpr int QT = 256;

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

// rank of pred among the block's flagged threads (ballot prefix), block total in *total
SPK_DEV int block_rank(bool pred, int* total) {
  __shared__ int wcount[QT / 32];
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) wcount[w] = __popc(m);
  __syncthreads();
  int before = 0, all = 0;
  for (int q = 0; q < QT / 32; ++q) {
    if (q < w) before += wcount[q];
    all += wcount[q];
  }
  __syncthreads();
  *total = all;
  return before + __popc(m & ((1u << lane) - 1u));
}

// unordered append with one atomic per block
SPK_DEV long long block_append(bool pred, unsigned long long* counter, int* rank) {
  __shared__ long long base;
  int tot;
  *rank = block_rank(pred, &tot);
  if (threadIdx.x == 0) base = tot ? (long long)atomicAdd(counter, (unsigned long long)tot) : 0;
  __syncthreads();
  return base;
}

// ---- certified radii -----------------------------------------------------------

__global__ void radii_init_kernel(long long n, const double* __restrict__ r_start, double floor_r, double* r,
                                  double* radii, int* idx, unsigned long long* count) {
  const long long i = (long long)blockIdx.x * QT + threadIdx.x;
  const bool live = i < n && r_start[i] >= floor_r;
  if (i < n) {
    r[i] = r_start[i];
    radii[i] = 0.0;
  }
  int rk;
  const long long base = block_append(live, count, &rk);
  if (live) idx[base + rk] = (int)i;
}

// cube of half-extent r centred on the point: centre p, axes diag(r)
// (spatial.py:330-333)
__global__ void radii_boxes_kernel(long long cap, const unsigned long long* __restrict__ na, int d,
                                   const int* __restrict__ idx, const double* __restrict__ pts,
                                   const double* __restrict__ r, double* centres, double* axes) {
  const long long q = (long long)blockIdx.x * QT + threadIdx.x;
  if (q >= (long long)*na || q >= cap) return;
  const long long i = idx[q];
  for (int k = 0; k < d; ++k) {
    centres[q * d + k] = pts[i * d + k];
    for (int j = 0; j < d; ++j) axes[(q * d + j) * d + k] = j == k ? r[i] : 0.0;
  }
}

__global__ void radii_update_kernel(long long cap, const unsigned long long* __restrict__ na,
                                    const int* __restrict__ idx, const double* __restrict__ lo,
                                    const double* __restrict__ hi, double floor_r, double* r, double* radii,
                                    int* nxt, unsigned long long* n_next) {
  const long long q = (long long)blockIdx.x * QT + threadIdx.x;
  bool keep = false;
  long long i = 0;
  if (q < (long long)*na && q < cap) {
    i = idx[q];
    if (lo[q] > 0.0 || hi[q] < 0.0) {
      radii[i] = r[i];
    } else {
      const double h = r[i] / 2.0;
      r[i] = h;
      keep = h >= floor_r;  // below the floor: radius stays 0
    }
  }
  int rk;
  const long long base = block_append(keep, n_next, &rk);
  if (keep) nxt[base + rk] = (int)i;
}

// ---- intersection ------------------------------------------------------------------

// per-node flags: bit0 survive, bit1 witness, 2 = tiny (inconclusive), 4 = split
__global__ void isect_mark_kernel(long long n, int d, const double* __restrict__ lo, const double* __restrict__ hi,
                                  const double* __restrict__ loa, const double* __restrict__ hia,
                                  const double* __restrict__ lob, const double* __restrict__ hib, double stop,
                                  uint8_t* flag, int* bsplit, int* btiny, unsigned long long* witness) {
  const long long i = (long long)blockIdx.x * QT + threadIdx.x;
  bool split = false, tiny = false;
  if (i < n) {
    const bool survive = loa[i] <= 0.0 && lob[i] <= 0.0;
    if (survive && hia[i] < 0.0 && hib[i] < 0.0) atomicMin(witness, (unsigned long long)i);
    double ext = 0.0;
    for (int k = 0; k < d; ++k) ext = fmax(ext, hi[i * d + k] - lo[i * d + k]);  // np.max of extents
    tiny = survive && ext < stop;
    split = survive && !tiny;
    flag[i] = (uint8_t)(split ? 4 : (tiny ? 2 : 0));
  }
  int ts, tt;
  block_rank(split, &ts);
  block_rank(tiny, &tt);
  if (threadIdx.x == 0) {
    bsplit[blockIdx.x] = ts;
    btiny[blockIdx.x] = tt;
  }
}

// exclusive scan of per-block counts (single block, sequential chunks)
__global__ void block_scan_kernel(int nblk, const int* __restrict__ in, long long* __restrict__ out,
                                  long long* __restrict__ total) {
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nblk; b0 += QT) {
    const int b = b0 + threadIdx.x;
    const long long v = b < nblk ? in[b] : 0;
    // inclusive warp scan + cross-warp
    long long x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    __shared__ long long wsum[QT / 32];
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    long long before = 0;
    for (int q = 0; q < w; ++q) before += wsum[q];
    if (b < nblk) out[b] = carry + before + x - v;
    __syncthreads();
    if (threadIdx.x == QT - 1) carry += before + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void isect_scatter_kernel(long long n, int d, const double* __restrict__ lo, const double* __restrict__ hi,
                                     const uint8_t* __restrict__ flag, const long long* __restrict__ off_split,
                                     const long long* __restrict__ off_tiny, const long long* __restrict__ k_total,
                                     double* child_lo, double* child_hi, double* tiny_lo, double* tiny_hi) {
  const long long i = (long long)blockIdx.x * QT + threadIdx.x;
  const uint8_t f = i < n ? flag[i] : 0;
  int tot;
  const int rs = block_rank(f == 4, &tot);
  const int rt = block_rank(f == 2, &tot);
  if (f == 2) {
    const long long j = off_tiny[blockIdx.x] + rt;
    for (int k = 0; k < d; ++k) {
      tiny_lo[j * d + k] = lo[i * d + k];
      tiny_hi[j * d + k] = hi[i * d + k];
    }
  }
  if (f != 4) return;
  const long long j = off_split[blockIdx.x] + rs, K = *k_total;
  // widest axis, ties to the lowest index; FP64 midpoint (spatial.py:189-199)
  int ax = 0;
  double best = -1.0;
  for (int k = 0; k < d; ++k) {
    const double e = hi[i * d + k] - lo[i * d + k];
    if (e > best) {
      best = e;
      ax = k;
    }
  }
  const double mid = 0.5 * (lo[i * d + ax] + hi[i * d + ax]);
  for (int k = 0; k < d; ++k) {
    const double l = lo[i * d + k], h = hi[i * d + k];
    child_lo[j * d + k] = l;
    child_hi[j * d + k] = k == ax ? mid : h;
    child_lo[(K + j) * d + k] = k == ax ? mid : l;
    child_hi[(K + j) * d + k] = h;
  }
}

// ---- bisection ------------------------------------------------------------------------

__global__ void bisect_mid_kernel(long long n, int d, const double* __restrict__ a, const double* __restrict__ b,
                                  double* mid) {
  const long long q = (long long)blockIdx.x * QT + threadIdx.x;
  if (q >= n * d) return;
  mid[q] = 0.5 * (a[q] + b[q]);
}

__global__ void bisect_update_kernel(long long n, int d, const double* __restrict__ fm, const double* __restrict__ mid,
                                     double* a, double* b) {
  const long long q = (long long)blockIdx.x * QT + threadIdx.x;
  if (q >= n * d) return;
  if (fm[q / d] < 0.0)
    a[q] = mid[q];
  else
    b[q] = mid[q];
}

}  // namespace
}  // namespace spk

using namespace spk;

extern "C" {

int spk_certified_radii(const spk_net* net, int policy, int n_keep, int precision, int64_t n, const double* points,
                        const double* r_start, double floor_r, double* radii, int64_t* stats, void* stream) {
  if (!net || (n > 0 && (!points || !r_start || !radii))) return fail(SPK_ERR_INVALID_PARAMETER, "null argument");
  if (n < 0) return fail(SPK_ERR_DIMENSION, "negative point count");
  if (n > (int64_t)INT32_MAX) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "too many points in one call");
  const int d = net->input_dim;
  if (d > MAX_AXES) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "certified radii support d <= 8");
  if (!(floor_r > 0.0)) return fail(SPK_ERR_INVALID_PARAMETER, "floor must be positive");
  if (stats) stats[0] = stats[1] = 0;
  if (n == 0) return SPK_OK;
  DeviceGuard g(net->device);
  cudaStream_t st = (cudaStream_t)stream;
  Scratch S(st);
  double* r = S.get<double>(n * 8);
  int* ia = S.get<int>(n * 4);
  int* ib = S.get<int>(n * 4);
  unsigned long long* cnt = S.get<unsigned long long>(16);
  double* cen = S.get<double>(n * d * 8);
  double* ax = S.get<double>(n * d * d * 8);
  double* blo = S.get<double>(n * 8);
  double* bhi = S.get<double>(n * 8);
  if (S.err != cudaSuccess) return cuda_fail(S.err, "radii alloc");
  const int blk = (int)((n + QT - 1) / QT);
  cudaMemsetAsync(cnt, 0, 16, st);
  radii_init_kernel<<<blk, QT, 0, st>>>(n, r_start, floor_r, r, radii, ia, cnt);
  unsigned long long na = 0;
  cudaError_t e = cudaMemcpyAsync(&na, cnt, 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "radii init");
  int* cur = ia;
  int* nxt = ib;
  unsigned long long* ncur = cnt;
  unsigned long long* nnext = cnt + 1;
  int64_t rounds = 0, bounds = 0;
  while (na > 0) {
    const int ab = (int)((na + QT - 1) / QT);
    radii_boxes_kernel<<<ab, QT, 0, st>>>((long long)na, ncur, d, cur, points, r, cen, ax);
    int rc = spk_bound_batch(net, policy, n_keep, precision, (int64_t)na, d, cen, ax, blo, bhi, nullptr, st);
    if (rc != SPK_OK) return rc;
    cudaMemsetAsync(nnext, 0, 8, st);
    radii_update_kernel<<<ab, QT, 0, st>>>((long long)na, ncur, cur, blo, bhi, floor_r, r, radii, nxt, nnext);
    bounds += (int64_t)na;
    ++rounds;
    e = cudaMemcpyAsync(&na, nnext, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "radii round");
    std::swap(cur, nxt);
    std::swap(ncur, nnext);
  }
  if (stats) {
    stats[0] = rounds;
    stats[1] = bounds;
  }
  e = cudaGetLastError();
  return e == cudaSuccess ? SPK_OK : cuda_fail(e, "radii kernels");
}

int spk_intersect(const spk_net* net_a, const spk_net* net_b, int policy, int n_keep, int precision,
                  const double* lo_root, const double* hi_root, double delta, int* kind, double* witness_lo,
                  double* witness_hi, int64_t* n_nodes, double* nodes_lo, double* nodes_hi, int64_t nodes_cap,
                  int64_t* stats, void* stream) {
  if (!net_a || !net_b || !lo_root || !hi_root || !kind || !n_nodes)
    return fail(SPK_ERR_INVALID_PARAMETER, "null argument");
  const int d = net_a->input_dim;
  if (net_b->input_dim != d) return fail(SPK_ERR_DIMENSION, "networks of different input dimension");
  if (d > MAX_AXES) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "intersection supports d <= 8");
  if (net_a->device != net_b->device) return fail(SPK_ERR_INVALID_PARAMETER, "networks on different devices");
  if (!(delta > 0.0)) return fail(SPK_ERR_INVALID_PARAMETER, "delta must be positive");
  DeviceGuard g(net_a->device);
  cudaStream_t st = (cudaStream_t)stream;
  const double stop = delta / std::sqrt((double)d);
  *kind = 0;
  *n_nodes = 0;
  Scratch S(st);
  long long* tot = S.get<long long>(16);
  unsigned long long* wit = S.get<unsigned long long>(8);
  // buffers grow with the frontier (stream-ordered pool; old blocks are
  // released with the scratch at the end)
  long long n = 1, capL = 0, capF = 1, capC = 0;
  double* flo = S.get<double>(d * 8);
  double* fhi = S.get<double>(d * 8);
  double *clo = nullptr, *chi = nullptr, *tlo = nullptr, *thi = nullptr;
  double *loa = nullptr, *hia = nullptr, *lob = nullptr, *hib = nullptr;
  uint8_t* flag = nullptr;
  int *bsplit = nullptr, *btiny = nullptr;
  long long *osplit = nullptr, *otiny = nullptr;
  if (S.err != cudaSuccess) return cuda_fail(S.err, "intersect alloc");
  cudaMemcpyAsync(flo, lo_root, d * 8, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(fhi, hi_root, d * 8, cudaMemcpyHostToDevice, st);
  std::vector<double> hlo, hhi;
  int64_t levels = 0, bounds = 0;
  int rc = SPK_OK;
  while (n > 0) {
    if (n > capL) {  // per-node level arrays
      const long long nc = std::max<long long>(n, 2 * capL);
      const long long nb = (nc + QT - 1) / QT;
      tlo = S.get<double>(nc * d * 8);
      thi = S.get<double>(nc * d * 8);
      loa = S.get<double>(nc * 8);
      hia = S.get<double>(nc * 8);
      lob = S.get<double>(nc * 8);
      hib = S.get<double>(nc * 8);
      flag = S.get<uint8_t>(nc);
      bsplit = S.get<int>(nb * 4);
      btiny = S.get<int>(nb * 4);
      osplit = S.get<long long>(nb * 8);
      otiny = S.get<long long>(nb * 8);
      if (S.err != cudaSuccess) return cuda_fail(S.err, "intersect level arrays");
      capL = nc;
    }
    if ((rc = bound_aabb_internal(net_a, policy, n_keep, precision, n, nullptr, flo, fhi, loa, hia, nullptr, st)))
      return rc;
    if ((rc = bound_aabb_internal(net_b, policy, n_keep, precision, n, nullptr, flo, fhi, lob, hib, nullptr, st)))
      return rc;
    bounds += 2 * n;
    ++levels;
    const int nb = (int)((n + QT - 1) / QT);
    cudaMemsetAsync(wit, 0xff, 8, st);
    isect_mark_kernel<<<nb, QT, 0, st>>>(n, d, flo, fhi, loa, hia, lob, hib, stop, flag, bsplit, btiny, wit);
    block_scan_kernel<<<1, QT, 0, st>>>(nb, bsplit, osplit, tot);
    block_scan_kernel<<<1, QT, 0, st>>>(nb, btiny, otiny, tot + 1);
    long long km[2];
    unsigned long long w = 0;
    cudaError_t e = cudaMemcpyAsync(km, tot, 16, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&w, wit, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "intersect level");
    if (w != ~0ull) {  // the first interior witness in frontier order
      *kind = 1;
      if (witness_lo && witness_hi) {
        cudaMemcpyAsync(witness_lo, flo + w * d, d * 8, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(witness_hi, fhi + w * d, d * 8, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
      }
      if (stats) {
        stats[0] = levels;
        stats[1] = bounds;
      }
      return SPK_OK;
    }
    const long long K = km[0], M = km[1];
    if (2 * K > capC) {
      const long long nc = std::max<long long>(2 * K, 2 * capC);
      clo = S.get<double>(nc * d * 8);
      chi = S.get<double>(nc * d * 8);
      if (S.err != cudaSuccess) return cuda_fail(S.err, "intersect children");
      capC = nc;
    }
    isect_scatter_kernel<<<nb, QT, 0, st>>>(n, d, flo, fhi, flag, osplit, otiny, tot, clo, chi, tlo, thi);
    if (M > 0) {
      const size_t old = hlo.size();
      hlo.resize(old + M * d);
      hhi.resize(old + M * d);
      cudaMemcpyAsync(hlo.data() + old, tlo, M * d * 8, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(hhi.data() + old, thi, M * d * 8, cudaMemcpyDeviceToHost, st);
    }
    std::swap(flo, clo);
    std::swap(fhi, chi);
    std::swap(capF, capC);
    n = 2 * K;
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "intersect scatter");
  }
  const long long m = (long long)(hlo.size() / d);
  *kind = m > 0 ? 2 : 0;
  *n_nodes = m;
  if (nodes_lo && nodes_hi)
    for (long long q = 0; q < std::min<long long>(m, nodes_cap) * d; ++q) {
      nodes_lo[q] = hlo[q];
      nodes_hi[q] = hhi[q];
    }
  if (stats) {
    stats[0] = levels;
    stats[1] = bounds;
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SPK_OK : cuda_fail(e, "intersect kernels");
}

int spk_bisect(const spk_net* net, int precision, int64_t n, double* a, double* b, int iters, double* out,
               void* stream) {
  if (!net || (n > 0 && (!a || !b || !out))) return fail(SPK_ERR_INVALID_PARAMETER, "null argument");
  if (n < 0 || iters < 0) return fail(SPK_ERR_DIMENSION, "negative size");
  if (n == 0) return SPK_OK;
  const int d = net->input_dim;
  DeviceGuard g(net->device);
  cudaStream_t st = (cudaStream_t)stream;
  Scratch S(st);
  double* fm = S.get<double>(n * 8);
  if (S.err != cudaSuccess) return cuda_fail(S.err, "bisect alloc");
  const int blk = (int)((n * d + QT - 1) / QT);
  for (int it = 0; it < iters; ++it) {
    bisect_mid_kernel<<<blk, QT, 0, st>>>(n, d, a, b, out);
    int rc = spk_eval_batch(net, precision, n, out, fm, st);
    if (rc != SPK_OK) return rc;
    bisect_update_kernel<<<blk, QT, 0, st>>>(n, d, fm, out, a, b);
  }
  bisect_mid_kernel<<<blk, QT, 0, st>>>(n, d, a, b, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SPK_OK : cuda_fail(e, "bisect kernels");
}

}  // extern "C"
