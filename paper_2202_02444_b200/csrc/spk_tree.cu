// K5: breadth-first k-d tree build (build_spatial_tree, spatial.py:214-289)
// as a level-synchronous frontier on the device.
//
// Per level: (1) the fused bound kernel classifies every frontier AABB
// (IN_AABB input, centre/half-extent formed in FP64 exactly like
// spatial.py:181-183); (2) spk_tree_mark decides split / tiny-leaf per node
// and counts splits per block with a warp ballot; (3) spk_tree_scatter
// finds its block offset, ranks split nodes inside the block with a
// ballot prefix, and writes the children: low halves at [0, K), high halves
// at [K, 2K) -- the reference's level layout (spatial.py:285-287) -- with
// the midpoint split on the widest axis computed in FP64 (spatial.py:189-199),
// so child AABBs are bit-identical to the reference's.  Tiny UNKNOWN leaves
// (convergence mode) get the 2d face-centre sign annotation
// (spatial.py:257-265) from one point-evaluation pass.
#include <algorithm>
#include <cmath>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "spk_kernels.cuh"
#include <cstdlib>

#include "spk_abi_internal.h"

#ifndef SPK_PAIR_ORDER
#define SPK_PAIR_ORDER 1  // bound tree levels in sibling-pair order (BoxInput::pair_order)
#endif

#ifndef SPK_TREE_SPECULATE
#define SPK_TREE_SPECULATE 1  // fixed-depth builds bound their latency-bound top levels in one launch
#endif
#ifndef SPK_MIRROR_EAGER_MIN
#define SPK_MIRROR_EAGER_MIN 4096  // levels at least this large are mirrored while the build runs
#endif
#ifndef SPK_SPEC_PER_SM
#define SPK_SPEC_PER_SM 16 // ... the levels of at most this many nodes per SM
#endif

namespace spk {

constexpr int TB_THREADS = 256;

struct TreeLevel {
  long long n = 0;
  double* lo = nullptr;      // n x d
  double* hi = nullptr;      // n x d
  double* blo = nullptr;     // bound lo (n)
  double* bhi = nullptr;     // bound hi (n)
  int8_t* label = nullptr;   // +1 / -1 / 0
  int8_t* face = nullptr;    // face-sign annotation (+1/-1, 0 = none)
  long long* parent = nullptr;
};

// per-node decision: flag 1 = split, 2 = tiny UNKNOWN leaf (convergence mode)
// band > 0 replaces "UNKNOWN" by "bound meets [-band, band]"
// (sample_near_surface's refinement rule, spatial.py:403-411)
__global__ void tree_mark_kernel(const long long* __restrict__ n_dev, int d, const double* __restrict__ lo,
                                 const double* __restrict__ hi, const int8_t* __restrict__ label,
                                 const double* __restrict__ blo, const double* __restrict__ bhi, double band,
                                 int depth, int max_depth, double stop_extent, uint8_t* __restrict__ flag,
                                 int* __restrict__ block_split, int* __restrict__ block_small, bool capped) {
  const long long n = *n_dev;
  const long long i = (long long)blockIdx.x * TB_THREADS + threadIdx.x;
  uint8_t f = 0;
  const bool open = i < n && (band > 0.0 ? (blo[i] <= band && bhi[i] >= -band) : label[i] == 0);
  if (open) {
    if (max_depth >= 0) {
      f = depth < max_depth ? 1 : 0;
    } else {
      double ext = 0.0;
      for (int k = 0; k < d; ++k) ext = fmax(ext, hi[i * d + k] - lo[i * d + k]);
      f = ext < stop_extent ? 2 : 1;
    }
    // level cap (segmented builds): nothing splits at the last level; open
    // nodes stay UNKNOWN internal nodes for the next segment, tiny ones
    // still become face-signed leaves
    if (capped && f == 1) f = 0;
  }
  if (i < n) flag[i] = f;
  __shared__ int ws[TB_THREADS / 32], wt[TB_THREADS / 32];
  const unsigned bs = __ballot_sync(0xffffffffu, f == 1);
  const unsigned bt = __ballot_sync(0xffffffffu, f == 2);
  if ((threadIdx.x & 31) == 0) {
    ws[threadIdx.x >> 5] = __popc(bs);
    wt[threadIdx.x >> 5] = __popc(bt);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0, b = 0;
    for (int w = 0; w < TB_THREADS / 32; ++w) { a += ws[w]; b += wt[w]; }
    block_split[blockIdx.x] = a;
    block_small[blockIdx.x] = b;
  }
}

// Exclusive offset of this block = sum of earlier blocks' counts.
__device__ long long block_offset(const int* __restrict__ counts, int upto) {
  long long s = 0;
  for (int b = threadIdx.x; b < upto; b += TB_THREADS) s += counts[b];
  __shared__ long long red[TB_THREADS / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  long long t = 0;
  for (int w = 0; w < TB_THREADS / 32; ++w) t += red[w];
  __syncthreads();
  return t;
}

// Rank of this thread's flag among the block's flagged threads (ballot prefix).
__device__ int block_rank(bool pred, int* total) {
  __shared__ int wcount[TB_THREADS / 32];
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) wcount[w] = __popc(m);
  __syncthreads();
  int before = 0, all = 0;
  for (int q = 0; q < TB_THREADS / 32; ++q) {
    if (q < w) before += wcount[q];
    all += wcount[q];
  }
  __syncthreads();
  *total = all;
  return before + __popc(m & ((1u << lane) - 1u));
}

// totals of the block counts -> K (splits), M (tiny leaves), next level size 2K
__global__ void tree_sum_kernel(int nblk, const int* __restrict__ block_split, const int* __restrict__ block_small,
                                long long* __restrict__ k_out, long long* __restrict__ m_out,
                                long long* __restrict__ next_n) {
  long long a = 0, b = 0;
  for (int q = threadIdx.x; q < nblk; q += TB_THREADS) {
    a += block_split[q];
    b += block_small[q];
  }
  __shared__ long long ra[TB_THREADS / 32], rb[TB_THREADS / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, off);
    b += __shfl_xor_sync(0xffffffffu, b, off);
  }
  if ((threadIdx.x & 31) == 0) {
    ra[threadIdx.x >> 5] = a;
    rb[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long ta = 0, tb = 0;
    for (int w = 0; w < TB_THREADS / 32; ++w) { ta += ra[w]; tb += rb[w]; }
    *k_out = ta;
    *m_out = tb;
    *next_n = 2 * ta;
  }
}

__global__ void tree_scatter_kernel(const long long* __restrict__ n_dev, int d, const double* __restrict__ lo,
                                    const double* __restrict__ hi, const uint8_t* __restrict__ flag,
                                    const int* __restrict__ block_split, const int* __restrict__ block_small,
                                    const long long* __restrict__ k_dev, double* __restrict__ child_lo,
                                    double* __restrict__ child_hi, long long* __restrict__ child_parent,
                                    long long* __restrict__ small_idx) {
  const long long n = *n_dev, n_split = *k_dev;
  const long long i = (long long)blockIdx.x * TB_THREADS + threadIdx.x;
  const long long off_s = block_offset(block_split, blockIdx.x);
  const long long off_t = block_offset(block_small, blockIdx.x);
  const uint8_t f = i < n ? flag[i] : 0;
  int tot;
  const int rs = block_rank(f == 1, &tot);
  const int rt = block_rank(f == 2, &tot);
  if (f == 2) small_idx[off_t + rt] = i;
  if (f != 1) return;
  const long long j = off_s + rs;
  // widest axis, ties to the lowest index (np.argmax, spatial.py:193)
  int ax = 0;
  double best = -1.0;
  for (int k = 0; k < d; ++k) {
    const double e = hi[i * d + k] - lo[i * d + k];
    if (e > best) { best = e; ax = k; }
  }
  const double mid = 0.5 * (lo[i * d + ax] + hi[i * d + ax]);
  for (int k = 0; k < d; ++k) {
    const double l = lo[i * d + k], h = hi[i * d + k];
    child_lo[j * d + k] = l;
    child_hi[j * d + k] = k == ax ? mid : h;
    child_lo[(n_split + j) * d + k] = k == ax ? mid : l;
    child_hi[(n_split + j) * d + k] = h;
  }
  child_parent[j] = i;
  child_parent[n_split + j] = i;
}

// Speculative top levels (fixed-depth builds).  The top levels of a tree hold
// a few hundred nodes each and their bound launches are latency-bound (~80 us
// whatever their size), while a node's AABB depends only on its path (widest
// axis, FP64 midpoint) and its bound only on its AABB.  So the complete binary
// tree of the first L levels is generated and bounded in ONE launch, and each
// of those levels then fetches its live nodes' bounds from it.  Level k of the
// complete tree (size n_roots 2^k, offset n_roots (2^k - 1)) is laid out like
// the reference's levels: child c of level k+1 has parent c mod size_k and is
// the high half when c >= size_k (tree_scatter_kernel with every node split).
__global__ void spec_boxes_kernel(long long n_roots, int L, int d, const double* __restrict__ root_lo,
                                  const double* __restrict__ root_hi, double* __restrict__ lo,
                                  double* __restrict__ hi) {
  const long long total = n_roots * ((1ll << L) - 1);
  const long long g = (long long)blockIdx.x * TB_THREADS + threadIdx.x;
  if (g >= total) return;
  int k = 0;
  while (n_roots * ((1ll << (k + 1)) - 1) <= g) ++k;
  long long i = g - n_roots * ((1ll << k) - 1);
  unsigned long long bits = 0;  // bit j-1: the node's ancestor at level j is a high half
  for (int j = k; j >= 1; --j) {
    const long long half = n_roots << (j - 1);
    if (i >= half) {
      bits |= 1ull << (j - 1);
      i -= half;
    }
  }
  double bl[MAX_AXES], bh[MAX_AXES];
  for (int q = 0; q < d; ++q) {
    bl[q] = root_lo[i * d + q];
    bh[q] = root_hi[i * d + q];
  }
  for (int j = 1; j <= k; ++j) {
    // tree_scatter_kernel's split: widest axis, ties to the lowest index, FP64 midpoint
    int ax = 0;
    double best = -1.0;
    for (int q = 0; q < d; ++q) {
      const double e = bh[q] - bl[q];
      if (e > best) { best = e; ax = q; }
    }
    const double mid = 0.5 * (bl[ax] + bh[ax]);
    if ((bits >> (j - 1)) & 1ull) bl[ax] = mid; else bh[ax] = mid;
  }
  for (int q = 0; q < d; ++q) {
    lo[g * d + q] = bl[q];
    hi[g * d + q] = bh[q];
  }
}

// live node i of a speculative level: its bound from the complete tree
// (cidx = its index within the complete level; nullptr at the roots)
__global__ void spec_fetch_kernel(const long long* __restrict__ n_dev, const long long* __restrict__ cidx,
                                  long long offset, const double* __restrict__ sblo, const double* __restrict__ sbhi,
                                  const int8_t* __restrict__ slab, double* __restrict__ blo, double* __restrict__ bhi,
                                  int8_t* __restrict__ label) {
  const long long n = *n_dev;
  const long long i = (long long)blockIdx.x * TB_THREADS + threadIdx.x;
  if (i >= n) return;
  const long long g = offset + (cidx ? cidx[i] : i);
  blo[i] = sblo[g];
  bhi[i] = sbhi[g];
  label[i] = slab[g];
}

// complete-level index of the next level's nodes: child c is the high half
// when c >= K (tree_scatter_kernel), of parent p = parent[c]
__global__ void spec_child_index_kernel(const long long* __restrict__ n_next, const long long* __restrict__ k_dev,
                                        const long long* __restrict__ parent, const long long* __restrict__ cidx,
                                        long long level_size, long long* __restrict__ cidx_next) {
  const long long n = *n_next, K = *k_dev;
  const long long c = (long long)blockIdx.x * TB_THREADS + threadIdx.x;
  if (c >= n) return;
  const long long p = parent[c];
  cidx_next[c] = (cidx ? cidx[p] : p) + (c >= K ? level_size : 0);
}

// Face centres of tiny leaves: (m, 2d, d) points (spatial.py:202-211).
__global__ void face_points_kernel(const long long* __restrict__ m_dev, int d, const long long* __restrict__ idx,
                                   const double* __restrict__ lo, const double* __restrict__ hi,
                                   double* __restrict__ pts, long long* __restrict__ np_out) {
  const long long m = *m_dev;
  const long long t = (long long)blockIdx.x * TB_THREADS + threadIdx.x;
  if (t == 0) *np_out = m * 2 * d;
  if (t >= m * 2 * d) return;
  const long long node = idx[t / (2 * d)];
  const int face = (int)(t % (2 * d));
  const int axis = face / 2;
  for (int k = 0; k < d; ++k) {
    const double l = lo[node * d + k], h = hi[node * d + k];
    const double c = (l + h) / 2.0, half = (h - l) / 2.0;
    double v = c;
    if (k == axis) v = (face & 1) ? c + half : c - half;
    pts[t * d + k] = v;
  }
}

__global__ void face_sign_kernel(const long long* __restrict__ m_dev, int d, const long long* __restrict__ idx,
                                 const double* __restrict__ vals, int8_t* __restrict__ face) {
  const long long m = *m_dev;
  const long long t = (long long)blockIdx.x * TB_THREADS + threadIdx.x;
  if (t >= m) return;
  bool neg = false, pos = false;
  for (int q = 0; q < 2 * d; ++q) {
    const double v = vals[t * 2 * d + q];
    neg |= v < 0.0;
    pos |= v >= 0.0;
  }
  face[idx[t]] = (neg && pos) ? 0 : (neg ? -1 : 1);
}

}  // namespace spk

struct spk_tree {
  int d = 0;
  int device = 0;
  int start_depth = 0;
  std::vector<spk::TreeLevel> levels;
  long long bound_evals = 0;
  cudaStream_t stream = nullptr;  // frees are ordered on the build stream
  long long launches = 0;   // kernels launched by the build
  double bound_ms = 0.0;    // CUDA-event time of the bound kernels
  // host mirror (SPK_TREE_HOST_MIRROR): per level one malloc block holding
  // lo, hi (n x d), bound_lo, bound_hi, label, face, parent back to back
  std::vector<char*> host;
  std::vector<long long> host_n;
  std::vector<long long> host_cap;  // row stride of each host block's sections (>= host_n)
  int precopied = -1;               // level whose AABBs / parents were copied before its bound ran
  bool device_released = false;  // spk_tree_release_device: only the host mirror remains
};

namespace spk {

// All tree memory comes from the device's stream-ordered pool
// (cudaMallocAsync): after the first build, a level costs no driver call.
static void free_level(TreeLevel& L, cudaStream_t st) {
  if (L.lo) cudaFreeAsync(L.lo, st);  // one block per level, see alloc_level
  L = TreeLevel();
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static int alloc_level(TreeLevel& L, long long n, int d, cudaStream_t st) {
  L.n = n;
  const size_t m = std::max<long long>(n, 1);
  const size_t b_lo = align_up(m * d * sizeof(double)), b_b = align_up(m * sizeof(double)),
               b_i8 = align_up(m), b_par = align_up(m * sizeof(long long));
  char* base = nullptr;
  cudaError_t e = cudaMallocAsync(&base, 2 * b_lo + 2 * b_b + 2 * b_i8 + b_par, st);
  if (e != cudaSuccess) return cuda_fail(e, "tree level alloc");
  L.lo = reinterpret_cast<double*>(base);
  L.hi = reinterpret_cast<double*>(base + b_lo);
  L.blo = reinterpret_cast<double*>(base + 2 * b_lo);
  L.bhi = reinterpret_cast<double*>(base + 2 * b_lo + b_b);
  L.label = reinterpret_cast<int8_t*>(base + 2 * b_lo + 2 * b_b);
  L.face = reinterpret_cast<int8_t*>(base + 2 * b_lo + 2 * b_b + b_i8);
  L.parent = reinterpret_cast<long long*>(base + 2 * b_lo + 2 * b_b + 2 * b_i8);
  return SPK_OK;
}

// per-thread pinned staging for the per-level block counts (grown, never freed)
static bool pinned_scratch(size_t bytes, void** out) {
  thread_local void* buf = nullptr;
  thread_local size_t cap = 0;
  if (bytes > cap) {
    if (buf) cudaFreeHost(buf);
    cap = std::max<size_t>(bytes, 1 << 16);
    if (cudaMallocHost(&buf, cap) != cudaSuccess) { buf = nullptr; cap = 0; return false; }
  }
  *out = buf;
  return true;
}

void keep_pool_memory(int device) {
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> lk(mu);
  if ((int)done.size() <= device) done.resize(device + 1, 0);
  if (done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[device] = 1;
}

// Host-mirror blocks of >= 1 MB come from a process-wide pool of pinned
// (page-locked, portable) blocks in power-of-two size classes: the
// device-to-host copies of large levels run as DMA at full PCIe rate instead
// of through pageable staging, and a block freed with its tree is reused by
// the next build (no cudaHostAlloc per build; a class is pinned from its
// second request on).  Smaller blocks use malloc.
// At most kPinnedKeep bytes stay cached.
namespace {
constexpr size_t kPinnedMin = 1u << 20;
constexpr size_t kPinnedKeep = (size_t)2 << 30;
std::mutex g_pin_mu;
std::vector<std::pair<size_t, char*>> g_pin_free;  // (class size, block)
size_t g_pin_cached = 0;
std::unordered_map<char*, size_t> g_pin_live;    // pinned blocks handed out -> class size
std::unordered_map<size_t, int> g_pin_seen;      // requests per size class

char* host_block(size_t bytes) {
  if (bytes < kPinnedMin) return static_cast<char*>(std::malloc(std::max<size_t>(bytes, 1)));
  size_t cls = kPinnedMin;
  while (cls < bytes) cls <<= 1;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  for (size_t i = 0; i < g_pin_free.size(); ++i) {
    if (g_pin_free[i].first == cls) {
      char* b = g_pin_free[i].second;
      g_pin_free.erase(g_pin_free.begin() + (long)i);
      g_pin_cached -= cls;
      g_pin_live[b] = cls;
      return b;
    }
  }
  // pinning costs ~3 ms per MB once; a size class is pinned from its second
  // request on (a one-shot build keeps pageable blocks, repeated builds reuse
  // pinned ones)
  if (g_pin_seen[cls]++ == 0) return static_cast<char*>(std::malloc(bytes));
  void* b = nullptr;
  if (cudaHostAlloc(&b, cls, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();  // fall back to pageable memory
    return static_cast<char*>(std::malloc(bytes));
  }
  g_pin_live[static_cast<char*>(b)] = cls;
  return static_cast<char*>(b);
}

void host_block_free(char* b) {
  if (!b) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  auto it = g_pin_live.find(b);
  if (it == g_pin_live.end()) {
    std::free(b);
    return;
  }
  const size_t cls = it->second;
  g_pin_live.erase(it);
  if (g_pin_cached + cls <= kPinnedKeep) {
    g_pin_free.emplace_back(cls, b);
    g_pin_cached += cls;
  } else {
    cudaFreeHost(b);
  }
}
}  // namespace

// Copy level `lv` of the build into host memory on the copy stream `cst`
// once the compute stream has passed event `done`: the host thread blocks on
// the (pageable) copy while the GPU already runs the next level's kernels.
static int mirror_level(spk_tree* tree, int lv, const TreeLevel& L, const long long* d_count, cudaEvent_t done,
                        cudaStream_t cst) {
  cudaStreamWaitEvent(cst, done, 0);
  long long n = 0;
  cudaError_t e = cudaMemcpyAsync(&n, d_count, sizeof(long long), cudaMemcpyDeviceToHost, cst);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cst);
  if (e != cudaSuccess) return cuda_fail(e, "tree mirror count");
  const size_t d = (size_t)tree->d, m = (size_t)n;
  const size_t sz[7] = {m * d * 8, m * d * 8, m * 8, m * 8, m, m, m * 8};
  size_t total = 0;
  for (size_t b : sz) total += b;
  char* h = host_block(total);
  if (!h) return fail(SPK_ERR_OUT_OF_MEMORY, "tree host mirror");
  const void* src[7] = {L.lo, L.hi, L.blo, L.bhi, L.label, L.face, L.parent};
  size_t off = 0;
  for (int q = 0; q < 7; ++q) {
    if (sz[q] && (e = cudaMemcpyAsync(h + off, src[q], sz[q], cudaMemcpyDeviceToHost, cst)) != cudaSuccess) break;
    off += sz[q];
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(cst);
  if (e != cudaSuccess) {
    host_block_free(h);
    return cuda_fail(e, "tree mirror copy");
  }
  if ((int)tree->host.size() <= lv) {
    tree->host.resize(lv + 1, nullptr);
    tree->host_n.resize(lv + 1, 0);
  }
  tree->host[lv] = h;
  tree->host_n[lv] = n;
  if ((int)tree->host_cap.size() <= lv) tree->host_cap.resize(lv + 1, 0);
  tree->host_cap[lv] = n;
  return SPK_OK;
}

// The levels the build did not mirror while it ran (the small ones, whose
// per-level count read and copy would leave the GPU waiting on the host
// between short launches): one count read, all copies, one synchronisation.
static int mirror_deferred(spk_tree* tree, const long long* d_cnt, cudaEvent_t done, cudaStream_t cst) {
  const int nl = (int)tree->levels.size();
  std::vector<int> todo;
  for (int l = 0; l < nl; ++l)
    if ((int)tree->host.size() <= l || tree->host[l] == nullptr) todo.push_back(l);
  if (todo.empty()) return SPK_OK;
  cudaStreamWaitEvent(cst, done, 0);
  std::vector<long long> n(nl);
  cudaError_t e = cudaMemcpyAsync(n.data(), d_cnt, nl * sizeof(long long), cudaMemcpyDeviceToHost, cst);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cst);
  if (e != cudaSuccess) return cuda_fail(e, "tree mirror counts");
  if ((int)tree->host.size() < nl) {
    tree->host.resize(nl, nullptr);
    tree->host_n.resize(nl, 0);
  }
  if ((int)tree->host_cap.size() < nl) tree->host_cap.resize(nl, 0);
  const size_t d = (size_t)tree->d;
  if (tree->precopied >= 0 && tree->precopied < nl && tree->host[tree->precopied]) {
    // AABBs and parents are on their way (cap-row sections): the bounds,
    // labels and faces of the live rows complete the block
    const int l = tree->precopied;
    const TreeLevel& L = tree->levels[l];
    const size_t m = (size_t)n[l], c = (size_t)tree->host_cap[l];
    char* h = tree->host[l];
    tree->host_n[l] = n[l];
    const size_t off_b = 2 * c * d * 8;
    if (m) {
      if (e == cudaSuccess) e = cudaMemcpyAsync(h + off_b, L.blo, m * 8, cudaMemcpyDeviceToHost, cst);
      if (e == cudaSuccess) e = cudaMemcpyAsync(h + off_b + c * 8, L.bhi, m * 8, cudaMemcpyDeviceToHost, cst);
      if (e == cudaSuccess) e = cudaMemcpyAsync(h + off_b + 2 * c * 8, L.label, m, cudaMemcpyDeviceToHost, cst);
      if (e == cudaSuccess) e = cudaMemcpyAsync(h + off_b + 2 * c * 8 + c, L.face, m, cudaMemcpyDeviceToHost, cst);
    }
  }
  for (int l : todo) {
    const TreeLevel& L = tree->levels[l];
    const size_t m = (size_t)n[l];
    const size_t sz[7] = {m * d * 8, m * d * 8, m * 8, m * 8, m, m, m * 8};
    size_t total = 0;
    for (size_t b : sz) total += b;
    char* h = host_block(total);
    if (!h) return fail(SPK_ERR_OUT_OF_MEMORY, "tree host mirror");
    tree->host[l] = h;
    tree->host_n[l] = n[l];
    tree->host_cap[l] = n[l];
    const void* src[7] = {L.lo, L.hi, L.blo, L.bhi, L.label, L.face, L.parent};
    size_t off = 0;
    for (int q = 0; q < 7 && e == cudaSuccess; ++q) {
      if (sz[q]) e = cudaMemcpyAsync(h + off, src[q], sz[q], cudaMemcpyDeviceToHost, cst);
      off += sz[q];
    }
    if (e != cudaSuccess) break;
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(cst);
  if (e != cudaSuccess) return cuda_fail(e, "tree mirror copy");
  return SPK_OK;
}

static void free_mirror(spk_tree* tree) {
  for (char* h : tree->host) host_block_free(h);
  tree->host.clear();
  tree->host_n.clear();
  tree->host_cap.clear();
  tree->precopied = -1;
}

}  // namespace spk

using namespace spk;

extern "C" {

int spk_tree_build(const spk_net* net, int policy, int n_keep, int precision, int64_t n_roots,
                   const double* root_lo, const double* root_hi, int start_depth, int max_depth, double delta,
                   void* stream, spk_tree** out) {
  return spk_tree_build_band(net, policy, n_keep, precision, n_roots, root_lo, root_hi, start_depth, max_depth,
                             delta, 0.0, stream, out);
}

int spk_tree_build_band(const spk_net* net, int policy, int n_keep, int precision, int64_t n_roots,
                        const double* root_lo, const double* root_hi, int start_depth, int max_depth,
                        double delta, double band, void* stream, spk_tree** out) {
  return spk_tree_build_ex(net, policy, n_keep, precision, n_roots, root_lo, root_hi, start_depth, max_depth,
                           delta, band, 0, stream, out);
}

int spk_tree_build_ex(const spk_net* net, int policy, int n_keep, int precision, int64_t n_roots,
                      const double* root_lo, const double* root_hi, int start_depth, int max_depth,
                      double delta, double band, int flags, void* stream, spk_tree** out) {
  if (!net || !out) return fail(SPK_ERR_INVALID_PARAMETER, "null argument");
  if (!(band >= 0.0)) return fail(SPK_ERR_INVALID_PARAMETER, "band must be >= 0");
  *out = nullptr;
  const int d = net->input_dim;
  if (d > MAX_AXES) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "tree build supports d <= 8");
  if (!(delta > 0.0)) return fail(SPK_ERR_INVALID_PARAMETER, "delta must be positive");
  if (max_depth > 60) return fail(SPK_ERR_DEPTH_OVERFLOW, "fixed depth exceeds 60");
  if (n_roots < 1 || start_depth < 0) return fail(SPK_ERR_INVALID_PARAMETER, "need >= 1 root, start_depth >= 0");
  for (long long q = 0; q < n_roots * d; ++q) {
    if (!std::isfinite(root_lo[q]) || !std::isfinite(root_hi[q]) || !(root_hi[q] > root_lo[q]))
      return fail(SPK_ERR_INVALID_PARAMETER, "bounds must be finite with positive extent");
  }
  DeviceGuard g(net->device);
  keep_pool_memory(net->device);
  cudaStream_t st = (cudaStream_t)stream;
  auto tree = new spk_tree();
  tree->stream = st;
  tree->d = d;
  tree->device = net->device;
  tree->start_depth = start_depth;
  const double stop = delta / std::sqrt((double)d);
  const bool fixed = max_depth >= 0;
  // SPK_TREE_LEVEL_CAP(c): at most c levels below the roots (segmented builds)
  const int level_cap = ((flags >> 8) & 0xff) - 1;
  // Level sizes stay on the device: kernels read their live count from
  // d_cnt[level] and are launched for a capacity bound (2x the previous
  // level).  The host only synchronises in convergence mode (to detect the
  // last level) or when a capacity bound would exceed kAsyncCap nodes.
  constexpr long long kAsyncCap = 1ll << 24;
  constexpr int kMaxLevels = 64;
  int rc = SPK_OK;
  long long* d_cnt = nullptr;  // [level] live count; [kMaxLevels + level] K; [2*kMaxLevels + level] M
  long long* d_np = nullptr;   // face-point count
  if (cudaMallocAsync(&d_cnt, 3 * kMaxLevels * sizeof(long long), st) != cudaSuccess ||
      cudaMallocAsync(&d_np, sizeof(long long), st) != cudaSuccess) {
    delete tree;
    return fail(SPK_ERR_OUT_OF_MEMORY, "tree counters");
  }
  cudaMemsetAsync(d_cnt, 0, 3 * kMaxLevels * sizeof(long long), st);
  {
    const long long r = n_roots;
    cudaMemcpyAsync(d_cnt, &r, sizeof(long long), cudaMemcpyHostToDevice, st);
  }
  TreeLevel cur;
  if ((rc = alloc_level(cur, n_roots, d, st)) != SPK_OK) { delete tree; return rc; }
  cudaMemcpyAsync(cur.lo, root_lo, n_roots * d * sizeof(double), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(cur.hi, root_hi, n_roots * d * sizeof(double), cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(cur.parent, 0xff, n_roots * sizeof(long long), st);  // -1
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEventCreate(&ev0);
  cudaEventCreate(&ev1);
  std::vector<cudaEvent_t> bound_ev;  // start/stop pairs, read once at the end
  int* counts = nullptr;
  uint8_t* flag = nullptr;
  long long* small_idx = nullptr;
  double* fpts = nullptr;
  double* fvals = nullptr;
  long long cap = 0, fcap = 0;
  std::vector<long long> caps;
  long long cur_cap = n_roots;  // capacity bound of the current level
  const bool mirror = (flags & SPK_TREE_HOST_MIRROR) != 0;
  cudaStream_t cst = nullptr;   // mirror copies
  std::vector<cudaEvent_t> level_done;
  if (mirror && cudaStreamCreateWithFlags(&cst, cudaStreamNonBlocking) != cudaSuccess) {
    delete tree;
    return fail(SPK_ERR_CUDA, "tree mirror stream");
  }
  // speculative top levels (fixed-depth builds of the fused policies): the
  // first spec_L levels whose complete size stays within 4 boxes per SM
  int spec_L = 0;
  {
    int mode_chk = policy == SPK_POLICY_INTERVAL || policy == SPK_POLICY_AFFINE_FIXED;
    const long long lim = SPK_TREE_SPECULATE ? (long long)SPK_SPEC_PER_SM * std::max(sm_count_for(net->device), 1) : 0;
    const int levels_left = fixed ? max_depth - start_depth + 1 : 0;
    for (long long sz = n_roots; mode_chk && spec_L < levels_left && spec_L < 20 && sz <= lim; sz *= 2) ++spec_L;
    if (level_cap >= 0) spec_L = std::min(spec_L, level_cap + 1);
    if (spec_L < 2) spec_L = 0;
  }
  double* spec_lo = nullptr;  // complete-tree AABBs (S x d) x 2, bounds (S) x 2, labels (S)
  double *spec_blo = nullptr, *spec_bhi = nullptr;
  int8_t* spec_lab = nullptr;
  long long* spec_idx[2] = {nullptr, nullptr};
  cudaEvent_t spec_e0 = nullptr, spec_e1 = nullptr;
  if (spec_L > 0) {
    const long long S = n_roots * ((1ll << spec_L) - 1), top = n_roots << (spec_L - 1);
    char* base = nullptr;
    const size_t b_box = align_up((size_t)S * d * sizeof(double)), b_b = align_up((size_t)S * sizeof(double)),
                 b_l = align_up((size_t)S), b_i = align_up((size_t)top * sizeof(long long));
    if (cudaMallocAsync(&base, 2 * b_box + 2 * b_b + b_l + 2 * b_i, st) != cudaSuccess) {
      rc = fail(SPK_ERR_OUT_OF_MEMORY, "speculative levels");
    } else {
      spec_lo = reinterpret_cast<double*>(base);
      spec_blo = reinterpret_cast<double*>(base + 2 * b_box);
      spec_bhi = reinterpret_cast<double*>(base + 2 * b_box + b_b);
      spec_lab = reinterpret_cast<int8_t*>(base + 2 * b_box + 2 * b_b);
      spec_idx[0] = reinterpret_cast<long long*>(base + 2 * b_box + 2 * b_b + b_l);
      spec_idx[1] = reinterpret_cast<long long*>(base + 2 * b_box + 2 * b_b + b_l + b_i);
      double* spec_hi = reinterpret_cast<double*>(base + b_box);
      spec_boxes_kernel<<<(int)((S + TB_THREADS - 1) / TB_THREADS), TB_THREADS, 0, st>>>(n_roots, spec_L, d, cur.lo,
                                                                                        cur.hi, spec_lo, spec_hi);
      cudaEventCreate(&spec_e0);
      cudaEventCreate(&spec_e1);
      cudaEventRecord(spec_e0, st);
      rc = bound_aabb_internal(net, policy, n_keep, precision, S, nullptr, spec_lo, spec_hi, spec_blo, spec_bhi,
                               spec_lab, st, 0);
      cudaEventRecord(spec_e1, st);
      tree->launches += 2;
    }
  }
  for (int depth = start_depth, lv = 0; rc == SPK_OK; ++depth, ++lv) {
    if (lv >= kMaxLevels) { rc = fail(SPK_ERR_DEPTH_OVERFLOW, "more than 64 tree levels"); break; }
    long long* n_dev = d_cnt + lv;
    long long* k_dev = d_cnt + kMaxLevels + lv;
    long long* m_dev = d_cnt + 2 * kMaxLevels + lv;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    bound_ev.push_back(e0);
    bound_ev.push_back(e1);
    cudaEventRecord(e0, st);
    // the last level of a fixed-depth mirrored build: its AABBs and parents
    // are final already (the previous scatter), so they go to the host while
    // its bound kernel runs (cap-row sections; the bounds follow after it)
    if (mirror && fixed && lv > 0 && cur_cap >= SPK_MIRROR_EAGER_MIN &&
        (depth >= max_depth || (level_cap >= 0 && lv >= level_cap))) {
      const size_t c = (size_t)cur_cap, dd = (size_t)d;
      char* h = host_block(2 * c * dd * 8 + 2 * c * 8 + 2 * c + c * 8);
      if (!h) { rc = fail(SPK_ERR_OUT_OF_MEMORY, "tree host mirror"); break; }
      if ((int)tree->host.size() <= lv) {
        tree->host.resize(lv + 1, nullptr);
        tree->host_n.resize(lv + 1, 0);
        tree->host_cap.resize(lv + 1, 0);
      }
      tree->host[lv] = h;
      tree->host_cap[lv] = cur_cap;
      tree->precopied = lv;
      cudaEvent_t ready;
      cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
      cudaEventRecord(ready, st);
      cudaStreamWaitEvent(cst, ready, 0);
      cudaEventDestroy(ready);
      cudaMemcpyAsync(h, cur.lo, c * dd * 8, cudaMemcpyDeviceToHost, cst);
      cudaMemcpyAsync(h + c * dd * 8, cur.hi, c * dd * 8, cudaMemcpyDeviceToHost, cst);
      cudaMemcpyAsync(h + 2 * c * dd * 8 + 2 * c * 8 + 2 * c, cur.parent, c * 8, cudaMemcpyDeviceToHost, cst);
    }
    // levels below the roots are [low children; high children]: bound them in
    // sibling-pair order (identical results; coherent live-row masks)
    if (lv < spec_L) {
      const long long* cidx = lv == 0 ? nullptr : spec_idx[lv & 1];
      spec_fetch_kernel<<<(int)((cur_cap + TB_THREADS - 1) / TB_THREADS), TB_THREADS, 0, st>>>(
          n_dev, cidx, n_roots * ((1ll << lv) - 1), spec_blo, spec_bhi, spec_lab, cur.blo, cur.bhi, cur.label);
    } else {
      rc = bound_aabb_internal(net, policy, n_keep, precision, cur_cap, n_dev, cur.lo, cur.hi, cur.blo, cur.bhi,
                               cur.label, st, (SPK_PAIR_ORDER && lv > 0) ? 1 : 0);
    }
    cudaEventRecord(e1, st);
    if (rc != SPK_OK) break;
    tree->launches += 4;
    cudaMemsetAsync(cur.face, 0, cur_cap, st);
    const int nb = (int)((cur_cap + TB_THREADS - 1) / TB_THREADS);
    if (cur_cap > cap) {
      if (counts) { cudaFreeAsync(counts, st); cudaFreeAsync(flag, st); cudaFreeAsync(small_idx, st); }
      cap = std::max<long long>(2 * cur_cap, 1024);
      const long long nbc = (cap + TB_THREADS - 1) / TB_THREADS;
      if (cudaMallocAsync(&counts, 2 * nbc * sizeof(int), st) != cudaSuccess ||
          cudaMallocAsync(&flag, cap, st) != cudaSuccess ||
          cudaMallocAsync(&small_idx, cap * sizeof(long long), st) != cudaSuccess) {
        rc = fail(SPK_ERR_OUT_OF_MEMORY, "tree scratch");
        break;
      }
    }
    int* bsplit = counts;
    int* bsmall = counts + nb;
    const bool capped = level_cap >= 0 && lv >= level_cap;
    tree_mark_kernel<<<nb, TB_THREADS, 0, st>>>(n_dev, d, cur.lo, cur.hi, cur.label, cur.blo, cur.bhi, band, depth,
                                                max_depth, stop, flag, bsplit, bsmall, capped);
    tree_sum_kernel<<<1, TB_THREADS, 0, st>>>(nb, bsplit, bsmall, k_dev, m_dev, d_cnt + lv + 1);
    // capacity of the next level
    const bool last_fixed = (fixed && depth >= max_depth) || capped;
    long long next_cap = last_fixed ? 0 : 2 * cur_cap;
    long long k_exact = -1;
    if (!fixed || next_cap > kAsyncCap) {
      long long km[2];
      cudaMemcpyAsync(&km[0], k_dev, sizeof(long long), cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(&km[1], m_dev, sizeof(long long), cudaMemcpyDeviceToHost, st);
      cudaError_t e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) { rc = cuda_fail(e, "tree level"); break; }
      k_exact = km[0];
      next_cap = 2 * km[0];
    }
    TreeLevel next;
    if (next_cap > 0 && (rc = alloc_level(next, next_cap, d, st)) != SPK_OK) break;
    // always launched: it also lists the tiny leaves (children only when K > 0)
    tree_scatter_kernel<<<nb, TB_THREADS, 0, st>>>(n_dev, d, cur.lo, cur.hi, flag, bsplit, bsmall, k_dev, next.lo,
                                                   next.hi, next.parent, small_idx);
    if (lv + 1 < spec_L && next_cap > 0) {
      spec_child_index_kernel<<<(int)((next_cap + TB_THREADS - 1) / TB_THREADS), TB_THREADS, 0, st>>>(
          d_cnt + lv + 1, k_dev, next.parent, lv == 0 ? nullptr : spec_idx[lv & 1], n_roots << lv,
          spec_idx[(lv + 1) & 1]);
      tree->launches += 1;
    }
    if (!fixed) {
      // tiny UNKNOWN leaves: face-centre signs (capacity = this level's bound)
      if (cur_cap * 2 * d > fcap) {
        if (fpts) { cudaFreeAsync(fpts, st); cudaFreeAsync(fvals, st); }
        fcap = cur_cap * 2 * d;
        if (cudaMallocAsync(&fpts, fcap * d * sizeof(double), st) != cudaSuccess ||
            cudaMallocAsync(&fvals, fcap * sizeof(double), st) != cudaSuccess) {
          rc = fail(SPK_ERR_OUT_OF_MEMORY, "face points");
          break;
        }
      }
      const long long np_cap = cur_cap * 2 * d;
      face_points_kernel<<<(int)((np_cap + TB_THREADS - 1) / TB_THREADS), TB_THREADS, 0, st>>>(
          m_dev, d, small_idx, cur.lo, cur.hi, fpts, d_np);
      rc = eval_internal(net, precision, np_cap, d_np, fpts, fvals, st);
      if (rc != SPK_OK) break;
      face_sign_kernel<<<(int)((cur_cap + TB_THREADS - 1) / TB_THREADS), TB_THREADS, 0, st>>>(m_dev, d, small_idx,
                                                                                               fvals, cur.face);
      tree->launches += 3;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { rc = cuda_fail(e, "tree kernels"); break; }
    caps.push_back(cur_cap);
    tree->levels.push_back(cur);
    cur = TreeLevel();
    if (mirror) {
      // this level is final once its kernels ran; copy the PREVIOUS level
      // now, while the GPU works on this one
      cudaEvent_t ev;
      cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      cudaEventRecord(ev, st);
      level_done.push_back(ev);
      // (small levels are mirrored in one batch after the build, mirror_deferred)
      if (lv >= 1 && caps[lv - 1] >= SPK_MIRROR_EAGER_MIN &&
          (rc = mirror_level(tree, lv - 1, tree->levels[lv - 1], d_cnt + lv - 1, level_done[lv - 1], cst)) !=
              SPK_OK)
        break;
    }
    if (next_cap == 0) break;  // no splits (exact) or last fixed depth
    cur = next;
    cur_cap = next_cap;
    (void)k_exact;
  }
  if (mirror && rc == SPK_OK && !tree->levels.empty()) {
    const int last = (int)tree->levels.size() - 1;
    rc = mirror_deferred(tree, d_cnt, level_done[last], cst);
  }
  for (auto ev : level_done) cudaEventDestroy(ev);
  if (cst) cudaStreamDestroy(cst);
  // live sizes of every level, one copy
  if (rc == SPK_OK) {
    std::vector<long long> sizes(tree->levels.size());
    cudaMemcpyAsync(sizes.data(), d_cnt, sizes.size() * sizeof(long long), cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_fail(e, "tree sizes");
    for (size_t l = 0; rc == SPK_OK && l < sizes.size(); ++l) {
      tree->levels[l].n = sizes[l];
      tree->bound_evals += sizes[l];
      float ms = 0.f;
      cudaEventElapsedTime(&ms, bound_ev[2 * l], bound_ev[2 * l + 1]);
      tree->bound_ms += ms;
    }
    // a fixed-depth build whose frontier emptied early ends at the last non-empty level
    while (rc == SPK_OK && !tree->levels.empty() && tree->levels.back().n == 0) {
      free_level(tree->levels.back(), st);
      tree->levels.pop_back();
      if (tree->host.size() > tree->levels.size()) {
        host_block_free(tree->host.back());
        tree->host.pop_back();
        tree->host_n.pop_back();
        if (tree->host_cap.size() > tree->host.size()) tree->host_cap.resize(tree->host.size());
        if (tree->precopied >= (int)tree->host.size()) tree->precopied = -1;
      }
    }
  }
  if (spec_e0) {
    float ms = 0.f;
    if (rc == SPK_OK && cudaEventElapsedTime(&ms, spec_e0, spec_e1) == cudaSuccess) tree->bound_ms += ms;
    cudaEventDestroy(spec_e0);
    cudaEventDestroy(spec_e1);
  }
  if (spec_lo) cudaFreeAsync(spec_lo, st);
  for (auto ev : bound_ev) cudaEventDestroy(ev);
  cudaFreeAsync(d_cnt, st);
  cudaFreeAsync(d_np, st);
  if (cur.lo) free_level(cur, st);
  if (counts) { cudaFreeAsync(counts, st); cudaFreeAsync(flag, st); cudaFreeAsync(small_idx, st); }
  if (fpts) { cudaFreeAsync(fpts, st); cudaFreeAsync(fvals, st); }
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  if (rc != SPK_OK) {
    for (auto& L : tree->levels) free_level(L, st);
    free_mirror(tree);
    delete tree;
    return rc;
  }
  *out = tree;
  return SPK_OK;
}

int spk_tree_destroy(spk_tree* tree) {
  if (!tree) return SPK_OK;
  DeviceGuard g(tree->device);
  for (auto& L : tree->levels) free_level(L, tree->stream);
  free_mirror(tree);
  delete tree;
  return SPK_OK;
}

int spk_tree_release_device(spk_tree* tree) {
  if (!tree) return fail(SPK_ERR_INVALID_PARAMETER, "null tree");
  if (tree->host.size() != tree->levels.size())
    return fail(SPK_ERR_INVALID_PARAMETER, "tree built without SPK_TREE_HOST_MIRROR");
  DeviceGuard g(tree->device);
  for (auto& L : tree->levels) {
    const long long n = L.n;
    free_level(L, tree->stream);
    L.n = n;  // sizes stay readable; device pointers are gone
  }
  tree->device_released = true;
  return SPK_OK;
}

int spk_tree_level_host(const spk_tree* tree, int level, int64_t* n, const double** lo, const double** hi,
                        const double** bound_lo, const double** bound_hi, const int8_t** label,
                        const int8_t** face, const int64_t** parent) {
  if (!tree || level < 0 || level >= (int)tree->levels.size())
    return fail(SPK_ERR_INVALID_PARAMETER, "bad tree level");
  if (level >= (int)tree->host.size() || !tree->host[level])
    return fail(SPK_ERR_INVALID_PARAMETER, "tree built without SPK_TREE_HOST_MIRROR");
  const size_t d = (size_t)tree->d;
  const size_t c = level < (int)tree->host_cap.size() ? (size_t)tree->host_cap[level] : (size_t)tree->host_n[level];
  const char* h = tree->host[level];
  if (n) *n = (int64_t)tree->host_n[level];
  // sections of c rows each (c = the level's row count, or its capacity for
  // a level copied before its count was known), live rows first
  if (lo) *lo = reinterpret_cast<const double*>(h);
  if (hi) *hi = reinterpret_cast<const double*>(h + c * d * 8);
  if (bound_lo) *bound_lo = reinterpret_cast<const double*>(h + 2 * c * d * 8);
  if (bound_hi) *bound_hi = reinterpret_cast<const double*>(h + 2 * c * d * 8 + c * 8);
  if (label) *label = reinterpret_cast<const int8_t*>(h + 2 * c * d * 8 + 2 * c * 8);
  if (face) *face = reinterpret_cast<const int8_t*>(h + 2 * c * d * 8 + 2 * c * 8 + c);
  if (parent) *parent = reinterpret_cast<const int64_t*>(h + 2 * c * d * 8 + 2 * c * 8 + 2 * c);
  return SPK_OK;
}

int spk_tree_info(const spk_tree* tree, int* n_levels, int64_t* n_nodes, int64_t* bound_evals) {
  if (!tree) return fail(SPK_ERR_INVALID_PARAMETER, "null tree");
  long long total = 0;
  for (auto& L : tree->levels) total += L.n;
  if (n_levels) *n_levels = (int)tree->levels.size();
  if (n_nodes) *n_nodes = total;
  if (bound_evals) *bound_evals = tree->bound_evals;
  return SPK_OK;
}

int spk_tree_level_copy(const spk_tree* tree, int level, double* lo, double* hi, double* bound_lo,
                        double* bound_hi, int8_t* label, int8_t* face, int64_t* parent) {
  if (!tree || level < 0 || level >= (int)tree->levels.size())
    return fail(SPK_ERR_INVALID_PARAMETER, "bad tree level");
  if (tree->device_released) return fail(SPK_ERR_INVALID_PARAMETER, "device levels released (host mirror only)");
  DeviceGuard g(tree->device);
  const TreeLevel& L = tree->levels[level];
  const size_t n = (size_t)L.n, d = (size_t)tree->d;
  struct { void* dst; const void* src; size_t bytes; } cp[] = {
      {lo, L.lo, n * d * sizeof(double)}, {hi, L.hi, n * d * sizeof(double)},
      {bound_lo, L.blo, n * sizeof(double)}, {bound_hi, L.bhi, n * sizeof(double)},
      {label, L.label, n}, {face, L.face, n}, {parent, L.parent, n * sizeof(int64_t)}};
  for (auto& c : cp) {
    if (!c.dst || !c.bytes) continue;
    cudaError_t e = cudaMemcpy(c.dst, c.src, c.bytes, cudaMemcpyDefault);
    if (e != cudaSuccess) return cuda_fail(e, "tree level copy");
  }
  return SPK_OK;
}

int spk_tree_stats(const spk_tree* tree, int64_t* launches, double* bound_ms) {
  if (!tree) return fail(SPK_ERR_INVALID_PARAMETER, "null tree");
  if (launches) *launches = tree->launches;
  if (bound_ms) *bound_ms = tree->bound_ms;
  return SPK_OK;
}

int spk_tree_level(const spk_tree* tree, int level, int64_t* n, const double** lo, const double** hi,
                   const double** bound_lo, const double** bound_hi, const int8_t** label, const int8_t** face,
                   const int64_t** parent) {
  if (!tree || level < 0 || level >= (int)tree->levels.size())
    return fail(SPK_ERR_INVALID_PARAMETER, "bad tree level");
  const TreeLevel& L = tree->levels[level];
  if (n) *n = L.n;
  if (tree->device_released && (lo || hi || bound_lo || bound_hi || label || face || parent))
    return fail(SPK_ERR_INVALID_PARAMETER, "device levels released (host mirror only)");
  if (lo) *lo = L.lo;
  if (hi) *hi = L.hi;
  if (bound_lo) *bound_lo = L.blo;
  if (bound_hi) *bound_hi = L.bhi;
  if (label) *label = L.label;
  if (face) *face = L.face;
  if (parent) *parent = reinterpret_cast<const int64_t*>(L.parent);
  return SPK_OK;
}

}  // extern "C"
