// K7: hierarchical marching cubes (extract_mesh, meshing.py:111-169).
//
// 1. Prune: integer index-range blocks, level by level (3*(m-l) levels):
//    world box from the linspace grid coordinates (meshing.py:23-26,
//    reproduced exactly: i*step + lo, last = hi), fused bound kernel,
//    keep lo <= 0 <= hi, split the widest index range at lo + size//2 with
//    the children interleaved (a0, b0, a1, b1, ...) as meshing.py:152-162
//    builds them; ballot/prefix compaction as in the tree build.
// 2. Dense stage per chunk of surviving blocks: the (S+1)^3 corner lattice of
//    every block (meshgrid 'ij' order, meshing.py:87-97); the chunk's distinct
//    grid corners (blocks share face lattices) go through the point-evaluation
//    pass once and are scattered back; per cell the case code (bit c set when corner c
//    < 0), triangle count from the reference's generated TRI_TABLE
//    (mc_tables.py:72-95), exclusive scan, and emission of every triangle
//    vertex as (global edge key, interpolated position) in exactly the
//    reference's visiting order (blocks, then cells in argwhere order, then
//    table order).
// 3. Dedup (meshing.py:38-52): stable key sort of all triangle vertices; the
//    first occurrence of a key fixes its position (the reference interpolates
//    from the first visiting cell's corner orientation), run heads become
//    vertices, every triangle vertex gets its run's id.
// Scans and the dedup sort use CUB (CUDA toolkit library code).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include <cub/cub.cuh>

#include "spk_kernels.cuh"
#include "spk_abi_internal.h"

namespace spk {

constexpr int MK = 256;

#ifndef SPK_MESH_DEDUP
#define SPK_MESH_DEDUP 1  // evaluate each distinct grid corner of a chunk once
#endif

struct GridDev {
  double lo[3], hi[3], step[3];
  int n;  // cells per axis
};

SPK_DEV double grid_coord(const GridDev& G, int axis, int i) {
  // np.linspace: arange * step + start, endpoint forced to stop
  return i == G.n ? G.hi[axis] : __dadd_rn(__dmul_rn((double)i, G.step[axis]), G.lo[axis]);
}

__constant__ int8_t c_tri[256 * 15];   // up to 5 triangles x 3 edges per case
__constant__ uint8_t c_ntri[256];
__constant__ int8_t c_corner[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                      {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
__constant__ int8_t c_edge[12][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6},
                                     {6, 7}, {7, 4}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};

__global__ void block_boxes_kernel(long long nb, const int* __restrict__ org, int sx, int sy, int sz, GridDev G,
                                   double* __restrict__ blo, double* __restrict__ bhi) {
  const long long q = (long long)blockIdx.x * MK + threadIdx.x;
  if (q >= nb) return;
  const int s[3] = {sx, sy, sz};
  for (int a = 0; a < 3; ++a) {
    const int i0 = org[q * 3 + a];
    blo[q * 3 + a] = grid_coord(G, a, i0);
    bhi[q * 3 + a] = grid_coord(G, a, i0 + s[a]);
  }
}

// keep = UNKNOWN (lo <= 0 <= hi); per-block counts of kept
__global__ void keep_count_kernel(long long nb, const int8_t* __restrict__ cls, int* __restrict__ bcnt) {
  const long long q = (long long)blockIdx.x * MK + threadIdx.x;
  const bool f = q < nb && cls[q] == 0;
  __shared__ int wc[MK / 32];
  const unsigned m = __ballot_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0) wc[threadIdx.x >> 5] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < MK / 32; ++w) s += wc[w];
    bcnt[blockIdx.x] = s;
  }
}

// kept block j (rank) -> children 2j (low half) and 2j+1 (high half) on
// axis `ax` at offset `half` (index units); or a plain compaction (ax < 0)
__global__ void keep_split_kernel(long long nb, const int8_t* __restrict__ cls, const int* __restrict__ org,
                                  const long long* __restrict__ boff, int ax, int half, int* __restrict__ out) {
  const long long q = (long long)blockIdx.x * MK + threadIdx.x;
  const bool f = q < nb && cls[q] == 0;
  __shared__ int wc[MK / 32];
  const unsigned m = __ballot_sync(0xffffffffu, f);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) wc[w] = __popc(m);
  __syncthreads();
  if (!f) return;
  int before = 0;
  for (int v = 0; v < w; ++v) before += wc[v];
  const long long j = boff[blockIdx.x] + before + __popc(m & ((1u << lane) - 1u));
  if (ax < 0) {
    for (int a = 0; a < 3; ++a) out[j * 3 + a] = org[q * 3 + a];
    return;
  }
  for (int a = 0; a < 3; ++a) {
    out[(2 * j) * 3 + a] = org[q * 3 + a];
    out[(2 * j + 1) * 3 + a] = org[q * 3 + a] + (a == ax ? half : 0);
  }
}

// corner lattice of each block, meshgrid('ij') order (k fastest)
__global__ void corner_points_kernel(long long nb, const int* __restrict__ org, int S, GridDev G,
                                     double* __restrict__ pts) {
  const int P = S + 1;
  const long long q = (long long)blockIdx.x * MK + threadIdx.x;
  if (q >= nb * P * P * P) return;
  const long long b = q / (P * P * P);
  const int r = (int)(q % (P * P * P));
  const int a = r / (P * P), bb = (r / P) % P, c = r % P;
  pts[q * 3 + 0] = grid_coord(G, 0, org[b * 3 + 0] + a);
  pts[q * 3 + 1] = grid_coord(G, 1, org[b * 3 + 1] + bb);
  pts[q * 3 + 2] = grid_coord(G, 2, org[b * 3 + 2] + c);
}

// global grid index of every corner of the chunk's lattices (the dedup key)
__global__ void corner_keys_kernel(long long nb, const int* __restrict__ org, int S, long long np1,
                                   unsigned long long* __restrict__ keys, long long* __restrict__ idx) {
  const int P = S + 1;
  const long long q = (long long)blockIdx.x * MK + threadIdx.x;
  if (q >= nb * P * P * P) return;
  const long long b = q / (P * P * P);
  const int r = (int)(q % (P * P * P));
  const int a = r / (P * P), bb = (r / P) % P, c = r % P;
  keys[q] = (unsigned long long)(((long long)(org[b * 3 + 0] + a) * np1 + (org[b * 3 + 1] + bb)) * np1 +
                                 (org[b * 3 + 2] + c));
  idx[q] = q;
}

// unique corners of a sorted key run: the head of each run writes its point
__global__ void unique_points_kernel(long long n, const unsigned long long* __restrict__ sk,
                                     const long long* __restrict__ sidx, const int* __restrict__ runid,
                                     const double* __restrict__ pts, double* __restrict__ upts) {
  const long long q = (long long)blockIdx.x * MK + threadIdx.x;
  if (q >= n || !(q == 0 || sk[q] != sk[q - 1])) return;
  const long long u = runid[q] - 1, src = sidx[q];
  for (int x = 0; x < 3; ++x) upts[u * 3 + x] = pts[src * 3 + x];
}

// every lattice corner takes its unique point's value
__global__ void scatter_values_kernel(long long n, const long long* __restrict__ sidx, const int* __restrict__ runid,
                                      const double* __restrict__ uvals, double* __restrict__ vals) {
  const long long q = (long long)blockIdx.x * MK + threadIdx.x;
  if (q < n) vals[sidx[q]] = uvals[runid[q] - 1];
}

SPK_DEV int cell_case(const double* __restrict__ v, int P, int a, int b, int c) {
  int code = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double x = v[((a + c_corner[k][0]) * P + (b + c_corner[k][1])) * P + (c + c_corner[k][2])];
    code |= (x < 0.0 ? 1 : 0) << k;
  }
  return code;
}

__global__ void cell_count_kernel(long long nb, int S, const double* __restrict__ vals, int* __restrict__ cnt) {
  const int P = S + 1;
  const long long q = (long long)blockIdx.x * MK + threadIdx.x;
  if (q >= nb * S * S * S) return;
  const long long b = q / (S * S * S);
  const int r = (int)(q % (S * S * S));
  const int a = r / (S * S), bb = (r / S) % S, c = r % S;
  cnt[q] = c_ntri[cell_case(vals + b * P * P * P, P, a, bb, c)];
}

__global__ void cell_emit_kernel(long long nb, int S, const int* __restrict__ org, const double* __restrict__ vals,
                                 const int* __restrict__ off, long long base_tri, GridDev G,
                                 unsigned long long* __restrict__ keys, double* __restrict__ pos) {
  const int P = S + 1;
  const long long q = (long long)blockIdx.x * MK + threadIdx.x;
  if (q >= nb * S * S * S) return;
  const long long b = q / (S * S * S);
  const int r = (int)(q % (S * S * S));
  const int a = r / (S * S), bb = (r / S) % S, c = r % S;
  const double* v = vals + b * P * P * P;
  const int code = cell_case(v, P, a, bb, c);
  const int nt = c_ntri[code];
  if (nt == 0) return;
  const long long np1 = (long long)G.n + 1;
  const int cell[3] = {org[b * 3 + 0] + a, org[b * 3 + 1] + bb, org[b * 3 + 2] + c};
  long long t0 = base_tri + off[q];
  for (int t = 0; t < nt; ++t) {
    for (int s = 0; s < 3; ++s) {
      const int e = c_tri[code * 15 + t * 3 + s];
      const int ca = c_edge[e][0], cb = c_edge[e][1];
      int ia[3], ib[3];
      for (int x = 0; x < 3; ++x) {
        ia[x] = cell[x] + c_corner[ca][x];
        ib[x] = cell[x] + c_corner[cb][x];
      }
      const double fa = v[((a + c_corner[ca][0]) * P + (bb + c_corner[ca][1])) * P + (c + c_corner[ca][2])];
      const double fb = v[((a + c_corner[cb][0]) * P + (bb + c_corner[cb][1])) * P + (c + c_corner[cb][2])];
      const double tt = __ddiv_rn(__dsub_rn(0.0, fa), __dsub_rn(fb, fa));
      const long long ent = (t0 + t) * 3 + s;
      int axis = 0;
      for (int x = 0; x < 3; ++x)
        if (ia[x] != ib[x]) axis = x;
      int lowc[3];
      for (int x = 0; x < 3; ++x) lowc[x] = min(ia[x], ib[x]);
      keys[ent] = (unsigned long long)(((long long)lowc[0] * np1 + lowc[1]) * np1 + lowc[2]) * 3ull + axis;
      for (int x = 0; x < 3; ++x) {
        const double pa = grid_coord(G, x, ia[x]), pb = grid_coord(G, x, ib[x]);
        pos[ent * 3 + x] = __dadd_rn(pa, __dmul_rn(tt, __dsub_rn(pb, pa)));
      }
    }
  }
}

__global__ void all_blocks_kernel(long long nb, int per_axis, int S, int* __restrict__ org) {
  const long long q = (long long)blockIdx.x * MK + threadIdx.x;
  if (q >= nb) return;
  const long long pa = per_axis;
  org[q * 3 + 0] = (int)(q / (pa * pa)) * S;
  org[q * 3 + 1] = (int)((q / pa) % pa) * S;
  org[q * 3 + 2] = (int)(q % pa) * S;
}

// first stream position of every vertex run (its head's entry index)
__global__ void run_first_kernel(long long n, const unsigned long long* __restrict__ sk,
                                 const long long* __restrict__ sidx, const int* __restrict__ runid,
                                 long long* __restrict__ first, int* __restrict__ run_iota) {
  const long long q = (long long)blockIdx.x * MK + threadIdx.x;
  if (q >= n) return;
  if (q == 0 || sk[q] != sk[q - 1]) {
    const int r = runid[q] - 1;
    first[r] = sidx[q];
    run_iota[r] = r;
  }
}

__global__ void invert_kernel(long long nv, const int* __restrict__ order, int* __restrict__ rank) {
  const long long q = (long long)blockIdx.x * MK + threadIdx.x;
  if (q < nv) rank[order[q]] = (int)q;
}

__global__ void iota_kernel(long long n, long long* __restrict__ v) {
  const long long q = (long long)blockIdx.x * MK + threadIdx.x;
  if (q < n) v[q] = q;
}

__global__ void run_head_kernel(long long n, const unsigned long long* __restrict__ sk, int* __restrict__ head) {
  const long long q = (long long)blockIdx.x * MK + threadIdx.x;
  if (q < n) head[q] = (q == 0 || sk[q] != sk[q - 1]) ? 1 : 0;
}

// head[] inclusive-scanned -> run ids; runs renumbered by first visit
// (the reference's vertex order); write vertices and triangle indices
__global__ void dedup_emit_kernel(long long n, const unsigned long long* __restrict__ sk,
                                  const long long* __restrict__ sidx, const int* __restrict__ runid,
                                  const int* __restrict__ rank, const double* __restrict__ pos,
                                  double* __restrict__ verts, unsigned long long* __restrict__ vkeys,
                                  long long* __restrict__ tris) {
  const long long q = (long long)blockIdx.x * MK + threadIdx.x;
  if (q >= n) return;
  const int id = rank[runid[q] - 1];
  const long long ent = sidx[q];
  tris[ent] = id;
  if (q == 0 || sk[q] != sk[q - 1]) {  // first (stable) occurrence fixes the position
    for (int x = 0; x < 3; ++x) verts[(long long)id * 3 + x] = pos[ent * 3 + x];
    vkeys[id] = sk[q];
  }
}

}  // namespace spk

struct spk_mesh {
  int device = 0;
  cudaStream_t stream = nullptr;
  long long n_vertices = 0, n_triangles = 0, n_blocks = 0, evals = 0, bound_evals = 0;
  long long block_first = 0, blocks_total = 0;  // this shard's slice of the surviving blocks
  double* verts = nullptr;                // n_vertices x 3
  unsigned long long* vkeys = nullptr;    // n_vertices (edge keys)
  long long* tris = nullptr;              // n_triangles x 3
  double eval_ms = 0.0, bound_ms = 0.0;
};

using namespace spk;

namespace {

struct Pool {
  cudaStream_t st;
  std::vector<void*> owned;
  cudaError_t err = cudaSuccess;
  template <typename P>
  P* get(size_t count) {
    void* p = nullptr;
    if (err == cudaSuccess) err = cudaMallocAsync(&p, std::max<size_t>(count * sizeof(P), 16), st);
    if (p) owned.push_back(p);
    return reinterpret_cast<P*>(p);
  }
  void release() {
    for (void* p : owned) cudaFreeAsync(p, st);
    owned.clear();
  }
  ~Pool() { release(); }  // stream-ordered frees: safe while kernels still read
};

// exclusive per-CUDA-block offsets of a small count array (host side)
int host_offsets(const int* d_cnt, int nblk, std::vector<long long>& offs, long long* total, long long* d_offs,
                 cudaStream_t st) {
  std::vector<int> h(nblk);
  cudaError_t e = cudaMemcpyAsync(h.data(), d_cnt, nblk * sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "mesh offsets");
  offs.resize(nblk);
  long long s = 0;
  for (int b = 0; b < nblk; ++b) {
    offs[b] = s;
    s += h[b];
  }
  *total = s;
  e = cudaMemcpyAsync(d_offs, offs.data(), nblk * sizeof(long long), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? SPK_OK : cuda_fail(e, "mesh offsets");
}

}  // namespace

extern "C" {

int spk_mesh_extract(const spk_net* net, int policy, int n_keep, int precision, const double* lo3, const double* hi3,
                     int m, int dense_levels, int prune, const int8_t* tri_table, const uint8_t* tri_count,
                     void* stream, spk_mesh** out) {
  return spk_mesh_extract_shard(net, policy, n_keep, precision, lo3, hi3, m, dense_levels, prune, tri_table,
                                tri_count, 0, 1, stream, out);
}

int spk_mesh_extract_shard(const spk_net* net, int policy, int n_keep, int precision, const double* lo3,
                           const double* hi3, int m, int dense_levels, int prune, const int8_t* tri_table,
                           const uint8_t* tri_count, int shard, int n_shards, void* stream, spk_mesh** out) {
  if (!net || !out || !tri_table || !tri_count) return fail(SPK_ERR_INVALID_PARAMETER, "null argument");
  if (n_shards < 1 || shard < 0 || shard >= n_shards) return fail(SPK_ERR_INVALID_PARAMETER, "bad shard index");
  *out = nullptr;
  if (net->input_dim != 3) return fail(SPK_ERR_DIMENSION, "meshing needs a 3-d network");
  if (m <= dense_levels || dense_levels < 0) return fail(SPK_ERR_INVALID_PARAMETER, "ResolutionTooSmall");
  if (m > 20) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "resolution exponent above 20");
  for (int a = 0; a < 3; ++a)
    if (!(hi3[a] > lo3[a]) || !std::isfinite(lo3[a]) || !std::isfinite(hi3[a]))
      return fail(SPK_ERR_INVALID_PARAMETER, "bounds must have positive extent");
  DeviceGuard g(net->device);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyToSymbolAsync(c_tri, tri_table, 256 * 15, 0, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyToSymbolAsync(c_ntri, tri_count, 256, 0, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "mesh tables");
  const int n = 1 << m;
  GridDev G;
  G.n = n;
  for (int a = 0; a < 3; ++a) {
    G.lo[a] = lo3[a];
    G.hi[a] = hi3[a];
    G.step[a] = (hi3[a] - lo3[a]) / (double)n;  // linspace: delta / div
  }
  auto mesh = new spk_mesh();
  mesh->device = net->device;
  mesh->stream = st;
  Pool pool{st};
  int rc = SPK_OK;
  cudaEvent_t ev0, ev1;
  cudaEventCreate(&ev0);
  cudaEventCreate(&ev1);

  // ---------------------------------------------------------------- prune
  int sz[3] = {n, n, n};
  int* org = pool.get<int>(3);
  {
    int z[3] = {0, 0, 0};
    cudaMemcpyAsync(org, z, sizeof(z), cudaMemcpyHostToDevice, st);
  }
  long long nb = 1;
  const int levels = prune ? 3 * (m - dense_levels) : 0;
  const int S = 1 << dense_levels;
  if (!prune) {  // dense extraction: every block of side 2^l, no bounds
    const long long pa = n / S;
    nb = pa * pa * pa;
    org = pool.get<int>(nb * 3);
    if (pool.err != cudaSuccess) rc = cuda_fail(pool.err, "mesh alloc");
    else all_blocks_kernel<<<(int)((nb + MK - 1) / MK), MK, 0, st>>>(nb, (int)pa, S, org);
  }
  for (int lev = 0; prune && lev <= levels && rc == SPK_OK && nb > 0; ++lev) {
    double* blo = pool.get<double>(nb * 3);
    double* bhi = pool.get<double>(nb * 3);
    double* rlo = pool.get<double>(nb);
    double* rhi = pool.get<double>(nb);
    int8_t* cls = pool.get<int8_t>(nb);
    const int nblk = (int)((nb + MK - 1) / MK);
    int* bcnt = pool.get<int>(nblk);
    long long* boff = pool.get<long long>(nblk);
    if (pool.err != cudaSuccess) { rc = cuda_fail(pool.err, "mesh alloc"); break; }
    block_boxes_kernel<<<nblk, MK, 0, st>>>(nb, org, sz[0], sz[1], sz[2], G, blo, bhi);
    cudaEventRecord(ev0, st);
    rc = spk_bound_aabb(net, policy, n_keep, precision, nb, blo, bhi, rlo, rhi, cls, st);
    cudaEventRecord(ev1, st);
    if (rc != SPK_OK) break;
    mesh->bound_evals += nb;
    keep_count_kernel<<<nblk, MK, 0, st>>>(nb, cls, bcnt);
    std::vector<long long> offs;
    long long kept = 0;
    if ((rc = host_offsets(bcnt, nblk, offs, &kept, boff, st)) != SPK_OK) break;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev0, ev1);
    mesh->bound_ms += ms;
    const bool last = lev == levels;
    int ax = -1, half = 0;
    if (!last) {
      ax = 0;
      for (int a = 1; a < 3; ++a)
        if (sz[a] > sz[ax]) ax = a;  // np.argmax: first maximum
      half = sz[ax] / 2;
    }
    const long long nn = last ? kept : 2 * kept;
    int* nxt = pool.get<int>(std::max<long long>(nn, 1) * 3);
    if (pool.err != cudaSuccess) { rc = cuda_fail(pool.err, "mesh alloc"); break; }
    if (kept > 0) keep_split_kernel<<<nblk, MK, 0, st>>>(nb, cls, org, boff, ax, half, nxt);
    org = nxt;
    nb = nn;
    if (!last) sz[ax] = half;  // blocks at a level share their sizes
  }
  // sharding (C4 across GPUs): every shard runs the (cheap)
  // prune redundantly and extracts a contiguous slice of the surviving blocks
  // in visiting order; the slices' triangles, concatenated in shard order, are
  // the unsharded visiting order (meshing.gather_mesh dedups the vertices)
  {
    const long long base = nb / n_shards, extra = nb % n_shards;
    const long long first = shard * base + std::min<long long>(shard, extra);
    const long long count = base + (shard < extra ? 1 : 0);
    mesh->blocks_total = nb;
    mesh->block_first = first;
    org = org + first * 3;
    nb = count;
  }
  mesh->n_blocks = nb;

  // ------------------------------------------------------ dense extraction
  std::vector<unsigned long long*> chunk_keys;
  std::vector<double*> chunk_pos;
  std::vector<long long> chunk_tris;
  long long total_tris = 0;
  const int P = S + 1;
  const long long cells_per = (long long)S * S * S, pts_per = (long long)P * P * P;
  const long long CH = std::max<long long>(1, std::min<long long>(nb, (16ll << 20) / pts_per));
  for (long long b0 = 0; rc == SPK_OK && b0 < nb; b0 += CH) {
    // per-chunk scratch (lattice points, values, counts, corner dedup) is
    // released at the end of the chunk (stream-ordered): memory stays
    // O(chunk), not O(mesh) -- a 1024^3 extraction has ~100 chunks
    Pool cp{st};
    const long long cb = std::min(CH, nb - b0);
    const int* corg = org + b0 * 3;
    double* pts = cp.get<double>(cb * pts_per * 3);
    double* vals = cp.get<double>(cb * pts_per);
    int* cnt = cp.get<int>(cb * cells_per);
    int* off = cp.get<int>(cb * cells_per);
    if (cp.err != cudaSuccess) { rc = cuda_fail(cp.err, "mesh alloc"); break; }
    const long long np_ = cb * pts_per, nc = cb * cells_per;
    corner_points_kernel<<<(int)((np_ + MK - 1) / MK), MK, 0, st>>>(cb, corg, S, G, pts);
    long long n_eval = np_;
    if (SPK_MESH_DEDUP && cb > 1) {
      // adjacent surviving blocks share their face lattices: evaluate every
      // distinct grid corner of the chunk once (sort by global index, unique,
      // evaluate, scatter back) -- the values are deterministic per point, so
      // the mesh is unchanged; ~30% fewer evaluations on dense regions
      const int gblk = (int)((np_ + MK - 1) / MK);
      unsigned long long* ck = cp.get<unsigned long long>(np_);
      unsigned long long* sk = cp.get<unsigned long long>(np_);
      long long* ci = cp.get<long long>(np_);
      long long* si = cp.get<long long>(np_);
      int* head = cp.get<int>(np_);
      int* runid = cp.get<int>(np_);
      if (cp.err != cudaSuccess) { rc = cuda_fail(cp.err, "mesh alloc"); break; }
      corner_keys_kernel<<<gblk, MK, 0, st>>>(cb, corg, S, (long long)G.n + 1, ck, ci);
      size_t tb = 0, tb2 = 0;
      const int key_bits = 64 - __builtin_clzll((unsigned long long)((long long)(G.n + 1) * (G.n + 1) * (G.n + 1)));
      cub::DeviceRadixSort::SortPairs(nullptr, tb, ck, sk, ci, si, (int)np_, 0, key_bits, st);
      cub::DeviceScan::InclusiveSum(nullptr, tb2, head, runid, (int)np_, st);
      void* tmp = cp.get<char>(std::max(tb, tb2));
      if (cp.err != cudaSuccess) { rc = cuda_fail(cp.err, "mesh alloc"); break; }
      cub::DeviceRadixSort::SortPairs(tmp, tb, ck, sk, ci, si, (int)np_, 0, key_bits, st);
      run_head_kernel<<<gblk, MK, 0, st>>>(np_, sk, head);
      cub::DeviceScan::InclusiveSum(tmp, tb2, head, runid, (int)np_, st);
      int nu = 0;
      cudaMemcpyAsync(&nu, runid + np_ - 1, 4, cudaMemcpyDeviceToHost, st);
      e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) { rc = cuda_fail(e, "mesh corner dedup"); break; }
      double* upts = cp.get<double>((long long)nu * 3);
      double* uvals = cp.get<double>(nu);
      if (cp.err != cudaSuccess) { rc = cuda_fail(cp.err, "mesh alloc"); break; }
      unique_points_kernel<<<gblk, MK, 0, st>>>(np_, sk, si, runid, pts, upts);
      cudaEventRecord(ev0, st);
      rc = spk_eval_batch(net, precision, nu, upts, uvals, st);
      cudaEventRecord(ev1, st);
      if (rc != SPK_OK) break;
      scatter_values_kernel<<<gblk, MK, 0, st>>>(np_, si, runid, uvals, vals);
      n_eval = nu;
    } else {
      cudaEventRecord(ev0, st);
      rc = spk_eval_batch(net, precision, np_, pts, vals, st);
      cudaEventRecord(ev1, st);
      if (rc != SPK_OK) break;
    }
    mesh->evals += n_eval;
    cell_count_kernel<<<(int)((nc + MK - 1) / MK), MK, 0, st>>>(cb, S, vals, cnt);
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, off, (int)nc, st);
    void* tmp = cp.get<char>(tmp_bytes);
    if (cp.err != cudaSuccess) { rc = cuda_fail(cp.err, "mesh alloc"); break; }
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, off, (int)nc, st);
    int last_cnt = 0, last_off = 0;
    cudaMemcpyAsync(&last_cnt, cnt + nc - 1, 4, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&last_off, off + nc - 1, 4, cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { rc = cuda_fail(e, "mesh scan"); break; }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev0, ev1);
    mesh->eval_ms += ms;
    const long long ntri = (long long)last_cnt + last_off;
    unsigned long long* keys = nullptr;
    double* pos = nullptr;
    if (ntri > 0) {
      keys = pool.get<unsigned long long>(ntri * 3);  // kept until the dedup below
      pos = pool.get<double>(ntri * 9);
      if (pool.err != cudaSuccess) { rc = cuda_fail(pool.err, "mesh alloc"); break; }
      cell_emit_kernel<<<(int)((nc + MK - 1) / MK), MK, 0, st>>>(cb, S, corg, vals, off, 0, G, keys, pos);
    }
    chunk_keys.push_back(keys);
    chunk_pos.push_back(pos);
    chunk_tris.push_back(ntri);
    total_tris += ntri;
  }

  // ------------------------------------------------------------- dedup
  if (rc == SPK_OK && total_tris > 0) {
    const long long ne = total_tris * 3;
    unsigned long long* keys = pool.get<unsigned long long>(ne);
    double* pos = pool.get<double>(ne * 3);
    if (pool.err != cudaSuccess) rc = cuda_fail(pool.err, "mesh alloc");
    long long at = 0;
    for (size_t c = 0; rc == SPK_OK && c < chunk_tris.size(); ++c) {
      if (!chunk_tris[c]) continue;
      cudaMemcpyAsync(keys + at, chunk_keys[c], chunk_tris[c] * 3 * 8, cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(pos + at * 3, chunk_pos[c], chunk_tris[c] * 9 * 8, cudaMemcpyDeviceToDevice, st);
      at += chunk_tris[c] * 3;
    }
    long long* idx = pool.get<long long>(ne);
    long long* sidx = pool.get<long long>(ne);
    unsigned long long* sk = pool.get<unsigned long long>(ne);
    int* head = pool.get<int>(ne);
    int* runid = pool.get<int>(ne);
    if (pool.err != cudaSuccess) rc = cuda_fail(pool.err, "mesh alloc");
    if (rc == SPK_OK) {
      const int nblk = (int)((ne + MK - 1) / MK);
      iota_kernel<<<nblk, MK, 0, st>>>(ne, idx);
      size_t tb = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, sk, idx, sidx, (int)ne, 0, 64, st);
      void* tmp = pool.get<char>(tb);
      size_t tb2 = 0;
      cub::DeviceScan::InclusiveSum(nullptr, tb2, head, runid, (int)ne, st);
      void* tmp2 = pool.get<char>(tb2);
      if (pool.err != cudaSuccess) rc = cuda_fail(pool.err, "mesh alloc");
      if (rc == SPK_OK) {
        cub::DeviceRadixSort::SortPairs(tmp, tb, keys, sk, idx, sidx, (int)ne, 0, 64, st);
        run_head_kernel<<<nblk, MK, 0, st>>>(ne, sk, head);
        cub::DeviceScan::InclusiveSum(tmp2, tb2, head, runid, (int)ne, st);
        int nv = 0;
        cudaMemcpyAsync(&nv, runid + ne - 1, 4, cudaMemcpyDeviceToHost, st);
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) rc = cuda_fail(e, "mesh dedup");
        mesh->n_vertices = nv;
        mesh->n_triangles = total_tris;
        // renumber runs by first visit: sort runs by their first stream position
        long long* first = pool.get<long long>(nv);
        long long* first_s = pool.get<long long>(nv);
        int* riota = pool.get<int>(nv);
        int* order = pool.get<int>(nv);
        int* rank = pool.get<int>(nv);
        size_t tb3 = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb3, first, first_s, riota, order, nv, 0, 64, st);
        void* tmp3 = pool.get<char>(tb3);
        if (pool.err != cudaSuccess) rc = cuda_fail(pool.err, "mesh alloc");
        if (rc == SPK_OK) {
          run_first_kernel<<<nblk, MK, 0, st>>>(ne, sk, sidx, runid, first, riota);
          cub::DeviceRadixSort::SortPairs(tmp3, tb3, first, first_s, riota, order, nv, 0, 64, st);
          invert_kernel<<<(nv + MK - 1) / MK, MK, 0, st>>>(nv, order, rank);
          e = cudaMallocAsync(&mesh->verts, std::max<long long>(nv, 1) * 24, st);
          if (e == cudaSuccess) e = cudaMallocAsync(&mesh->vkeys, std::max<long long>(nv, 1) * 8, st);
          if (e == cudaSuccess) e = cudaMallocAsync(&mesh->tris, ne * 8, st);
          if (e != cudaSuccess) rc = cuda_fail(e, "mesh output alloc");
          else
            dedup_emit_kernel<<<nblk, MK, 0, st>>>(ne, sk, sidx, runid, rank, pos, mesh->verts, mesh->vkeys,
                                                    mesh->tris);
        }
      }
    }
  }
  if (rc == SPK_OK) {
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_fail(e, "mesh");
  }
  pool.release();
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  if (rc != SPK_OK) {
    if (mesh->verts) cudaFreeAsync(mesh->verts, st);
    if (mesh->vkeys) cudaFreeAsync(mesh->vkeys, st);
    if (mesh->tris) cudaFreeAsync(mesh->tris, st);
    delete mesh;
    return rc;
  }
  *out = mesh;
  return SPK_OK;
}

int spk_mesh_info(const spk_mesh* mesh, int64_t* n_vertices, int64_t* n_triangles, int64_t* n_blocks,
                  int64_t* point_evals, int64_t* bound_evals) {
  if (!mesh) return fail(SPK_ERR_INVALID_PARAMETER, "null mesh");
  if (n_vertices) *n_vertices = mesh->n_vertices;
  if (n_triangles) *n_triangles = mesh->n_triangles;
  if (n_blocks) *n_blocks = mesh->n_blocks;
  if (point_evals) *point_evals = mesh->evals;
  if (bound_evals) *bound_evals = mesh->bound_evals;
  return SPK_OK;
}

int spk_mesh_shard_info(const spk_mesh* mesh, int64_t* block_first, int64_t* blocks_total) {
  if (!mesh) return fail(SPK_ERR_INVALID_PARAMETER, "null mesh");
  if (block_first) *block_first = mesh->block_first;
  if (blocks_total) *blocks_total = mesh->blocks_total;
  return SPK_OK;
}

int spk_mesh_copy(const spk_mesh* mesh, double* vertices, int64_t* triangles, uint64_t* vertex_keys) {
  if (!mesh) return fail(SPK_ERR_INVALID_PARAMETER, "null mesh");
  DeviceGuard g(mesh->device);
  cudaError_t e = cudaSuccess;
  if (vertices && mesh->n_vertices) e = cudaMemcpy(vertices, mesh->verts, mesh->n_vertices * 24, cudaMemcpyDefault);
  if (e == cudaSuccess && triangles && mesh->n_triangles)
    e = cudaMemcpy(triangles, mesh->tris, mesh->n_triangles * 24, cudaMemcpyDefault);
  if (e == cudaSuccess && vertex_keys && mesh->n_vertices)
    e = cudaMemcpy(vertex_keys, mesh->vkeys, mesh->n_vertices * 8, cudaMemcpyDefault);
  return e == cudaSuccess ? SPK_OK : cuda_fail(e, "mesh copy");
}

int spk_mesh_destroy(spk_mesh* mesh) {
  if (!mesh) return SPK_OK;
  DeviceGuard g(mesh->device);
  if (mesh->verts) cudaFreeAsync(mesh->verts, mesh->stream);
  if (mesh->vkeys) cudaFreeAsync(mesh->vkeys, mesh->stream);
  if (mesh->tris) cudaFreeAsync(mesh->tris, mesh->stream);
  delete mesh;
  return SPK_OK;
}

}  // extern "C"
