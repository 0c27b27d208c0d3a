// Persistent bound / point-evaluation kernels built on spk_pass.cuh and
// their host launchers.  Instantiated per (precision, MMAX) in
// spk_inst_*.cu so nvcc compiles them in parallel.
#pragma once
#include <mutex>
#include "spk_pass.cuh"

namespace spk {

enum InputKind : int { IN_BOXES = 0, IN_AABB = 1, IN_RANDOM = 2, IN_POINTS = 3 };

struct BoxInput {
  int kind;
  int s;                   // axes per box (IN_BOXES)
  const double* a;         // centres / AABB lo / points
  const double* b;         // axes / AABB hi
  long long first;         // IN_RANDOM: stream offset
  unsigned long long seed; // IN_RANDOM
  double half;             // IN_RANDOM: cube half-extent
  const long long* n_dev;  // optional device-side count (<= the launch's n): sync-free loops
  int pair_order = 0;      // tree levels [low halves; high halves]: slot 2p+c processes node p + c*n/2,
                           // so a box group holds two sibling boxes (coherent live-row masks)
  const int* perm = nullptr;  // optional processing order: slot gb processes box perm[gb] (spk_order.cu)
  int spread = 0;             // small batch spread over every SM (see spread_node)
  int small = 0;              // few-hundred-box batch: the SM = 1 tile (Cfg), FP32, width 256
  long long spread_n = 0;     // spread: host-side box count (capacity when n_dev is given)
};

// Node processed by slot `gb` of a launch over n boxes (identity unless a
// processing order is given).  Every box's bound is independent of the others,
// so the order never changes a result.
SPK_DEV long long node_of(const BoxInput& in, long long gb, long long n) {
  if (gb >= n) return -1;
  if (in.perm) return in.perm[gb];
  if (!in.pair_order || (n & 1)) return gb;
  return (gb >> 1) + (gb & 1) * (n >> 1);
}

// Spread mode (a batch with fewer box groups than the grid has): the kernel
// runs one tile per CTA over grid x NB slots and box group p (TB boxes) goes
// to CTA p mod grid, group slot p / grid -- the first groups land on warp 0 of
// every CTA, i.e. one SM sub-partition each, instead of filling a few CTAs.
// Empty slots return -1 (their groups skip the K loops through the live-row
// masks).  Boxes of a group: siblings (p, p + n/2) under pair_order, else
// p*TB + c.
template <int TB, int NBG>
SPK_DEV long long spread_node(const BoxInput& in, long long slot, long long n, int grid) {
  constexpr int NB = TB * NBG;
  const long long cta = slot / NB;
  const int r = (int)(slot % NB), grp = r / TB, c = r % TB;
  const long long p = (long long)grp * grid + cta;
  long long node;
  if (in.pair_order && TB == 2 && !(n & 1)) {
    node = p < (n >> 1) ? p + c * (n >> 1) : -1;
  } else {
    node = p * TB + c;
  }
  return (node >= 0 && node < n) ? node : -1;
}

struct BoundOutput {
  double* lo;   // bounds (or point values)
  double* hi;   // may be null for points
  int8_t* cls;  // may be null
};

#ifndef SPK_RELU_SPECIAL
#define SPK_RELU_SPECIAL 1  // FP32 affine passes of ReLU-only nets run a ReLU-specialised kernel
#endif
#ifndef SPK_ELU_POINT
#define SPK_ELU_POINT 1  // ELU-only nets: FP32 point passes with the activation constant-folded (RL = 2)
#endif
#ifndef SPK_PREFETCH_INPUTS
#define SPK_PREFETCH_INPUTS 0  // L2 prefetch of the next tile's inputs (prefetch_tile; measured: C1 +-0, C2 tree +2% -- off)
#endif

// splitmix64 finaliser; the C5 box stream.
SPK_DEV unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
SPK_DEV double random_coord(unsigned long long seed, long long idx, int k, int d) {
  const unsigned long long z = mix64(seed + 0x9E3779B97F4A7C15ull * (unsigned long long)(idx * d + k + 1));
  return (double)(z >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

// Inputs of one tile of NB boxes -> X rows [0, d) (packed columns), zeros
// in rows [d, MMAX).  Shared by the fixed-shape and the symbol-carrying kernels.
template <typename T, int C, int MMAX, int MODE, int SM = 0>
SPK_DEV void prep_inputs(const NetDev<T>& net, const BoxInput& in, long long n, long long g0, T* X, int tid,
                         bool pack) {
  using CF = Cfg<T, C, MMAX, SM>;
  constexpr int NB = CF::NB, CP = CF::CP;
  const int d = net.d;
  // the first layer reads rows [0, d) plus the zero pad row of its
  // double-buffered k-pair; every other row is rewritten by its epilogue
  const int rows = ((d + 1) & ~1) < MMAX ? ((d + 1) & ~1) : MMAX;
  for (int q = tid; q < rows * NB; q += NT) {
    const int k = q / NB, b = q % NB;
    const long long gb = in.spread ? spread_node<CF::TB, CF::NBG>(in, g0 + b, n, (int)gridDim.x)
                                   : node_of(in, g0 + b, n);
    T packed[CP];
#pragma unroll
    for (int c = 0; c < CP; ++c) packed[c] = T(0);
    if (k < d && gb >= 0) {
      State<T, C, MODE> st;
      double centre;
      double ax[MAX_AXES];
#pragma unroll
      for (int j = 0; j < MAX_AXES; ++j) ax[j] = 0.0;
      int n_ax = 0;
      if (in.kind == IN_BOXES || in.kind == IN_POINTS) {
        centre = in.a[gb * d + k];
        if (in.kind == IN_BOXES) {
          n_ax = in.s < MAX_AXES ? in.s : MAX_AXES;
#pragma unroll
          for (int j = 0; j < MAX_AXES; ++j)
            if (j < n_ax) ax[j] = in.b[(gb * in.s + j) * d + k];
        }
      } else if (in.kind == IN_AABB) {
        const double l = in.a[gb * d + k], h = in.b[gb * d + k];
        centre = (l + h) / 2.0;  // spatial.py:182-183, exact halving
        n_ax = d < MAX_AXES ? d : MAX_AXES;
#pragma unroll
        for (int j = 0; j < MAX_AXES; ++j)
          if (j == k) ax[j] = (h - l) / 2.0;
      } else {
        centre = random_coord(in.seed, in.first + gb, k, d);
        n_ax = d < MAX_AXES ? d : MAX_AXES;
#pragma unroll
        for (int j = 0; j < MAX_AXES; ++j)
          if (j == k) ax[j] = in.half;
      }
      input_state<T, C, MODE>(centre, ax, n_ax, 1, st);
      if (pack) {
        for (int a = 0; a < net.n_pre; ++a) apply_act<T, C, MODE>(st, net.pre_act[a]);
        pack_next<T, C, MODE>(st, net.gamma_first, packed);
      } else {
        packed[0] = st.base;
        if (MODE == MODE_AFFINE) {
#pragma unroll
          for (int j = 0; j < State<T, C, MODE>::S; ++j) packed[1 + j] = st.A[j];
        }
        packed[C - 1] = st.e;
      }
    }
    T* dst = X + CF::xrow(k) + (b / CF::TB) * CF::GS;
#pragma unroll
    for (int c = 0; c < CP; ++c)
      if (!CF::IL || c < C) dst[CF::xcol(b % CF::TB, c)] = packed[c];
  }
}

// L2 prefetch of a future tile's FP64 inputs (box corners / centres + axes):
// the first layer of a tile otherwise waits on DRAM latency with every warp
// idle (C1: ~6% long-scoreboard stalls).  Contiguous slot ranges only (natural
// order, or the two sibling halves of a tree level); no registers held.
SPK_DEV void prefetch_l2(const void* p, size_t bytes, int tid) {
  const char* c = reinterpret_cast<const char*>((reinterpret_cast<uintptr_t>(p)) & ~uintptr_t(127));
  const char* e = reinterpret_cast<const char*>(p) + bytes;
  for (const char* q = c + (size_t)tid * 128; q < e; q += (size_t)NT * 128)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
}
template <int NB>
SPK_DEV void prefetch_tile(const BoxInput& in, int d, long long g0, long long n, int tid) {
  if (SPK_PREFETCH_INPUTS == 0 || g0 >= n || in.perm || in.spread || in.n_dev) return;
  if (in.kind != IN_BOXES && in.kind != IN_AABB && in.kind != IN_POINTS) return;
  const long long cnt = (g0 + NB < n ? NB : n - g0);
  const int sb = in.kind == IN_BOXES ? in.s : (in.kind == IN_AABB ? 1 : 0);
  auto range = [&](long long first, long long count) {
    prefetch_l2(in.a + first * d, (size_t)count * d * 8, tid);
    if (sb) prefetch_l2(in.b + first * sb * d, (size_t)count * sb * d * 8, tid);
  };
  if (in.pair_order && !(n & 1)) {  // slots 2p+c -> nodes p + c n/2
    range(g0 >> 1, (cnt + 1) >> 1);
    range((g0 >> 1) + (n >> 1), (cnt + 1) >> 1);
  } else {
    range(g0, cnt);
  }
}

template <typename T, int C, int MODE>
SPK_DEV void emit_bounds(const BoundOutput& out, long long gb, const State<T, C, MODE>& st) {
  double lo, hi;
  final_bounds<T, C, MODE>(st, lo, hi);
  out.lo[gb] = lo;
  if (out.hi) out.hi[gb] = hi;
  if (out.cls) out.cls[gb] = (int8_t)(lo > 0.0 ? 1 : (hi < 0.0 ? -1 : 0));
}

template <typename T, int C, int MMAX, int MODE, int SM = 0, int RL = 0>
__global__ void __launch_bounds__(NT, (Cfg<T, C, MMAX, SM>::MINB))
    bound_kernel(const NetDev<T> net, const BoxInput in, const BoundOutput out, const long long n_cap) {
  using CF = Cfg<T, C, MMAX, SM>;
  // real box count; spread mode runs over grid x NB slots
  const long long n = in.n_dev ? *in.n_dev : (in.spread ? in.spread_n : n_cap);
  constexpr int NB = CF::NB;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  T* Wst = X + CF::XS;
  T* NBUF = Wst + CF::NS * CF::TILE;
  uint64_t* full = reinterpret_cast<uint64_t*>(NBUF + CF::NBUF);
  const int tid = threadIdx.x;

  const long long n_slots = in.spread ? (long long)gridDim.x * NB : n;
  const long long nbt = (n_slots + NB - 1) / NB;
  const long long mine = blockIdx.x < nbt ? (nbt - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  unsigned* released = reinterpret_cast<unsigned*>(full + 16);
  if (tid == 0) {
    for (int s = 0; s < CF::NS; ++s) {
      mbar_init(&full[s], 1);
      released[s] = 0u;
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int per_pass = net.tiles_per_pass / CF::TSCALE;
  WRing<T, C, MMAX, SM> ring{Wst, full, released, net.wtiles, per_pass, mine * per_pass, 0};
  if (CF::LIVE) ring.live = reinterpret_cast<uint32_t*>(released + 16);
  ring.prologue(tid);

  for (long long tile = blockIdx.x; tile < nbt; tile += gridDim.x) {
    const long long g0 = tile * NB;
    if (CF::TEAMSYNC) csync();  // every team is done with the previous tile's X
    prep_inputs<T, C, MMAX, MODE, SM>(net, in, n, g0, X, tid, true);
    prefetch_tile<NB>(in, net.d, g0 + (long long)gridDim.x * NB, n, tid);
    auto node = [&](int b) -> long long {
      return in.spread ? spread_node<CF::TB, CF::NBG>(in, g0 + b, n, (int)gridDim.x) : node_of(in, g0 + b, n);
    };
    // a box group without boxes (spread padding, the tail tile) marks no live rows
    if (CF::LIVE) ring.group_empty = node((tid / CF::NG) * CF::TB) < 0;
    csync();
    auto emit = [&](int b, const State<T, C, MODE>& st) {
      const long long nd = node(b);
      if (nd >= 0) emit_bounds<T, C, MODE>(out, nd, st);
    };
    run_layers<T, C, MMAX, MODE, decltype(emit)&, SM, RL>(net, X, NBUF, ring, tid, emit);
  }
}

// ------------------------------------------------------------- launchers
template <typename T, int C, int MMAX, int MODE, int SM = 0, int RL = 0>
cudaError_t launch_bound(const NetDev<T>& net, const BoxInput& in, const BoundOutput& out, long long n,
                         int sm_count, cudaStream_t stream) {
  using CF = Cfg<T, C, MMAX, SM>;
  auto kfn = bound_kernel<T, C, MMAX, MODE, SM, RL>;
  static std::atomic<unsigned long long> optin{0};
  if (cudaError_t e = smem_optin((const void*)kfn, (int)CF::SMEM, optin)) return e;
  if (n <= 0) return cudaSuccess;
  const long long nbt = (n + CF::NB - 1) / CF::NB;
  const long long slots = (long long)sm_count * CF::MINB;
  const int grid = in.spread ? sm_count : (int)(nbt < slots ? nbt : slots);
  kfn<<<grid, NT, CF::SMEM, stream>>>(net, in, out, n);
  return cudaGetLastError();
}

// Per-(T, MMAX) dispatch on mode and S; defined in spk_inst_<T>_<MMAX>.cu.
template <typename T, int MMAX>
cudaError_t dispatch_bound(int mode, int S, const NetDev<T>& net, const BoxInput& in,
                           const BoundOutput& out, long long n, int sm_count, cudaStream_t stream);

template <typename T, int MMAX>
struct KTOf {
  static constexpr int KT = Cfg<T, 1, MMAX>::KT_BASE;   // host tile rows
  static constexpr int PAD = Cfg<T, 1, MMAX>::KT_PAD;   // layers padded to a multiple of this
  static constexpr int SUB = Cfg<T, 1, MMAX>::SUB;
};

#define SPK_DEFINE_DISPATCH(T, MMAX)                                                                  \
  template <>                                                                                         \
  cudaError_t dispatch_bound<T, MMAX>(int mode, int S, const NetDev<T>& net, const BoxInput& in,       \
                                      const BoundOutput& out, long long n, int sm, cudaStream_t st) { \
    if constexpr (sizeof(T) == 4 && MMAX == 256) {                                                    \
      if (in.small && mode == MODE_INTERVAL)                                                          \
        return launch_bound<T, 2, MMAX, MODE_INTERVAL, 1>(net, in, out, n, sm, st);                   \
      if (in.small && mode == MODE_AFFINE && S == 3)                                                  \
        return net.relu_net == 1 ? launch_bound<T, 5, MMAX, MODE_AFFINE, 1, 1>(net, in, out, n, sm, st) \
                            : launch_bound<T, 5, MMAX, MODE_AFFINE, 1>(net, in, out, n, sm, st);       \
    }                                                                                                 \
    /* ReLU-only nets, FP32 affine cubes (the configs): the specialised pass */                       \
    if constexpr (sizeof(T) == 4 && SPK_RELU_SPECIAL)                                                 \
      if (mode == MODE_AFFINE && S == 3 && net.relu_net == 1)                                         \
        return launch_bound<T, 5, MMAX, MODE_AFFINE, 0, 1>(net, in, out, n, sm, st);                  \
    if constexpr (sizeof(T) == 4 && SPK_ELU_POINT)                                                    \
      if (mode == MODE_POINT && net.relu_net == 2)                                                    \
        return launch_bound<T, 1, MMAX, MODE_POINT, 0, 2>(net, in, out, n, sm, st);                   \
    if (mode == MODE_POINT) return launch_bound<T, 1, MMAX, MODE_POINT>(net, in, out, n, sm, st);      \
    if (mode == MODE_INTERVAL) return launch_bound<T, 2, MMAX, MODE_INTERVAL>(net, in, out, n, sm, st); \
    switch (S) {                                                                                      \
      case 0: return launch_bound<T, 2, MMAX, MODE_AFFINE>(net, in, out, n, sm, st);                  \
      case 1: return launch_bound<T, 3, MMAX, MODE_AFFINE>(net, in, out, n, sm, st);                  \
      case 2: return launch_bound<T, 4, MMAX, MODE_AFFINE>(net, in, out, n, sm, st);                  \
      case 3: return launch_bound<T, 5, MMAX, MODE_AFFINE>(net, in, out, n, sm, st);                  \
      default: return launch_bound<T, MAX_AXES + 2, MMAX, MODE_AFFINE>(net, in, out, n, sm, st);      \
    }                                                                                                 \
  }

}  // namespace spk
