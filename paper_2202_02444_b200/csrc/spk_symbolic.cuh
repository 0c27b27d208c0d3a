// K3: symbol-carrying policies -- affine-truncate:n_keep and affine-full
// (range_core.py:595-619; definitional truncate/condense :433-464).
//
// Same fused pass as the fixed-shape kernel (dense layers = one contraction
// over all C = KC + 2 columns of the tile: base, KC symbol columns, error),
// with a block-cooperative epilogue per activation:
//   A. every (neuron, box): interval of the current form, sound rule
//      (alpha, beta, gamma), base/coefficients scaled by alpha, rounding into
//      the error channel; gamma becomes the candidate new symbol of that
//      neuron (a diagonal column, never materialised);
//   B. per box: L1 norm of every live old symbol over all neurons (warp
//      shuffles + fixed-order cross-warp sum, deterministic);
//   C. per box, one warp: keep the n_keep largest candidates by (norm desc,
//      index asc) -- the reference's stable argsort: a 32-step
//      binary search for the n_keep-th largest norm bit pattern with warp
//      REDUX counts, then ballot prefixes keep ties in index order; kept
//      symbols stay in index order;
//   D. every (neuron, box): rebuild the row in the kept order and fold the
//      dropped |coefficients| into the error channel with round-up adds.
// affine-full is the same path with nothing ever dropped (capacity KC must
// hold s + sum of activation widths).  The symbol count is uniform across
// boxes (it depends only on layer widths), so every box has the same layout.
#pragma once
#include <type_traits>
#include "spk_kernels.cuh"

namespace spk {

struct SymParams {
  int n_keep;  // truncate: kept symbols; full: capacity
  int full;    // 1 = affine-full (never drop)
  int s0;      // symbols of the input boxes
};

template <typename T, int KC, int MMAX>
struct SymCfg {
  static constexpr int C = KC + 2;
  using CF = Cfg<T, C, MMAX>;
  static constexpr int NB = CF::NB;
  static constexpr int NWB = CF::NG >= 32 ? CF::NG / 32 : 1;  // warps per box (partials)
  static constexpr int CAND = KC + MMAX;                        // max candidates per activation
  // extra shared memory after X / W ring / narrow buffer
  static constexpr size_t EXTRA = sizeof(T) * (size_t)NB * MMAX      // NEWG: gamma of new symbols
                                  + sizeof(T) * (size_t)NB * NWB * KC      // partial norms
                                  + sizeof(int) * (size_t)NB * KC * 2;     // KEPT, SLOTOLD
  static constexpr size_t SMEM = CF::SMEM + EXTRA + 64;
};

// Apply one activation to all rows of the tile (steps A-D above).
template <typename T, int KC, int MMAX>
SPK_DEV void sym_activation(int act, int m_out, int& nsym, const SymParams& P, T* __restrict__ X,
                            T* __restrict__ NEWG, T* __restrict__ PART, int* __restrict__ KEPT,
                            int* __restrict__ SLOTOLD, int tid) {
  using SC = SymCfg<T, KC, MMAX>;
  using CF = typename SC::CF;
  constexpr int C = SC::C, TI = CF::TI, CP = CF::CP, NB = CF::NB, NG = CF::NG;
  static_assert(CF::TB == 1, "symbolic tiles hold one box per thread");
  if (act == ACT_IDENTITY) return;  // range_core.py:586-587
  const int ng = tid % NG, bg = tid / NG;
  const int n_old = nsym;

  // ---- A: rule, scale, candidate gammas, partial norms
  T pn[KC];
#pragma unroll
  for (int j = 0; j < KC; ++j) pn[j] = T(0);
#pragma unroll
  for (int ti = 0; ti < TI; ++ti) {
    const int i = CF::neuron(ng, ti);
    T* row = X + CF::xrow(i) + bg * CP;
    if (i >= m_out) {
      continue;
    }
    T A[KC];
    T base = row[0], e = row[C - 1];
    T rA = T(0);
#pragma unroll
    for (int j = 0; j < KC; ++j) {
      A[j] = row[1 + j];
      rA = Num<T>::add_ru(rA, fabs(A[j]));
    }
    const T r = Num<T>::add_ru(rA, e);
    T a, b, g;
    const int kind = affine_rule<T>(act, Num<T>::sub_rd(base, r), Num<T>::add_ru(base, r), a, b, g);
    if (kind == 1) {
      base = T(0);
      e = T(0);
#pragma unroll
      for (int j = 0; j < KC; ++j) A[j] = T(0);
      g = T(0);
    } else if (kind == 2) {
      const T nb = Num<T>::fma_rn(a, base, b);
#pragma unroll
      for (int j = 0; j < KC; ++j) A[j] = Num<T>::mul_rn(a, A[j]);
      const T aa = fabs(a);
      T ne = Num<T>::mul_ru(aa, e);
      ne = Num<T>::fma_ru(Num<T>::RHO, Num<T>::add_ru(fabs(nb), Num<T>::mul_ru(aa, rA)), ne);
      e = Num<T>::add_ru(ne, Num<T>::TINY);
      base = nb;
    }
    row[0] = base;
    row[C - 1] = e;
#pragma unroll
    for (int j = 0; j < KC; ++j) {
      row[1 + j] = A[j];
      pn[j] += fabs(A[j]);
    }
    NEWG[bg * MMAX + i] = g;
  }
  // ---- B: per-box norms of the old symbols (deterministic reduction)
  constexpr int LANES = NG < 32 ? NG : 32;
#pragma unroll
  for (int j = 0; j < KC; ++j) {
#pragma unroll
    for (int off = LANES / 2; off > 0; off >>= 1) pn[j] += __shfl_xor_sync(0xffffffffu, pn[j], off);
  }
  if (ng % LANES == 0) {
#pragma unroll
    for (int j = 0; j < KC; ++j) PART[(bg * SC::NWB + ng / 32) * KC + j] = pn[j];
  }
  csync();

  // ---- C: selection, one warp per box
  const int total = n_old + m_out;
  const bool keep_all = P.full || total <= P.n_keep;
  const int n_new = keep_all ? total : P.n_keep;
  const int warp = tid >> 5, lane = tid & 31;
  for (int b = warp; b < NB; b += NT / 32) {
    int* kept = KEPT + b * KC;
    int* slot_old = SLOTOLD + b * KC;
    if (keep_all) {
      for (int p = lane; p < KC; p += 32) {
        kept[p] = p < total ? p : -1;
        slot_old[p] = p < n_old ? p : -1;
      }
      continue;
    }
    // candidate c: c < n_old -> old symbol norm, else gamma of neuron c - n_old
    auto norm_of = [&](int c) -> T {
      if (c < n_old) {
        T v = T(0);
        for (int w = 0; w < SC::NWB; ++w) v += PART[(b * SC::NWB + w) * KC + c];
        return v;
      }
      return fabs(NEWG[b * MMAX + (c - n_old)]);
    };
    // Top-n_keep by (norm desc, index asc) -- the reference's stable argsort
    // (SPEC.md:215).  Norms are >= 0, so their IEEE bit patterns order like
    // the values: binary-search the n_keep-th largest key K with warp-wide
    // counts (REDUX), keep every key > K and the lowest-index keys == K.
    using KeyT = typename std::conditional<sizeof(T) == 4, unsigned, unsigned long long>::type;
    constexpr int PER = (SC::CAND + 31) / 32;
    constexpr int KBITS = 8 * (int)sizeof(KeyT);
    KeyT key[PER];
    bool valid[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int c = lane + 32 * q;
      valid[q] = c < total;
      const T v = valid[q] ? norm_of(c) : T(0);
      if constexpr (sizeof(T) == 4) key[q] = __float_as_uint((float)v);
      else key[q] = (KeyT)__double_as_longlong((double)v);
    }
    KeyT klo = 0, khi = ~(KeyT)0;
    for (int it = 0; it < KBITS && klo < khi; ++it) {
      const KeyT mid = klo + (khi - klo) / 2 + 1;
      unsigned cnt = 0;
#pragma unroll
      for (int q = 0; q < PER; ++q) cnt += (valid[q] && key[q] >= mid) ? 1u : 0u;
      cnt = __reduce_add_sync(0xffffffffu, cnt);
      if (cnt >= (unsigned)P.n_keep) klo = mid;
      else khi = mid - 1;
    }
    const KeyT kth = klo;
    unsigned greater = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) greater += (valid[q] && key[q] > kth) ? 1u : 0u;
    greater = __reduce_add_sync(0xffffffffu, greater);
    const int need_eq = P.n_keep - (int)greater;
    // kept flags in index order (candidate c = lane + 32 q: q-major, lane-minor)
    const unsigned lt = (1u << lane) - 1u;
    int eq_seen = 0, kept_seen = 0;
    for (int p = lane; p < KC; p += 32) slot_old[p] = -1;
    __syncwarp();
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const bool eq = valid[q] && key[q] == kth;
      const unsigned meq = __ballot_sync(0xffffffffu, eq);
      const bool keep = (valid[q] && key[q] > kth) || (eq && eq_seen + __popc(meq & lt) < need_eq);
      eq_seen += __popc(meq);
      const unsigned mk = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int slot = kept_seen + __popc(mk & lt);
        const int c = lane + 32 * q;
        kept[slot] = c;
        if (c < n_old) slot_old[c] = slot;
      }
      kept_seen += __popc(mk);
    }
    for (int p = P.n_keep + lane; p < KC; p += 32) kept[p] = -1;
  }
  csync();

  // ---- D: rebuild rows in kept order, fold dropped columns into e
#pragma unroll
  for (int ti = 0; ti < TI; ++ti) {
    const int i = CF::neuron(ng, ti);
    if (i >= m_out) continue;
    T* row = X + CF::xrow(i) + bg * CP;
    const int* kept = KEPT + bg * KC;
    const int* slot_old = SLOTOLD + bg * KC;
    const T g = NEWG[bg * MMAX + i];
    T e = row[C - 1];
    T nA[KC];
    bool mine_kept = false;
#pragma unroll
    for (int p = 0; p < KC; ++p) {
      const int src = kept[p];
      T v = T(0);
      if (src >= 0 && src < n_old) v = row[1 + src];
      if (src == n_old + i) { v = g; mine_kept = true; }
      nA[p] = v;
    }
#pragma unroll
    for (int j = 0; j < KC; ++j)
      if (j < n_old && slot_old[j] < 0) e = Num<T>::add_ru(e, fabs(row[1 + j]));
    if (!mine_kept) e = Num<T>::add_ru(e, fabs(g));
#pragma unroll
    for (int p = 0; p < KC; ++p) row[1 + p] = nA[p];
    row[C - 1] = e;
  }
  nsym = n_new;
  csync();
}

// Hidden dense layer + its activations + packing for the next layer.
template <typename T, int KC, int MMAX>
SPK_DEV void sym_layer(const LayerDev<T>& L, int& nsym, const SymParams& P, T* __restrict__ X,
                       WRing<T, KC + 2, MMAX>& ring, T* NEWG, T* PART, int* KEPT, int* SLOTOLD, int tid) {
  using SC = SymCfg<T, KC, MMAX>;
  using CF = typename SC::CF;
  constexpr int C = SC::C, TI = CF::TI, TB = CF::TB, CP = CF::CP;
  const int ng = tid % CF::NG, bg = tid / CF::NG;
  T acc[TI][TB][C];
  dense_kloop<T, C, MMAX>(L, X, ring, tid, acc);
  // raw state -> rows (the K loop is done: every thread passed the last barrier)
#pragma unroll
  for (int ti = 0; ti < TI; ++ti) {
    const int i = CF::neuron(ng, ti);
    T* row = X + CF::xrow(i) + bg * CP;
    const bool valid = i < L.m_out;
    const T be = valid ? L.berr[i] : T(0);
#pragma unroll
    for (int c = 0; c < CP; ++c) {
      T v = T(0);
      if (valid && c < C) v = (c == C - 1) ? Num<T>::add_ru(acc[ti][0][C - 1], be) : acc[ti][0][c];
      row[c] = v;
    }
  }
  csync();
  for (int a = 0; a < L.n_act; ++a)
    sym_activation<T, KC, MMAX>(L.act[a], L.m_out, nsym, P, X, NEWG, PART, KEPT, SLOTOLD, tid);
  // pack: v = e + gamma' (|base| + sum|A| + e) for the next dense layer
#pragma unroll
  for (int ti = 0; ti < TI; ++ti) {
    const int i = CF::neuron(ng, ti);
    if (i >= L.m_out) continue;
    T* row = X + CF::xrow(i) + bg * CP;
    T rA = T(0);
#pragma unroll
    for (int j = 0; j < KC; ++j) rA = Num<T>::add_ru(rA, fabs(row[1 + j]));
    const T e = row[C - 1];
    row[C - 1] = Num<T>::fma_ru(L.gamma_next, Num<T>::add_ru(Num<T>::add_ru(fabs(row[0]), rA), e), e);
  }
  csync();
}

template <typename T, int KC, int MMAX>
__global__ void __launch_bounds__(NT, 1)
    sym_bound_kernel(const NetDev<T> net, const BoxInput in, const BoundOutput out, const long long n_cap,
                     const SymParams P) {
  const long long n = in.n_dev ? *in.n_dev : n_cap;
  using SC = SymCfg<T, KC, MMAX>;
  using CF = typename SC::CF;
  constexpr int C = SC::C, NB = CF::NB;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  T* Wst = X + CF::XS;
  T* NBUF = Wst + CF::NS * CF::TILE;
  T* NEWG = NBUF + CF::NBUF;
  T* PART = NEWG + (size_t)NB * MMAX;
  int* KEPT = reinterpret_cast<int*>(PART + (size_t)NB * SC::NWB * KC);
  int* SLOTOLD = KEPT + NB * KC;
  uint64_t* full = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(SLOTOLD + NB * KC) + 15) & ~(uintptr_t)15);  // full[16], empty[16]
  const int tid = threadIdx.x;

  const long long nbt = (n + NB - 1) / NB;
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
  const int per_pass = net.tiles_per_pass / Cfg<T, C, MMAX>::TSCALE;
  WRing<T, C, MMAX> ring{Wst, full, released, net.wtiles, per_pass, mine * per_pass, 0};
  ring.prologue(tid);

  for (long long tile = blockIdx.x; tile < nbt; tile += gridDim.x) {
    const long long g0 = tile * NB;
    if (CF::TEAMSYNC) csync();  // the final (team-local) layer of the previous tile is done
    prep_inputs<T, C, MMAX, MODE_AFFINE>(net, in, n, g0, X, tid, true);
    csync();
    int nsym = P.s0;
    for (int l = 0; l < net.n_layers; ++l) {
      const LayerDev<T>& L = net.L[l];
      if (l == net.n_layers - 1) {
        // final width-1 layer: activations after it only widen the error
        // channel, which leaves lo/hi identical to appending a symbol
        auto emit = [&](int b, const State<T, C, MODE_AFFINE>& st) {
          if (g0 + b < n) emit_bounds<T, C, MODE_AFFINE>(out, node_of(in, g0 + b, n), st);
        };
        narrow_layer<T, C, MMAX, MODE_AFFINE>(L, X, NBUF, tid, true, T(0), emit);
      } else {
        sym_layer<T, KC, MMAX>(L, nsym, P, X, ring, NEWG, PART, KEPT, SLOTOLD, tid);
      }
    }
  }
}

template <typename T, int KC, int MMAX>
cudaError_t launch_sym(const NetDev<T>& net, const BoxInput& in, const BoundOutput& out, long long n,
                       const SymParams& P, int sm_count, cudaStream_t stream) {
  using SC = SymCfg<T, KC, MMAX>;
  auto kfn = sym_bound_kernel<T, KC, MMAX>;
  static std::atomic<unsigned long long> optin{0};
  if (cudaError_t e = smem_optin((const void*)kfn, (int)SC::SMEM, optin)) return e;
  if (n <= 0) return cudaSuccess;
  const long long nbt = (n + SC::NB - 1) / SC::NB;
  const int grid = (int)(nbt < sm_count ? nbt : sm_count);
  kfn<<<grid, NT, SC::SMEM, stream>>>(net, in, out, n, P);
  return cudaGetLastError();
}

template <typename T, int MMAX>
cudaError_t dispatch_sym(int kc, const NetDev<T>& net, const BoxInput& in, const BoundOutput& out, long long n,
                         const SymParams& P, int sm, cudaStream_t st);

#define SPK_DEFINE_SYM_DISPATCH(T, MMAX, KCMAX)                                                         \
  template <>                                                                                          \
  cudaError_t dispatch_sym<T, MMAX>(int kc, const NetDev<T>& net, const BoxInput& in,                   \
                                    const BoundOutput& out, long long n, const SymParams& P, int sm,    \
                                    cudaStream_t st) {                                                  \
    if (kc <= 8) return launch_sym<T, 8, MMAX>(net, in, out, n, P, sm, st);                             \
    if (kc <= 16 || KCMAX <= 16) return launch_sym<T, 16, MMAX>(net, in, out, n, P, sm, st);            \
    return launch_sym<T, (KCMAX > 16 ? KCMAX : 16), MMAX>(net, in, out, n, P, sm, st);                  \
  }

}  // namespace spk
