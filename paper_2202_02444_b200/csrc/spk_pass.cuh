// Fused all-layer network pass over a tile of boxes (the K1/K2/K4 kernels).
//
// One CTA owns NB boxes for the whole network.  Their state lives in shared
// memory as X[k][box][c]: for point evaluation c = {x}; for interval
// arithmetic c = {centre, v}; for affine-fixed c = {base, A_1..A_S, v},
// where v = e + gamma*(|base| + sum|A|) is the error channel pre-inflated by
// the rounding budget of the next dense layer.  A dense layer is then ONE
// contraction of W against all C columns of all NB boxes:
//     base' = W base + b,   A' = W A   (FFMA, round-to-nearest)
//     e'    = |W| v + berr               (FFMA.RP with |W| operand modifier)
// which is exactly the reference's per-layer GEMM (range_core.py:573-582)
// with the error GEMV folded in, plus a rigorous FP32 rounding budget.  The
// epilogue applies the activation rule (range_core.py:583-603) and the
// affine-fixed fold, and writes the next layer's X in place.  The final
// dense layer (width 1) is a warp reduction that emits lo/hi (and the sign
// class).  W streams from L2 through a 3-stage cp.async.bulk (TMA bulk copy)
// + mbarrier ring of KT x MMAX tiles, so the layer loop never waits on HBM.
//
// Register tile per thread: TI consecutive output neurons x TB boxes x C
// columns; all C columns of one (neuron, box) pair are owned by one thread,
// which lets the activation rule run straight out of registers.
#pragma once
#include <type_traits>
#include "spk_common.cuh"
#include "spk_rules.cuh"

namespace spk {

constexpr int MAX_LAYERS = 24;
// Box axes of the fused affine pass: s <= 3 run tiles with exactly s symbol
// columns; 4 <= s <= MAX_AXES run the MAX_AXES-column tile with zero columns
// for the missing axes (exact zeros: identical bounds).  Higher-dimensional
// nets (input_dim <= MAX_AXES) thereby get the reference's exact affine
// forms of their boxes (range_core.py:547-568 is generic in d).
constexpr int MAX_AXES = 8;
constexpr int MAX_ACTS = 4;
constexpr int NT = 256;         // threads per CTA (8 warps)
constexpr int NARROW_MAX = 4;   // dense layers this narrow use the warp-reduction path
#ifndef SPK_SPEC_PREFETCH
#define SPK_SPEC_PREFETCH 1  // unconditional 2-ahead fragment prefetch (see Cfg::SMEM)
#endif
#ifndef SPK_INLINE_POINT_ACT
#define SPK_INLINE_POINT_ACT 1
#endif
#ifndef SPK_F64_DIRECT
#define SPK_F64_DIRECT 1
#endif
#ifndef SPK_SCALAR_UNROLL
#define SPK_SCALAR_UNROLL 8
#endif
#ifndef SPK_SUB_F32
#define SPK_SUB_F32 32  // FP32 blocked-summation length (rounding budget gamma_{SUB + m/SUB + 1})
#endif
#ifndef SPK_NARROW_2CTA
#define SPK_NARROW_2CTA 1
#endif
#ifndef SPK_UNROLL_BLOCK
#define SPK_UNROLL_BLOCK 1  // FP32 K loop: each full blocked-summation chunk fully unrolled
#endif
#ifndef SPK_LIVE_ROWS
#define SPK_LIVE_ROWS 1  // skip all-zero X rows (ReLU-inactive neurons) in the FP32 K loop (Cfg::LIVE)
#endif
#ifndef SPK_LIVE_WARP
#define SPK_LIVE_WARP 1  // narrow nets: warp-union live-row masks (Cfg::LIVE)
#endif
#ifndef SPK_PACKED_ERR
#define SPK_PACKED_ERR 1  // FP32 error column on FFMA2.RP over neuron pairs (bit-identical sums)
#endif
#ifndef SPK_PACKED_ERR_MINW
#define SPK_PACKED_ERR_MINW 128  // measured (round 2): C2 tree -1.2%, C5 width 512 -2.5%, width 64 +2.5%, width 32 +-0
#endif
#ifndef SPK_2CTA_MAXW
#define SPK_2CTA_MAXW 64  // widest FP32 net on the one-box-per-thread, 2-CTA/SM tile (64: C5_64 +3% with masks)
#endif
#ifndef SPK_KT_F32_W64
#define SPK_KT_F32_W64 32  // W tile rows of FP32 width-64 nets (32: live-row masks apply; C5_64 +11%)
#endif
#ifndef SPK_LIVE_DENSE_NARROW
#define SPK_LIVE_DENSE_NARROW 28  // the same for the warp-union masks of narrow nets
#endif
#ifndef SPK_AT32_512
#define SPK_AT32_512 1  // FP32 width-512 affine tile: 32-row W tiles, 2 stages, interleaved X, live-row masks (C5_512 -19%)
#endif
#ifndef SPK_LIVE_DENSE
#define SPK_LIVE_DENSE 28  // tiles with more live rows than this run the unrolled chunk (18: +8%, 23: +1%)
#endif
#ifndef SPK_TEAM_SYNC
#define SPK_TEAM_SYNC 1  // layer boundaries synchronise teams, not the CTA (Cfg::TEAMSYNC)
#endif
#ifndef SPK_TEAM_MIN_NS
#define SPK_TEAM_MIN_NS 4  // ring depth from which layer boundaries are team-local
#endif
#ifndef SPK_KT_POINT512
#define SPK_KT_POINT512 1  // Cfg::PT32: 32-row W tiles for FP32 width-512 point passes (C4 evaluation -10.7%)
#endif
#ifndef SPK_DEFER_RELEASE
#define SPK_DEFER_RELEASE 1  // WRing::DEFER: examine the release atomic one tile later
#endif
#ifndef SPK_DEFER_MIN_NS
#define SPK_DEFER_MIN_NS 4  // ... on rings of at least this many stages
#endif
#ifndef SPK_LIVE_F64
#define SPK_LIVE_F64 1  // live-row masks on the FP64 wide tiles (scalar K loop)
#endif
#ifndef SPK_LIVE_DENSE_F64
#define SPK_LIVE_DENSE_F64 12  // FP64 tiles (KT rows) with more live rows than this x KT/16 run dense
#endif
#ifndef SPK_IL_X
#define SPK_IL_X 0  // interleaved box-group columns on the wide FP32 affine tile (Cfg::IL; measured C2 +12% with the 4th ring stage and team-local syncs, +5.7% without: off)
#endif
#ifndef SPK_X_SKEW
#define SPK_X_SKEW 0  // skewed X rows on wide FP32 tiles (conflict-free epilogue stores; measured C2 +0.8%: off)
#endif
#ifndef SPK_FUSE_FINAL
#define SPK_FUSE_FINAL 1  // ReLU-specialised passes: width-1 output layer folded into the last epilogue
#endif
#ifndef SPK_ONE_BLOCK
#define SPK_ONE_BLOCK 1  // FP32 nets of width <= SPK_SUB_F32: accumulate onto the bias, no partials
#endif
#ifndef SPK_ONE_BLOCK_W64
#define SPK_ONE_BLOCK_W64 0  // width-64 FP32 nets: one summation block per layer + running-error layer (measured: C5_64 +7.5% time for only 1.3x tighter -- off)
#endif
#ifndef SPK_NARROW_TI4
#define SPK_NARROW_TI4 0  // FP32 width-32 affine tile: 4 neurons/thread, 3 CTAs/SM (Cfg::TI4; measured: 80-register cap spills, C1 0.307 -> 0.451 ms)
#endif
#ifndef SPK_RUNERR
#define SPK_RUNERR 1  // FP32 affine K loops: running (a-posteriori) rounding bound of the base column
#endif
#ifndef SPK_F64_BASE
#define SPK_F64_BASE 0  // ... in FP64 instead (DFMA base column on those layers; measured C2 +20%, excess 5.4 -> 4.6%: off)
#endif
#ifndef SPK_FUSED_RELU
#define SPK_FUSED_RELU 1  // affine-fixed ReLU layers: fused rule + pack, straddle branch behind a warp vote
#endif
#ifndef SPK_FUSED_RELU_VOTE
#define SPK_FUSED_RELU_VOTE 0  // the straddle branch behind a warp vote (measured: predicated is 2-4% faster)
#endif
#ifndef SPK_PACKED_F32
#define SPK_PACKED_F32 1  // FP32 K loop on FFMA2 (sm_100a packed f32x2)
#endif
constexpr int kScalarUnroll = SPK_SCALAR_UNROLL;  // FP64 K loop unroll (A/B knob)
constexpr int NSTAGE_MIN = 3;   // W tile ring depth floor (deeper when tiles are small)
constexpr size_t SMEM_BUDGET = 210 * 1024;  // leaves room for the symbolic kernel's extras
constexpr size_t SMEM_MAX_OPTIN = 227 * 1024;  // sm_100 opt-in limit of dynamic shared memory per CTA
constexpr size_t SMEM_BUDGET_IL = 225 * 1024;  // interleaved bound tiles (no symbolic extras)

enum Mode : int {
  MODE_POINT = 0,
  MODE_INTERVAL = 1,
  MODE_AFFINE = 2,
  MODE_MI = 3,  // ray march round: point value + interval bound   (columns: x, c, v)
  MODE_MA = 4   // ray march round: point value + affine-fixed S=1 (columns: x, base, A, v)
};
// bound part of a mode, and the column offset of the bound state
constexpr int bound_mode(int m) { return m == MODE_MI ? MODE_INTERVAL : (m == MODE_MA ? MODE_AFFINE : m); }
constexpr int pv_off(int m) { return m >= MODE_MI ? 1 : 0; }

template <typename T>
struct LayerDev {
  int m_in, m_out;
  int narrow;
  int ntiles;
  int n_act;
  int act[MAX_ACTS];
  const T* w;        // narrow layers: W row-major (m_out x m_in)
  const T* bias;     // m_out
  const T* berr;     // m_out: rounding budget of the bias term, rounded up
  T gamma_next;      // rounding budget factor of the NEXT dense layer (0 after the last)
  T gamma_base_next; // the same for |base| when the next layer's K loop bounds the base
                     // column's rounding a posteriori (runerr): weight rounding only
  int runerr;        // FP32 affine K loops: this layer runs the running-error form
};

template <typename T>
struct NetDev {
  int d;
  int n_layers;
  int n_pre;
  int pre_act[MAX_ACTS];
  T gamma_first;
  int tiles_per_pass;
  int relu_net;      // every dense layer's activations are exactly [] or [ReLU], none before the first
  const T* wtiles;   // generic layers' k-tiles, each KT x MMAX (row k = column k of W)
  LayerDev<T> L[MAX_LAYERS];
};

// SM = 1: the small-batch tile (a box pair per CTA, one neuron per thread,
// two CTAs per SM).  A batch of a few hundred boxes (the top tree levels) is
// latency-bound -- one warp's K-loop chain per layer -- so the 256 output
// neurons of a layer are spread over all 256 threads instead of 32.
template <typename T, int C, int MMAX, int SM = 0>
struct Cfg {
  static constexpr int VEC = 16 / (int)sizeof(T);  // elements per 16-byte vector
  // FP32 width-32 nets with affine columns: 4 neurons per thread and three
  // CTAs per SM (SPK_NARROW_TI4) -- their K loops are 32 steps long, so the
  // tile is latency-bound and more resident warps pay more than register
  // reuse of W across neurons
  static constexpr bool TI4 = SPK_NARROW_TI4 && SM == 0 && sizeof(T) == 4 && MMAX <= 32 && C >= 3 && C <= 6;
  // register tile: TI neurons x TB boxes x C columns per thread
  static constexpr int TI = SM ? 1
                               : (TI4 ? 4
                                      : (C <= 6 ? (sizeof(T) == 4 ? 8 : 4)
                                                : (C <= 20 ? VEC : (VEC / 2 > 0 ? VEC / 2 : 1))));
  // narrow nets (MMAX = 32) with affine columns: one box per thread and two
  // CTAs per SM -- their K loops are short, so latency hiding across CTAs
  // matters more than register reuse across boxes (measured: 4x32 -19%
  // time; at width 64 the 1-CTA, 2-box tile was 17% faster without live-row
  // masks, and the 2-CTA tile is 3% faster with them: FP32 only)
  static constexpr int MINB =
      SM ? 2
         : (TI4 ? 3
                : ((SPK_NARROW_2CTA && (MMAX <= 32 || (sizeof(T) == 4 && MMAX <= SPK_2CTA_MAXW)) && C >= 3 && C <= 6)
                       ? 2
                       : 1));
  static constexpr int TB = SM ? 2
                               : (C == 1 ? (sizeof(T) == 4 ? 8 : 4)
                                         : (C == 2 ? 4 : (C <= 6 ? (MINB == 2 ? 1 : 2) : 1)));
  static constexpr int CP = C == 1 ? 1 : (C == 2 ? 2 : (C <= 4 ? 4 : (C <= 6 ? (TB == 1 ? 8 : 6)
                                                                         : ((C + VEC - 1) / VEC) * VEC)));
  static constexpr int NG = MMAX / TI;
  static constexpr int NBG = NT / NG;
  static constexpr int NB = NBG * TB;
  static constexpr int KT_RAW = 32768 / (MMAX * (int)sizeof(T));
  // FP32 width-512 point passes (X is one column: 72 KB): 32-row W tiles in
  // a 2-stage ring instead of 16-row tiles in 5 -- half the per-tile ring
  // traffic (mbarrier waits and release atomics were ~20% of the stall
  // samples); same blocked-sum order, bit-identical values
  //
  // The host lays W out once per network in KT_BASE-row tiles with every
  // layer padded to a multiple of KT_PAD rows (the largest KT of any kernel
  // of this width), so a kernel with KT = TSCALE * KT_BASE reads the same
  // array as whole pairs of tiles: its tile counts are the host's / TSCALE.
  static constexpr bool PT32 = SPK_KT_POINT512 && sizeof(T) == 4 && MMAX == 512 && C == 1 && SM == 0;
  // FP32 width-512 affine cubes (SPK_AT32_512): the same 32-row tiles in a
  // 2-stage ring, which fits beside X in its interleaved layout (Cfg::IL,
  // 90 KB) and makes the live-row masks available at this width
  static constexpr bool AT32 = SPK_AT32_512 && sizeof(T) == 4 && MMAX == 512 && C == 5 && SM == 0;
  static constexpr int KT_BASE = (sizeof(T) == 4 && MMAX == 64) ? SPK_KT_F32_W64
                                 : (KT_RAW > MMAX ? MMAX : (KT_RAW < 1 ? 1 : KT_RAW));
  static constexpr int KT_PAD = (SPK_KT_POINT512 && sizeof(T) == 4 && MMAX == 512 && SM == 0) ? 32 : KT_BASE;
  static constexpr int KT = (PT32 || AT32) ? 32 : KT_BASE;
  static constexpr int TSCALE = KT / KT_BASE;
  static_assert(KT % KT_BASE == 0 && KT_PAD % KT == 0, "host tile layout");
  // blocked-sum length (FP32); width-64 nets sum each layer as one block
  // (the single-block loop: no partial registers, which lets the narrow
  // 128-register tile carry the running-error layer)
  static constexpr int SUB = sizeof(T) == 4 ? ((MMAX == 64 && SPK_ONE_BLOCK_W64) ? 64 : SPK_SUB_F32) : 1 << 20;
  static constexpr int TILE = KT * MMAX;                 // elements per W tile
  // Interleaved box-group columns (SPK_IL_X; FP32 affine cubes on the wide
  // two-box tile): a box group's 10 values per X row are [b0.base b0.A1 b0.A2
  // b0.A3 | b1.base b1.A1 b1.A2 b1.A3 | b0.err b1.err] -- the K loop's f32x2
  // pairs stay 8-byte aligned without the per-box pad column (CP = 6), so X
  // shrinks by 1/6 and the W ring gains a stage (3 -> 4 at width 256, which
  // also enables the team-local layer boundaries); 5 LDS.64 / STS.64 per
  // row segment instead of 3 LDS.128 / STS.128.
  static constexpr bool IL = (SPK_IL_X || AT32) && sizeof(T) == 4 && C == 5 && TB == 2 && SM == 0;
  static constexpr int GS = IL ? 10 : TB * CP;           // elements of a box group's row segment
  // offset of column c of the group's box tb within its row segment
  SPK_DEV static constexpr int xcol(int tb, int c) { return IL ? (c < 4 ? tb * 4 + c : 8 + tb) : tb * CP + c; }
  // X row stride (elements): 16-byte aligned rows, and an odd number of
  // 16-byte units per row so the epilogue's vector stores spread over banks
  static constexpr int RS0 = ((NBG * GS * (int)sizeof(T) + 15) / 16) * 16 / (int)sizeof(T);
  // a thread's TI neurons: TI/G groups of G consecutive neurons (G elements
  // = one vector load); group q of neuron-group ng starts at q*NG*G + ng*G,
  // so a warp's vector loads of a W row are contiguous (bank-conflict free)
  static constexpr int G = TI < VEC ? TI : VEC;
  // Skewed rows (wide FP32 tiles, SPK_X_SKEW): in the epilogue the lanes of a
  // warp write rows G = 4 apart, so with any row stride that is a multiple of
  // 16 bytes only 2 of the 8 16-byte bank slots are hit (measured: 73% of the
  // epilogue's store wavefronts were conflict replays on the C2 level).  Row r
  // is shifted by ((r / 4) mod 8) 16-byte units: 8 consecutive lanes then hit
  // 8 distinct slots, for 28 extra floats per row.  Readers of a whole row
  // (the K loop: broadcast) only add the row's shift.
  static constexpr int SKEW0 =
      (SPK_X_SKEW && sizeof(T) == 4 && SM == 0 && NG >= 32 && G == 4 && KT % 32 == 0) ? 16 / (int)sizeof(T) : 0;
  static constexpr size_t SKEW_BYTES =
      sizeof(T) * ((size_t)MMAX * (RS0 + 7 * SKEW0) + (size_t)NSTAGE_MIN * KT * MMAX + NB * NARROW_MAX * CP + MMAX) +
      4096;
  static constexpr int SKEW = (SKEW0 && SKEW_BYTES <= SMEM_MAX_OPTIN) ? SKEW0 : 0;
  static constexpr int RS = SKEW ? RS0 + 7 * SKEW
                                 : (((RS0 * (int)sizeof(T) / 16) % 2 == 1) ? RS0 : RS0 + 16 / (int)sizeof(T));
  static constexpr int XS = MMAX * RS;                   // elements of X
  // element offset of X row r
  SPK_DEV static int xrow(int r) { return r * RS + (SKEW ? ((r >> 2) & 7) * SKEW : 0); }
  // (K loops address row t*KT + kk as xrow(t*KT) + xrow(kk): needs KT % 32 == 0)
  static constexpr int NBUF = NB * NARROW_MAX * CP;      // narrow-layer staging
  // W ring depth: as many KT x MMAX tiles as fit beside X (small nets keep
  // every tile of the network resident and never re-stream W)
  // (the interleaved tiles are never used by the symbolic kernel, whose
  // extras the 210 KB budget leaves room for; upper bound of the live-row
  // mask area, exact size LIVE_BYTES below)
  static constexpr long long LIVE_BYTES_EST = 2ll * NBG * (MMAX / 32 > 0 ? MMAX / 32 : 1) * 4 + (NT / 32) * 40 * 4;
  static constexpr long long NS_FIT =
      ((long long)(IL ? SMEM_BUDGET_IL : SMEM_BUDGET) / MINB - (long long)sizeof(T) * (XS + NBUF) - 1024 -
       (long long)LIVE_BYTES_EST) /
      ((long long)sizeof(T) * TILE);
  static constexpr int NS_MIN = (PT32 || AT32) ? 2 : NSTAGE_MIN;
  static constexpr int NS = NS_FIT < NS_MIN ? NS_MIN : (NS_FIT > 16 ? 16 : (int)NS_FIT);
  // + one W row of slack: the K loops prefetch the fragment two rows ahead
  // unconditionally (a predicated prefetch made ptxas copy fragments), so the
  // last step may read one row past the last ring stage (values unused)
  // Live-row masks: one bit per X row per box group, set by the epilogue when
  // any of the group's columns for that neuron is nonzero.  A ReLU-inactive
  // neuron (slope 0) leaves an all-zero row, and FMAs with an exact zero
  // change neither the round-to-nearest sums nor the round-up error column,
  // so the K loop may skip those rows with identical results.  FP32 wide nets
  // (a warp-uniform box group: NG >= 32) with 32-row W tiles (at width 512 the
  // 16-row tiles measured 10% slower masked on random cubes).
  // Narrow nets (NG < 32: a warp holds 32/NG box groups) use one mask per
  // warp -- the union over its box groups, so a skipped row is zero for every
  // box the warp computes (needs a G-neuron group's mask word fixed by ti).
  // FP64 wide tiles (SPK_LIVE_F64): the 16-row W tiles (width 256) use their
  // half of the 32-row mask word, same exactness argument (C2 FP64 build
  // 105.3 -> 96.7 ms); the 8-row tiles of width 512 lost 4% to the list
  // overhead (C5_512 FP64 1289 -> 1339 ms) and stay dense.
  static constexpr bool LIVE =
      SPK_LIVE_ROWS && C >= 2 &&
      ((sizeof(T) == 4 && KT == 32 && (NG >= 32 || (SPK_LIVE_WARP && C >= 3 && 32 % (NG * G) == 0))) ||
       (sizeof(T) == 8 && SPK_LIVE_F64 && SM == 0 && NG >= 32 && KT >= 16 && KT <= 32 && 32 % KT == 0));
  static constexpr int LW = MMAX / 32;  // mask words per box group
  static constexpr int LLIST = 40;  // per-warp live-row list (<= 32 rows + 2 pad entries)
  static constexpr size_t LIVE_BYTES = LIVE ? (size_t)2 * NBG * LW * 4 + (size_t)(NT / 32) * LLIST * 4 : 0;
  static constexpr size_t SMEM = sizeof(T) * (size_t)(XS + NS * TILE + NBUF + MMAX) + 2 * 16 * 8 + 64 + LIVE_BYTES;
  static_assert(NG >= 1 && NG <= NT && NT % NG == 0, "tile shape");
  static_assert(!SKEW || KT % 32 == 0, "skewed rows need 32-row W tiles");
  static_assert((TB * CP * sizeof(T)) % 16 == 0, "vector loads of X");
  static_assert(TI % G == 0, "W vector groups");
  SPK_DEV static int neuron(int ng, int ti) { return (ti / G) * (NG * G) + ng * G + (ti % G); }
  // A box group's X columns are read (K loop) and rewritten (epilogue) only
  // by the threads that own it: the NG threads tid in [bg*NG, (bg+1)*NG).
  // Those form a "team" -- TEAM = NG/32 whole warps, or (NG <= 32) one warp
  // holding 32/NG box groups -- which is all a layer boundary has to
  // synchronise (named barrier per team, or __syncwarp); the W ring keeps the
  // teams within NS tiles of each other.
  static constexpr int TEAM = NG >= 32 ? NG / 32 : 1;            // warps per team
  static constexpr int TEAM_BOXES = NG >= 32 ? TB : (32 / NG) * TB;  // boxes per team
  static constexpr int NTEAMS = NT / (32 * TEAM);
  static_assert(TEAM == 1 || NTEAMS <= 14, "named barriers 2..15");
  // Team-local layer boundaries pay off when the W ring is deep enough to
  // absorb the teams' drift (measured: +4-5% with >= 4 stages; with the
  // 3-stage ring of 8x256 affine tiles a leading team stalls on refills that
  // wait for the slowest one, -3%), so shallow rings keep the CTA barrier.
  static constexpr bool TEAMSYNC = SPK_TEAM_SYNC && NS >= SPK_TEAM_MIN_NS;
};

// copy N bytes (N in {4, 8, 16}) between 16/8/4-aligned addresses as one access
template <int N> struct VecOf;
template <> struct VecOf<16> { using type = float4; };
template <> struct VecOf<8> { using type = float2; };
template <> struct VecOf<4> { using type = float; };

// A thread's TI per-neuron parameters (bias, bias budget) as TI/G vector loads
// of G consecutive neurons (the arrays are 16-byte aligned and zero-padded to
// a multiple of 4 entries, spk_abi.cu); groups wholly past m_out read zeros.
template <typename T, int TI, int G, int NG>
SPK_DEV void load_group(const T* __restrict__ p, int m_out, int ng, T (&out)[TI]) {
  using GV = typename VecOf<G * (int)sizeof(T)>::type;
#pragma unroll
  for (int q = 0; q < TI / G; ++q) {
    const int i0 = q * (NG * G) + ng * G;
    if (i0 < m_out) {
      const GV v = __ldg(reinterpret_cast<const GV*>(p + i0));
      const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
      for (int j = 0; j < G; ++j) out[q * G + j] = e[j];
    } else {
#pragma unroll
      for (int j = 0; j < G; ++j) out[q * G + j] = T(0);
    }
  }
}

// ------------------------------------------------------------ mbarrier/TMA
SPK_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
SPK_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
SPK_DEV void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
SPK_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
SPK_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// barrier among the NT compute threads only (the producer warp never joins)
SPK_DEV void csync() { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); }
// barrier among the warps of one team (see Cfg::TEAM)
template <int TEAM>
SPK_DEV void team_sync(int tid) {
  if (TEAM == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(2 + (tid >> 5) / TEAM), "n"(TEAM * 32) : "memory");
  }
}


SPK_DEV void tma_bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Ring of W tiles.  Tile g of the CTA's global sequence is tile
// (g mod tiles_per_pass) of the network; all warps consume every tile in
// order.  Each warp releases a stage with one shared-memory atomic; the last
// of the 8 warps to release it issues the refill (cp.async.bulk into the same
// stage), so warps never synchronise with each other per tile and no extra
// producer warp (which would cost ~25% of the register file) is needed.  When
// the whole network fits in the ring (tiles_per_pass <= NS) every tile is
// loaded once and stays resident for the CTA's lifetime.
template <typename T, int C, int MMAX, int SM = 0>
struct WRing {
  using CF = Cfg<T, C, MMAX, SM>;
  T* stages;
  uint64_t* full;
  unsigned* released;  // per-stage count of warps done with the current round
  const T* src;
  int per_pass;
  long long total;  // tiles this CTA will consume
  long long next;   // next tile to consume
  int st = 0;        // ring stage of `next` (next % NS, or next % per_pass when resident)
  uint32_t ph = 0;   // mbarrier phase parity of `next` ((next / NS) & 1)
  uint32_t* live = nullptr;  // live-row masks [2][NBG][LW] (Cfg::LIVE), set by the kernel
  bool group_empty = false;  // this thread's box group holds no box in the current tile

  SPK_DEV bool resident() const { return per_pass <= CF::NS; }
  SPK_DEV void issue(long long g) const {
    const int s = resident() ? (int)(g % per_pass) : (int)(g % CF::NS);
    const T* src_t = src + (size_t)(g % per_pass) * CF::TILE;
    tma_bulk_load(stages + (size_t)s * CF::TILE, src_t, CF::TILE * sizeof(T), &full[s]);
  }
  SPK_DEV void prologue(int tid) const {
    if (tid == 0 && total > 0) {
      const long long n0 = resident() ? per_pass : (total < CF::NS ? total : CF::NS);
      for (long long g = 0; g < n0; ++g) issue(g);
    }
  }
  SPK_DEV const T* acquire() const {
    mbar_wait(&full[st], resident() ? 0u : ph);  // resident stages complete once and stay complete
    return stages + (size_t)st * CF::TILE;
  }
  // Deferred release decision (SPK_DEFER_RELEASE, rings of >= 4 stages):
  // lane 0 examines its atomic's result at the warp's next release (or at
  // settle(), after the layer's last tile), so the shared-memory atomic's
  // round trip overlaps a tile of FMAs instead of stalling the warp.  The
  // refill goes out one tile later, which the deep ring absorbs; the stage's
  // counter is reset before its refill is issued, and no warp can release the
  // stage again before that refill lands, so the count stays exact.
  // measured: C5 width 64 -2%; width-512 point pass +1%, and on the 3-stage
  // rings (C2, C5 width 512) +6%: on for narrow nets only
  static constexpr bool DEFER = SPK_DEFER_RELEASE && CF::NS >= SPK_DEFER_MIN_NS && MMAX <= 64;
  unsigned pend_old = 0u;
  int pend_st = -1;
  long long pend_next = 0;
  SPK_DEV void settle() {
    if (DEFER && pend_st >= 0) {
      if (pend_old == NT / 32 - 1) {
        released[pend_st] = 0u;
        if (pend_next + CF::NS < total) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(pend_next + CF::NS);
        }
      }
      pend_st = -1;
    }
  }
  // the calling warp is done reading the current stage
  SPK_DEV void release(int tid) {
    if (!resident()) {
      __syncwarp();
      if ((tid & 31) == 0) {
        if constexpr (DEFER) {
          settle();
          pend_old = atomicAdd(&released[st], 1u);
          pend_st = st;
          pend_next = next;
        } else if (atomicAdd(&released[st], 1u) == NT / 32 - 1) {
          released[st] = 0u;
          if (next + CF::NS < total) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(next + CF::NS);
          }
        }
      }
    }
    ++next;
    // stage / phase advance incrementally (no 64-bit division per tile)
    if (++st == (resident() ? per_pass : CF::NS)) {
      st = 0;
      ph ^= 1u;
    }
  }
};

// --------------------------------------------------------------- epilogue
// Per-(neuron, box) state between layers.
template <typename T, int C, int MODE>
struct State {
  static constexpr int BM = bound_mode(MODE);
  static constexpr int OFF = pv_off(MODE);
  static constexpr int S = BM == MODE_AFFINE ? C - 2 - OFF : 0;
  T base;       // value / centre / affine base
  T A[S > 0 ? S : 1];
  T e;          // interval radius / affine error (not yet pre-inflated)
  T pv;         // march modes: point value at the probe
};

template <typename T, int C, int MODE>
SPK_DEV T sum_abs_A(const State<T, C, MODE>& st) {
  // starts from |A_0| (RU(0 + |A_0|) = |A_0| exactly): one dependent add less
  constexpr int S = State<T, C, MODE>::S;
  if constexpr (S == 0) return T(0);
  T r = fabs(st.A[0]);
#pragma unroll
  for (int j = 1; j < S; ++j) r = Num<T>::add_ru(r, fabs(st.A[j]));
  return r;
}

// Non-ReLU affine activations (ELU / sin / tanh).  Inline (a by-reference
// call would force the state into local memory on every path); the rule
// itself -- the FP64 transcendental part -- is out of line (spk_rules.cuh).
template <typename T, int C, int MODE>
SPK_DEV void apply_affine_general(State<T, C, MODE>& st, int act) {
  const T rA = sum_abs_A(st);
  const T r = Num<T>::add_ru(rA, st.e);
  const T lo = Num<T>::sub_rd(st.base, r), hi = Num<T>::add_ru(st.base, r);
  T a, b, g;
  const int kind = affine_rule<T>(act, lo, hi, a, b, g);
  if (kind == 0) return;
  if (kind == 1) {
    st.base = T(0);
#pragma unroll
    for (int j = 0; j < State<T, C, MODE>::S; ++j) st.A[j] = T(0);
    st.e = T(0);
    return;
  }
  const T nb = Num<T>::fma_rn(a, st.base, b);
#pragma unroll
  for (int j = 0; j < State<T, C, MODE>::S; ++j) st.A[j] = Num<T>::mul_rn(a, st.A[j]);
  const T aa = fabs(a);
  T e = Num<T>::fma_ru(aa, st.e, g);
  // rounding of a*base+b and of the a*A_j products
  e = Num<T>::fma_ru(Num<T>::RHO, Num<T>::add_ru(fabs(nb), Num<T>::mul_ru(aa, rA)), e);
  st.e = Num<T>::add_ru(e, Num<T>::TINY);
  st.base = nb;
}

// Apply one activation to the state (sound rules; range_core.py:583-603 for
// affine-fixed, :639-641 for interval, network.py:149-160 for points).
template <typename T, int C, int MODE>
SPK_DEV void apply_act(State<T, C, MODE>& st, int act) {
  if (act == ACT_IDENTITY) return;  // skipped, range_core.py:586-587
  constexpr int BM = bound_mode(MODE);
  if (MODE >= MODE_MI) st.pv = act_value<T>(act, st.pv);
  if (BM == MODE_POINT) {
    st.base = act_value<T>(act, st.base);
  } else if (BM == MODE_INTERVAL) {
    const T lo = Num<T>::sub_rd(st.base, st.e), hi = Num<T>::add_ru(st.base, st.e);
    T L, H;
    interval_image<T>(act, lo, hi, L, H);
    const T c = Num<T>::fma_rn(L, T(0.5), Num<T>::mul_rn(H, T(0.5)));
    st.base = c;
    st.e = fmax(Num<T>::sub_ru(H, c), Num<T>::sub_ru(c, L));
  } else if (act == ACT_RELU) {
    // Branch-free ReLU (no divergence between active / inactive / straddling
    // lanes): slope a = 1 (lo >= 0), 0 (hi <= 0), else hi/(hi-lo) clamped;
    // the remainder bound below is exact-zero for a = 0 or 1, and the
    // rounding terms are only charged where a rounding can occur (straddle).
    const T rA = sum_abs_A(st);
    const T r = Num<T>::add_ru(rA, st.e);
    const T lo = Num<T>::sub_rd(st.base, r), hi = Num<T>::add_ru(st.base, r);
    const bool on = lo >= T(0), off = hi <= T(0), mix = !(on || off);
    T a = fmin(fmax(Num<T>::div_fast(hi, hi - lo), T(0)), T(1));
    a = on ? T(1) : (off ? T(0) : a);
    const T ru = mix ? fmax(Num<T>::mul_ru(-a, lo), Num<T>::fma_ru(-a, hi, hi)) : T(0);
    const T b = Num<T>::mul_rn(ru, T(0.5));
    const T g = fmax(b, Num<T>::sub_ru(ru, b));
    const T nb = Num<T>::fma_rn(a, st.base, b);
#pragma unroll
    for (int j = 0; j < State<T, C, MODE>::S; ++j) st.A[j] = Num<T>::mul_rn(a, st.A[j]);
    T e = Num<T>::fma_ru(a, st.e, g);
    const T rnd = Num<T>::fma_ru(Num<T>::RHO, Num<T>::add_ru(fabs(nb), Num<T>::mul_ru(a, rA)), Num<T>::TINY);
    st.e = mix ? Num<T>::add_ru(e, rnd) : e;
    st.base = nb;
  } else {
    apply_affine_general<T, C, MODE>(st, act);
  }
}
// Column values handed to the next dense layer.
template <typename T, int C, int MODE>
SPK_DEV void pack_next(const State<T, C, MODE>& st, T gamma_next, T* out, T gamma_base = T(-1)) {
  constexpr int BM = bound_mode(MODE), OFF = pv_off(MODE);
  if (MODE >= MODE_MI) out[0] = st.pv;
  out[OFF] = st.base;
  // v = e + gamma' (|base| + sum|A| + e): gamma' covers the next layer's
  // FMA rounding and (FP32) the rounding of the FP64 weights to T.
  if (BM == MODE_INTERVAL) {
    out[OFF + 1] = Num<T>::fma_ru(gamma_next, Num<T>::add_ru(fabs(st.base), st.e), st.e);
  } else if (BM == MODE_AFFINE) {
    const T rA = sum_abs_A(st);
#pragma unroll
    for (int j = 0; j < State<T, C, MODE>::S; ++j) out[OFF + 1 + j] = st.A[j];
    if (gamma_base >= T(0)) {
      // the next K loop bounds the base column's FMA rounding itself (RUNERR):
      // only the weights' FP64 -> T rounding is charged on |base| here
      out[C - 1] = Num<T>::fma_ru(gamma_next, Num<T>::add_ru(rA, st.e), Num<T>::fma_ru(gamma_base, fabs(st.base), st.e));
    } else {
      out[C - 1] = Num<T>::fma_ru(gamma_next, Num<T>::add_ru(Num<T>::add_ru(fabs(st.base), rA), st.e), st.e);
    }
  }
}

// ReLU rule + pack for the next layer, fused (affine-fixed layers whose only
// activation is ReLU -- the hot epilogue).  Identical to apply_act(ACT_RELU)
// followed by pack_next on active (lo >= 0) and inactive (hi <= 0) neurons,
// which take a short select-only path; straddling neurons (the only ones
// that need the slope division and the remainder / rounding terms) run in a
// branch guarded by a warp vote, so a warp without a straddling (neuron,
// box) skips it.  Returns whether the packed columns can be nonzero (the
// live-row mask bit): inactive neurons pack exact (+-)zeros.
template <typename T, int C, int MODE>
SPK_DEV bool relu_affine_pack(State<T, C, MODE>& st, T gamma_next, T* out, T gamma_base = T(-1)) {
  constexpr int S = State<T, C, MODE>::S;
  const T rA = sum_abs_A(st);
  const T r = Num<T>::add_ru(rA, st.e);
  const T lo = Num<T>::sub_rd(st.base, r), hi = Num<T>::add_ru(st.base, r);
  const bool on = lo >= T(0), off = hi <= T(0), mix = !(on || off);
  // on: (1, 0, 0) leaves the state exactly as it is; off: everything 0
  T nb = on ? st.base : T(0);
  T e = on ? st.e : T(0);
  T rA2 = on ? rA : T(0);
  // inactive: 0 * A (the reference's signed zeros); active and straddling
  // lanes keep A (exact times 1; straddling lanes scale it below)
  const T keep = off ? T(0) : T(1);
#pragma unroll
  for (int j = 0; j < S; ++j) st.A[j] = Num<T>::mul_rn(keep, st.A[j]);
  if (SPK_FUSED_RELU_VOTE ? __any_sync(__activemask(), mix) : true) {
    if (mix) {
      T a = fmin(fmax(Num<T>::div_fast(hi, hi - lo), T(0)), T(1));
      const T ru = fmax(Num<T>::mul_ru(-a, lo), Num<T>::fma_ru(-a, hi, hi));
      const T b = Num<T>::mul_rn(ru, T(0.5));
      const T g = fmax(b, Num<T>::sub_ru(ru, b));
      nb = Num<T>::fma_rn(a, st.base, b);
#pragma unroll
      for (int j = 0; j < S; ++j) st.A[j] = Num<T>::mul_rn(a, st.A[j]);
      e = Num<T>::fma_ru(a, st.e, g);
      const T rnd = Num<T>::fma_ru(Num<T>::RHO, Num<T>::add_ru(fabs(nb), Num<T>::mul_ru(a, rA)), Num<T>::TINY);
      e = Num<T>::add_ru(e, rnd);
      rA2 = sum_abs_A(st);
    }
  }
  st.base = nb;
  st.e = e;
  constexpr int OFF = pv_off(MODE);
  out[OFF] = nb;
#pragma unroll
  for (int j = 0; j < S; ++j) out[OFF + 1 + j] = st.A[j];
  out[C - 1] = gamma_base >= T(0)
                   ? Num<T>::fma_ru(gamma_next, Num<T>::add_ru(rA2, e), Num<T>::fma_ru(gamma_base, fabs(nb), e))
                   : Num<T>::fma_ru(gamma_next, Num<T>::add_ru(Num<T>::add_ru(fabs(nb), rA2), e), e);
  return !off;
}

// Final bound of a width-1 output: lo/hi rounded outward.
template <typename T, int C, int MODE>
SPK_DEV void final_bounds(const State<T, C, MODE>& st, double& lo, double& hi) {
  constexpr int BM = bound_mode(MODE);
  if (BM == MODE_POINT) {
    lo = hi = (double)st.base;
  } else if (BM == MODE_INTERVAL) {
    lo = (double)Num<T>::sub_rd(st.base, st.e);
    hi = (double)Num<T>::add_ru(st.base, st.e);
  } else {
    const T r = Num<T>::add_ru(sum_abs_A(st), st.e);
    lo = (double)Num<T>::sub_rd(st.base, r);
    hi = (double)Num<T>::add_ru(st.base, r);
  }
}

// State of one (neuron, box) from its accumulated columns (+ the bias term's
// rounding budget be on the error column; march modes carry the point value
// in column 0).
template <typename T, int C, int MODE>
SPK_DEV State<T, C, MODE> state_from(const T* col, T be) {
  constexpr int BM = bound_mode(MODE), OFF = pv_off(MODE);
  State<T, C, MODE> st;
  st.pv = OFF ? col[0] : T(0);
  st.base = col[OFF];
  if (BM == MODE_AFFINE) {
#pragma unroll
    for (int j = 0; j < State<T, C, MODE>::S; ++j) st.A[j] = col[OFF + 1 + j];
  }
  st.e = (BM == MODE_POINT) ? T(0) : Num<T>::add_ru(col[C - 1], be);
  return st;
}

// ------------------------------------------------------------ dense layers
// Generic layer: register-tiled contraction over the W ring.  The
// round-to-nearest columns are summed in blocks of SUB k-steps (fresh
// partials added to the running sums), so the rounding budget is
// gamma_{SUB + ceil(m_in/SUB) + 1} instead of gamma_{m_in + 1}.
template <typename T, int C, int MMAX, int BIAS2 = -1, bool TEAMS = false, int SM = 0>
SPK_DEV void dense_kloop_scalar(const LayerDev<T>& L, const T* __restrict__ X, WRing<T, C, MMAX, SM>& ring, int tid,
                                T (&acc)[Cfg<T, C, MMAX, SM>::TI][Cfg<T, C, MMAX, SM>::TB][C],
                                const uint32_t* live = nullptr) {
  using CF = Cfg<T, C, MMAX, SM>;
  constexpr int TI = CF::TI, TB = CF::TB, CP = CF::CP, KT = CF::KT;
  const int ng = tid % CF::NG, bg = tid / CF::NG;
  // RN columns accumulate in SUB-step partial sums (blocked summation, the
  // blocks may span W tiles): rounding budget gamma_{SUB + ceil(m_in/SUB) + 1}
  // instead of gamma_{m_in + 1}.  The RU error column needs no blocking.
  // With one block (FP64: SUB = 2^20) the partials ARE the accumulators: the
  // dot product accumulates in place and the bias is added last -- the same
  // operation order as flushing one block onto the bias, 2 x TI x TB x (C-1)
  // fewer registers.
  constexpr bool DIRECT = SPK_F64_DIRECT && CF::SUB >= (1 << 20);
  constexpr int CR = C > 1 ? C - 1 : 1;
  constexpr int SUBIN = KT < CF::SUB ? KT : CF::SUB;
  constexpr int PTI = DIRECT ? 1 : TI, PTB = DIRECT ? 1 : TB;

  T bias_r[TI];
  if (!DIRECT) load_group<T, TI, CF::G, CF::NG>(L.bias, L.m_out, ng, bias_r);
#pragma unroll
  for (int ti = 0; ti < TI; ++ti) {
    const T b0 = DIRECT ? T(0) : bias_r[ti];
#pragma unroll
    for (int tb = 0; tb < TB; ++tb) {
      acc[ti][tb][0] = b0;
#pragma unroll
      for (int c = 1; c < C; ++c) acc[ti][tb][c] = (c == BIAS2) ? b0 : T(0);
    }
  }
  T part[PTI][PTB][CR];
#pragma unroll
  for (int ti = 0; ti < PTI; ++ti)
#pragma unroll
    for (int tb = 0; tb < PTB; ++tb)
#pragma unroll
      for (int c = 0; c < CR; ++c) part[ti][tb][c] = T(0);
  int since = 0;
  auto flush = [&]() {
    if (DIRECT) return;
#pragma unroll
    for (int ti = 0; ti < PTI; ++ti)
#pragma unroll
      for (int tb = 0; tb < PTB; ++tb)
#pragma unroll
        for (int c = 0; c < CR; ++c) {
          acc[ti][tb][c] += part[ti][tb][c];
          part[ti][tb][c] = T(0);
        }
  };

  // fragment loads for one k-step (W: TI values, X: TB*CP values)
  auto load_frag = [&](const T* __restrict__ Ws, const T* __restrict__ Xt, int kk, T* w, T* x) {
    using WV = typename VecOf<CF::G * (int)sizeof(T)>::type;
    WV* wd = reinterpret_cast<WV*>(w);
#pragma unroll
    for (int q = 0; q < TI / CF::G; ++q)
      wd[q] = *reinterpret_cast<const WV*>(Ws + kk * MMAX + q * (CF::NG * CF::G) + ng * CF::G);
    const float4* xp = reinterpret_cast<const float4*>(Xt + CF::xrow(kk));
    float4* xd = reinterpret_cast<float4*>(x);
#pragma unroll
    for (int q = 0; q < (int)(TB * CP * sizeof(T) / 16); ++q) xd[q] = xp[q];
  };
  auto fma_step = [&](const T* w, const T* x) {
#pragma unroll
    for (int ti = 0; ti < TI; ++ti) {
#pragma unroll
      for (int tb = 0; tb < TB; ++tb) {
        T* dst = DIRECT ? acc[ti][tb] : part[DIRECT ? 0 : ti][DIRECT ? 0 : tb];
        if (C == 1) {
          dst[0] = Num<T>::fma_rn(w[ti], x[tb * CP], dst[0]);
        } else {
#pragma unroll
          for (int c = 0; c < C - 1; ++c) dst[c] = Num<T>::fma_rn(w[ti], x[tb * CP + c], dst[c]);
          acc[ti][tb][C - 1] = Num<T>::fma_ru(fabs(w[ti]), x[tb * CP + C - 1], acc[ti][tb][C - 1]);
        }
      }
    }
  };

  // element-wise fragment loads (no type-punned register arrays: punning
  // FP64 fragments through float4 made ptxas stage them in local memory)
  auto load_frag_e = [&](const T* __restrict__ Ws, const T* __restrict__ Xt, int kk, T* w, T* x) {
    using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
#pragma unroll
    for (int q = 0; q < TI / CF::G; ++q) {
      const T* src = Ws + kk * MMAX + q * (CF::NG * CF::G) + ng * CF::G;
#pragma unroll
      for (int e = 0; e < CF::G; e += 2) {
        const V2 v = *reinterpret_cast<const V2*>(src + e);
        w[q * CF::G + e] = v.x;
        w[q * CF::G + e + 1] = v.y;
      }
    }
    const V2* xp = reinterpret_cast<const V2*>(Xt + CF::xrow(kk));
#pragma unroll
    for (int q = 0; q < TB * CP / 2; ++q) {
      const V2 v = xp[q];
      x[2 * q] = v.x;
      x[2 * q + 1] = v.y;
    }
  };
  // one block (DIRECT): every full chunk of CH k-steps fully unrolled with
  // statically indexed double-buffered fragments (no register rotation)
  constexpr int CH = KT < 32 ? KT : 32;
  constexpr bool UNROLLED = SPK_UNROLL_BLOCK && DIRECT && (KT % CH) == 0 && (CF::G % 2) == 0 &&
                            ((TB * CP) % 2) == 0;

  for (int t = 0; t < L.ntiles / CF::TSCALE; ++t) {
    const T* __restrict__ Ws = ring.acquire();
    const T* __restrict__ Xt = X + CF::xrow(t * KT) + bg * CF::GS;
    // rows past m_in are zero in X and W: stop at m_in (rounded to the
    // double-buffer pair), e.g. 4 k-steps instead of KT for the 3-input layer
    int k_end = L.m_in - t * KT;
    k_end = k_end > KT ? KT : ((k_end + 1) & ~1);
    if constexpr (CF::LIVE && DIRECT) {
      // live-row masks (FP64): rows that are exactly zero for the whole box
      // group are skipped -- an FMA with an exact zero leaves the in-place
      // accumulators unchanged -- so sparse tiles run a row list
      if (live != nullptr) {
        const uint32_t word = live[(t * KT) >> 5];
        uint32_t m = KT >= 32 ? word : ((word >> ((t * KT) & 31)) & ((1u << (KT & 31)) - 1u));
        if (__popc(m) <= SPK_LIVE_DENSE_F64 * KT / 16) {
          if (m != 0u) {
            if (__popc(m) & 1) m |= ~m & (m + 1u);  // pad to pairs with an exactly-zero row (< KT)
            const int cnt = __popc(m), lane = tid & 31;
            int* lst = reinterpret_cast<int*>(ring.live + 2 * CF::NBG * CF::LW) + (tid >> 5) * CF::LLIST;
            __syncwarp();
            if ((m >> lane) & 1u) lst[__popc(m & ((1u << lane) - 1u))] = lane;
            if (lane < 2) lst[cnt + lane] = 0;  // prefetch past the last pair reads row 0 (unused)
            __syncwarp();
            T w0[TI], x0[TB * CP], w1[TI], x1[TB * CP];
            int2 kk = *reinterpret_cast<const int2*>(lst);
            load_frag_e(Ws, Xt, kk.x, w0, x0);
#pragma unroll 1
            for (int p = 0; p < cnt; p += 2) {
              load_frag_e(Ws, Xt, kk.y, w1, x1);
              const int2 nx = *reinterpret_cast<const int2*>(lst + p + 2);
              fma_step(w0, x0);
              load_frag_e(Ws, Xt, nx.x, w0, x0);
              fma_step(w1, x1);
              kk = nx;
            }
          }
          ring.release(tid);
          continue;
        }
      }
    }
    if (UNROLLED && k_end == KT) {
#pragma unroll 1
      for (int k0 = 0; k0 < KT; k0 += CH) {
        T wf[2][TI], xf[2][TB * CP];
        load_frag_e(Ws, Xt, k0, wf[0], xf[0]);
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          if (j + 1 < CH) load_frag_e(Ws, Xt, k0 + j + 1, wf[(j + 1) & 1], xf[(j + 1) & 1]);
          fma_step(wf[j & 1], xf[j & 1]);
        }
      }
      ring.release(tid);
      continue;
    }
#pragma unroll 1
    for (int k0 = 0; k0 < k_end; k0 += SUBIN) {
      const int k1 = k0 + SUBIN < k_end ? k0 + SUBIN : k_end;
      // register double buffering: fragments of step kk+1 load while step kk
      // computes (FP64: unroll 8 measured fastest; unroll 1 is 1.7x slower)
      T w0[TI], x0[TB * CP], w1[TI], x1[TB * CP];
      load_frag(Ws, Xt, k0, w0, x0);
#pragma unroll kScalarUnroll
      for (int kk = k0; kk < k1; kk += 2) {
        load_frag(Ws, Xt, kk + 1, w1, x1);
        fma_step(w0, x0);
        if (SPK_SPEC_PREFETCH || kk + 2 < k1) load_frag(Ws, Xt, kk + 2, w0, x0);  // row k1 <= KT: in bounds
        fma_step(w1, x1);
      }
      since += SUBIN;
      if (since >= CF::SUB) {
        flush();
        since = 0;
      }
    }
    ring.release(tid);  // this warp is done with the stage
  }
  ring.settle();
  if (since > 0) flush();
  if (DIRECT) {
    T bias_r[TI];
    load_group<T, TI, CF::G, CF::NG>(L.bias, L.m_out, ng, bias_r);
#pragma unroll
    for (int ti = 0; ti < TI; ++ti) {
      const T b0 = bias_r[ti];
#pragma unroll
      for (int tb = 0; tb < TB; ++tb) {
        acc[ti][tb][0] = acc[ti][tb][0] + b0;
        if (BIAS2 > 0 && BIAS2 < C - 1) acc[ti][tb][BIAS2 > 0 && BIAS2 < C ? BIAS2 : 0] += b0;
      }
    }
  }
  // every thread of the team finished reading X before its epilogue rewrites it
  if (TEAMS) {
    team_sync<CF::TEAM>(tid);
  } else {
    csync();
  }
}


// ------------------------------------------------------------ packed FP32
// sm_100a FFMA2 / FADD2 (fma.rn.f32x2 / add.rn.f32x2): two FP32 lanes per
// instruction; the scalar weight is broadcast by ptxas's `.F32` operand form
// (no duplicate move), so acc(c, c+1) += w * x(c, c+1) is one issue slot.
typedef unsigned long long f32x2;
SPK_DEV f32x2 f2_fma(float w, f32x2 x, f32x2 acc) {
  asm("{.reg .b64 wd;\n mov.b64 wd, {%1, %1};\n fma.rn.f32x2 %0, wd, %2, %0;}" : "+l"(acc) : "f"(w), "l"(x));
  return acc;
}
// error column of two neurons: acc(i, i+1) += RU(|w_i| * x), RU(|w_i+1| * x)
// -- one FFMA2.RP with the |.| operand modifier and x broadcast (.F32)
SPK_DEV f32x2 f2_fma_ru_abs(float w0, float w1, float x, f32x2 acc) {
  asm("{.reg .b64 wd, xd;\n mov.b64 wd, {%1, %2};\n mov.b64 xd, {%3, %3};\n fma.rp.f32x2 %0, wd, xd, %0;}"
      : "+l"(acc)
      : "f"(fabsf(w0)), "f"(fabsf(w1)), "f"(x));
  return acc;
}
SPK_DEV f32x2 f2_fma2(f32x2 w, f32x2 x, f32x2 acc) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(w), "l"(x));
  return acc;
}
SPK_DEV f32x2 f2_mul(float w, f32x2 x) {
  f32x2 r;
  asm("{.reg .b64 wd;\n mov.b64 wd, {%1, %1};\n mul.rn.f32x2 %0, wd, %2;}" : "=l"(r) : "f"(w), "l"(x));
  return r;
}
SPK_DEV f32x2 f2_add(f32x2 a, f32x2 b) {
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(a) : "l"(b));
  return a;
}
SPK_DEV void f2_split(f32x2 v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
SPK_DEV f32x2 f2_pack(float lo, float hi) {
  f32x2 v;
  asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(lo), "f"(hi));
  return v;
}

// FP32 K loop with packed FMAs.  Columns of one box: NP round-to-nearest
// pairs, an optional odd RN column, and the round-up error column (scalar
// FFMA.RP with the |W| operand modifier).  Point evaluation (C == 1) pairs
// adjacent boxes instead.  Same blocked-summation budget as the scalar loop.
// RE (running error): on the layers the host flags (LayerDev::runerr) the
// base column (low lane of pair 0) also accumulates Wilkinson's a-posteriori
// bound sum_k |s_k| of its partial and flushed sums (one FFMA.RP per step),
// and the loop charges u/(1-u) * that sum to the error column -- instead of
// the a-priori gamma_n * sum |W| |base| that pack_next would otherwise put on
// v (~6x tighter per layer).  The extra op sits on the saturated FP32 pipe
// (+24% when every layer does it), so only the leading wide layers, whose
// budgets dominate the FP32 excess of deep affine-fixed nets through the
// non-cancelling error channel (x10 per layer, tools/excess_attrib.py), take
// this form of the loop.
template <int C, int MMAX, int BIAS2 = -1, bool TEAMS = false, int SM = 0, bool RE = false>
SPK_DEV void dense_kloop_f32(const LayerDev<float>& L, const float* __restrict__ X, WRing<float, C, MMAX, SM>& ring,
                             int tid, float (&acc)[Cfg<float, C, MMAX, SM>::TI][Cfg<float, C, MMAX, SM>::TB][C],
                             const uint32_t* live = nullptr) {
  using CF = Cfg<float, C, MMAX, SM>;
  constexpr int TI = CF::TI, TB = CF::TB, CP = CF::CP, KT = CF::KT;
  constexpr bool POINT = C == 1;
  constexpr int NRN = POINT ? 1 : C - 1;           // round-to-nearest columns per box
  constexpr int NP = POINT ? TB / 2 : NRN / 2;     // packed pairs (per box; boxes for POINT)
  constexpr int NBOX = POINT ? 1 : TB;             // pair groups
  constexpr bool ODD = !POINT && (NRN % 2 == 1);
  constexpr int XQ = CF::GS / 2;                   // x fragment as f32x2 words
  // f32x2 word and lane of column c of the group's box tb (Cfg::xcol)
  constexpr auto xword = [](int tb, int c) { return CF::xcol(tb, c) / 2; };
  constexpr auto xlane = [](int tb, int c) { return CF::xcol(tb, c) % 2; };
  static_assert(POINT ? (TB % 2 == 0) : (CP % 2 == 0), "pair alignment");
  constexpr bool RUN = RE && !POINT && NP >= 1 && BIAS2 < 0;
  static_assert(RE == RUN, "running error bound: affine columns (base in pair 0) only");
  // runtime per layer (LayerDev::runerr, set by the host for the leading wide
  // layers whose budgets dominate): the K loop below exists in both forms
  const bool re_layer = RUN && L.runerr;
  // F64B: the running-error layers accumulate their base column in FP64
  // instead (one DFMA per (neuron, box) and k-step on the FP64 pipe, beside
  // the FP32 pipe's packed columns): the FP64 sum's own rounding (<= gamma_n
  // of 2^-53, <= 1e-13 relative for n <= 513) is charged a priori by the pack
  // (LayerDev::gamma_base_next = weight rounding + 1e-13), and the final FP64 -> FP32
  // rounding of the base is charged exactly, |b64 - RN(b64)|, so the layer's
  // base column costs ~u |base| instead of Wilkinson's u sum_k |s_k|.  Skipped
  // all-zero rows add exact zeros, so results stay order-independent.
  constexpr bool F64B = RUN && SPK_F64_BASE;
  float erun[RUN && !F64B ? TI : 1][RUN && !F64B ? TB : 1];
  double base64[F64B ? TI : 1][F64B ? TB : 1];
#pragma unroll
  for (int ti = 0; ti < (RUN && !F64B ? TI : 1); ++ti)
#pragma unroll
    for (int tb = 0; tb < (RUN && !F64B ? TB : 1); ++tb) erun[ti][tb] = 0.f;
  const int ng = tid % CF::NG, bg = tid / CF::NG;

  constexpr int NPA = NP > 0 ? NP : 1;
  f32x2 accp[TI][NBOX][NPA], partp[TI][NBOX][NPA];
  float acco[TI][TB], parto[TI][TB], acce[TI][TB];
  // error column packed over neuron pairs (SPK_PACKED_ERR; FFMA2.RP, same
  // per-lane rounding and order as the scalar FFMA.RP, so identical sums)
  constexpr bool PE = SPK_PACKED_ERR && !POINT && TI % 2 == 0 && MMAX >= SPK_PACKED_ERR_MINW;
  f32x2 acce2[PE ? TI / 2 : 1][TB];
#pragma unroll
  for (int j = 0; j < (PE ? TI / 2 : 1); ++j)
#pragma unroll
    for (int tb = 0; tb < TB; ++tb) acce2[j][tb] = 0ull;
  float bias_r[TI];
  load_group<float, TI, CF::G, CF::NG>(L.bias, L.m_out, ng, bias_r);
#pragma unroll
  for (int ti = 0; ti < TI; ++ti) {
    const float b0 = bias_r[ti];
#pragma unroll
    for (int g = 0; g < NBOX; ++g)
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        // the bias enters the base column (column 0, or every box for POINT)
        accp[ti][g][p] = POINT ? f2_pack(b0, b0)
                               : (p == 0 ? f2_pack(b0, BIAS2 == 1 ? b0 : 0.f) : f2_pack(0.f, 0.f));
      }
#pragma unroll
    for (int tb = 0; tb < TB; ++tb) {
      acco[ti][tb] = (ODD && NP == 0) ? b0 : 0.f;  // C == 2: the odd column is the base
      acce[ti][tb] = 0.f;
      if constexpr (F64B) base64[ti][tb] = (double)b0;
    }
  }
  constexpr int SUBIN = KT < CF::SUB ? KT : CF::SUB;
  // every SUBIN chunk starts a fresh blocked-summation block (KT a multiple of SUB)
  constexpr bool ALWAYS_FRESH = (KT % CF::SUB) == 0;
  // nets no wider than one summation block (width <= SUB, e.g. C1's 4x32):
  // every layer is a single block, so the products accumulate straight onto
  // the bias -- an (m_in + 1)-term chain inside the same gamma_{m_in + 2}
  // budget -- with no partial registers, zeroing or flushes
  constexpr bool ONEBLK = SPK_ONE_BLOCK && MMAX <= CF::SUB;
  int since = 0;
  // partial sums -> running sums (a fresh block re-initialises the partials)
  auto flush = [&](auto rec) {
    if (ONEBLK) return;
    constexpr bool REC = decltype(rec)::value && RUN;
#pragma unroll
    for (int ti = 0; ti < TI; ++ti) {
#pragma unroll
      for (int g = 0; g < NBOX; ++g) {
#pragma unroll
        for (int p = 0; p < NP; ++p) accp[ti][g][p] = f2_add(accp[ti][g][p], partp[ti][g][p]);
        if (REC && !F64B) {  // the flush's own rounding: u |acc_new|
          float b_, a_;
          f2_split(accp[ti][g][0], b_, a_);
          erun[ti][g] = __fadd_ru(erun[ti][g], fabsf(b_));
        }
      }
      if (ODD) {
#pragma unroll
        for (int tb = 0; tb < TB; ++tb) acco[ti][tb] += parto[ti][tb];
      }
    }
  };
  auto zero_parts = [&]() {
    if (ONEBLK) return;
#pragma unroll
    for (int ti = 0; ti < TI; ++ti) {
#pragma unroll
      for (int g = 0; g < NBOX; ++g)
#pragma unroll
        for (int p = 0; p < NP; ++p) partp[ti][g][p] = 0ull;
#pragma unroll
      for (int tb = 0; tb < TB; ++tb) parto[ti][tb] = 0.f;
    }
  };
  auto load_frag = [&](const float* __restrict__ Ws, const float* __restrict__ Xt, int kk, float* w, f32x2* xq) {
    using WV = typename VecOf<CF::G * 4>::type;
    WV* wd = reinterpret_cast<WV*>(w);
#pragma unroll
    for (int q = 0; q < TI / CF::G; ++q)
      wd[q] = *reinterpret_cast<const WV*>(Ws + kk * MMAX + q * (CF::NG * CF::G) + ng * CF::G);
    if constexpr (CF::IL) {  // 40-byte segments: 8-byte aligned words
      const unsigned long long* x8 = reinterpret_cast<const unsigned long long*>(Xt + CF::xrow(kk));
#pragma unroll
      for (int q = 0; q < XQ; ++q) xq[q] = x8[q];
    } else {
      const ulonglong2* xp = reinterpret_cast<const ulonglong2*>(Xt + CF::xrow(kk));
#pragma unroll
      for (int q = 0; q < XQ / 2; ++q) {
        const ulonglong2 v = xp[q];
        xq[2 * q] = v.x;
        xq[2 * q + 1] = v.y;
      }
    }
  };
  // one k-step; FIRST: the first step of a fresh block writes the partials
  // (RN(w*x) == RN(w*x + 0): the same sums as zero-initialised partials)
  auto fma_step = [&](const float* w, const f32x2* xq, auto first, auto rec) {
    constexpr bool FIRST = decltype(first)::value;
    constexpr bool REC = decltype(rec)::value && RUN;
#pragma unroll
    for (int ti = 0; ti < TI; ++ti) {
#pragma unroll
      for (int g = 0; g < NBOX; ++g)
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const f32x2 xv = xq[POINT ? p : xword(g, 2 * p)];
          f32x2& dst = ONEBLK ? accp[ti][g][p] : partp[ti][g][p];
          dst = (FIRST && !ONEBLK) ? f2_mul(w[ti], xv) : f2_fma(w[ti], xv, dst);
          if (REC && p == 0) {
            // Wilkinson's running bound sum_k |s_k|.  Only steps whose base
            // input is nonzero can round (an exact-zero x leaves s_k ==
            // s_(k-1)): gating on it keeps the bound independent of which
            // all-zero rows the live-row masks skip -- results stay identical
            // for any batch composition
            float b_, a_, x0_, x1_;
            f2_split(xv, x0_, x1_);
            if constexpr (F64B) {
              base64[ti][g] = __fma_rn((double)w[ti], (double)x0_, base64[ti][g]);
            } else {
              f2_split(ONEBLK ? accp[ti][g][0] : partp[ti][g][0], b_, a_);
              erun[ti][g] = __fmaf_ru(fabsf(b_), x0_ != 0.f ? 1.f : 0.f, erun[ti][g]);
            }
          }
        }
      if (!POINT) {
#pragma unroll
        for (int tb = 0; tb < TB; ++tb) {
          float lo, hi;
          f2_split(xq[xword(tb, C - 1)], lo, hi);
          const float xe = xlane(tb, C - 1) == 0 ? lo : hi;
          if (!PE) {
            acce[ti][tb] = __fmaf_ru(fabsf(w[ti]), xe, acce[ti][tb]);
          } else if (ti % 2 == 1) {
            acce2[ti / 2][tb] = f2_fma_ru_abs(w[ti - 1], w[ti], xe, acce2[ti / 2][tb]);
          }
          if (ODD) {
            float ol, oh;
            f2_split(xq[xword(tb, 2 * NP)], ol, oh);
            const float xo = xlane(tb, 2 * NP) == 0 ? ol : oh;
            float& dso = ONEBLK ? acco[ti][tb] : parto[ti][tb];
            dso = (FIRST && !ONEBLK) ? __fmul_rn(w[ti], xo) : __fmaf_rn(w[ti], xo, dso);
          }
        }
      }
    }
  };
  using F0 = std::integral_constant<bool, false>;
  using F1 = std::integral_constant<bool, true>;
  // a full SUBIN chunk, fully unrolled: constant shared-memory offsets, no
  // loop control, fragments double-buffered one step ahead
  auto full_chunk = [&](const float* __restrict__ Ws, const float* __restrict__ Xt, int k0, auto fresh, auto rec) {
    float wf[2][TI];
    f32x2 xf[2][XQ];
    load_frag(Ws, Xt, k0, wf[0], xf[0]);
#pragma unroll
    for (int j = 0; j < SUBIN; ++j) {
      if (j + 1 < SUBIN) load_frag(Ws, Xt, k0 + j + 1, wf[(j + 1) & 1], xf[(j + 1) & 1]);
      if (j == 0 && decltype(fresh)::value) {
        fma_step(wf[0], xf[0], F1{}, rec);
      } else {
        fma_step(wf[j & 1], xf[j & 1], F0{}, rec);
      }
    }
  };

  auto tiles = [&](auto rec) {
  for (int t = 0; t < L.ntiles / CF::TSCALE; ++t) {
    const float* __restrict__ Ws = ring.acquire();
    const float* __restrict__ Xt = X + CF::xrow(t * KT) + bg * CF::GS;
    int k_end = L.m_in - t * KT;
    k_end = k_end > KT ? KT : ((k_end + 1) & ~1);
    // live rows of this tile only (bits past m_in are never set); a dense tile
    // takes the unrolled chunk instead (a masked step costs more than an unrolled one)
    uint32_t m = 0u;
    if (CF::LIVE && live != nullptr) {
      const uint32_t word = live[(t * KT) >> 5];
      m = KT == 32 ? word : ((word >> ((t * KT) & 31)) & ((1u << (KT & 31)) - 1u));
    }
    if (CF::LIVE && live != nullptr && __popc(m) <= (CF::NG < 32 ? SPK_LIVE_DENSE_NARROW : SPK_LIVE_DENSE)) {
      if (since == 0) zero_parts();
      if (m != 0u) {
        // an odd count gets one exactly-zero row (one exists: KT is even); the
        // warp writes the tile's live rows as a list (lane l holds bit l) and
        // the loop runs over row pairs read from it (broadcast LDS.64), with
        // the single-exit shape and unconditional prefetch of the dense loop
        if (__popc(m) & 1) m |= ~m & (m + 1u);
        const int cnt = __popc(m), lane = tid & 31;
        int* lst = reinterpret_cast<int*>(ring.live + 2 * CF::NBG * CF::LW) + (tid >> 5) * CF::LLIST;
        __syncwarp();
        if ((m >> lane) & 1u) lst[__popc(m & ((1u << lane) - 1u))] = lane;
        if (lane < 2) lst[cnt + lane] = 0;  // prefetch past the last pair reads row 0 (unused)
        __syncwarp();
        float w0[TI], w1[TI];
        f32x2 x0[XQ], x1[XQ];
        int2 kk = *reinterpret_cast<const int2*>(lst);
        load_frag(Ws, Xt, kk.x, w0, x0);
#pragma unroll 1
        for (int p = 0; p < cnt; p += 2) {
          load_frag(Ws, Xt, kk.y, w1, x1);
          const int2 nx = *reinterpret_cast<const int2*>(lst + p + 2);
          fma_step(w0, x0, F0{}, rec);
          load_frag(Ws, Xt, nx.x, w0, x0);
          fma_step(w1, x1, F0{}, rec);
          kk = nx;
        }
      }
      since += KT;
      if (since >= CF::SUB) {
        flush(rec);
        since = 0;
      }
      ring.release(tid);
      continue;
    }
#pragma unroll 1
    for (int k0 = 0; k0 < k_end; k0 += SUBIN) {
      const int k1 = k0 + SUBIN < k_end ? k0 + SUBIN : k_end;
      // (interval, C == 2: the rolled loop measured 2% faster)
      if (SPK_UNROLL_BLOCK && C != 2 && k1 - k0 == SUBIN) {
        if (ALWAYS_FRESH || since == 0) {
          full_chunk(Ws, Xt, k0, F1{}, rec);
        } else {
          full_chunk(Ws, Xt, k0, F0{}, rec);
        }
      } else {
        if (since == 0) zero_parts();
        float w0[TI], w1[TI];
        f32x2 x0[XQ], x1[XQ];
        load_frag(Ws, Xt, k0, w0, x0);
#pragma unroll 1
        for (int kk = k0; kk < k1; kk += 2) {
          load_frag(Ws, Xt, kk + 1, w1, x1);
          fma_step(w0, x0, F0{}, rec);
          if (SPK_SPEC_PREFETCH || kk + 2 < k1) load_frag(Ws, Xt, kk + 2, w0, x0);  // row k1 <= KT: in bounds
          fma_step(w1, x1, F0{}, rec);
        }
      }
      since += SUBIN;
      if (since >= CF::SUB) {
        flush(rec);
        since = 0;
      }
    }
    ring.release(tid);
  }
  ring.settle();
  if (since > 0) flush(rec);
  };
  if (RUN && re_layer) {
    tiles(std::integral_constant<bool, RUN>{});
  } else {
    tiles(F0{});
  }
  if (TEAMS) {
    team_sync<CF::TEAM>(tid);
  } else {
    csync();
  }
  // unpack into the scalar accumulator layout of the epilogue
#pragma unroll
  for (int ti = 0; ti < TI; ++ti) {
    if (POINT) {
#pragma unroll
      for (int p = 0; p < NP; ++p) f2_split(accp[ti][0][p], acc[ti][2 * p][0], acc[ti][2 * p + 1][0]);
    } else {
#pragma unroll
      for (int tb = 0; tb < TB; ++tb) {
#pragma unroll
        for (int p = 0; p < NP; ++p) f2_split(accp[ti][tb][p], acc[ti][tb][2 * p], acc[ti][tb][2 * p + 1]);
        if (ODD) acc[ti][tb][2 * NP] = acco[ti][tb];
        if (PE) {
          float e0, e1;
          f2_split(acce2[ti / 2][tb], e0, e1);
          acc[ti][tb][C - 1] = (ti % 2 == 0) ? e0 : e1;
        } else {
          acc[ti][tb][C - 1] = acce[ti][tb];
        }
        if constexpr (F64B) {
          if (re_layer) {
            // the FP64 base rounded to FP32, its rounding charged exactly
            const double b64 = base64[ti][tb];
            const float b32 = __double2float_rn(b64);
            acc[ti][tb][0] = b32;
            acc[ti][tb][C - 1] = __fadd_ru(acc[ti][tb][C - 1], __double2float_ru(fabs(b64 - (double)b32)));
          }
        } else if (RUN && re_layer) {
          // base column rounding <= u/(1-u) sum |s| with u/(1-u) <= 0x1.000002p-24
          acc[ti][tb][C - 1] = __fmaf_ru(erun[ti][RUN ? tb : 0], 0x1.000002p-24f, acc[ti][tb][C - 1]);
        }
      }
    }
  }
}

// BIAS2 >= 0: a second column that also starts from the bias (march modes:
// the point value in column 0 and the bound's base in column 1)
template <typename T, int C, int MMAX, int BIAS2 = -1, bool TEAMS = false, int SM = 0, bool RE = false>
SPK_DEV void dense_kloop(const LayerDev<T>& L, const T* __restrict__ X, WRing<T, C, MMAX, SM>& ring, int tid,
                         T (&acc)[Cfg<T, C, MMAX, SM>::TI][Cfg<T, C, MMAX, SM>::TB][C], const uint32_t* live = nullptr) {
  if constexpr (sizeof(T) == 4 && SPK_PACKED_F32) {
    dense_kloop_f32<C, MMAX, BIAS2, TEAMS, SM, RE>(L, X, ring, tid, acc, live);
  } else {
    dense_kloop_scalar<T, C, MMAX, BIAS2, TEAMS, SM>(L, X, ring, tid, acc, live);
  }
}

// RL = 2 (point passes): the hidden layers' activations are all ELU, one
// each -- the epilogue applies it without the runtime activation loop.
// RL = 1: the net's activations are all ReLU, one per hidden layer
// (NetDev::relu_net, checked by the host): the ELU / sin / tanh rules and the
// runtime activation dispatch are compiled out -- a smaller kernel (fewer
// instruction-cache misses, fewer registers) for the configs' ReLU nets.
struct NoEmit {
  template <class S> SPK_DEV void operator()(int, const S&) const {}
};

// FF (fused final): this is the last hidden layer and the next one is the
// width-1 output layer without activations (Lf).  Instead of writing X and
// running narrow_layer, each thread folds its packed neurons straight into the
// output's columns (RN FMA chain over its TI neurons, RU error column), the NG
// threads of a box group combine them with a butterfly, and the group's first
// lane emits the bound: chain length TI + log2(NG) + 1, inside the output
// layer's rounding budget (spk_abi.cu).  No X stores, no staging, no syncs.
template <typename T, int C, int MMAX, int MODE, int SM = 0, int RL = 0, bool FF = false, class Emit = NoEmit>
SPK_DEV void generic_layer(const LayerDev<T>& L, T* __restrict__ X, WRing<T, C, MMAX, SM>& ring, int tid,
                           bool last, T gamma_next, int lidx, const LayerDev<T>* Lf = nullptr,
                           Emit* emit = nullptr) {
  using CF = Cfg<T, C, MMAX, SM>;
  constexpr int TI = CF::TI, TB = CF::TB, CP = CF::CP;
  const int ng = tid % CF::NG, bg = tid / CF::NG;
  static_assert(!FF || (CF::NG <= 32 && MODE == MODE_AFFINE), "fused final layer: box group within a warp");
  T wf[FF ? TI : 1];
  T fin[FF ? TB : 1][FF ? C : 1];
  if constexpr (FF) {
    load_group<T, TI, CF::G, CF::NG>(Lf->w, Lf->m_in, ng, wf);
#pragma unroll
    for (int tb = 0; tb < TB; ++tb)
#pragma unroll
      for (int c = 0; c < C; ++c) fin[tb][c] = T(0);
  }
  // live-row masks (Cfg::LIVE; bound modes): this layer reads parity lidx&1
  // (written by the previous epilogue; the first layer reads every row) and
  // its epilogue fills the other parity, cleared here -- its last reader
  // (the previous layer's K loop) finished before the previous epilogue
  constexpr bool LV = CF::LIVE && (MODE == MODE_AFFINE || MODE == MODE_INTERVAL);
  uint32_t* m_nxt = nullptr;
  const uint32_t* m_cur = nullptr;
  // one warp per box group holding 4-neuron groups at 4*lane (NG == 32, G == 4):
  // the masks are assembled with shuffles and stored whole, no clearing/atomics
  constexpr bool WMASK = LV && CF::NG == 32 && CF::G == 4;
  // one neuron per thread over the whole CTA (SM = 1 tile): warp w holds
  // neurons 32w..32w+31 = mask word w, one ballot
  constexpr bool BMASK = LV && CF::TI == 1 && CF::NG == NT;
  // narrow nets (NG < 32): every box group of a warp stores the warp's union
  // (redux.sync per G-neuron group, accumulated per word, stored whole)
  constexpr bool XMASK = LV && CF::NG < 32;
  uint32_t xw[CF::LW];
#pragma unroll
  for (int w = 0; w < CF::LW; ++w) xw[w] = 0u;
  if (LV && ring.live != nullptr) {
    m_nxt = ring.live + (size_t)(((lidx + 1) & 1) * CF::NBG + bg) * CF::LW;
    if (lidx > 0) m_cur = ring.live + (size_t)((lidx & 1) * CF::NBG + bg) * CF::LW;
    if (!WMASK && !BMASK && !XMASK && ng < CF::LW) m_nxt[ng] = 0u;
  }
  // layer parameters the epilogue needs, read before the K loop so their
  // latency hides behind it (dynamically indexed parameter / global reads at
  // the epilogue stalled every warp at once); the common single-ReLU layer
  // takes a constant-folded rule
  const int nact = L.n_act;
  const bool relu_only = (RL == 1) ? nact == 1 : (nact == 1 && L.act[0] == ACT_RELU);
  T be_r[TI];
  if (MODE != MODE_POINT) {
    load_group<T, TI, CF::G, CF::NG>(L.berr, L.m_out, ng, be_r);
  } else {
#pragma unroll
    for (int ti = 0; ti < TI; ++ti) be_r[ti] = T(0);
  }
  T acc[TI][TB][C];
  // running-error K loop (affine-fixed, FP32): this layer bounds its base
  // column's rounding itself, so the packs feeding a generic layer of this
  // instantiation charge only the weight rounding on |base| (gamma_base_next)
  // (wide-net tiles only: on the 2-CTA/SM tiles of narrow nets -- 128-register
  // cap -- the second form of the loop cost 15-25%, for little: their excess
  // is already small; consistency is per instantiation, so a tile without RE
  // packs with the full budget and ignores the runerr flags)
  // (the small tile, SM = 1, runs the same bound as the big tiles of its
  // width, so every processing order of a batch stays bit-identical)
  constexpr bool RE = SPK_RUNERR && SPK_PACKED_F32 && sizeof(T) == 4 && MODE == MODE_AFFINE && C >= 3 &&
                      (CF::MINB == 1 || SM == 1 || (MMAX == 64 && MMAX <= CF::SUB));
  const T gamma_base = RE ? L.gamma_base_next : T(-1);
  dense_kloop<T, C, MMAX, (MODE >= MODE_MI ? 1 : -1), CF::TEAMSYNC, SM, RE>(L, X, ring, tid, acc, m_cur);

  // epilogue: activation rules, write next X in place (one contiguous
  // TB*CP vector per neuron: the thread's boxes are adjacent in the row)
  if (MODE == MODE_POINT) {
    // point values: ReLU unrolled; any other activation through ONE rolled
    // loop per neuron so its (large) code exists once (instruction cache)
#pragma unroll
    for (int ti = 0; ti < TI; ++ti) {
      const int i = CF::neuron(ng, ti);
      T out[TB * CP];
#pragma unroll
      for (int tb = 0; tb < TB; ++tb) out[tb * CP] = i < L.m_out ? acc[ti][tb][0] : T(0);
      if constexpr (RL == 2) {  // ELU-only net: one ELU per hidden layer, none on the output
        if (nact == 1) {
#pragma unroll
          for (int tb = 0; tb < TB; ++tb) out[tb * CP] = elu_value<T>(out[tb * CP]);
        }
      } else
      for (int a = 0; a < nact; ++a) {
        const int act = relu_only ? ACT_RELU : L.act[a];
        if (act == ACT_RELU) {
#pragma unroll
          for (int tb = 0; tb < TB; ++tb) out[tb * CP] = fmax(out[tb * CP], T(0));
        } else if (act == ACT_ELU) {  // small inline code (elu_value): unrolled, registers only
#pragma unroll
          for (int tb = 0; tb < TB; ++tb) out[tb * CP] = elu_value<T>(out[tb * CP]);
        } else if (act != ACT_IDENTITY) {
#pragma unroll 1
          for (int tb = 0; tb < TB; ++tb)
            out[tb * CP] = SPK_INLINE_POINT_ACT ? act_value_inline<T>(act, out[tb * CP])
                                                : act_value_slow<T>(act, out[tb * CP]);
        }
      }
      if (i >= L.m_out) {
#pragma unroll
        for (int tb = 0; tb < TB; ++tb) out[tb * CP] = T(0);
      }
      float4* dst = reinterpret_cast<float4*>(X + CF::xrow(i) + bg * TB * CP);
      const float4* srcv = reinterpret_cast<const float4*>(out);
#pragma unroll
      for (int q = 0; q < (int)(TB * CP * sizeof(T) / 16); ++q) dst[q] = srcv[q];
    }
    if (CF::TEAMSYNC) {
      team_sync<CF::TEAM>(tid);
    } else {
      csync();
    }
    return;
  }
  uint32_t live_bits = 0u;
#pragma unroll
  for (int ti = 0; ti < TI; ++ti) {
    const int i = CF::neuron(ng, ti);
    const bool valid = i < L.m_out;
    const T be = be_r[ti];
    T out[TB * CP];
#pragma unroll
    for (int c = 0; c < TB * CP; ++c) out[c] = T(0);
    // fused ReLU epilogue (affine-fixed): live bit from the rule itself
    constexpr bool FUSED_RELU = SPK_FUSED_RELU && MODE == MODE_AFFINE;
    bool nz_rule = false;
#pragma unroll
    for (int tb = 0; tb < TB; ++tb) {
      if (valid) {
        State<T, C, MODE> st = state_from<T, C, MODE>(acc[ti][tb], be);
        if (FUSED_RELU && relu_only) {
          nz_rule |= relu_affine_pack<T, C, MODE>(st, gamma_next, out + tb * CP, gamma_base);
          if constexpr (FF) {
#pragma unroll
            for (int c = 0; c < C - 1; ++c) fin[tb][c] = Num<T>::fma_rn(wf[ti], out[tb * CP + c], fin[tb][c]);
            fin[tb][C - 1] = Num<T>::fma_ru(fabs(wf[ti]), out[tb * CP + C - 1], fin[tb][C - 1]);
          }
          continue;
        }
        if (relu_only) {
          apply_act<T, C, MODE>(st, ACT_RELU);
        } else if (RL != 1) {
          for (int a = 0; a < nact; ++a) apply_act<T, C, MODE>(st, L.act[a]);
        }
        pack_next<T, C, MODE>(st, gamma_next, out + tb * CP, gamma_base);
        if constexpr (FF) {
#pragma unroll
          for (int c = 0; c < C - 1; ++c) fin[tb][c] = Num<T>::fma_rn(wf[ti], out[tb * CP + c], fin[tb][c]);
          fin[tb][C - 1] = Num<T>::fma_ru(fabs(wf[ti]), out[tb * CP + C - 1], fin[tb][C - 1]);
        }
        if (LV) {
#pragma unroll
          for (int c = 0; c < CP; ++c) nz_rule |= out[tb * CP + c] != T(0);
        }
      }
    }
    if constexpr (FF) continue;  // nothing goes back to X
    if constexpr (CF::IL) {
      // interleaved segment: 5 pairs (Cfg::xcol)
      float2* d2 = reinterpret_cast<float2*>(X + CF::xrow(i) + bg * CF::GS);
      d2[0] = make_float2(out[0], out[1]);
      d2[1] = make_float2(out[2], out[3]);
      d2[2] = make_float2(out[CP + 0], out[CP + 1]);
      d2[3] = make_float2(out[CP + 2], out[CP + 3]);
      d2[4] = make_float2(out[4], out[CP + 4]);
    } else {
      float4* dst = reinterpret_cast<float4*>(X + CF::xrow(i) + bg * TB * CP);
      const float4* srcv = reinterpret_cast<const float4*>(out);
#pragma unroll
      for (int q = 0; q < (int)(TB * CP * sizeof(T) / 16); ++q) dst[q] = srcv[q];
    }
    if (LV) {
      const bool nz = nz_rule && !ring.group_empty;
      live_bits |= (nz ? 1u : 0u) << (ti % CF::G);
      if (ti % CF::G == CF::G - 1) {  // a group of G consecutive neurons: one word, one atomic
        const int i0 = i - (CF::G - 1);
        if (BMASK) {
          const uint32_t v = __ballot_sync(0xffffffffu, live_bits != 0u);
          if (m_nxt != nullptr && (tid & 31) == 0) m_nxt[i0 >> 5] = v;
        } else if (XMASK) {
          // neurons (ti/G)*NG*G + ng*G + r: the word is fixed by ti (NG*G divides 32)
          xw[((ti / CF::G) * CF::NG * CF::G) >> 5] |= __reduce_or_sync(0xffffffffu, live_bits << (i0 & 31));
        } else if (WMASK) {
          // the warp owns every neuron of its box group: OR the nibbles of the
          // 8 lanes sharing a 32-bit word with shuffles, one plain store each
          uint32_t v = live_bits << (i0 & 31);
          v |= __shfl_xor_sync(0xffffffffu, v, 1);
          v |= __shfl_xor_sync(0xffffffffu, v, 2);
          v |= __shfl_xor_sync(0xffffffffu, v, 4);
          if (m_nxt != nullptr && (ng & 7) == 0) m_nxt[i0 >> 5] = v;
        } else if (m_nxt != nullptr && live_bits != 0u) {
          atomicOr(&m_nxt[i0 >> 5], live_bits << (i0 & 31));
        }
        live_bits = 0u;
      }
    }
  }
  if constexpr (FF) {
    // the box group's NG lanes (consecutive, NG | 32) combine their partials
#pragma unroll
    for (int off = 1; off < CF::NG; off <<= 1) {
#pragma unroll
      for (int tb = 0; tb < TB; ++tb)
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const T o = __shfl_xor_sync(0xffffffffu, fin[tb][c], off);
          fin[tb][c] = c == C - 1 ? Num<T>::add_ru(fin[tb][c], o) : fin[tb][c] + o;
        }
    }
    if (ng == 0) {
#pragma unroll
      for (int tb = 0; tb < TB; ++tb) {
        fin[tb][0] += Lf->bias[0];
        State<T, C, MODE> st = state_from<T, C, MODE>(fin[tb], Lf->berr[0]);
        (*emit)(bg * TB + tb, st);
      }
    }
  } else if (XMASK && m_nxt != nullptr && ng == 0) {
#pragma unroll
    for (int w = 0; w < CF::LW; ++w) m_nxt[w] = xw[w];
  }
  if (CF::TEAMSYNC) {
    team_sync<CF::TEAM>(tid);
  } else {
    csync();
  }
  (void)last;
}

// Narrow layer (m_out <= NARROW_MAX, e.g. the final width-1 layer): LP
// lanes per (box, neuron) item stride over k, then a butterfly over the LP
// lanes.  LP = 32 for wide nets; narrow nets (MMAX <= 64) use LP = 4 -- 8
// items per warp, a 2-level butterfly -- since their k loops are short.
// Rounding budget gamma_n, n = max(ceil(m_in/32) + 6, ceil(m_in/LP) + 3)
// (spk_abi.cu: the same budget covers the 32-lane order of K3F).
template <int MMAX>
constexpr int narrow_lanes() { return MMAX <= 64 ? 4 : 32; }

template <typename T, int C, int MMAX, int MODE, class Emit, int SM = 0, int RL = 0>
SPK_DEV void narrow_layer(const LayerDev<T>& L, T* __restrict__ X, T* __restrict__ NBUF, int tid,
                          bool last, T gamma_next, Emit&& emit) {
  using CF = Cfg<T, C, MMAX, SM>;
  constexpr int CP = CF::CP, KT = CF::KT;
  constexpr int LP = narrow_lanes<MMAX>(), IPW = 32 / LP;  // lanes per item, items per warp
  // team mode: a team reduces and finishes only its own boxes (the X columns
  // it owns); otherwise the whole CTA shares the tile's boxes
  constexpr bool TM = CF::TEAMSYNC;
  constexpr int NW = TM ? CF::TEAM : NT / 32;            // warps sharing the items
  const int warp = tid >> 5, lane = tid & 31, sub = lane / LP, l = lane % LP;
  const int team = TM ? warp / CF::TEAM : 0;
  const int tw = TM ? warp % CF::TEAM : warp;             // warp index within the team
  const int tl = TM ? tid - team * CF::TEAM * 32 : tid;   // thread index within the team
  const int b0 = TM ? team * CF::TEAM_BOXES : 0;
  const int nbox = TM ? CF::TEAM_BOXES : CF::NB;
  auto sync = [&]() {
    if (TM) {
      team_sync<CF::TEAM>(tid);
    } else {
      csync();
    }
  };
  const int items = nbox * L.m_out;
  const bool one = L.m_out == 1;
  for (int it0 = tw * IPW; it0 < items; it0 += NW * IPW) {
    const int it = it0 + sub;
    const bool live = it < items;
    const int b = b0 + (one ? it : it / L.m_out), i = one ? 0 : it % L.m_out;
    const T* wrow = L.w + (size_t)i * L.m_in;
    T p[C];
#pragma unroll
    for (int c = 0; c < C; ++c) p[c] = T(0);
    if (live) {
      for (int k = l; k < L.m_in; k += LP) {
        const T wk = __ldg(wrow + k);
        const T* xk = X + CF::xrow(k) + (b / CF::TB) * CF::GS;
        const int bt = b % CF::TB;
        if (C == 1) {
          p[0] = Num<T>::fma_rn(wk, xk[CF::xcol(bt, 0)], p[0]);
        } else {
#pragma unroll
          for (int c = 0; c < C - 1; ++c) p[c] = Num<T>::fma_rn(wk, xk[CF::xcol(bt, c)], p[c]);
          p[C - 1] = Num<T>::fma_ru(fabs(wk), xk[CF::xcol(bt, C - 1)], p[C - 1]);
        }
      }
    }
#pragma unroll
    for (int off = LP / 2; off > 0; off >>= 1) {
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const T o = __shfl_xor_sync(0xffffffffu, p[c], off);
        p[c] = (C > 1 && c == C - 1) ? Num<T>::add_ru(p[c], o) : p[c] + o;
      }
    }
    if (live && l == 0) {
      T* dst = NBUF + ((size_t)b * NARROW_MAX + i) * CP;
#pragma unroll
      for (int c = 0; c < C; ++c) dst[c] = p[c];
    }
  }
  sync();
  // epilogue
  for (int it = tl; it < items; it += NW * 32) {
    const int b = b0 + it / L.m_out, i = it % L.m_out;
    const T* src = NBUF + ((size_t)b * NARROW_MAX + i) * CP;
    T col[C];
#pragma unroll
    for (int c = 0; c < C; ++c) col[c] = src[c];
    col[0] += L.bias[i];
    if (pv_off(MODE)) col[1] += L.bias[i];  // march modes: the bound's base column too
    State<T, C, MODE> st = state_from<T, C, MODE>(col, L.berr[i]);
    for (int a = 0; a < L.n_act; ++a) apply_act<T, C, MODE>(st, RL == 1 ? (int)ACT_RELU : L.act[a]);
    if (last) {
      emit(b, st);
    } else {
      T out[CP];
#pragma unroll
      for (int c = 0; c < CP; ++c) out[c] = T(0);
      pack_next<T, C, MODE>(st, gamma_next, out);
      T* dst = X + CF::xrow(i) + (b / CF::TB) * CF::GS;
#pragma unroll
      for (int c = 0; c < CP; ++c)
        if (!CF::IL || c < C) dst[CF::xcol(b % CF::TB, c)] = out[c];
    }
  }
  if (!last) {
    // zero the rows a following generic layer reads beyond m_out (own columns)
    const int r_end = ((L.m_out + KT - 1) / KT) * KT;
    const int w = (nbox / CF::TB) * CF::GS;  // the team's boxes are whole groups
    const int n = (r_end - L.m_out) * w;
    for (int q = tl; q < n; q += NW * 32) X[CF::xrow(L.m_out + q / w) + (b0 / CF::TB) * CF::GS + q % w] = T(0);
  }
  sync();
}

// ---------------------------------------------------------------- the pass
// Runs every layer for the CTA's current tile.  X rows [0, d) must hold the
// packed input columns and rows [d, MMAX) zeros; `emit(b, state)` receives
// each box's final width-1 state.
template <typename T, int C, int MMAX, int MODE, class Emit, int SM = 0, int RL = 0>
SPK_DEV void run_layers(const NetDev<T>& net, T* X, T* NBUF, WRing<T, C, MMAX, SM>& ring, int tid,
                        Emit&& emit) {
  using CF = Cfg<T, C, MMAX, SM>;
  // ReLU-specialised affine passes fold the width-1 output layer into the
  // last hidden layer's epilogue (generic_layer FF)
  // (narrow nets only: at width 256 the 5-level butterfly per thread cost
  // +11% on the C2 tree vs the narrow layer's 32-lane split, and the small
  // tile would need the same order to stay bit-identical)
  constexpr bool FUSE = SPK_FUSE_FINAL && RL == 1 && MODE == MODE_AFFINE && CF::NG <= 32 && MMAX <= 64;
  for (int l = 0; l < net.n_layers; ++l) {
    const LayerDev<T>& L = net.L[l];
    const bool last = (l == net.n_layers - 1);
    if (L.narrow) {
      narrow_layer<T, C, MMAX, MODE, Emit, SM, RL>(L, X, NBUF, tid, last, L.gamma_next, emit);
    } else if (FUSE && l + 2 == net.n_layers && net.L[l + 1].narrow && net.L[l + 1].m_out == 1 &&
               net.L[l + 1].n_act == 0) {
      using E = typename std::remove_reference<Emit>::type;
      generic_layer<T, C, MMAX, MODE, SM, RL, FUSE, E>(L, X, ring, tid, false, L.gamma_next, l, &net.L[l + 1],
                                                       &emit);
      break;
    } else {
      generic_layer<T, C, MMAX, MODE, SM, RL>(L, X, ring, tid, last, L.gamma_next, l);
    }
  }
}

// Sound FP64 -> T conversion of one input coordinate of an affine/interval
// state.  Returns the packed columns for X given the centre coordinate and
// the s axis components along this dimension (n_ax of them).
template <typename T, int C, int MODE>
SPK_DEV void input_state(double centre, const double* ax, int n_ax, int stride, State<T, C, MODE>& st) {
  st.base = Num<T>::from_d_rn(centre);
  if (MODE == MODE_POINT) { st.e = T(0); return; }
  T err = conv_err<T>(centre, st.base);
  if (MODE == MODE_INTERVAL) {
    double r = 0.0;
    for (int j = 0; j < n_ax; ++j) r = __dadd_ru(r, fabs(ax[j * stride]));
    st.e = Num<T>::add_ru(Num<T>::from_d_ru(r), err);
  } else {
    constexpr int S = State<T, C, MODE>::S;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const double a = j < n_ax ? ax[j * stride] : 0.0;
      st.A[j] = Num<T>::from_d_rn(a);
      err = Num<T>::add_ru(err, conv_err<T>(a, st.A[j]));
    }
    // axes beyond the compiled S are folded into the error channel (sound)
    for (int j = S; j < n_ax; ++j) {
      err = Num<T>::add_ru(err, Num<T>::from_d_ru(fabs(ax[j * stride])));
    }
    st.e = err;
  }
}

}  // namespace spk
