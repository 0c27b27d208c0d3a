// Fused range-marching round (K6 fast path for interval / affine-fixed).
//
// One network pass per round evaluates, for every active ray, BOTH the
// convergence probe f(p + (t+delta) r) and the bound over the segment
// [t, t+sigma] (rays.py:117-133): column 0 of the state is the point value,
// the remaining columns the interval (c, v) or affine S=1 (base, A, v)
// state.  Inputs are generated in the prep stage from the FP64 ray state
// with the reference's expressions, and the emit stage applies the FP64
// update (flip test, sigma *= eta+/eta-, t += max(safety sigma*, delta),
// rays.py:121-137) -- so a round is one kernel plus the compaction.
#pragma once
#include "spk_kernels.cuh"

namespace spk {

struct MarchParamsDev {
  double t_max, sigma0, eta_plus, eta_minus, delta, safety;
};

struct MarchState {
  const int* idx;        // active ray indices (compacted)
  const double* origins;
  long long ostride;     // 0: every ray shares origins[0..2]
  const double* dirs;
  double* t;
  double* sig;
  double* steps;
  uint8_t* hit;
  double* t_out;
  const uint8_t* neg0;
  uint8_t* live;
  unsigned long long* certified;
};

template <typename T, int C, int MMAX, int MODE>
__global__ void __launch_bounds__(NT, (Cfg<T, C, MMAX>::MINB))
    march_round_kernel(const NetDev<T> net, const MarchState M, const MarchParamsDev P, const long long n) {
  using CF = Cfg<T, C, MMAX>;
  constexpr int NB = CF::NB, CP = CF::CP;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  T* Wst = X + CF::XS;
  T* NBUF = Wst + CF::NS * CF::TILE;
  uint64_t* full = reinterpret_cast<uint64_t*>(NBUF + CF::NBUF);
  unsigned* released = reinterpret_cast<unsigned*>(full + 16);
  const int tid = threadIdx.x;
  const long long nbt = (n + NB - 1) / NB;
  const long long mine = blockIdx.x < nbt ? (nbt - 1 - blockIdx.x) / gridDim.x + 1 : 0;
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
  if (CF::LIVE) ring.live = reinterpret_cast<uint32_t*>(released + 16);
  ring.prologue(tid);

  for (long long tile = blockIdx.x; tile < nbt; tile += gridDim.x) {
    const long long g0 = tile * NB;
    if (CF::TEAMSYNC) csync();  // every team is done with the previous tile's X
    // ---- probe point + segment box of every ray in the tile -> X rows 0..3
    for (int q = tid; q < 4 * NB; q += NT) {
      const int k = q / NB, b = q % NB;
      T packed[CP];
#pragma unroll
      for (int c = 0; c < CP; ++c) packed[c] = T(0);
      const long long j = g0 + b;
      if (k < 3 && j < n) {
        const int i = M.idx[j];
        const double p = M.origins[i * M.ostride + k], r = M.dirs[(long long)i * 3 + k];
        const double ti = M.t[i], si = M.sig[i];
        const double probe = __dadd_rn(p, __dmul_rn(__dadd_rn(ti, P.delta), r));
        const double centre = __dadd_rn(p, __dmul_rn(__dadd_rn(ti, __ddiv_rn(si, 2.0)), r));
        const double axis = __dmul_rn(__ddiv_rn(si, 2.0), r);
        State<T, C, MODE> st;
        st.pv = Num<T>::from_d_rn(probe);
        st.base = Num<T>::from_d_rn(centre);
        T err = conv_err<T>(centre, st.base);
        if (MODE == MODE_MA) {
          st.A[0] = Num<T>::from_d_rn(axis);
          st.e = Num<T>::add_ru(err, conv_err<T>(axis, st.A[0]));
        } else {
          st.e = Num<T>::add_ru(Num<T>::from_d_ru(fabs(axis)), err);
        }
        for (int a = 0; a < net.n_pre; ++a) apply_act<T, C, MODE>(st, net.pre_act[a]);
        pack_next<T, C, MODE>(st, net.gamma_first, packed);
      }
      T* dst = X + CF::xrow(k) + b * CP;
#pragma unroll
      for (int c = 0; c < CP; ++c) dst[c] = packed[c];
    }
    csync();
    auto emit = [&](int b, const State<T, C, MODE>& st) {
      const long long j = g0 + b;
      if (j >= n) return;
      const int i = M.idx[j];
      M.steps[i] = __dadd_rn(M.steps[i], 1.0);
      const double fv = (double)st.pv;
      if ((fv < 0.0) != (M.neg0[i] != 0)) {  // sign flip a delta ahead: hit at t
        M.hit[i] = 1;
        M.t_out[i] = M.t[i];
        M.live[i] = 0;
        return;
      }
      double lo, hi;
      final_bounds<T, C, MODE>(st, lo, hi);
      const bool known = (lo > 0.0) || (hi < 0.0);
      const double sa = M.sig[i];
      const double star = known ? sa : 0.0;
      M.sig[i] = known ? __dmul_rn(sa, P.eta_plus) : __dmul_rn(sa, P.eta_minus);
      const double nt = __dadd_rn(M.t[i], fmax(__dmul_rn(P.safety, star), P.delta));
      M.t[i] = nt;
      M.live[i] = nt < P.t_max ? 1 : 0;
      if (known) atomicAdd(M.certified, 1ull);
    };
    run_layers<T, C, MMAX, MODE>(net, X, NBUF, ring, tid, emit);
  }
}

template <typename T, int C, int MMAX, int MODE>
cudaError_t launch_march_round(const NetDev<T>& net, const MarchState& M, const MarchParamsDev& P, long long n,
                               int sm_count, cudaStream_t stream) {
  using CF = Cfg<T, C, MMAX>;
  auto kfn = march_round_kernel<T, C, MMAX, MODE>;
  static std::atomic<unsigned long long> optin{0};
  if (cudaError_t e = smem_optin((const void*)kfn, (int)CF::SMEM, optin)) return e;
  if (n <= 0) return cudaSuccess;
  const long long nbt = (n + CF::NB - 1) / CF::NB;
  const long long slots = (long long)sm_count * CF::MINB;
  const int grid = (int)(nbt < slots ? nbt : slots);
  kfn<<<grid, NT, CF::SMEM, stream>>>(net, M, P, n);
  return cudaGetLastError();
}

template <typename T>
cudaError_t dispatch_march_round(int mmax, bool affine, const NetDev<T>& net, const MarchState& M,
                                 const MarchParamsDev& P, long long n, int sm, cudaStream_t st);

#define SPK_MARCH_CASE(T, MM)                                                                          \
  case MM:                                                                                            \
    return affine ? launch_march_round<T, 4, MM, MODE_MA>(net, M, P, n, sm, st)                       \
                  : launch_march_round<T, 3, MM, MODE_MI>(net, M, P, n, sm, st);

#define SPK_DEFINE_MARCH_DISPATCH(T)                                                                   \
  template <>                                                                                         \
  cudaError_t dispatch_march_round<T>(int mmax, bool affine, const NetDev<T>& net, const MarchState& M, \
                                      const MarchParamsDev& P, long long n, int sm, cudaStream_t st) { \
    switch (mmax) {                                                                                   \
      SPK_MARCH_CASE(T, 32)                                                                           \
      SPK_MARCH_CASE(T, 64)                                                                           \
      SPK_MARCH_CASE(T, 128)                                                                          \
      SPK_MARCH_CASE(T, 256)                                                                          \
      default:                                                                                        \
        return affine ? launch_march_round<T, 4, 512, MODE_MA>(net, M, P, n, sm, st)                  \
                      : launch_march_round<T, 3, 512, MODE_MI>(net, M, P, n, sm, st);                 \
    }                                                                                                 \
  }

}  // namespace spk
