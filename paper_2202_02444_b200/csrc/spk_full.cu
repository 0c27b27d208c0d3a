// K3F: affine-full with a large symbol capacity (range_core.py:595-603 with
// PolicyKind.FULL: every activation appends diag(gamma) as new symbols and
// nothing is ever condensed; capacity s + sum of hidden activation widths,
// _plan_symbol_capacity range_core.py:530-544).
//
// The register-tiled symbolic kernel (spk_symbolic.cuh) holds <= 32
// symbols; the reference's DEFAULT policy for trees, meshes and the
// volumetric queries is affine-full, which on the 7x32 fixtures needs 227
// symbols and on an 8x256 net 1795.  This kernel trades tiling for
// capacity: one persistent CTA works on one box at a time, its symbol
// matrix A[k][i] (column 0 = base, columns 1.. = symbols, neuron-contiguous
// rows of stride MMAX) lives in a per-CTA global scratch (L1/L2 resident for
// small nets) and is ping-ponged between two buffers per dense layer:
//   dense      A'[k][o] = sum_i W[o][i] A[k][i] over every column k, with the
//              fused pass's blocked summation (SUB-term FMA chains, partial
//              sums added in order, bias last) so the network's
//              pre-computed sound rounding budgets (gamma', berr) apply
//              unchanged; error e'[o] = RU(sum_i |W[o][i]| v[i]) + berr[o];
//   activation per neuron: r = RU(sum_k |A[k][o]|) + e, sound rule
//              (alpha, beta, gamma) on [base - r, base + r], base/A scaled,
//              products' rounding into e, gamma appended as a new one-hot
//              symbol column (never dropped);
//   pack       v = e + gamma'(|base| + sum|A| + e) for the next layer;
//   final      width-1 layer by warp butterfly (the narrow path's order),
//              final activations fold gamma into e (same lo/hi), outward
//              rounded lo/hi.
// affine-truncate beyond the register tile (n_keep > 16 on widths > 64, > 32
// otherwise) runs here too: after each activation's append, per-symbol L1
// norms (one warp per symbol), rank = #(larger norm, or equal norm and lower
// index) -- the reference's stable argsort, range_core.py:604-619 -- the
// n_keep best kept in their original order, the dropped |coefficients| added
// to the error channel with round-up adds.
// FP32: sound like every other kernel; FP64: the reference's algorithm.
#include <algorithm>
#include <string>

#include "spk_kernels.cuh"
#include "spk_abi_internal.h"

namespace spk {

constexpr int FULL_MMAX = 512;

struct FullParams {
  int mmax, kt, sub, ncol_cap, s0;
  int n_keep;  // affine-truncate: symbols kept after every activation (0 = affine-full)
  long long toff[MAX_LAYERS];  // first W^T tile row of every generic layer
};

// RA[o] = RU(sum_{k >= 1} |A[k][o]|), deterministic split over the CTA
template <typename T>
SPK_DEV void symbol_norms(const T* __restrict__ A, int ncol, int m, int M, T* PART, T* RA, int tid) {
  if (m >= NT) {
    for (int o = tid; o < m; o += NT) {
      T s = T(0);
      for (int k = 1; k < ncol; ++k) s = Num<T>::add_ru(s, fabs(A[(size_t)k * M + o]));
      RA[o] = s;
    }
  } else {
    const int P = NT / m, part = tid / m, o = tid % m;
    if (part < P) {
      T s = T(0);
      for (int k = 1 + part; k < ncol; k += P) s = Num<T>::add_ru(s, fabs(A[(size_t)k * M + o]));
      PART[part * m + o] = s;
    }
    __syncthreads();
    for (int q = tid; q < m; q += NT) {
      T s = T(0);
      for (int p = 0; p < P; ++p) s = Num<T>::add_ru(s, PART[p * m + q]);
      RA[q] = s;
    }
  }
  __syncthreads();
}

template <typename T>
__global__ void __launch_bounds__(NT) full_bound_kernel(const NetDev<T> net, const BoxInput in,
                                                        const BoundOutput out, const long long n_cap,
                                                        const FullParams P, T* __restrict__ scratch) {
  const long long n = in.n_dev ? *in.n_dev : n_cap;
  __shared__ T E[FULL_MMAX], V[FULL_MMAX], RA[FULL_MMAX], ALPHA[FULL_MMAX], NEWG[FULL_MMAX];
  __shared__ T PART[NT];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, M = P.mmax, d = net.d;
  T* buf0 = scratch + (size_t)blockIdx.x * (2 * (size_t)P.ncol_cap * M + 2 * P.ncol_cap);
  T* buf1 = buf0 + (size_t)P.ncol_cap * M;
  T* NRM = buf1 + (size_t)P.ncol_cap * M;            // truncate: per-symbol L1 norms
  int* POS = reinterpret_cast<int*>(NRM + P.ncol_cap);  // truncate: kept flag per symbol

  for (long long slot = blockIdx.x; slot < n; slot += gridDim.x) {
    // optional processing order (fp32-refine re-bounds a subset in place)
    const long long box = in.perm ? (long long)in.perm[slot] : slot;
    T* cur = buf0;
    T* nxt = buf1;
    // ---- input state (prep_inputs' forms), packed for the first layer
    const int s0 = P.s0;
    if (tid < d) {
      const int k = tid;
      double centre;
      constexpr int CI = MAX_AXES + 2;  // base, up to MAX_AXES axis symbols, error
      double ax[MAX_AXES];
      for (int j = 0; j < MAX_AXES; ++j) ax[j] = 0.0;
      int n_ax = 0;
      if (in.kind == IN_BOXES) {
        centre = in.a[box * d + k];
        n_ax = in.s < MAX_AXES ? in.s : MAX_AXES;
        for (int j = 0; j < n_ax; ++j) ax[j] = in.b[(box * in.s + j) * d + k];
      } else if (in.kind == IN_AABB) {
        const double l = in.a[box * d + k], h = in.b[box * d + k];
        centre = (l + h) / 2.0;
        n_ax = d < MAX_AXES ? d : MAX_AXES;
        ax[k] = (h - l) / 2.0;
      } else {
        centre = random_coord(in.seed, in.first + box, k, d);
        n_ax = d < MAX_AXES ? d : MAX_AXES;
        ax[k] = in.half;
      }
      State<T, CI, MODE_AFFINE> st;
      input_state<T, CI, MODE_AFFINE>(centre, ax, n_ax, 1, st);
      T packed[CI];
      pack_next<T, CI, MODE_AFFINE>(st, net.gamma_first, packed);
      cur[k] = packed[0];
      for (int j = 0; j < s0; ++j) cur[(size_t)(1 + j) * M + k] = j < MAX_AXES ? packed[1 + j] : T(0);
      V[k] = packed[CI - 1];
    }
    __syncthreads();
    int ncol = 1 + s0, m_in = d;
    for (int l = 0; l < net.n_layers; ++l) {
      const LayerDev<T>& L = net.L[l];
      const int m = L.m_out;
      if (L.narrow) {
        // ---- final layer: warp per (column, output), lanes stride inputs
        for (int it = warp; it < ncol * m; it += NT / 32) {
          const int k = it / m, o = it % m;
          const T* wrow = L.w + (size_t)o * m_in;
          const T* a = cur + (size_t)k * M;
          T p = T(0);
          for (int i = lane; i < m_in; i += 32) p = Num<T>::fma_rn(__ldg(wrow + i), a[i], p);
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
          if (lane == 0) nxt[(size_t)k * M + o] = k == 0 ? p + L.bias[o] : p;
        }
        for (int o = warp; o < m; o += NT / 32) {
          const T* wrow = L.w + (size_t)o * m_in;
          T p = T(0);
          for (int i = lane; i < m_in; i += 32) p = Num<T>::fma_ru(fabs(__ldg(wrow + i)), V[i], p);
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) p = Num<T>::add_ru(p, __shfl_xor_sync(0xffffffffu, p, off));
          if (lane == 0) E[o] = Num<T>::add_ru(p, L.berr[o]);
        }
        __syncthreads();
        // ---- final activations (gamma folded into e) and the bounds; one
        // warp per output neuron
        for (int o = warp; o < m; o += NT / 32) {
          T base = nxt[o], e = E[o];
          for (int a = 0; a < L.n_act; ++a) {
            if (L.act[a] == ACT_IDENTITY) continue;
            T rA = T(0);
            for (int k = 1 + lane; k < ncol; k += 32) rA = Num<T>::add_ru(rA, fabs(nxt[(size_t)k * M + o]));
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) rA = Num<T>::add_ru(rA, __shfl_xor_sync(0xffffffffu, rA, off));
            const T r = Num<T>::add_ru(rA, e);
            T al, be, ga;
            const int kind = affine_rule<T>(L.act[a], Num<T>::sub_rd(base, r), Num<T>::add_ru(base, r), al, be, ga);
            if (kind == 1) {
              base = T(0);
              e = T(0);
              al = T(0);
            } else if (kind == 2) {
              const T nb = Num<T>::fma_rn(al, base, be);
              const T aa = fabs(al);
              T ne = Num<T>::fma_ru(aa, e, ga);
              ne = Num<T>::fma_ru(Num<T>::RHO, Num<T>::add_ru(fabs(nb), Num<T>::mul_ru(aa, rA)), ne);
              e = Num<T>::add_ru(ne, Num<T>::TINY);
              base = nb;
            } else {
              al = T(1);
            }
            if (al != T(1))
              for (int k = 1 + lane; k < ncol; k += 32) nxt[(size_t)k * M + o] = Num<T>::mul_rn(al, nxt[(size_t)k * M + o]);
            __syncwarp();
          }
          T rA = T(0);
          for (int k = 1 + lane; k < ncol; k += 32) rA = Num<T>::add_ru(rA, fabs(nxt[(size_t)k * M + o]));
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) rA = Num<T>::add_ru(rA, __shfl_xor_sync(0xffffffffu, rA, off));
          if (lane == 0 && o == 0) {
            const T r = Num<T>::add_ru(rA, e);
            const double lo = (double)Num<T>::sub_rd(base, r), hi = (double)Num<T>::add_ru(base, r);
            out.lo[box] = lo;
            if (out.hi) out.hi[box] = hi;
            if (out.cls) out.cls[box] = (int8_t)(lo > 0.0 ? 1 : (hi < 0.0 ? -1 : 0));
          }
        }
        __syncthreads();
        break;
      }
      // ---- hidden dense layer over every column (blocked summation)
      const T* wt = net.wtiles + P.toff[l] * (long long)M;
      for (int q = tid; q < ncol * m; q += NT) {
        const int k = q / m, o = q % m;
        const T* a = cur + (size_t)k * M;
        T tot = T(0);
        for (int i0 = 0; i0 < m_in; i0 += P.sub) {
          const int i1 = min(i0 + P.sub, m_in);
          T p = T(0);
          for (int i = i0; i < i1; ++i) p = Num<T>::fma_rn(wt[(size_t)i * M + o], a[i], p);
          tot = i0 == 0 ? p : tot + p;
        }
        if (k == 0) tot += L.bias[o];
        nxt[(size_t)k * M + o] = tot;
      }
      for (int o = tid; o < m; o += NT) {
        T e = T(0);
        for (int i = 0; i < m_in; ++i) e = Num<T>::fma_ru(fabs(wt[(size_t)i * M + o]), V[i], e);
        E[o] = Num<T>::add_ru(e, L.berr[o]);
      }
      __syncthreads();
      T* t = cur;
      cur = nxt;
      nxt = t;
      m_in = m;
      // ---- activations: rule, scale, append gamma as new symbols
      for (int a = 0; a < L.n_act; ++a) {
        const int act = L.act[a];
        if (act == ACT_IDENTITY) continue;  // range_core.py:586-587
        symbol_norms<T>(cur, ncol, m, M, PART, RA, tid);
        for (int o = tid; o < m; o += NT) {
          T base = cur[o], e = E[o];
          const T rA = RA[o];
          const T r = Num<T>::add_ru(rA, e);
          T al, be, ga;
          const int kind = affine_rule<T>(act, Num<T>::sub_rd(base, r), Num<T>::add_ru(base, r), al, be, ga);
          if (kind == 1) {
            base = T(0);
            e = T(0);
            al = T(0);
            ga = T(0);
          } else if (kind == 2) {
            const T nb = Num<T>::fma_rn(al, base, be);
            const T aa = fabs(al);
            T ne = Num<T>::mul_ru(aa, e);
            ne = Num<T>::fma_ru(Num<T>::RHO, Num<T>::add_ru(fabs(nb), Num<T>::mul_ru(aa, rA)), ne);
            e = Num<T>::add_ru(ne, Num<T>::TINY);
            base = nb;
          } else {
            al = T(1);
            ga = T(0);
          }
          cur[o] = base;
          E[o] = e;
          ALPHA[o] = al;
          NEWG[o] = ga;
        }
        __syncthreads();
        const int total = (ncol - 1 + m) * m;
        for (int q = tid; q < total; q += NT) {
          const int k = 1 + q / m, o = q % m;
          T* p = cur + (size_t)k * M + o;
          if (k < ncol) {
            const T al = ALPHA[o];
            if (al != T(1)) *p = Num<T>::mul_rn(al, *p);
          } else {
            *p = (k - ncol == o) ? NEWG[o] : T(0);
          }
        }
        ncol += m;
        __syncthreads();
        if (P.n_keep > 0 && ncol - 1 > P.n_keep) {
          // ---- affine-truncate (range_core.py:604-619): keep the n_keep
          // symbols of largest L1 norm over the components, ties to the lower
          // index (stable argsort), in their original order; the dropped
          // |coefficients| move into the error channel.  Symbol k is row 1+k-1.
          const int ncand = ncol - 1;
          for (int k = warp; k < ncand; k += NT / 32) {
            const T* row = cur + (size_t)(1 + k) * M;
            T s = T(0);
            for (int o = lane; o < m; o += 32) s += fabs(row[o]);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            if (lane == 0) NRM[k] = s;
          }
          __syncthreads();
          for (int k = tid; k < ncand; k += NT) {
            const T nk = NRM[k];
            int rank = 0;
            for (int j = 0; j < ncand; ++j) {
              const T nj = NRM[j];
              rank += (nj > nk || (nj == nk && j < k)) ? 1 : 0;
            }
            POS[k] = rank < P.n_keep ? 1 : 0;
          }
          __syncthreads();
          for (int k = tid; k < ncand; k += NT) {
            int pos = -1;
            if (POS[k] > 0) {
              pos = 0;
              for (int j = 0; j < k; ++j) pos += POS[j] > 0 ? 1 : 0;
            }
            NRM[k] = (T)pos;  // the norms are dead; POS (read here) stays intact
          }
          __syncthreads();
          for (int o = tid; o < m; o += NT) {
            T dropped = T(0);
            for (int k = 0; k < ncand; ++k)
              if (NRM[k] < T(0)) dropped = Num<T>::add_ru(dropped, fabs(cur[(size_t)(1 + k) * M + o]));
            E[o] = Num<T>::add_ru(E[o], dropped);
            nxt[o] = cur[o];
          }
          for (int q = tid; q < ncand * m; q += NT) {
            const int k = q / m, o = q % m;
            const int pos = (int)NRM[k];
            if (pos >= 0) nxt[(size_t)(1 + pos) * M + o] = cur[(size_t)(1 + k) * M + o];
          }
          __syncthreads();
          T* t2 = cur;
          cur = nxt;
          nxt = t2;
          ncol = 1 + P.n_keep;
        }
      }
      // ---- pack: v = e + gamma'(|base| + sum|A| + e)
      symbol_norms<T>(cur, ncol, m, M, PART, RA, tid);
      for (int o = tid; o < m; o += NT) {
        const T e = E[o];
        V[o] = Num<T>::fma_ru(L.gamma_next, Num<T>::add_ru(Num<T>::add_ru(fabs(cur[o]), RA[o]), e), e);
      }
      __syncthreads();
    }
  }
}

template <typename T>
static int launch_full_t(const spk_net* cnet, const BoxInput& in, const BoundOutput& out, long long n, int s0,
                         int need, int n_keep, cudaStream_t st) {
  spk_net* net = const_cast<spk_net*>(cnet);
  NetDev<T> nd_copy;
  const NetDev<T>* nd = &nd_copy;
  if (int rc = get_dev<T>(net, &nd_copy)) return rc;
  FullParams P;
  P.mmax = net->mmax;
  switch (net->mmax) {
    case 32: P.kt = KTOf<T, 32>::KT; P.sub = KTOf<T, 32>::SUB; break;
    case 64: P.kt = KTOf<T, 64>::KT; P.sub = KTOf<T, 64>::SUB; break;
    case 128: P.kt = KTOf<T, 128>::KT; P.sub = KTOf<T, 128>::SUB; break;
    case 256: P.kt = KTOf<T, 256>::KT; P.sub = KTOf<T, 256>::SUB; break;
    default: P.kt = KTOf<T, 512>::KT; P.sub = KTOf<T, 512>::SUB; break;
  }
  P.ncol_cap = 1 + need;
  P.s0 = s0;
  P.n_keep = n_keep;
  long long t = 0;
  for (int l = 0; l < nd->n_layers && l < MAX_LAYERS; ++l) {
    P.toff[l] = t * P.kt;  // rows of W^T (each MMAX wide) before layer l
    t += nd->L[l].ntiles;
  }
  const int sm = sm_count_for(net->device);
  if (sm <= 0) return fail(SPK_ERR_CUDA, "no CUDA device");
  if (n <= 0) return SPK_OK;
  const long long grid = std::min<long long>(n, (long long)sm * 4);
  T* scratch = nullptr;
  const size_t bytes = (size_t)grid * (2 * (size_t)P.ncol_cap * P.mmax + 2 * P.ncol_cap) * sizeof(T);
  cudaError_t e = cudaMallocAsync(&scratch, bytes, st);
  if (e != cudaSuccess) return cuda_fail(e, "affine-full scratch");
  full_bound_kernel<T><<<(int)grid, NT, 0, st>>>(*nd, in, out, n, P, scratch);
  e = cudaGetLastError();
  cudaFreeAsync(scratch, st);
  if (e != cudaSuccess) return cuda_fail(e, "affine-full kernel");
  return SPK_OK;
}

int launch_full(const spk_net* net, int precision, const BoxInput& in, const BoundOutput& out, long long n, int s0,
                int need, int n_keep, cudaStream_t st) {
  if (net->mmax > FULL_MMAX) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "affine-full: layer width beyond 512");
  if (s0 > MAX_AXES) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "more than 8 box axes");
  if ((int)net->layers.size() > MAX_LAYERS) return fail(SPK_ERR_UNSUPPORTED_SHAPE, "too many layers");
  DeviceGuard g(net->device);
  return precision == SPK_FP64 ? launch_full_t<double>(net, in, out, n, s0, need, n_keep, st)
                               : launch_full_t<float>(net, in, out, n, s0, need, n_keep, st);
}

}  // namespace spk
