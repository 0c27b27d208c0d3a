// Spatial processing order for large box batches.
//
// The fused pass skips X rows that are exactly zero for every box of a box
// group (live-row masks, spk_pass.cuh): ReLU-inactive neurons.  Boxes that are
// close in space share their inactive sets, so a batch of independent boxes in
// arbitrary order (C5's random cubes, a user's range_bound_batch) is bounded
// in Morton order of the box centres: keys from the centres quantised to
// 2^10 cells per axis over the batch's bounding box, one CUB radix sort of
// (key, index), and the kernel reads box perm[slot] and writes its bound back
// to the same index.  Each box's bound does not depend on its neighbours, so
// the results are identical to the natural order.
#include <cub/cub.cuh>

#include "spk_abi_internal.h"
#include "spk_kernels.cuh"

namespace spk {

namespace {

SPK_DEV unsigned long long ordered_bits(double x) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
SPK_DEV double from_ordered(unsigned long long o) {
  const unsigned long long u = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
  return __longlong_as_double((long long)u);
}

SPK_DEV double centre_of(const BoxInput& in, long long gb, int k, int d) {
  if (in.kind == IN_RANDOM) return random_coord(in.seed, in.first + gb, k, d);
  if (in.kind == IN_AABB) return 0.5 * (in.a[gb * d + k] + in.b[gb * d + k]);
  return in.a[gb * d + k];  // IN_BOXES / IN_POINTS: centres
}

// per-axis min / max of the centres (ordered-integer atomics)
__global__ void centre_range_kernel(BoxInput in, int d, long long n_cap, unsigned long long* mn,
                                    unsigned long long* mx) {
  const long long n = in.n_dev ? (*in.n_dev < n_cap ? *in.n_dev : n_cap) : n_cap;
  unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0ull, 0ull, 0ull};
  for (long long gb = blockIdx.x * (long long)blockDim.x + threadIdx.x; gb < n; gb += (long long)gridDim.x * blockDim.x) {
    for (int k = 0; k < d; ++k) {
      const unsigned long long o = ordered_bits(centre_of(in, gb, k, d));
      lo[k] = o < lo[k] ? o : lo[k];
      hi[k] = o > hi[k] ? o : hi[k];
    }
  }
  for (int k = 0; k < d; ++k) {
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo[k], off);
      const unsigned long long b = __shfl_xor_sync(0xffffffffu, hi[k], off);
      lo[k] = a < lo[k] ? a : lo[k];
      hi[k] = b > hi[k] ? b : hi[k];
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&mn[k], lo[k]);
      atomicMax(&mx[k], hi[k]);
    }
  }
}

SPK_DEV unsigned int spread3(unsigned int v) {  // 10 bits -> every third bit
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000FFu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

__global__ void morton_kernel(BoxInput in, int d, long long n_cap, const unsigned long long* mn,
                              const unsigned long long* mx, unsigned int* keys, int* idx) {
  // slots past a device-side count sort last (key above every 30-bit code)
  const long long n = in.n_dev ? (*in.n_dev < n_cap ? *in.n_dev : n_cap) : n_cap;
  double lo[3], inv[3];
  for (int k = 0; k < d; ++k) {
    lo[k] = from_ordered(mn[k]);
    const double w = from_ordered(mx[k]) - lo[k];
    inv[k] = w > 0.0 ? 1023.999 / w : 0.0;
  }
  for (long long gb = blockIdx.x * (long long)blockDim.x + threadIdx.x; gb < n_cap;
       gb += (long long)gridDim.x * blockDim.x) {
    if (gb >= n) {
      keys[gb] = 0xFFFFFFFFu;
      idx[gb] = (int)gb;
      continue;
    }
    unsigned int key = 0u;
    for (int k = 0; k < d; ++k) {
      double q = (centre_of(in, gb, k, d) - lo[k]) * inv[k];
      q = q < 0.0 ? 0.0 : (q > 1023.0 ? 1023.0 : q);  // NaN-safe clamp
      key |= spread3((unsigned int)q) << (2 - k);
    }
    keys[gb] = key;
    idx[gb] = (int)gb;
  }
}

}  // namespace

// Morton processing order of a batch of n (capacity; in.n_dev, when given, is
// the live count: the other slots sort last) boxes, n < 2^31.  *perm points
// into *scratch, which the caller releases with cudaFreeAsync on `st`.
int spatial_order(const BoxInput& in, int d, long long n, int sm, cudaStream_t st, int** perm, void** scratch) {
  *perm = nullptr;
  *scratch = nullptr;
  if (n <= 0 || n >= (1ll << 31) || d < 1 || d > 3) return SPK_OK;
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (unsigned int*)nullptr, (unsigned int*)nullptr,
                                  (int*)nullptr, (int*)nullptr, (int)n, 0, 32, st);
  const size_t nb = (size_t)n;
  const size_t bytes = 64 + 2 * nb * 4 + 2 * nb * 4 + tmp_bytes + 256;
  char* base = nullptr;
  cudaError_t e = cudaMallocAsync(&base, bytes, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(spatial order)");
  unsigned long long* mn = reinterpret_cast<unsigned long long*>(base);
  unsigned long long* mx = mn + 4;
  unsigned int* k0 = reinterpret_cast<unsigned int*>(base + 64);
  unsigned int* k1 = k0 + nb;
  int* i0 = reinterpret_cast<int*>(k1 + nb);
  int* i1 = i0 + nb;
  void* tmp = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(i1 + nb) + 255) & ~(uintptr_t)255);
  static const unsigned long long init[8] = {~0ull, ~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull, 0ull};
  e = cudaMemcpyAsync(mn, init, sizeof(init), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "spatial order init");
  const int grid = (int)std::min<long long>((n + 255) / 256, (long long)(sm > 0 ? sm : 148) * 8);
  centre_range_kernel<<<grid, 256, 0, st>>>(in, d, n, mn, mx);
  morton_kernel<<<grid, 256, 0, st>>>(in, d, n, mn, mx, k0, i0);
  e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, i0, i1, (int)n, 0, 32, st);
  if (e != cudaSuccess) return cuda_fail(e, "spatial order sort");
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "spatial order kernels");
  *perm = i1;
  *scratch = base;
  return SPK_OK;
}

}  // namespace spk
