// Host-pointer entry point: the reference's range_bound_batch contract
// (NumPy in, NumPy out; range_core.py:547) with the host<->device copies
// inside.  Chunks are double-buffered through pinned staging on two streams
// so the PCIe copies and the CPU-side staging memcpy overlap the kernels.
#include <algorithm>
#include <cstring>

#include "spk_kernels.cuh"
#include "spk_abi_internal.h"

namespace spk {

namespace {
struct Slot {
  cudaStream_t st = nullptr;
  cudaEvent_t done = nullptr;
  double *h_in = nullptr, *h_lo = nullptr, *h_hi = nullptr;
  int8_t* h_cls = nullptr;
  double *d_in = nullptr, *d_lo = nullptr, *d_hi = nullptr;
  int8_t* d_cls = nullptr;
  long long first = -1, count = 0;
};
}  // namespace

int host_pipeline(const spk_net* net, int policy, int n_keep, int precision, long long n, int s,
                  const double* centers, const double* axes, double* lo, double* hi, int8_t* cls) {
  DeviceGuard g(net->device);
  const int d = net->input_dim;
  const long long chunk = std::min<long long>(n, 1 << 20);
  const size_t in_per_box = (size_t)d * (1 + s);
  Slot slots[2];
  int rc = SPK_OK;
  auto check = [&](cudaError_t e, const char* w) {
    if (e != cudaSuccess && rc == SPK_OK) rc = cuda_fail(e, w);
    return rc == SPK_OK;
  };
  for (auto& sl : slots) {
    if (!check(cudaStreamCreateWithFlags(&sl.st, cudaStreamNonBlocking), "stream")) break;
    if (!check(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming), "event")) break;
    if (!check(cudaMallocHost(&sl.h_in, chunk * in_per_box * sizeof(double)), "pinned")) break;
    if (!check(cudaMallocHost(&sl.h_lo, chunk * sizeof(double)), "pinned")) break;
    if (!check(cudaMallocHost(&sl.h_hi, chunk * sizeof(double)), "pinned")) break;
    if (!check(cudaMallocHost(&sl.h_cls, chunk), "pinned")) break;
    if (!check(cudaMalloc(&sl.d_in, chunk * in_per_box * sizeof(double)), "device")) break;
    if (!check(cudaMalloc(&sl.d_lo, chunk * sizeof(double)), "device")) break;
    if (!check(cudaMalloc(&sl.d_hi, chunk * sizeof(double)), "device")) break;
    if (!check(cudaMalloc(&sl.d_cls, chunk), "device")) break;
  }
  auto drain = [&](Slot& sl) {
    if (sl.first < 0) return;
    check(cudaEventSynchronize(sl.done), "sync");
    std::memcpy(lo + sl.first, sl.h_lo, sl.count * sizeof(double));
    std::memcpy(hi + sl.first, sl.h_hi, sl.count * sizeof(double));
    if (cls) std::memcpy(cls + sl.first, sl.h_cls, sl.count);
    sl.first = -1;
  };
  long long i = 0;
  for (long long start = 0; rc == SPK_OK && start < n; start += chunk, ++i) {
    Slot& sl = slots[i & 1];
    drain(sl);
    const long long cnt = std::min(chunk, n - start);
    // staging layout: centres (cnt x d) then axes (cnt x s x d)
    std::memcpy(sl.h_in, centers + start * d, cnt * d * sizeof(double));
    if (s > 0) std::memcpy(sl.h_in + cnt * d, axes + start * s * d, cnt * s * d * sizeof(double));
    if (!check(cudaMemcpyAsync(sl.d_in, sl.h_in, cnt * in_per_box * sizeof(double), cudaMemcpyHostToDevice,
                               sl.st), "H2D"))
      break;
    rc = spk_bound_batch(net, policy, n_keep, precision, cnt, s, sl.d_in, sl.d_in + cnt * d, sl.d_lo, sl.d_hi,
                         sl.d_cls, sl.st);
    if (rc != SPK_OK) break;
    check(cudaMemcpyAsync(sl.h_lo, sl.d_lo, cnt * sizeof(double), cudaMemcpyDeviceToHost, sl.st), "D2H");
    check(cudaMemcpyAsync(sl.h_hi, sl.d_hi, cnt * sizeof(double), cudaMemcpyDeviceToHost, sl.st), "D2H");
    check(cudaMemcpyAsync(sl.h_cls, sl.d_cls, cnt, cudaMemcpyDeviceToHost, sl.st), "D2H");
    check(cudaEventRecord(sl.done, sl.st), "event");
    sl.first = start;
    sl.count = cnt;
  }
  for (auto& sl : slots) drain(sl);
  for (auto& sl : slots) {
    if (sl.st) cudaStreamSynchronize(sl.st);
    cudaFreeHost(sl.h_in); cudaFreeHost(sl.h_lo); cudaFreeHost(sl.h_hi); cudaFreeHost(sl.h_cls);
    cudaFree(sl.d_in); cudaFree(sl.d_lo); cudaFree(sl.d_hi); cudaFree(sl.d_cls);
    if (sl.done) cudaEventDestroy(sl.done);
    if (sl.st) cudaStreamDestroy(sl.st);
  }
  return rc;
}

}  // namespace spk
