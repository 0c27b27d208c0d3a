// Host-pointer entry point: the reference's range_bound_batch contract
// (NumPy in, NumPy out; range_core.py:547) with the host<->device copies
// inside.  Chunks are double-buffered through pinned staging on two streams
// so the PCIe copies and the CPU-side staging memcpy overlap the kernels.
#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include "spk_kernels.cuh"
#include "spk_abi_internal.h"

namespace spk {

namespace {
// Grow-only buffer: pinned host or device memory, reused across calls.
template <bool PINNED>
struct Buf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t reserve(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    release();
    const size_t want = std::max<size_t>(bytes + bytes / 4, 1 << 16);
    cudaError_t e = PINNED ? cudaMallocHost(&p, want) : cudaMalloc(&p, want);
    if (e != cudaSuccess) { p = nullptr; return e; }
    cap = want;
    return cudaSuccess;
  }
  void release() {
    if (p) { if (PINNED) cudaFreeHost(p); else cudaFree(p); }
    p = nullptr;
    cap = 0;
  }
  template <typename T> T* as() const { return static_cast<T*>(p); }
};

struct Slot {
  cudaStream_t st = nullptr;
  cudaEvent_t done = nullptr;
  Buf<true> h_in, h_out;   // staging: centres + axes / lo, hi, cls
  Buf<false> d_in, d_out;
  long long first = -1, count = 0;
};

// Per-thread, per-device staging: the reference calls range_bound_batch in
// 4096-box chunks (spatial.py:38) from ThreadPoolExecutor workers
// (rays.py:170-181), so every call must neither allocate nor synchronise the
// device (cudaFree would) and concurrent threads must not share buffers.
// Streams, events and grow-only buffers live as long as the thread.
struct HostCtx {
  int device = -1;
  Slot slots[2];
  bool ready = false;
  ~HostCtx() {
    if (!ready) return;
    int prev = 0;
    if (cudaGetDevice(&prev) != cudaSuccess) return;  // runtime already torn down
    cudaSetDevice(device);
    for (auto& sl : slots) {
      if (sl.st) cudaStreamSynchronize(sl.st);
      sl.h_in.release(); sl.h_out.release(); sl.d_in.release(); sl.d_out.release();
      if (sl.done) cudaEventDestroy(sl.done);
      if (sl.st) cudaStreamDestroy(sl.st);
    }
    cudaSetDevice(prev);
  }
};

HostCtx* host_ctx(int device) {
  thread_local std::vector<std::unique_ptr<HostCtx>> per_device;
  if ((int)per_device.size() <= device) per_device.resize(device + 1);
  if (!per_device[device]) per_device[device].reset(new HostCtx);
  return per_device[device].get();
}
}  // namespace

int host_pipeline(const spk_net* net, int policy, int n_keep, int precision, long long n, int s,
                  const double* centers, const double* axes, double* lo, double* hi, int8_t* cls) {
  DeviceGuard g(net->device);
  const int d = net->input_dim;
  const long long chunk = std::min<long long>(n, 1 << 20);
  const size_t in_bytes = (size_t)chunk * d * (1 + s) * sizeof(double);
  const size_t out_bytes = (size_t)chunk * (2 * sizeof(double) + 1);
  HostCtx* ctx = host_ctx(net->device);
  int rc = SPK_OK;
  auto check = [&](cudaError_t e, const char* w) {
    if (e != cudaSuccess && rc == SPK_OK) rc = cuda_fail(e, w);
    return rc == SPK_OK;
  };
  if (!ctx->ready) {
    ctx->device = net->device;
    for (auto& sl : ctx->slots) {
      if (!check(cudaStreamCreateWithFlags(&sl.st, cudaStreamNonBlocking), "stream")) return rc;
      if (!check(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming), "event")) return rc;
    }
    ctx->ready = true;
  }
  const int used = n > chunk ? 2 : 1;
  for (int k = 0; k < used; ++k) {
    Slot& sl = ctx->slots[k];
    if (!check(sl.h_in.reserve(in_bytes), "pinned") || !check(sl.h_out.reserve(out_bytes), "pinned") ||
        !check(sl.d_in.reserve(in_bytes), "device") || !check(sl.d_out.reserve(out_bytes), "device"))
      return rc;
    sl.first = -1;
  }
  auto drain = [&](Slot& sl) {
    if (sl.first < 0) return;
    check(cudaEventSynchronize(sl.done), "sync");
    const double* h = sl.h_out.as<double>();
    std::memcpy(lo + sl.first, h, sl.count * sizeof(double));
    std::memcpy(hi + sl.first, h + sl.count, sl.count * sizeof(double));
    if (cls) std::memcpy(cls + sl.first, reinterpret_cast<const int8_t*>(h + 2 * sl.count), sl.count);
    sl.first = -1;
  };
  long long i = 0;
  for (long long start = 0; rc == SPK_OK && start < n; start += chunk, ++i) {
    Slot& sl = ctx->slots[i % used];
    drain(sl);
    if (rc != SPK_OK) break;
    const long long cnt = std::min(chunk, n - start);
    // staging layout: centres (cnt x d) then axes (cnt x s x d); results lo, hi, cls
    double* hin = sl.h_in.as<double>();
    double* din = sl.d_in.as<double>();
    double* dout = sl.d_out.as<double>();
    std::memcpy(hin, centers + start * d, cnt * d * sizeof(double));
    if (s > 0) std::memcpy(hin + cnt * d, axes + start * s * d, cnt * s * d * sizeof(double));
    if (!check(cudaMemcpyAsync(din, hin, cnt * d * (1 + s) * sizeof(double), cudaMemcpyHostToDevice, sl.st),
               "H2D"))
      break;
    rc = spk_bound_batch(net, policy, n_keep, precision, cnt, s, din, din + cnt * d, dout, dout + cnt,
                         reinterpret_cast<int8_t*>(dout + 2 * cnt), sl.st);
    if (rc != SPK_OK) break;
    check(cudaMemcpyAsync(sl.h_out.p, dout, cnt * (2 * sizeof(double) + 1), cudaMemcpyDeviceToHost, sl.st), "D2H");
    check(cudaEventRecord(sl.done, sl.st), "event");
    sl.first = start;
    sl.count = cnt;
  }
  for (int k = 0; k < used; ++k) {
    if (rc == SPK_OK) {
      drain(ctx->slots[k]);
    } else {  // leave the slots idle for the next call
      cudaStreamSynchronize(ctx->slots[k].st);
      ctx->slots[k].first = -1;
    }
  }
  return rc;
}

}  // namespace spk
