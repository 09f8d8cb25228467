// gemm() / gemm_async() / gemm_batch(): the public entry points around
// execute().  Operands may live in host memory (the reference's callers use
// host Matrix objects): each host operand's byte window is copied into HBM,
// the plan's views are rebased into the copy, and C's window is copied back.
//
// gemm_batch() runs a list of independent gemm calls with the host staging
// pipelined across calls on three streams -- copy-in, compute, copy-out --
// so the PCIe transfers of one call overlap the kernels of its neighbours.
// Ordering is that of calling gemm() on each element in turn: a call whose
// host inputs overlap an earlier call's host output waits for that copy-out;
// device-resident operands are ordered by the single compute stream.
#include <algorithm>
#include <mutex>
#include <vector>

#include "driver.hpp"

namespace mdgemm {

namespace {

bool is_device_ptr(const void* ptr) {
  if (!ptr) return false;
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

// Per-device copy-in / compute / copy-out streams (blocking streams, so they
// stay ordered with the legacy default stream other libraries use).
struct Streams {
  cudaStream_t in = nullptr, compute = nullptr, out = nullptr;
};

Streams device_streams() {
  static std::mutex mu;
  static std::vector<Streams> cache;
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lock(mu);
  if (cache.size() <= static_cast<size_t>(dev)) cache.resize(dev + 1);
  Streams& s = cache[dev];
  if (!s.compute) {
    cuda_check(cudaStreamCreate(&s.in), "stream");
    cuda_check(cudaStreamCreate(&s.compute), "stream");
    cuda_check(cudaStreamCreate(&s.out), "stream");
  }
  return s;
}

struct Window {
  const std::byte* lo = nullptr;
  const std::byte* hi = nullptr;
  bool overlaps(const Window& o) const { return lo < o.hi && o.lo < hi; }
};

struct Inflight {
  std::vector<void*> buffers;
  cudaEvent_t in_done = nullptr, comp_done = nullptr, out_done = nullptr;
  Window c_host;  // host window written by this call's copy-out (empty if none)
};

constexpr size_t kDepth = 3;  // calls allowed in flight (bounds staging memory)

}  // namespace

void gemm_async(Scalar alpha, const MatrixView& a, const MatrixView& b, Scalar beta, const MatrixView& c,
                const Config& cfg, void* stream, FlopCounter* fc) {
  if (ranges_overlap(c, a) || ranges_overlap(c, b)) throw Error("gemm: C must not alias A or B");
  const ExecutionPlan p = plan(alpha, a, b, beta, c, cfg);
  execute(p, cfg.numerics, stream, fc);
}

void gemm_batch(const std::vector<GemmCall>& calls, const Config& cfg, FlopCounter* fc) {
  // Every plan first: policy and shape errors surface before any device work.
  std::vector<ExecutionPlan> plans;
  plans.reserve(calls.size());
  for (const GemmCall& g : calls) {
    if (ranges_overlap(g.c, g.a) || ranges_overlap(g.c, g.b)) throw Error("gemm: C must not alias A or B");
    plans.push_back(plan(g.alpha, g.a, g.b, g.beta, g.c, cfg));
  }
  const Streams S = device_streams();
  std::vector<Inflight> fl(calls.size());
  auto event = [] {
    cudaEvent_t e = nullptr;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    return e;
  };
  auto cleanup = [&] {
    cudaStreamSynchronize(S.in);
    cudaStreamSynchronize(S.compute);
    cudaStreamSynchronize(S.out);
    for (Inflight& f : fl) {
      for (void* q : f.buffers) cudaFree(q);  // normally already released stream-ordered
      f.buffers.clear();
      for (cudaEvent_t e : {f.in_done, f.comp_done, f.out_done})
        if (e) cudaEventDestroy(e);
    }
  };
  try {
    for (size_t i = 0; i < calls.size(); ++i) {
      ExecutionPlan p = plans[i];
      Inflight& f = fl[i];
      f.in_done = event();
      f.comp_done = event();
      f.out_done = event();
      if (i >= kDepth) cuda_check(cudaStreamWaitEvent(S.in, fl[i - kDepth].out_done, 0), "throttle");
      const MatrixView* originals[3] = {&calls[i].a, &calls[i].b, &calls[i].c};
      const bool needed = p.m > 0 && p.n > 0;
      const bool need[3] = {needed && p.k > 0, needed && p.k > 0, needed};
      Window win[3];
      std::byte* dev[3] = {nullptr, nullptr, nullptr};
      for (int r = 0; r < 3; ++r) {
        const auto [lo, hi] = byte_range(*originals[r]);
        win[r] = Window{lo, hi};
        if (!need[r] || hi <= lo || is_device_ptr(lo)) continue;
        // read-after-write on host memory written by an earlier copy-out
        for (size_t h = 0; h < i; ++h)
          if (fl[h].c_host.overlaps(win[r])) cuda_check(cudaStreamWaitEvent(S.in, fl[h].out_done, 0), "dependency");
        void* d = nullptr;
        const size_t bytes = static_cast<size_t>(hi - lo);
        cuda_check(cudaMallocAsync(&d, bytes, S.in), "staging allocation");
        f.buffers.push_back(d);
        dev[r] = static_cast<std::byte*>(d);
        cuda_check(cudaMemcpyAsync(d, lo, bytes, cudaMemcpyHostToDevice, S.in), "H2D staging");
      }
      auto rebase = [&](MatrixView& v) {
        for (int r = 0; r < 3; ++r)
          if (dev[r] && v.base >= win[r].lo && v.base < win[r].hi) {
            v.base = dev[r] + (v.base - win[r].lo);
            return;
          }
      };
      rebase(p.a);
      rebase(p.b);
      rebase(p.c);
      cuda_check(cudaEventRecord(f.in_done, S.in), "event");
      cuda_check(cudaStreamWaitEvent(S.compute, f.in_done, 0), "dependency");
      execute(p, cfg.numerics, S.compute, fc);
      cuda_check(cudaEventRecord(f.comp_done, S.compute), "event");
      cuda_check(cudaStreamWaitEvent(S.out, f.comp_done, 0), "dependency");
      if (dev[2]) {
        f.c_host = win[2];
        cuda_check(cudaMemcpyAsync(const_cast<std::byte*>(win[2].lo), dev[2], static_cast<size_t>(win[2].hi - win[2].lo),
                                   cudaMemcpyDeviceToHost, S.out),
                   "D2H staging");
      }
      for (void* q : f.buffers) cuda_check(cudaFreeAsync(q, S.out), "staging release");
      f.buffers.clear();
      cuda_check(cudaEventRecord(f.out_done, S.out), "event");
    }
    cuda_check(cudaStreamSynchronize(S.out), "gemm synchronisation");
    cuda_check(cudaStreamSynchronize(S.compute), "gemm synchronisation");
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}

void gemm(Scalar alpha, const MatrixView& a, const MatrixView& b, Scalar beta, const MatrixView& c,
          const Config& cfg, FlopCounter* fc) {
  gemm_batch({GemmCall{alpha, a, b, beta, c}}, cfg, fc);
}

}  // namespace mdgemm
