// gemm() / gemm_async() / gemm_batch(): the public entry points around
// execute().  Operands may live in host memory (the reference's callers use
// host Matrix objects): each host operand's byte window is copied into HBM,
// the plan's views are rebased into the copy, and C's window is copied back.
//
// gemm_batch() runs a list of gemm calls with the semantics of calling gemm()
// on each in order, but
//   * host staging is pipelined across calls (copy-in / compute / copy-out
//     streams), so one call's PCIe traffic overlaps its neighbours' kernels;
//   * calls that do not touch each other's memory run concurrently on
//     several compute streams, so small problems share the GPU, one call's
//     tail overlaps the next call's head, and FP64 (DMMA) and FP32 (FFMA2)
//     kernels can co-reside on an SM (different pipes).
// Ordering is preserved wherever it matters: a call waits for every earlier
// call whose device write window overlaps its device reads or writes (or vice
// versa), and host inputs that an earlier call's copy-out writes are read
// only after that copy-out.
#include <algorithm>
#include <cstdlib>
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

constexpr int kComputeStreams = 8;  // at most; MDGEMM_STREAMS picks how many a batch uses
constexpr size_t kDepth = 3;  // host-staged calls allowed in flight (bounds staging memory)

// Per-device copy-in / compute / copy-out streams (blocking streams, so they
// stay ordered with the legacy default stream other libraries use).
struct Streams {
  cudaStream_t in = nullptr, out = nullptr;
  cudaStream_t compute[kComputeStreams] = {};
};

Streams device_streams() {
  static std::mutex mu;
  static std::vector<Streams> cache;
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lock(mu);
  if (cache.size() <= static_cast<size_t>(dev)) cache.resize(dev + 1);
  Streams& s = cache[dev];
  if (!s.in) {
    cuda_check(cudaStreamCreate(&s.in), "stream");
    cuda_check(cudaStreamCreate(&s.out), "stream");
    for (cudaStream_t& c : s.compute) cuda_check(cudaStreamCreate(&c), "stream");
  }
  return s;
}

struct Window {
  const std::byte* lo = nullptr;
  const std::byte* hi = nullptr;
  bool empty() const { return hi <= lo; }
  bool overlaps(const Window& o) const { return !empty() && !o.empty() && lo < o.hi && o.lo < hi; }
};

struct Call {
  ExecutionPlan plan;
  Window win[3];       // A, B, C byte windows as the caller gave them
  bool host[3] = {};   // operand lives in host memory (staged)
  bool active = false; // m, n > 0
  // device footprint (unstaged operands only)
  Window dev_read[3];
  Window dev_write;
  Window host_write;   // host window written by the copy-out
  std::vector<void*> buffers;
  cudaEvent_t in_done = nullptr, comp_done = nullptr, out_done = nullptr;
  int stream = 0;
};

cudaEvent_t new_event() {
  cudaEvent_t e = nullptr;
  cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  return e;
}

// Grow the device's stream-ordered pool ONCE, up front, to what the batch
// can hold at a time: one workspace arena per concurrent stream plus the
// host staging windows in flight.  Growing it inside the batch maps memory
// while calls are being enqueued, which stalled whole steps of the cfg2
// sweep by 200-350 ms (measured).
void reserve_for_batch(const std::vector<GemmCall>& calls, size_t arena_bytes, int nstreams) {
  size_t stage = 0;
  for (const GemmCall& g : calls) {
    size_t st = 0;
    for (const MatrixView* v : {&g.a, &g.b, &g.c}) {
      const auto [lo, hi] = byte_range(*v);
      if (hi > lo && !is_device_ptr(lo)) st += static_cast<size_t>(hi - lo);
    }
    stage = std::max(stage, st);
  }
  const size_t want = arena_bytes * static_cast<size_t>(nstreams) + stage * (kDepth + 1);
  int dev = 0;
  if (want == 0 || cudaGetDevice(&dev) != cudaSuccess) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
  uint64_t keep = ~0ULL;  // the pool must keep what is reserved (driver.cpp sets the same)
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  static std::mutex mu;
  static std::vector<size_t> reserved;
  std::lock_guard<std::mutex> lock(mu);
  if (reserved.size() <= static_cast<size_t>(dev)) reserved.resize(dev + 1, 0);
  if (want <= reserved[dev]) return;
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return;
  const size_t bytes = std::min(want, free_b / 2);  // never take more than half of what is free
  void* ptr = nullptr;
  if (bytes > reserved[dev] && cudaMallocAsync(&ptr, bytes, cudaStreamLegacy) == cudaSuccess) {
    cudaFreeAsync(ptr, cudaStreamLegacy);  // the pool keeps it (release threshold: never)
    reserved[dev] = bytes;
  }
  cudaGetLastError();
}

void run_batch(const std::vector<GemmCall>& calls, const Config& cfg, cudaStream_t user, bool sync, FlopCounter* fc) {
  // Every plan first: policy and shape errors surface before any device work.
  std::vector<Call> cs(calls.size());
  for (size_t i = 0; i < calls.size(); ++i) {
    const GemmCall& g = calls[i];
    if (ranges_overlap(g.c, g.a) || ranges_overlap(g.c, g.b)) throw Error("gemm: C must not alias A or B");
    cs[i].plan = plan(g.alpha, g.a, g.b, g.beta, g.c, cfg);
  }
  const Streams S = device_streams();
  static const int nstreams = [] {  // tuning: MDGEMM_STREAMS = 1..8 concurrent compute streams
    const char* f = std::getenv("MDGEMM_STREAMS");
    const int v = f ? std::atoi(f) : 4;  // default four concurrent streams
    return v < 1 ? 1 : (v > kComputeStreams ? kComputeStreams : v);
  }();
  // Workspaces (packed operands, stream-K / split-K partials): one arena per
  // compute stream, reused by that stream's calls in stream order, sized for
  // the largest call, instead of a pool allocation per call.
  const bool shared = cs.size() > 1;
  size_t arena_want = 0;
  for (const Call& c : cs) arena_want = std::max(arena_want, workspace_bytes(c.plan, cfg.numerics, shared));
  reserve_for_batch(calls, arena_want, std::min<int>(nstreams, static_cast<int>(cs.size())));
  void* arena[kComputeStreams] = {};
  size_t arena_size[kComputeStreams] = {};
  // fork from the caller's stream
  cudaEvent_t fork = new_event();
  cuda_check(cudaEventRecord(fork, user), "event");
  cuda_check(cudaStreamWaitEvent(S.in, fork, 0), "fork");
  for (cudaStream_t c : S.compute) cuda_check(cudaStreamWaitEvent(c, fork, 0), "fork");
  cuda_check(cudaStreamWaitEvent(S.out, fork, 0), "fork");

  auto cleanup = [&](bool wait) {
    if (wait) {
      cudaStreamSynchronize(S.in);
      for (cudaStream_t c : S.compute) cudaStreamSynchronize(c);
      cudaStreamSynchronize(S.out);
    }
    for (int s = 0; s < kComputeStreams; ++s)
      if (arena[s]) cudaFree(arena[s]);
    for (Call& c : cs) {
      for (void* q : c.buffers) cudaFree(q);
      c.buffers.clear();
      for (cudaEvent_t e : {c.in_done, c.comp_done, c.out_done})
        if (e) cudaEventDestroy(e);  // destruction is deferred until the event completes
    }
    cudaEventDestroy(fork);
  };
  try {
    size_t staged = 0;  // host-staged calls issued so far (for the in-flight throttle)
    std::vector<size_t> staged_ids;
    int rr = 0;
    double queued[kComputeStreams] = {};  // estimated work placed on each compute stream
    for (size_t i = 0; i < calls.size(); ++i) {
      Call& c = cs[i];
      ExecutionPlan& p = c.plan;
      c.active = p.m > 0 && p.n > 0;
      c.in_done = new_event();
      c.comp_done = new_event();
      c.out_done = new_event();
      const MatrixView* originals[3] = {&calls[i].a, &calls[i].b, &calls[i].c};
      const bool need[3] = {c.active && p.k > 0, c.active && p.k > 0, c.active};
      bool any_host = false;
      for (int r = 0; r < 3; ++r) {
        const auto [lo, hi] = byte_range(*originals[r]);
        c.win[r] = Window{lo, hi};
        if (!need[r] || c.win[r].empty()) continue;
        c.host[r] = !is_device_ptr(lo);
        any_host = any_host || c.host[r];
        if (!c.host[r]) c.dev_read[r] = c.win[r];
      }
      if (need[2] && !c.host[2]) c.dev_write = c.win[2];

      // Device-memory conflicts with earlier calls: for every compute stream
      // the most recent conflicting call (waiting for it covers the earlier
      // ones on that stream).  The call joins the stream of its latest
      // conflict -- a dependency chain stays on one stream -- or, without
      // conflicts, the next stream round-robin.
      auto conflicts = [&](const Call& e) {
        if (e.dev_write.overlaps(c.dev_write)) return true;
        for (int r = 0; r < 3; ++r)
          if (e.dev_write.overlaps(c.dev_read[r]) || c.dev_write.overlaps(e.dev_read[r])) return true;
        return false;
      };
      long latest[kComputeStreams];
      std::fill(latest, latest + kComputeStreams, -1L);
      long newest = -1;
      int unresolved = nstreams;
      for (long h = static_cast<long>(i) - 1; h >= 0 && unresolved > 0; --h) {
        const Call& e = cs[static_cast<size_t>(h)];
        if (latest[e.stream] >= 0 || !conflicts(e)) continue;
        latest[e.stream] = h;
        --unresolved;
        newest = std::max(newest, h);
      }
      if (newest >= 0) {
        c.stream = cs[static_cast<size_t>(newest)].stream;
      } else {  // a new chain: the stream with the least queued work (ties round-robin)
        c.stream = rr;
        for (int q = 1; q < nstreams; ++q) {
          const int s = (rr + q) % nstreams;
          if (queued[s] < queued[c.stream]) c.stream = s;
        }
        rr = (rr + 1) % nstreams;
      }
      // estimated device time of the call: useful flops at its pipe's rate
      // (FP32 FFMA2 about twice the FP64 DMMA rate) plus the operand bytes
      queued[c.stream] += (p.comp_prec == Precision::Single ? 0.5 : 1.0) * static_cast<double>(p.m) *
                              static_cast<double>(p.n) * static_cast<double>(p.k) +
                          1e3 * static_cast<double>(p.m + p.n);
      cudaStream_t cst = S.compute[c.stream];

      // ---- copy-in of host operands
      std::byte* dev[3] = {nullptr, nullptr, nullptr};
      if (any_host) {
        if (staged >= kDepth)
          cuda_check(cudaStreamWaitEvent(S.in, cs[staged_ids[staged - kDepth]].out_done, 0), "throttle");
        staged_ids.push_back(i);
        ++staged;
        for (int r = 0; r < 3; ++r) {
          if (!need[r] || !c.host[r] || c.win[r].empty()) continue;
          for (size_t h = 0; h < i; ++h)  // host read-after-write through an earlier copy-out
            if (cs[h].host_write.overlaps(c.win[r])) cuda_check(cudaStreamWaitEvent(S.in, cs[h].out_done, 0), "dep");
          for (size_t h = 0; h < i; ++h)  // device-resident C of an earlier call copied from the same host bytes
            if (cs[h].dev_write.overlaps(c.win[r])) cuda_check(cudaStreamWaitEvent(S.in, cs[h].comp_done, 0), "dep");
          void* d = nullptr;
          const size_t bytes = static_cast<size_t>(c.win[r].hi - c.win[r].lo);
          cuda_check(cudaMallocAsync(&d, bytes, S.in), "staging allocation");
          c.buffers.push_back(d);
          dev[r] = static_cast<std::byte*>(d);
          cuda_check(cudaMemcpyAsync(d, c.win[r].lo, bytes, cudaMemcpyHostToDevice, S.in), "H2D staging");
        }
        cuda_check(cudaEventRecord(c.in_done, S.in), "event");
        cuda_check(cudaStreamWaitEvent(cst, c.in_done, 0), "dependency");
      }
      auto rebase = [&](MatrixView& v) {
        for (int r = 0; r < 3; ++r)
          if (dev[r] && v.base >= c.win[r].lo && v.base < c.win[r].hi) {
            v.base = dev[r] + (v.base - c.win[r].lo);
            return;
          }
      };
      rebase(p.a);
      rebase(p.b);
      rebase(p.c);

      // ---- device-memory dependencies on earlier calls on other streams
      for (int s = 0; s < kComputeStreams; ++s)
        if (s != c.stream && latest[s] >= 0)
          cuda_check(cudaStreamWaitEvent(cst, cs[static_cast<size_t>(latest[s])].comp_done, 0), "dependency");

      // (the planning-time size saw host operand addresses; a staged call's
      // tensor-map alignment can differ, so re-check and grow in stream order)
      const size_t ws_need = c.active ? workspace_bytes(p, cfg.numerics, shared) : 0;
      if (ws_need > arena_size[c.stream]) {
        if (arena[c.stream]) {
          cuda_check(cudaFreeAsync(arena[c.stream], cst), "workspace release");
          arena[c.stream] = nullptr;
          arena_size[c.stream] = 0;
        }
        const size_t bytes = std::max(ws_need, arena_want);
        cuda_check(cudaMallocAsync(&arena[c.stream], bytes, cst), "workspace allocation");
        arena_size[c.stream] = bytes;
      }
      execute_scheduled(p, cfg.numerics, cst, fc, shared, arena[c.stream], arena_size[c.stream]);
      cuda_check(cudaEventRecord(c.comp_done, cst), "event");

      // ---- copy-out of a host C, release of staging
      if (any_host) {
        cuda_check(cudaStreamWaitEvent(S.out, c.comp_done, 0), "dependency");
        if (dev[2]) {
          c.host_write = c.win[2];
          cuda_check(cudaMemcpyAsync(const_cast<std::byte*>(c.win[2].lo), dev[2],
                                     static_cast<size_t>(c.win[2].hi - c.win[2].lo), cudaMemcpyDeviceToHost, S.out),
                     "D2H staging");
        }
        for (void* q : c.buffers) cuda_check(cudaFreeAsync(q, S.out), "staging release");
        c.buffers.clear();
        cuda_check(cudaEventRecord(c.out_done, S.out), "event");
      } else {
        cuda_check(cudaEventRecord(c.out_done, cst), "event");
      }
    }
    // the arenas go back to the pool after each stream's last call
    for (int s = 0; s < kComputeStreams; ++s)
      if (arena[s]) {
        cuda_check(cudaFreeAsync(arena[s], S.compute[s]), "workspace release");
        arena[s] = nullptr;
      }
    // join back into the caller's stream
    for (const Call& c : cs) cuda_check(cudaStreamWaitEvent(user, c.out_done, 0), "join");
    if (sync) cuda_check(cudaStreamSynchronize(user), "gemm synchronisation");
  } catch (...) {
    cleanup(true);
    throw;
  }
  cleanup(false);
}

}  // namespace

void gemm_async(Scalar alpha, const MatrixView& a, const MatrixView& b, Scalar beta, const MatrixView& c,
                const Config& cfg, void* stream, FlopCounter* fc) {
  if (ranges_overlap(c, a) || ranges_overlap(c, b)) throw Error("gemm: C must not alias A or B");
  const ExecutionPlan p = plan(alpha, a, b, beta, c, cfg);
  execute(p, cfg.numerics, stream, fc);
}

void gemm_batch(const std::vector<GemmCall>& calls, const Config& cfg, FlopCounter* fc) {
  run_batch(calls, cfg, cudaStreamLegacy, true, fc);
}

void gemm_batch_async(const std::vector<GemmCall>& calls, const Config& cfg, void* stream, FlopCounter* fc) {
  run_batch(calls, cfg, stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy, false, fc);
}

void gemm(Scalar alpha, const MatrixView& a, const MatrixView& b, Scalar beta, const MatrixView& c,
          const Config& cfg, FlopCounter* fc) {
  gemm_batch({GemmCall{alpha, a, b, beta, c}}, cfg, fc);
}

}  // namespace mdgemm
