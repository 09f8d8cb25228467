// gemm() / gemm_async() / gemm_batch(): the public entry points around
// execute().  Operands may live in host memory (the reference's callers use
// host Matrix objects): each host operand's byte window is copied into HBM,
// the plan's views are rebased into the copy, and C's window is copied back.
//
// gemm_batch() runs a list of gemm calls with the semantics of calling gemm()
// on each in order, but
//   * a host byte window is copied into HBM once per batch and stays
//     resident: later calls reading it use the device copy, later calls
//     updating it update the device copy, and it goes back to the host once,
//     after its last writer (residents are evicted least-recently-used when
//     they outgrow half of the free device memory);
//   * host copies run on their own streams, so PCIe traffic overlaps the
//     kernels of neighbouring calls;
//   * calls that do not touch each other's memory run concurrently on
//     several compute streams, so small problems share the GPU, one call's
//     tail overlaps the next call's head, and FP64 (DMMA) and FP32 (FFMA2)
//     kernels can co-reside on an SM (different pipes).
// Ordering is preserved wherever it matters: a call waits for every earlier
// call whose device write window (the caller's device memory or a resident
// copy) overlaps its reads or writes, or vice versa.
#include <algorithm>
#include <atomic>
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
  bool contains(const Window& o) const { return !o.empty() && lo <= o.lo && o.hi <= hi; }
  size_t bytes() const { return empty() ? 0 : static_cast<size_t>(hi - lo); }
};

struct Call {
  ExecutionPlan plan;
  Window win[3];       // A, B, C byte windows as the caller gave them
  bool host[3] = {};   // operand lives in host memory (staged)
  bool active = false; // m, n > 0
  // device footprint: the caller's device memory, or the resident copy of a host operand
  Window dev_read[3];
  Window dev_write;
  cudaEvent_t comp_done = nullptr;
  int stream = 0;
};

// A host byte window kept in HBM for the rest of the batch.  Live residents
// are pairwise disjoint in host space and each holds the CURRENT value of its
// host bytes (the host copy is stale while `dirty`).  A call whose host
// operand lies inside a resident reads / writes the resident directly, so an
// operand that many calls of a batch share crosses PCIe once, and a C that
// later calls update goes back to the host once, after its last writer.
struct Resident {
  Window host;
  std::byte* dev = nullptr;
  bool live = true;
  bool dirty = false;
  long last_writer = -1;
  long last_use[kComputeStreams];  // latest call using it, per compute stream
  uint64_t touched = 0;            // LRU stamp
  cudaEvent_t staged = nullptr;    // H2D complete (recorded on the copy-in stream)
  Resident() { std::fill(last_use, last_use + kComputeStreams, -1L); }
};

std::atomic<uint64_t> g_h2d_bytes{0}, g_d2h_bytes{0};

cudaEvent_t new_event() {
  cudaEvent_t e = nullptr;
  cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  return e;
}

// Distinct host bytes a batch reads or writes (union of its host windows).
size_t unique_host_bytes(std::vector<Window> w) {
  std::sort(w.begin(), w.end(), [](const Window& x, const Window& y) { return x.lo < y.lo; });
  size_t total = 0;
  const std::byte* lo = nullptr;
  const std::byte* hi = nullptr;
  for (const Window& x : w) {
    if (x.empty()) continue;
    if (hi && x.lo <= hi) {
      hi = std::max(hi, x.hi);
      continue;
    }
    if (hi) total += static_cast<size_t>(hi - lo);
    lo = x.lo;
    hi = x.hi;
  }
  if (hi) total += static_cast<size_t>(hi - lo);
  return total;
}

// Grow the device's stream-ordered pool ONCE, up front, to what the batch
// can hold at a time: one workspace arena per concurrent stream plus the
// resident host windows.  Growing it inside the batch maps memory while
// calls are being enqueued, which stalled whole steps of the cfg2 sweep by
// 200-350 ms (measured).  Returns the byte budget for residents.
size_t reserve_for_batch(size_t host_bytes, size_t arena_bytes, int nstreams) {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  size_t free_b = 0, total_b = 0;
  cuda_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
  static std::mutex mu;
  static std::vector<size_t> reserved;
  std::lock_guard<std::mutex> lock(mu);
  if (reserved.size() <= static_cast<size_t>(dev)) reserved.resize(dev + 1, 0);
  // residents may use what the pool already holds plus half of what is free
  const size_t arenas = arena_bytes * static_cast<size_t>(nstreams);
  const size_t room = reserved[dev] + free_b / 2;
  size_t budget = room > arenas ? room - arenas : 0;
  if (const char* f = std::getenv("MDGEMM_RESIDENT_MB"))  // tests: force evictions
    budget = std::min(budget, static_cast<size_t>(std::atof(f) * (1 << 20)));
  const size_t want = arenas + std::min(host_bytes, budget);
  cudaMemPool_t pool;
  if (want == 0 || want <= reserved[dev] || cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return budget;
  uint64_t keep = ~0ULL;  // the pool must keep what is reserved (driver.cpp sets the same)
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  void* ptr = nullptr;
  if (cudaMallocAsync(&ptr, want, cudaStreamLegacy) == cudaSuccess) {
    cudaFreeAsync(ptr, cudaStreamLegacy);  // the pool keeps it (release threshold: never)
    reserved[dev] = want;
  }
  cudaGetLastError();
  return budget;
}

void run_batch(const std::vector<GemmCall>& calls, const Config& cfg, cudaStream_t user, bool sync, FlopCounter* fc) {
  // Every plan first: policy and shape errors surface before any device work.
  std::vector<Call> cs(calls.size());
  for (size_t i = 0; i < calls.size(); ++i) {
    const GemmCall& g = calls[i];
    if (ranges_overlap(g.c, g.a) || ranges_overlap(g.c, g.b)) throw Error("gemm: C must not alias A or B");
    cs[i].plan = plan(g.alpha, g.a, g.b, g.beta, g.c, cfg);
  }
  // operand windows, and which live in host memory
  std::vector<Window> host_windows;
  for (size_t i = 0; i < calls.size(); ++i) {
    Call& c = cs[i];
    const ExecutionPlan& p = c.plan;
    c.active = p.m > 0 && p.n > 0;
    const MatrixView* originals[3] = {&calls[i].a, &calls[i].b, &calls[i].c};
    const bool need[3] = {c.active && p.k > 0, c.active && p.k > 0, c.active};
    for (int r = 0; r < 3; ++r) {
      if (!need[r]) continue;
      const auto [lo, hi] = byte_range(*originals[r]);
      c.win[r] = Window{lo, hi};
      if (c.win[r].empty()) continue;
      c.host[r] = !is_device_ptr(lo);
      if (c.host[r]) host_windows.push_back(c.win[r]);
    }
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
  const size_t budget = reserve_for_batch(unique_host_bytes(host_windows), arena_want,
                                          std::min<int>(nstreams, static_cast<int>(cs.size())));
  void* arena[kComputeStreams] = {};
  size_t arena_size[kComputeStreams] = {};
  std::vector<Resident> res;
  size_t resident_bytes = 0;
  uint64_t clock = 0;
  std::vector<cudaEvent_t> extra_events;  // write-back events, destroyed at the end
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
      for (Resident& r : res)
        if (r.live && r.dev) cudaFree(r.dev);
    }
    for (int s = 0; s < kComputeStreams; ++s)
      if (arena[s]) cudaFree(arena[s]);
    for (Call& c : cs)
      if (c.comp_done) cudaEventDestroy(c.comp_done);  // destruction is deferred until the event completes
    for (Resident& r : res)
      if (r.staged) cudaEventDestroy(r.staged);
    for (cudaEvent_t e : extra_events) cudaEventDestroy(e);
    cudaEventDestroy(fork);
  };
  // Copy a dirty resident back to its host bytes after its last writer; the
  // copy-in stream waits for it (later staging may read those host bytes).
  auto write_back = [&](Resident& r) {
    if (!r.dirty) return;
    cuda_check(cudaStreamWaitEvent(S.out, cs[static_cast<size_t>(r.last_writer)].comp_done, 0), "dependency");
    cuda_check(cudaMemcpyAsync(const_cast<std::byte*>(r.host.lo), r.dev, r.host.bytes(), cudaMemcpyDeviceToHost, S.out),
               "D2H staging");
    g_d2h_bytes.fetch_add(r.host.bytes(), std::memory_order_relaxed);
    r.dirty = false;
  };
  // Drop a resident in the middle of the batch: write it back, then free it on
  // the copy-in stream once every call using it has finished.
  auto retire = [&](Resident& r) {
    if (r.dirty) {
      write_back(r);
      cudaEvent_t wb = new_event();
      extra_events.push_back(wb);
      cuda_check(cudaEventRecord(wb, S.out), "event");
      cuda_check(cudaStreamWaitEvent(S.in, wb, 0), "dependency");
    }
    for (int s = 0; s < kComputeStreams; ++s)
      if (r.last_use[s] >= 0)
        cuda_check(cudaStreamWaitEvent(S.in, cs[static_cast<size_t>(r.last_use[s])].comp_done, 0), "dependency");
    cuda_check(cudaFreeAsync(r.dev, S.in), "staging release");
    resident_bytes -= r.host.bytes();
    r.live = false;
  };
  try {
    int rr = 0;
    double queued[kComputeStreams] = {};  // estimated work placed on each compute stream
    for (size_t i = 0; i < calls.size(); ++i) {
      Call& c = cs[i];
      ExecutionPlan& p = c.plan;
      c.comp_done = new_event();

      // ---- host operands: find or stage their residents.  Operands of this
      // call that overlap each other, and residents that straddle an edge of
      // one, merge into one hull window; afterwards every live resident
      // overlapping a hull either contains it (a hit) or lies inside it.
      std::vector<Window> hulls;
      for (int r = 0; r < 3; ++r)
        if (c.host[r]) hulls.push_back(c.win[r]);
      for (bool changed = true; changed;) {
        changed = false;
        for (size_t x = 0; x < hulls.size() && !changed; ++x) {
          for (size_t y = x + 1; y < hulls.size() && !changed; ++y)
            if (hulls[x].overlaps(hulls[y])) {
              hulls[x] = Window{std::min(hulls[x].lo, hulls[y].lo), std::max(hulls[x].hi, hulls[y].hi)};
              hulls.erase(hulls.begin() + static_cast<long>(y));
              changed = true;
            }
          for (const Resident& e : res)
            if (!changed && e.live && e.host.overlaps(hulls[x]) && !e.host.contains(hulls[x]) &&
                !hulls[x].contains(e.host)) {
              hulls[x] = Window{std::min(hulls[x].lo, e.host.lo), std::max(hulls[x].hi, e.host.hi)};
              changed = true;
            }
        }
      }
      std::vector<size_t> mine;  // residents this call uses
      std::vector<Window> misses;
      for (const Window& h : hulls) {
        size_t hit = res.size();
        for (size_t e = 0; e < res.size() && hit == res.size(); ++e)
          if (res[e].live && res[e].host.contains(h)) hit = e;
        if (hit == res.size()) misses.push_back(h);
        else mine.push_back(hit);
      }
      for (const Window& h : misses) {
        for (Resident& e : res)  // residents inside the new hull go back to the host first
          if (e.live && h.contains(e.host)) retire(e);
        // make room: least recently used residents this call does not use
        while (resident_bytes + h.bytes() > budget) {
          Resident* lru = nullptr;
          for (size_t e = 0; e < res.size(); ++e)
            if (res[e].live && std::find(mine.begin(), mine.end(), e) == mine.end() &&
                (!lru || res[e].touched < lru->touched))
              lru = &res[e];
          if (!lru) break;  // nothing left to evict: go over budget rather than fail
          retire(*lru);
        }
        Resident nr;
        nr.host = h;
        void* d = nullptr;
        cuda_check(cudaMallocAsync(&d, h.bytes(), S.in), "staging allocation");
        nr.dev = static_cast<std::byte*>(d);
        cuda_check(cudaMemcpyAsync(d, h.lo, h.bytes(), cudaMemcpyHostToDevice, S.in), "H2D staging");
        g_h2d_bytes.fetch_add(h.bytes(), std::memory_order_relaxed);
        nr.staged = new_event();
        cuda_check(cudaEventRecord(nr.staged, S.in), "event");
        resident_bytes += h.bytes();
        res.push_back(nr);
        mine.push_back(res.size() - 1);
      }
      for (size_t e : mine) res[e].touched = ++clock;
      // device windows of every operand (resident copies for host operands)
      std::byte* dev_base[3] = {nullptr, nullptr, nullptr};
      const Resident* holder[3] = {nullptr, nullptr, nullptr};
      for (int r = 0; r < 3; ++r) {
        if (c.win[r].empty()) continue;
        Window dw = c.win[r];
        if (c.host[r]) {
          for (size_t e : mine)
            if (res[e].host.contains(c.win[r])) holder[r] = &res[e];
          dev_base[r] = holder[r]->dev + (c.win[r].lo - holder[r]->host.lo);
          dw = Window{dev_base[r], dev_base[r] + c.win[r].bytes()};
        }
        if (r < 2) c.dev_read[r] = dw;
        else c.dev_write = dw;
      }

      // Device-memory conflicts with earlier calls: for every compute stream
      // the most recent conflicting call (waiting for it covers the earlier
      // ones on that stream).  The call joins the stream of its latest
      // conflict -- a dependency chain stays on one stream -- or, without
      // conflicts, the stream with the least queued work.
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

      // ---- the call waits for its residents' copy-in and for conflicting calls on other streams
      for (size_t e : mine) cuda_check(cudaStreamWaitEvent(cst, res[e].staged, 0), "dependency");
      for (int s = 0; s < kComputeStreams; ++s)
        if (s != c.stream && latest[s] >= 0)
          cuda_check(cudaStreamWaitEvent(cst, cs[static_cast<size_t>(latest[s])].comp_done, 0), "dependency");
      auto rebase = [&](MatrixView& v) {
        for (int r = 0; r < 3; ++r)
          if (dev_base[r] && v.base >= c.win[r].lo && v.base < c.win[r].hi) {
            v.base = dev_base[r] + (v.base - c.win[r].lo);
            return;
          }
      };
      rebase(p.a);
      rebase(p.b);
      rebase(p.c);

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
      for (size_t e : mine) res[e].last_use[c.stream] = static_cast<long>(i);
      if (holder[2]) {
        Resident& w = res[static_cast<size_t>(holder[2] - res.data())];
        w.dirty = true;
        w.last_writer = static_cast<long>(i);
      }
    }
    // host results go back once, after their last writer; then the residents
    // are released once every compute stream is done with them
    for (Resident& r : res)
      if (r.live) write_back(r);
    long last_on[kComputeStreams];
    std::fill(last_on, last_on + kComputeStreams, -1L);
    for (size_t i = 0; i < cs.size(); ++i) last_on[cs[i].stream] = static_cast<long>(i);
    for (int s = 0; s < kComputeStreams; ++s)
      if (last_on[s] >= 0) cuda_check(cudaStreamWaitEvent(S.out, cs[static_cast<size_t>(last_on[s])].comp_done, 0), "join");
    for (Resident& r : res)
      if (r.live) {
        cuda_check(cudaFreeAsync(r.dev, S.out), "staging release");
        r.live = false;
      }
    // the arenas go back to the pool after each stream's last call
    for (int s = 0; s < kComputeStreams; ++s)
      if (arena[s]) {
        cuda_check(cudaFreeAsync(arena[s], S.compute[s]), "workspace release");
        arena[s] = nullptr;
      }
    // join back into the caller's stream
    cudaEvent_t done = new_event();
    extra_events.push_back(done);
    cuda_check(cudaEventRecord(done, S.out), "event");
    cuda_check(cudaStreamWaitEvent(user, done, 0), "join");
    if (sync) cuda_check(cudaStreamSynchronize(user), "gemm synchronisation");
  } catch (...) {
    cleanup(true);
    throw;
  }
  cleanup(false);
}

}  // namespace

void staging_bytes(uint64_t* h2d, uint64_t* d2h) {
  if (h2d) *h2d = g_h2d_bytes.load(std::memory_order_relaxed);
  if (d2h) *d2h = g_d2h_bytes.load(std::memory_order_relaxed);
}

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
