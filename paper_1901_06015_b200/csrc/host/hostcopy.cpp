// Host <-> HBM copies of operands that live in PAGEABLE host memory (a
// std::vector, a reference Matrix: what a drop-in caller of gemm() hands
// over).  DMA can only read pinned memory, so cudaMemcpyAsync on pageable
// memory goes through the driver's small bounce buffers one at a time, with
// the host blocked: a few GB/s.  The library keeps its own ring of pinned
// chunks per process instead:
//
//   H2D  host threads memcpy chunk i of the source into a free ring slot while
//        the copy engine moves chunk i-1 to HBM (cudaMemcpyAsync from pinned
//        memory, stream-ordered on the caller's copy stream);
//   D2H  the copy engine fills slot i while the host threads drain slot i-1
//        into the destination; returns once the bytes are in place (as a
//        pageable cudaMemcpyAsync does).
//
// Pinned (cudaHostAlloc / cudaHostRegister) and device memory keep the plain
// asynchronous copy, and so do windows below one chunk's worth of benefit.
// The memcpy into / out of a slot is split over a small pool of host threads
// (one thread moves ~10 GB/s; PCIe 5 x16 needs several).
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "driver.hpp"

namespace mdgemm {

namespace {

constexpr size_t kChunk = size_t(8) << 20;    // bytes per ring slot
constexpr int kSlots = 4;                      // ring depth
constexpr size_t kDirect = size_t(1) << 20;   // below this the driver's path is as good

// Chunk of a window: a quarter of it (so even a small window pipelines its
// host memcpy against the DMA of the previous chunk), 256 KB .. one slot.
size_t chunk_of(size_t n) {
  const size_t q = ((n / 4) + 65535) & ~size_t(65535);
  return std::min(kChunk, std::max(q, size_t(256) << 10));
}

// A fixed pool of memcpy helpers: run(dst, src, n) splits the range over the
// helpers and the calling thread and returns when all parts are copied.  The
// helpers spin for a while on the job counter before they sleep (a helper
// woken from a futex on a busy host takes longer than a 1 MB memcpy).
class CopyPool {
 public:
  CopyPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    int n = static_cast<int>(std::min(hw / 2, 7u));
    if (const char* f = std::getenv("MDGEMM_COPY_THREADS")) n = std::max(0, std::atoi(f) - 1);
    for (int i = 0; i < n; ++i) workers_.emplace_back([this, i] { loop(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> l(mu_);
      stop_.store(true);
    }
    cv_.notify_all();
    for (std::thread& t : workers_) t.join();
  }
  void run(void* dst, const void* src, size_t n) {
    const int parts = static_cast<int>(workers_.size()) + 1;
    if (parts == 1 || n < (size_t(512) << 10)) {
      std::memcpy(dst, src, n);
      return;
    }
    dst_ = static_cast<char*>(dst);
    src_ = static_cast<const char*>(src);
    n_ = n;
    per_ = ((n + parts - 1) / parts + 63) & ~size_t(63);
    pending_.store(parts - 1, std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> l(mu_);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    part(parts - 1);
    while (pending_.load(std::memory_order_acquire) != 0) std::this_thread::yield();
  }

 private:
  void part(int i) {
    const size_t lo = std::min(n_, static_cast<size_t>(i) * per_), hi = std::min(n_, lo + per_);
    if (hi > lo) std::memcpy(dst_ + lo, src_ + lo, hi - lo);
  }
  void loop(int i) {
    uint64_t seen = 0;
    for (;;) {
      bool got = false;
      for (int spin = 0; spin < 20000 && !got; ++spin) {  // ~ tens of microseconds
        if (stop_.load(std::memory_order_relaxed)) return;
        got = gen_.load(std::memory_order_acquire) != seen;
      }
      if (!got) {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [&] { return stop_.load() || gen_.load() != seen; });
        if (stop_.load()) return;
      }
      seen = gen_.load(std::memory_order_acquire);
      part(i);
      pending_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::atomic<bool> stop_{false};
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> pending_{0};
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t n_ = 0, per_ = 0;
};

struct Ring {
  std::mutex mu;  // one staging copy at a time per process (gemm is reentrant)
  void* slot[kSlots] = {};
  // per device (events belong to one), and the event a slot's last copy recorded
  std::vector<std::vector<cudaEvent_t>> ev;
  cudaEvent_t last[kSlots] = {};
  bool ready = false;
};

Ring& ring() {
  static Ring r;
  return r;
}

CopyPool& pool() {
  static CopyPool p;
  return p;
}

// (lock held) pinned slots, allocated on first use; the current device's events
std::vector<cudaEvent_t>& ensure(Ring& r) {
  if (!r.ready) {
    for (int s = 0; s < kSlots; ++s)
      cuda_check(cudaHostAlloc(&r.slot[s], kChunk, cudaHostAllocPortable), "pinned staging allocation");
    r.ready = true;
  }
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  if (r.ev.size() <= static_cast<size_t>(dev)) r.ev.resize(dev + 1);
  if (r.ev[dev].empty()) {
    r.ev[dev].resize(kSlots);
    for (cudaEvent_t& e : r.ev[dev]) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  }
  return r.ev[dev];
}

// wait until slot k's previous copy is done, then record its next one on st
void claim(Ring& r, int k) {
  if (r.last[k]) cuda_check(cudaEventSynchronize(r.last[k]), "staging slot");
}
void release(Ring& r, std::vector<cudaEvent_t>& ev, int k, cudaStream_t st) {
  cuda_check(cudaEventRecord(ev[k], st), "event");
  r.last[k] = ev[k];
}

}  // namespace

bool host_pageable(const void* p) {
  static const bool ring_on = [] {  // tuning / A-B: MDGEMM_PAGEABLE_RING=0 = the driver's pageable copies
    const char* f = std::getenv("MDGEMM_PAGEABLE_RING");
    return !(f && std::atoi(f) == 0);
  }();
  if (!p || !ring_on) return false;
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return attr.type == cudaMemoryTypeUnregistered;
}

void h2d_copy(void* dst, const void* src, size_t n, cudaStream_t st) {
  if (n < kDirect || !host_pageable(src)) {
    cuda_check(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st), "H2D staging");
    return;
  }
  Ring& r = ring();
  std::lock_guard<std::mutex> lock(r.mu);
  std::vector<cudaEvent_t>& ev = ensure(r);
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  const size_t ch = chunk_of(n);
  for (size_t off = 0, i = 0; off < n; off += ch, ++i) {
    const int k = static_cast<int>(i % kSlots);
    const size_t len = std::min(ch, n - off);
    claim(r, k);  // the slot's previous copy has left it
    pool().run(r.slot[k], s + off, len);
    cuda_check(cudaMemcpyAsync(d + off, r.slot[k], len, cudaMemcpyHostToDevice, st), "H2D staging");
    release(r, ev, k, st);
  }
}

void d2h_copy(void* dst, const void* src, size_t n, cudaStream_t st) {
  if (n < kDirect || !host_pageable(dst)) {
    cuda_check(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st), "D2H staging");
    return;
  }
  Ring& r = ring();
  std::lock_guard<std::mutex> lock(r.mu);
  std::vector<cudaEvent_t>& ev = ensure(r);
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  const size_t ch = chunk_of(n);
  const size_t chunks = (n + ch - 1) / ch;
  auto issue = [&](size_t i) {
    const int k = static_cast<int>(i % kSlots);
    const size_t off = i * ch, len = std::min(ch, n - off);
    claim(r, k);
    cuda_check(cudaMemcpyAsync(r.slot[k], s + off, len, cudaMemcpyDeviceToHost, st), "D2H staging");
    release(r, ev, k, st);
  };
  for (size_t i = 0; i < std::min<size_t>(chunks, kSlots); ++i) issue(i);
  for (size_t i = 0; i < chunks; ++i) {
    const int k = static_cast<int>(i % kSlots);
    const size_t off = i * ch, len = std::min(ch, n - off);
    claim(r, k);  // chunk i has arrived in its slot
    pool().run(d + off, r.slot[k], len);
    if (i + kSlots < chunks) issue(i + kSlots);
  }
}

void trim_host_staging() {
  Ring& r = ring();
  std::lock_guard<std::mutex> lock(r.mu);
  if (!r.ready) return;
  for (int s = 0; s < kSlots; ++s) {
    if (r.last[s]) cudaEventSynchronize(r.last[s]);
    cudaFreeHost(r.slot[s]);
    r.slot[s] = nullptr;
    r.last[s] = nullptr;
  }
  r.ready = false;  // the events stay (they belong to their devices)
}

}  // namespace mdgemm
