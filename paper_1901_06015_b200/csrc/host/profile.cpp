// Launch accounting and optional per-kernel CUDA-event timing.  Events are
// recorded on the launch stream around each kernel and resolved only in
// mdg_profile_end(), so profiling adds no synchronisation to the timed work.
#include "profile.hpp"

#include <atomic>
#include <vector>

namespace mdgemm::prof {

namespace {

std::atomic<uint64_t> g_launches{0};

struct Record {
  int kind;
  cudaEvent_t start, stop;
  double work;
  int kind2;
  double work2;
};

struct ThreadLog {
  bool on = false;
  std::vector<Record> records;
  std::vector<cudaEvent_t> spare;

  cudaEvent_t take() {
    if (!spare.empty()) {
      cudaEvent_t e = spare.back();
      spare.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};

thread_local ThreadLog g_log;

}  // namespace

Scope::Scope(int kind, cudaStream_t stream, double work) : kind_(kind), stream_(stream), work_(work) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (!g_log.on) return;
  start_ = g_log.take();
  cudaEventRecord(start_, stream_);
}

Scope::Scope(int kind, cudaStream_t stream, double work, int kind2, double work2) : Scope(kind, stream, work) {
  kind2_ = kind2;
  work2_ = work2;
}

Scope::~Scope() {
  if (!start_) return;
  cudaEvent_t stop = g_log.take();
  cudaEventRecord(stop, stream_);
  g_log.records.push_back(Record{kind_, start_, stop, work_, kind2_, work2_});
}

uint64_t launches() { return g_launches.load(std::memory_order_relaxed); }

void begin() {
  g_log.on = true;
  g_log.records.clear();
}

void end(mdg_kernel_stats_t* out) {
  for (int k = 0; k < MDG_KERNEL_KINDS; ++k) out[k] = mdg_kernel_stats_t{0, 0.0, 0.0};
  for (Record& r : g_log.records) {
    float ms = 0.0f;
    cudaEventSynchronize(r.stop);
    cudaEventElapsedTime(&ms, r.start, r.stop);
    mdg_kernel_stats_t& s = out[r.kind];
    s.launches += 1;
    s.total_ms += ms;
    s.work += r.work;
    if (r.kind2 >= 0) {
      out[r.kind2].total_ms += ms;
      out[r.kind2].work += r.work2;
    }
    g_log.spare.push_back(r.start);
    g_log.spare.push_back(r.stop);
  }
  g_log.records.clear();
  g_log.on = false;
}

}  // namespace mdgemm::prof
