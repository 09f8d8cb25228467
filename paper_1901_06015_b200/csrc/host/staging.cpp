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
#include <cstdio>
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
namespace {
std::mutex g_reserve_mu;
std::vector<size_t> g_reserved;  // bytes the library's pool holds per device
}  // namespace

void reset_reservation_impl() {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lock(g_reserve_mu);
  if (g_reserved.size() > static_cast<size_t>(dev)) g_reserved[dev] = 0;
}

size_t reserve_for_batch(size_t host_bytes, size_t arena_bytes, int nstreams) {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lock(g_reserve_mu);
  std::vector<size_t>& reserved = g_reserved;
  if (reserved.size() <= static_cast<size_t>(dev)) reserved.resize(dev + 1, 0);
  // Device operands only and the pool already holds the arenas: nothing to
  // decide (and no cudaMemGetInfo, which stalled lone-call enqueues)
  if (host_bytes == 0 && arena_bytes * static_cast<size_t>(nstreams) <= reserved[dev]) return 0;
  size_t free_b = 0, total_b = 0;
  cuda_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
  // residents may use what the pool already holds plus half of what is free
  const size_t arenas = arena_bytes * static_cast<size_t>(nstreams);
  const size_t room = reserved[dev] + free_b / 2;
  size_t budget = room > arenas ? room - arenas : 0;
  if (const char* f = std::getenv("MDGEMM_RESIDENT_MB"))  // tests: force evictions
    budget = std::min(budget, static_cast<size_t>(std::atof(f) * (1 << 20)));
  const size_t want = arenas + std::min(host_bytes, budget);
  if (want == 0 || want <= reserved[dev]) return budget;
  void* ptr = nullptr;  // the library's pool keeps what is reserved (driver.cpp: workspace_pool)
  if (ws_alloc(&ptr, want, cudaStreamLegacy) == cudaSuccess) {
    cudaFreeAsync(ptr, cudaStreamLegacy);  // the pool keeps it (release threshold: never)
    reserved[dev] = want;
  }
  cudaGetLastError();
  return budget;
}

// ------------------------------------------------------------- dual-pipe mode
// A batch whose calls include both computation precisions runs on the
// dual-pipe kernel (gemm_dual.cu): calls are list-scheduled into launches,
// each pairing FP64 (DMMA) jobs with FP32 (FFMA2) jobs whose estimated
// durations match, so both pipes of every SM work at once.  A launch holds
// only calls whose dependencies (device-memory conflicts, as in the stream
// scheduler) completed in earlier launches; launches run in order on one
// stream, their packs on other streams into rotating arenas (dual_arenas,
// three by default: the packs run up to two launches ahead, on the SMs each
// launch leaves free -- driver.cpp: dual_grid).  Calls the
// kernel does not take (EXACT numerics, k = 0, ...) run in the same order
// through execute().  Host operands are staged once up front (only when no
// two host windows of the batch partially overlap and they fit the resident
// budget; otherwise the batch takes the stream scheduler below).
namespace {

// device rates of the two groups while both run, measured per launch on the
// cfg2 sweep (MDGEMM_DUAL_LOG: group end times): 27.3 + 30.7 TFLOP/s
// (tools/dual_probe's register-light loops: 28.7 + 34.9)
constexpr double kDualRateD = 27.3e12, kDualRateF = 30.7e12;

// A call's tile range [t0, t1) inside one launch: a long call may be split
// over consecutive launches (its tiles are independent; each launch packs its
// operands again) so that every launch pairs equal FP64 and FP32 work.
struct Piece {
  size_t call;
  int32_t t0, t1;
};
struct Unit {
  std::vector<Piece> d, f;  // dual jobs
  long classic = -1;        // or one call through execute()
  size_t bytes = 0;         // packed operand bytes of the dual jobs
};

constexpr int kMaxDualArenas = 4;
int dual_arenas() {  // MDGEMM_DUAL_ARENAS: packed-operand arenas of a dual batch (2..4)
  static const int n = [] {
    const char* f = std::getenv("MDGEMM_DUAL_ARENAS");
    const int v = f ? std::atoi(f) : 3;
    return std::min(kMaxDualArenas, std::max(2, v));
  }();
  return n;
}

int dual_mode() {
  const char* f = std::getenv("MDGEMM_DUAL");  // 0 off, 1 auto, 2 force (even one-precision batches)
  return f ? std::atoi(f) : 1;
}

// Everything the host decides about a dual-pipe batch before any device work.
struct DualPlan {
  std::vector<int> kind;          // per call: 0 through execute(), 1 FP64 (D) job, 2 FP32 (F) job
  std::vector<DualPrep> prep;     // pack geometry of the dual jobs
  std::vector<double> est;        // estimated device time of a whole call at the co-run rate
  std::vector<long> ab_writer;    // latest call writing what this call's A/B read (its packs wait for it)
  std::vector<Unit> units;        // the launches, in order
  std::vector<long> unit_of;      // last launch holding a piece of the call
  std::vector<long> first_unit;   // first one
  std::vector<Window> all;        // distinct host windows (each becomes one resident copy)
  size_t host_bytes = 0;
  size_t arena_bytes = 0;         // largest launch's packed operands
  // estimated times (co-run rates): the longest dependency path through each call, the longest
  // of all, and the larger of the two groups' total work (the span of a perfectly paired batch)
  std::vector<double> through;
  double critical = 0.0, span = 0.0;
};

}  // namespace

// Dependency DAG (device-memory conflicts) + list schedule into launches.
// Host only; false when the batch is not for the dual kernel.
bool dual_schedule(std::vector<Call>& cs, const Config& cfg, DualPlan& P) {
  const int mode = dual_mode();
  const size_t n = cs.size();
  if (mode == 0 || n < 2 || cfg.numerics != Numerics::Fast) return false;
  P.kind.assign(n, 0);
  std::vector<int>& kind = P.kind;
  size_t nd = 0, nf = 0;
  for (size_t i = 0; i < n; ++i)
    if (dual_eligible(cs[i].plan, cfg.numerics)) {
      kind[i] = cs[i].plan.comp_prec == Precision::Single ? 2 : 1;
      (kind[i] == 1 ? nd : nf) += 1;
    }
  if (mode == 1 && (nd == 0 || nf == 0)) return false;
  if (nd + nf == 0) return false;

  // ---- host windows: per-call hulls; any two overlapping hulls must be identical
  std::vector<std::vector<Window>> hulls(n);
  std::vector<Window>& all = P.all;
  for (size_t i = 0; i < n; ++i) {
    std::vector<Window>& hs = hulls[i];
    for (int r = 0; r < 3; ++r)
      if (cs[i].host[r]) hs.push_back(cs[i].win[r]);
    for (bool changed = true; changed;) {
      changed = false;
      for (size_t x = 0; x < hs.size() && !changed; ++x)
        for (size_t y = x + 1; y < hs.size() && !changed; ++y)
          if (hs[x].overlaps(hs[y])) {
            hs[x] = Window{std::min(hs[x].lo, hs[y].lo), std::max(hs[x].hi, hs[y].hi)};
            hs.erase(hs.begin() + static_cast<long>(y));
            changed = true;
          }
    }
    all.insert(all.end(), hs.begin(), hs.end());
  }
  std::sort(all.begin(), all.end(), [](const Window& a, const Window& b) {
    return a.lo != b.lo ? a.lo < b.lo : a.hi < b.hi;
  });
  all.erase(std::unique(all.begin(), all.end(), [](const Window& a, const Window& b) { return a.lo == b.lo && a.hi == b.hi; }),
            all.end());
  size_t& host_bytes = P.host_bytes;
  for (size_t x = 0; x < all.size(); ++x) {
    host_bytes += all[x].bytes();
    if (x + 1 < all.size() && all[x].overlaps(all[x + 1])) return false;
  }

  // ---- device windows (host operands at their future resident copies) and dependencies
  // Residents are laid out later; for conflict analysis a host window stands for itself
  // (host and device address ranges never mix within one window).
  for (size_t i = 0; i < n; ++i) {
    Call& c = cs[i];
    for (int r = 0; r < 3; ++r) {
      if (c.win[r].empty()) continue;
      if (r < 2) c.dev_read[r] = c.win[r];
      else c.dev_write = c.win[r];
    }
  }
  struct WinState {
    Window w;
    long writer = -1;
    std::vector<long> readers;
  };
  std::vector<WinState> ws;
  std::vector<std::vector<long>> succ(n);
  std::vector<int> npred(n, 0);
  P.ab_writer.assign(n, -1);
  std::vector<long>& ab_writer = P.ab_writer;
  for (size_t i = 0; i < n; ++i) {
    const Call& c = cs[i];
    std::vector<long> preds;
    for (const WinState& w : ws) {
      for (int r = 0; r < 2; ++r)
        if (w.writer >= 0 && w.w.overlaps(c.dev_read[r])) {
          preds.push_back(w.writer);
          ab_writer[i] = std::max(ab_writer[i], w.writer);
        }
      if (w.w.overlaps(c.dev_write)) {
        if (w.writer >= 0) preds.push_back(w.writer);
        preds.insert(preds.end(), w.readers.begin(), w.readers.end());
      }
    }
    std::sort(preds.begin(), preds.end());
    preds.erase(std::unique(preds.begin(), preds.end()), preds.end());
    for (long h : preds) succ[static_cast<size_t>(h)].push_back(static_cast<long>(i));
    npred[i] = static_cast<int>(preds.size());
    auto find = [&](const Window& x) -> WinState& {
      for (WinState& w : ws)
        if (w.w.lo == x.lo && w.w.hi == x.hi) return w;
      ws.push_back(WinState{x, -1, {}});
      return ws.back();
    };
    for (int r = 0; r < 2; ++r)
      if (!c.dev_read[r].empty()) find(c.dev_read[r]).readers.push_back(static_cast<long>(i));
    if (!c.dev_write.empty()) {
      for (WinState& w : ws)
        if (w.w.overlaps(c.dev_write)) {
          w.writer = static_cast<long>(i);
          w.readers.clear();
        }
      WinState& mine = find(c.dev_write);
      mine.writer = static_cast<long>(i);
      mine.readers.clear();
    }
  }

  // ---- list schedule
  double rate_d = kDualRateD, rate_f = kDualRateF;
  if (const char* f = std::getenv("MDGEMM_DUAL_RATES")) {  // tuning: "D,F" in TFLOP/s
    double a = 0, b = 0;
    if (std::sscanf(f, "%lf,%lf", &a, &b) == 2 && a > 0 && b > 0) {
      rate_d = a * 1e12;
      rate_f = b * 1e12;
    }
  }
  P.prep.assign(n, DualPrep{});
  P.est.assign(n, 0.0);
  std::vector<DualPrep>& prep = P.prep;
  std::vector<double>& est = P.est;
  size_t max_call_bytes = 0;
  for (size_t i = 0; i < n; ++i)
    if (kind[i]) {
      prep[i] = dual_prepare(cs[i].plan);
      est[i] = prep[i].tile_flops / (kind[i] == 1 ? rate_d : rate_f);
      max_call_bytes = std::max(max_call_bytes, prep[i].bytes);
    }
  const size_t unit_cap = std::max(max_call_bytes, size_t{6} << 30);  // packed bytes per launch
  // priority: the longest remaining dependency path (critical path first), so
  // long chains advance early and the last launches still pair both pipes
  std::vector<double> tail(n, 0.0);
  for (size_t i = n; i-- > 0;) {
    double t = 0.0;
    for (long s2 : succ[i]) t = std::max(t, tail[static_cast<size_t>(s2)]);
    tail[i] = t + (kind[i] ? est[i] : 1e-5);
  }
  auto by_priority = [&](size_t x, size_t y) { return tail[x] != tail[y] ? tail[x] > tail[y] : x < y; };
  {
    std::vector<double> head(n, 0.0);  // longest path that ends where call i starts
    double sum_d = 0, sum_f = 0;
    for (size_t i = 0; i < n; ++i) {
      const double e = kind[i] ? est[i] : 1e-5;
      for (long s2 : succ[i]) head[static_cast<size_t>(s2)] = std::max(head[static_cast<size_t>(s2)], head[i] + e);
      (kind[i] == 1 ? sum_d : sum_f) += kind[i] ? est[i] : 0.0;
    }
    P.through.resize(n);
    for (size_t i = 0; i < n; ++i) {
      P.through[i] = head[i] + tail[i];
      P.critical = std::max(P.critical, P.through[i]);
    }
    P.span = std::max(sum_d, sum_f);
  }
  std::vector<Unit>& units = P.units;
  P.unit_of.assign(n, -1);
  P.first_unit.assign(n, -1);
  std::vector<long>& unit_of = P.unit_of;
  std::vector<long>& first_unit = P.first_unit;
  std::vector<int32_t> next_tile(n, 0);
  auto rem_est = [&](size_t i) {
    return est[i] * static_cast<double>(prep[i].tiles - next_tile[i]) / static_cast<double>(prep[i].tiles);
  };
  std::vector<size_t> ready;
  for (size_t i = 0; i < n; ++i)
    if (npred[i] == 0) ready.push_back(i);
  std::sort(ready.begin(), ready.end(), by_priority);
  size_t done = 0;
  size_t left_d = 0, left_f = 0;  // dual calls not finished yet, per kind
  for (size_t i = 0; i < n; ++i) (kind[i] == 1 ? left_d : left_f) += kind[i] != 0;
  while (done < n) {
    Unit u;
    auto it = std::find_if(ready.begin(), ready.end(), [&](size_t i) { return kind[i] == 0; });
    if (it != ready.end()) {
      u.classic = static_cast<long>(*it);
    } else {
      double td = 0, tf = 0;
      for (size_t i : ready) (kind[i] == 1 ? td : tf) += rem_est(i);
      // Only one kind ready while the other kind still has work to come (all
      // chains at the same phase, e.g. the first launch): take about half of
      // the ready work, in whole calls, so the next launch pairs the rest with
      // the successors of this half.  Otherwise pair min(td, tf) of each.
      const bool one_sided = (td > 0) != (tf > 0);
      const bool other_left = td > 0 ? left_f > 0 : left_d > 0;
      const bool halve = one_sided && other_left;
      static const double part = [] {  // tuning: MDGEMM_DUAL_ONESIDED = share of one-sided ready work taken
        const char* f = std::getenv("MDGEMM_DUAL_ONESIDED");
        const double v = f ? std::atof(f) : 0.5;
        return v > 0.0 && v <= 1.0 ? v : 0.5;
      }();
      const double target_d = (td > 0 && tf > 0) ? std::min(td, tf) : (halve ? td * part : td);
      const double target_f = (td > 0 && tf > 0) ? std::min(td, tf) : (halve ? tf * part : tf);
      // in priority order, whole remaining ranges that keep each side within
      // 5 % of its target; then a side that fell short takes part of its next
      // call's tiles
      double ad = 0, af = 0;
      auto room = [&](size_t i) {
        const std::vector<Piece>& lst = kind[i] == 1 ? u.d : u.f;
        if (lst.size() >= static_cast<size_t>(mdg::DUAL_MAX_JOBS)) return false;
        return (u.d.empty() && u.f.empty()) || u.bytes + prep[i].bytes <= unit_cap;
      };
      auto take = [&](size_t i, int32_t nt) {
        const bool isd = kind[i] == 1;
        (isd ? u.d : u.f).push_back(Piece{i, next_tile[i], next_tile[i] + nt});
        (isd ? ad : af) += est[i] * nt / prep[i].tiles;
        u.bytes += prep[i].bytes;
      };
      std::vector<char> used(ready.size(), 0);
      for (size_t x = 0; x < ready.size(); ++x) {
        const size_t i = ready[x];
        const bool isd = kind[i] == 1;
        const double acc = isd ? ad : af, target = isd ? target_d : target_f;
        if (room(i) && acc + rem_est(i) <= target * 1.05) {
          take(i, prep[i].tiles - next_tile[i]);
          used[x] = 1;
        }
      }
      for (size_t x = 0; x < ready.size(); ++x) {
        const size_t i = ready[x];
        const bool isd = kind[i] == 1;
        const double acc = isd ? ad : af, target = isd ? target_d : target_f;
        if (used[x] || !room(i) || (acc >= target * 0.95 && !(isd ? u.d : u.f).empty())) continue;
        const int32_t left = prep[i].tiles - next_tile[i];
        const double per_tile = est[i] / prep[i].tiles;
        const int32_t want = static_cast<int32_t>(std::ceil((target - acc) / per_tile));
        // (halving keeps whole calls: their successors are what the next launch pairs with)
        take(i, halve ? left : std::max<int32_t>(1, std::min(left, want)));
        used[x] = 1;
      }
    }
    const long uid = static_cast<long>(units.size());
    std::vector<size_t> finished;
    for (std::vector<Piece>* lst : {&u.d, &u.f})
      for (const Piece& pc : *lst) {
        if (first_unit[pc.call] < 0) first_unit[pc.call] = uid;
        unit_of[pc.call] = uid;
        next_tile[pc.call] = pc.t1;
        if (pc.t1 == prep[pc.call].tiles) finished.push_back(pc.call);
      }
    if (u.classic >= 0) {
      unit_of[static_cast<size_t>(u.classic)] = uid;
      first_unit[static_cast<size_t>(u.classic)] = uid;
      finished.push_back(static_cast<size_t>(u.classic));
    }
    for (size_t i : finished) {
      ready.erase(std::find(ready.begin(), ready.end(), i));
      if (kind[i] == 1) --left_d;
      if (kind[i] == 2) --left_f;
    }
    done += finished.size();
    std::vector<size_t> newly;
    for (size_t i : finished)
      for (long s : succ[i])
        if (--npred[static_cast<size_t>(s)] == 0) newly.push_back(static_cast<size_t>(s));
    ready.insert(ready.end(), newly.begin(), newly.end());
    std::sort(ready.begin(), ready.end(), by_priority);
    // longest k first: the virtual tile order front-loads the longest tiles
    auto by_k = [&](const Piece& x, const Piece& y) { return prep[x.call].lpad > prep[y.call].lpad; };
    std::stable_sort(u.d.begin(), u.d.end(), by_k);
    std::stable_sort(u.f.begin(), u.f.end(), by_k);
    units.push_back(std::move(u));
  }
  size_t& arena_bytes = P.arena_bytes;
  for (const Unit& u : units) arena_bytes = std::max(arena_bytes, u.bytes);
  if (const char* logp = std::getenv("MDGEMM_DUAL_LOG")) {  // tuning: the launch schedule
    if (FILE* f = std::fopen(logp, "a")) {
      std::fprintf(f, "batch %zu calls -> %zu launches\n", n, units.size());
      for (const Unit& u : units) {
        double td = 0, tf = 0;
        for (const Piece& pc : u.d) td += est[pc.call] * (pc.t1 - pc.t0) / prep[pc.call].tiles;
        for (const Piece& pc : u.f) tf += est[pc.call] * (pc.t1 - pc.t0) / prep[pc.call].tiles;
        std::fprintf(f, "  D %2zu jobs %8.3f ms | F %2zu jobs %8.3f ms | classic %ld | %.2f GB\n", u.d.size(), td * 1e3,
                     u.f.size(), tf * 1e3, u.classic, u.bytes / 1e9);
      }
      std::fclose(f);
    }
  }
  return true;
}

// Issue a scheduled dual batch: host copies, packs, launches, write-backs.
void dual_emit(std::vector<Call>& cs, const Config& cfg, const Streams& S, const DualPlan& plan, cudaStream_t user,
               bool sync, FlopCounter* fc) {
  const size_t n = cs.size();
  const std::vector<DualPrep>& prep = plan.prep;
  const std::vector<double>& est = plan.est;
  const std::vector<long>& ab_writer = plan.ab_writer;
  const std::vector<Unit>& units = plan.units;
  const std::vector<long>& unit_of = plan.unit_of;
  const std::vector<long>& first_unit = plan.first_unit;
  const std::vector<Window>& all = plan.all;
  const size_t arena_bytes = plan.arena_bytes;

  // ---- emission
  // K: the dual launches (and classic units) in order; P: packs, fanned out to
  // PX so the many small pack kernels of a launch overlap each other
  cudaStream_t K = S.compute[0], P = S.compute[1];
  const cudaStream_t PX[2] = {S.compute[2], S.compute[3]};
  std::vector<cudaEvent_t> events;
  auto ev = [&]() {
    events.push_back(new_event());
    return events.back();
  };
  std::vector<std::pair<Window, std::byte*>> residents;  // host window -> device copy
  // Packed-operand arenas, used round robin by the launches: the packs of
  // launch u go into arena u % n once launch u - n is done with it, so they may
  // run that many launches ahead (on the SMs a dual launch leaves free).
  void* arena[kMaxDualArenas] = {};
  const int narenas = dual_arenas();
  int* counters = nullptr;
  bool failed = true;
  auto cleanup = [&](bool wait) {
    if (wait) {
      cudaStreamSynchronize(S.in);
      cudaStreamSynchronize(K);
      cudaStreamSynchronize(P);
      for (cudaStream_t q : PX) cudaStreamSynchronize(q);
      cudaStreamSynchronize(S.out);
      for (auto& r : residents) cudaFree(r.second);
      for (void* a : arena)
        if (a) cudaFree(a);
      if (counters) cudaFree(counters);
    }
    for (cudaEvent_t e : events) cudaEventDestroy(e);
    for (Call& c : cs)
      if (c.comp_done) cudaEventDestroy(c.comp_done);
  };
  try {
    cudaEvent_t fork = ev();
    cuda_check(cudaEventRecord(fork, user), "event");
    for (cudaStream_t st : {S.in, K, P, PX[0], PX[1], S.out}) cuda_check(cudaStreamWaitEvent(st, fork, 0), "fork");
    // host operands: one resident copy per distinct window, copied in the
    // order the schedule first needs them; every launch waits only for the
    // copies of its own operands, and a host C goes back right after the last
    // launch writing it
    std::vector<long> first_use(all.size(), -1), last_write(all.size(), -1);
    std::vector<std::vector<size_t>> call_res(n);
    for (size_t i = 0; i < n; ++i)
      for (int r = 0; r < 3; ++r) {
        if (!cs[i].host[r]) continue;
        for (size_t x = 0; x < all.size(); ++x)
          if (all[x].contains(cs[i].win[r])) {
            call_res[i].push_back(x);
            const long u = unit_of[i];
            if (first_use[x] < 0 || first_unit[i] < first_use[x]) first_use[x] = first_unit[i];
            if (r == 2) last_write[x] = std::max(last_write[x], u);
          }
      }
    std::vector<size_t> order(all.size());
    for (size_t x = 0; x < all.size(); ++x) order[x] = x;
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return first_use[a] < first_use[b]; });
    std::vector<cudaEvent_t> staged(all.size(), nullptr);
    std::vector<char> pageable_out(all.size(), 0);
    for (size_t x = 0; x < all.size(); ++x) pageable_out[x] = last_write[x] >= 0 && host_pageable(all[x].lo);
    residents.resize(all.size());
    for (size_t x : order) {
      void* d = nullptr;
      cuda_check(ws_alloc(&d, all[x].bytes(), S.in), "staging allocation");
      residents[x] = {all[x], static_cast<std::byte*>(d)};
      h2d_copy(d, all[x].lo, all[x].bytes(), S.in);
      g_h2d_bytes.fetch_add(all[x].bytes(), std::memory_order_relaxed);
      staged[x] = ev();
      cuda_check(cudaEventRecord(staged[x], S.in), "event");
    }
    auto rebase = [&](size_t i) {
      Call& c = cs[i];
      ExecutionPlan& p = c.plan;
      for (int r = 0; r < 3; ++r) {
        if (!c.host[r]) continue;
        std::byte* base = nullptr;
        for (auto& rs : residents)
          if (rs.first.contains(c.win[r])) base = rs.second + (c.win[r].lo - rs.first.lo);
        for (MatrixView* v : {&p.a, &p.b, &p.c})
          if (v->base >= c.win[r].lo && v->base < c.win[r].hi) v->base = base + (v->base - c.win[r].lo);
      }
    };
    // the streams wait for the copies a unit's calls read (once per resident and stream)
    std::vector<char> waited_k(all.size(), 0), waited_p(all.size(), 0);
    auto wait_inputs = [&](const std::vector<size_t>& members, bool on_p) {
      for (size_t i : members)
        for (size_t x : call_res[i]) {
          std::vector<char>& w = on_p ? waited_p : waited_k;
          if (w[x]) continue;
          w[x] = 1;
          cuda_check(cudaStreamWaitEvent(on_p ? P : K, staged[x], 0), "dependency");
        }
    };
    for (size_t i = 0; i < n; ++i) rebase(i);
    if (arena_bytes > 0)
      for (int a = 0; a < narenas; ++a) cuda_check(ws_alloc(&arena[a], arena_bytes, P), "workspace allocation");
    // per-launch tile counters of the dynamic tile order (MDGEMM_DUAL_DYNAMIC=1; the
    // default static boustrophedon order measured 0.7 % faster on the cfg2 sweep: the
    // atomic fetch at every tile start delays the producer's first copies)
    const bool dynamic = [] {
      const char* f = std::getenv("MDGEMM_DUAL_DYNAMIC");
      return f ? std::atoi(f) != 0 : false;
    }();
    if (dynamic && !units.empty()) {
      cuda_check(ws_alloc(reinterpret_cast<void**>(&counters), units.size() * 2 * sizeof(int), K), "tile counters");
      cuda_check(cudaMemsetAsync(counters, 0, units.size() * 2 * sizeof(int), K), "tile counters");
    }
    std::vector<cudaEvent_t> k_done(units.size(), nullptr);
    std::vector<mdg::PackGroup> pack_groups(2);  // (26 KB each: kernel parameters of the group launches)
    const char* log_path = std::getenv("MDGEMM_DUAL_LOG");
    const bool log_units = log_path != nullptr;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> unit_ev(units.size(), {nullptr, nullptr});
    unsigned long long* timing_buf = nullptr;
    for (auto& pr : unit_ev) {
      pr.first = nullptr;
      pr.second = nullptr;
    }
    for (size_t ui = 0; ui < units.size(); ++ui) {
      const Unit& u = units[ui];
      std::vector<size_t> members;
      for (const std::vector<Piece>* lst : {&u.d, &u.f})
        for (const Piece& pc : *lst) members.push_back(pc.call);
      if (u.classic >= 0) members.push_back(static_cast<size_t>(u.classic));
      wait_inputs(members, false);
      if (u.classic < 0) wait_inputs(members, true);
      if (u.classic >= 0) {
        Call& c = cs[static_cast<size_t>(u.classic)];
        execute_scheduled(c.plan, cfg.numerics, K, fc, true, nullptr, 0, nullptr, cfg.splitk);
      } else {
        // packs: after the kernel that last used this arena and after writers of the A/B read
        if (ui >= static_cast<size_t>(narenas) && k_done[ui - narenas])
          cuda_check(cudaStreamWaitEvent(P, k_done[ui - narenas], 0), "arena reuse");
        long abw = -1;
        for (size_t i : members)
          if (ab_writer[i] >= 0) abw = std::max(abw, unit_of[static_cast<size_t>(ab_writer[i])]);
        if (abw >= 0 && k_done[static_cast<size_t>(abw)])
          cuda_check(cudaStreamWaitEvent(P, k_done[static_cast<size_t>(abw)], 0), "dependency");
        // fan out: the FP32 jobs' packs on PX[0] (P's dependencies), P joins it;
        // all packs of a group are one launch (pack_group_kernel)
        cudaEvent_t pgo = ev();
        cuda_check(cudaEventRecord(pgo, P), "event");
        cuda_check(cudaStreamWaitEvent(PX[0], pgo, 0), "fork");
        mdg::DualDesc dd{};
        double flops_d = 0, flops_f = 0;
        char* w = static_cast<char*>(arena[ui % narenas]);
        size_t off = 0;
        for (int grp = 0; grp < 2; ++grp) {
          const std::vector<Piece>& lst = grp == 0 ? u.d : u.f;
          mdg::DualJob* jobs = grp == 0 ? dd.d : dd.f;
          mdg::PackGroup& pg = pack_groups[grp];
          pg.n = 0;
          double traffic = 0;
          int32_t tiles = 0;
          for (size_t x = 0; x < lst.size(); ++x) {
            const size_t i = lst[x].call;
            dual_describe(cs[i].plan, w + off, &jobs[x], &pg, &traffic);
            off += prep[i].bytes;
            jobs[x].tile0 = tiles;
            jobs[x].tile_begin = lst[x].t0;
            tiles += lst[x].t1 - lst[x].t0;
            const ExecutionPlan& p = cs[i].plan;
            (grp == 0 ? flops_d : flops_f) += 2.0 * p.m * p.n * p.k * (lst[x].t1 - lst[x].t0) / prep[i].tiles;
          }
          dual_pack_group(pg, traffic, grp == 0 ? P : PX[0]);
          (grp == 0 ? dd.nd : dd.nf) = static_cast<int32_t>(lst.size());
          (grp == 0 ? dd.tiles_d : dd.tiles_f) = tiles;
        }
        {
          cudaEvent_t j = ev();
          cuda_check(cudaEventRecord(j, PX[0]), "event");
          cuda_check(cudaStreamWaitEvent(P, j, 0), "join");
        }
        cudaEvent_t packed = ev();
        cuda_check(cudaEventRecord(packed, P), "event");
        cuda_check(cudaStreamWaitEvent(K, packed, 0), "dependency");
        if (log_units) {  // (no host synchronisation: the schedule is timed as it runs)
          if (!timing_buf) {
            cuda_check(cudaMalloc(&timing_buf, units.size() * 3 * 8), "timing buffer");
            cuda_check(cudaMemsetAsync(timing_buf, 0, units.size() * 3 * 8, K), "timing buffer");
          }
          dd.timing = timing_buf + 3 * ui;
          cuda_check(cudaEventCreate(&unit_ev[ui].first), "event");
          cuda_check(cudaEventCreate(&unit_ev[ui].second), "event");
          events.push_back(unit_ev[ui].first);
          events.push_back(unit_ev[ui].second);
          cuda_check(cudaEventRecord(unit_ev[ui].first, K), "event");
        }
        dd.counters = counters ? counters + 2 * ui : nullptr;
        dual_launch(dd, flops_d, flops_f, K);
        if (log_units) cuda_check(cudaEventRecord(unit_ev[ui].second, K), "event");
        if (fc)
          for (const std::vector<Piece>* lst : {&u.d, &u.f})
            for (const Piece& pc : *lst)
              if (pc.t1 == prep[pc.call].tiles) fc->add(reference_flops(cs[pc.call].plan));
      }
      k_done[ui] = ev();
      cuda_check(cudaEventRecord(k_done[ui], K), "event");
      // host results this launch wrote for the last time (pageable ones after
      // the last launch: their copy-out holds the host thread)
      bool any = false;
      for (size_t x = 0; x < all.size(); ++x)
        if (last_write[x] == static_cast<long>(ui) && !pageable_out[x]) {
          if (!any) cuda_check(cudaStreamWaitEvent(S.out, k_done[ui], 0), "dependency");
          any = true;
          d2h_copy(const_cast<std::byte*>(all[x].lo), residents[x].second, all[x].bytes(), S.out);
          g_d2h_bytes.fetch_add(all[x].bytes(), std::memory_order_relaxed);
        }
    }
    // results back to the host (every host C, after the last launch), residents released
    cuda_check(cudaStreamWaitEvent(S.out, k_done.empty() ? fork : k_done.back(), 0), "join");
    for (size_t x = 0; x < all.size(); ++x)
      if (last_write[x] >= 0 && pageable_out[x]) {
        d2h_copy(const_cast<std::byte*>(all[x].lo), residents[x].second, all[x].bytes(), S.out);
        g_d2h_bytes.fetch_add(all[x].bytes(), std::memory_order_relaxed);
      }
    for (auto& rs : residents) cuda_check(cudaFreeAsync(rs.second, S.out), "staging release");
    residents.clear();
    for (void*& a : arena)
      if (a) {
        cuda_check(cudaFreeAsync(a, S.out), "workspace release");
        a = nullptr;
      }
    if (counters) {
      cuda_check(cudaFreeAsync(counters, S.out), "tile counters");
      counters = nullptr;
    }
    cudaEvent_t done = ev();
    cuda_check(cudaEventRecord(done, S.out), "event");
    cuda_check(cudaStreamWaitEvent(user, done, 0), "join");
    if (sync) cuda_check(cudaStreamSynchronize(user), "gemm synchronisation");
    if (log_units) {  // measured device time of every launch next to its estimate
      cuda_check(cudaEventSynchronize(done), "event");
      std::vector<unsigned long long> tm(units.size() * 3, 0);
      if (timing_buf) {
        cuda_check(cudaMemcpy(tm.data(), timing_buf, tm.size() * 8, cudaMemcpyDeviceToHost), "timing");
        cudaFree(timing_buf);
      }
      if (FILE* f = std::fopen(log_path, "a")) {
        for (size_t ui = 0; ui < units.size(); ++ui) {
          if (!unit_ev[ui].first) continue;
          float ms = 0;
          cudaEventElapsedTime(&ms, unit_ev[ui].first, unit_ev[ui].second);
          double td = 0, tf = 0, fd = 0, ff = 0;
          for (int grp = 0; grp < 2; ++grp)
            for (const Piece& pc : grp == 0 ? units[ui].d : units[ui].f) {
              const double frac = static_cast<double>(pc.t1 - pc.t0) / prep[pc.call].tiles;
              const ExecutionPlan& q = cs[pc.call].plan;
              (grp == 0 ? td : tf) += est[pc.call] * frac;
              (grp == 0 ? fd : ff) += 2.0 * q.m * q.n * q.k * frac;
            }
          const unsigned long long t0 = ~tm[3 * ui];
          const double dend = tm[3 * ui + 1] > t0 ? (tm[3 * ui + 1] - t0) * 1e-6 : 0.0;
          const double fend = tm[3 * ui + 2] > t0 ? (tm[3 * ui + 2] - t0) * 1e-6 : 0.0;
          float gap = 0;  // idle kernel stream before this launch (its packs, host enqueue)
          if (ui > 0 && unit_ev[ui - 1].second) cudaEventElapsedTime(&gap, unit_ev[ui - 1].second, unit_ev[ui].first);
          std::fprintf(f,
                       "  launch %3zu: D %2zu est %7.3f end %7.3f | F %2zu est %7.3f end %7.3f | measured %7.3f ms | "
                       "%.1f + %.1f TF/s | gap %.3f ms\n",
                       ui, units[ui].d.size(), td * 1e3, dend, units[ui].f.size(), tf * 1e3, fend, ms, fd / ms / 1e9,
                       ff / ms / 1e9, gap);
        }
        std::fclose(f);
      }
    }
    failed = false;
  } catch (...) {
    cleanup(true);
    throw;
  }
  cleanup(failed);
}

// Long dependency chains.  Calls updating one C run one after another, and a
// chain alternating FP64 and FP32 calls keeps one pipe idle whenever nothing
// else is left to pair it with: when the batch's longest dependency path
// exceeds kChainShare of its paired span, the calls on such paths are cut into
// column panels (B and C column slices, the multi-GPU split of multi.cpp) --
// independent sub-chains that the list scheduler pairs with each other.  Every
// C element keeps its k order, so the bits do not change.  Device operands
// with unit-stride C columns only (panels of other layouts share byte windows).
constexpr double kChainShare = 0.25;
constexpr int64_t kMinPanelColumns = 256, kPanelAlign = 128;
constexpr int kMaxPanels = 8;

int chain_split_mode() {  // MDGEMM_CHAIN_SPLIT: 0 off, 1 auto (default), 2..8 force that many panels
  static const int v = [] {
    const char* f = std::getenv("MDGEMM_CHAIN_SPLIT");
    return f ? std::max(0, std::min(kMaxPanels, std::atoi(f))) : 1;
  }();
  return v;
}

MatrixView column_panel(const MatrixView& v, int64_t j0, int64_t nb) {
  MatrixView out = v;
  out.base = v.base + static_cast<size_t>(j0 * v.cs) * dtype_size(v.dtype);
  out.n = nb;
  return out;
}

// The batch with the calls on long paths cut into column panels; empty when
// nothing is to be split.
std::vector<GemmCall> split_long_chains(const std::vector<GemmCall>& calls, const DualPlan& plan) {
  const int mode = chain_split_mode();
  std::vector<GemmCall> out;
  if (mode == 0 || plan.host_bytes != 0 || plan.span <= 0) return out;
  const double limit = kChainShare * plan.span;
  if (mode == 1 && plan.critical <= limit) return out;
  const int panels = mode >= 2 ? mode : static_cast<int>(std::min<double>(kMaxPanels, std::ceil(plan.critical / limit)));
  bool any = false;
  for (size_t i = 0; i < calls.size(); ++i) {
    const GemmCall& g = calls[i];
    const int64_t n = g.c.n;
    const int pc = static_cast<int>(std::min<int64_t>(panels, n / kMinPanelColumns));
    const bool cut = plan.kind[i] != 0 && g.c.rs == 1 && pc >= 2 && g.b.n == n &&
                     (mode >= 2 || plan.through[i] > limit);
    if (!cut) {
      out.push_back(g);
      continue;
    }
    any = true;
    for (int r = 0; r < pc; ++r) {
      int64_t j0 = 0, nb = 0;
      shard_columns(n, pc, r, kPanelAlign, &j0, &nb);
      if (nb == 0) continue;
      out.push_back(GemmCall{g.alpha, g.a, column_panel(g.b, j0, nb), g.beta, column_panel(g.c, j0, nb)});
    }
  }
  if (!any) out.clear();
  return out;
}

// Estimated device time of a scheduled batch: per launch, the paired part of
// its two groups at the co-run rates, what one group has beyond the other at
// that group's rate alone (measured: FP64 31.5, FP32 50 TFLOP/s in the dual
// kernel), and a fixed cost per launch (ramp-up, the last tiles' tail).
double estimated_makespan(const DualPlan& plan) {
  constexpr double kAloneD = 27.3 / 31.5, kAloneF = 30.7 / 50.0, kPerLaunch = 0.3e-3;
  double t = 0;
  for (const Unit& u : plan.units) {
    if (u.classic >= 0) continue;
    double td = 0, tf = 0;
    for (const Piece& pc : u.d) td += plan.est[pc.call] * (pc.t1 - pc.t0) / plan.prep[pc.call].tiles;
    for (const Piece& pc : u.f) tf += plan.est[pc.call] * (pc.t1 - pc.t0) / plan.prep[pc.call].tiles;
    const double paired = std::min(td, tf);
    t += paired + (td - paired) * kAloneD + (tf - paired) * kAloneF + kPerLaunch;
  }
  return t;
}

bool run_batch(const std::vector<GemmCall>& calls, const Config& cfg, cudaStream_t user, bool sync, FlopCounter* fc,
               const double* better_than = nullptr);

// better_than: run only if the schedule's estimate beats this time (the finer batch of a caller
// that has a schedule of its own); otherwise nothing is issued and the result is false.
bool try_run_dual(std::vector<Call>& cs, const Config& cfg, const Streams& S, cudaStream_t user, bool sync,
                  FlopCounter* fc, const std::vector<GemmCall>& calls, const double* better_than) {
  DualPlan plan;
  if (!dual_schedule(cs, cfg, plan)) return false;
  if (better_than) {
    if (estimated_makespan(plan) >= *better_than) return false;
  } else {
    const std::vector<GemmCall> finer = split_long_chains(calls, plan);
    if (!finer.empty()) {
      const double mine = estimated_makespan(plan);
      if (run_batch(finer, cfg, user, sync, fc, &mine)) return true;
    }
  }
  const size_t budget = reserve_for_batch(plan.host_bytes, plan.arena_bytes, dual_arenas());
  if (plan.host_bytes > budget) {  // does not fit: the stream scheduler evicts as it goes
    for (Call& c : cs) c.dev_read[0] = c.dev_read[1] = c.dev_write = Window{};
    return false;
  }
  dual_emit(cs, cfg, S, plan, user, sync, fc);
  return true;
}

bool run_batch(const std::vector<GemmCall>& calls, const Config& cfg, cudaStream_t user, bool sync, FlopCounter* fc,
               const double* better_than) {
  // Every plan first: policy and shape errors surface before any device work.
  std::vector<Call> cs(calls.size());
  try {
    for (size_t i = 0; i < calls.size(); ++i) {
      const GemmCall& g = calls[i];
      if (ranges_overlap(g.c, g.a) || ranges_overlap(g.c, g.b)) throw Error("gemm: C must not alias A or B");
      cs[i].plan = plan(g.alpha, g.a, g.b, g.beta, g.c, cfg);
    }
  } catch (const Error&) {
    if (better_than) return false;  // a panel the planner rejects: the caller keeps its calls whole
    throw;
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
  if (try_run_dual(cs, cfg, S, user, sync, fc, calls, better_than)) return true;
  if (better_than) return false;  // a finer batch that does not beat its caller's schedule
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
  for (const Call& c : cs) arena_want = std::max(arena_want, workspace_bytes(c.plan, cfg.numerics, shared, cfg.splitk));
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
    d2h_copy(const_cast<std::byte*>(r.host.lo), r.dev, r.host.bytes(), S.out);
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
        cuda_check(ws_alloc(&d, h.bytes(), S.in), "staging allocation");
        nr.dev = static_cast<std::byte*>(d);
        h2d_copy(d, h.lo, h.bytes(), S.in);
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
      const size_t ws_need = c.active ? workspace_bytes(p, cfg.numerics, shared, cfg.splitk) : 0;
      if (ws_need > arena_size[c.stream]) {
        if (arena[c.stream]) {
          cuda_check(cudaFreeAsync(arena[c.stream], cst), "workspace release");
          arena[c.stream] = nullptr;
          arena_size[c.stream] = 0;
        }
        const size_t bytes = std::max(ws_need, arena_want);
        cuda_check(ws_alloc(&arena[c.stream], bytes, cst), "workspace allocation");
        arena_size[c.stream] = bytes;
      }
      execute_scheduled(p, cfg.numerics, cst, fc, shared, arena[c.stream], arena_size[c.stream], nullptr, cfg.splitk);
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
  return true;
}

}  // namespace

std::vector<DualPiece> dual_schedule_pieces(const std::vector<GemmCall>& calls, const Config& cfg,
                                            std::vector<int32_t>* call_tiles) {
  std::vector<Call> cs(calls.size());
  for (size_t i = 0; i < calls.size(); ++i) {
    const GemmCall& g = calls[i];
    if (ranges_overlap(g.c, g.a) || ranges_overlap(g.c, g.b)) throw Error("gemm: C must not alias A or B");
    cs[i].plan = plan(g.alpha, g.a, g.b, g.beta, g.c, cfg);
    Call& c = cs[i];
    const ExecutionPlan& p = c.plan;
    c.active = p.m > 0 && p.n > 0;
    const MatrixView* originals[3] = {&g.a, &g.b, &g.c};
    const bool need[3] = {c.active && p.k > 0, c.active && p.k > 0, c.active};
    for (int r = 0; r < 3; ++r) {
      if (!need[r]) continue;
      const auto [lo, hi] = byte_range(*originals[r]);
      c.win[r] = Window{lo, hi};
      c.host[r] = !c.win[r].empty();  // addresses only: no device is touched
    }
  }
  DualPlan dp;
  std::vector<DualPiece> out;
  if (call_tiles) call_tiles->assign(calls.size(), 0);
  if (!dual_schedule(cs, cfg, dp)) return out;
  for (size_t i = 0; i < calls.size(); ++i)
    if (call_tiles && dp.kind[i]) (*call_tiles)[i] = dp.prep[i].tiles;
  for (size_t u = 0; u < dp.units.size(); ++u) {
    const Unit& un = dp.units[u];
    if (un.classic >= 0) out.push_back(DualPiece{static_cast<int32_t>(u), static_cast<int32_t>(un.classic), 0, 0, 0});
    for (int grp = 0; grp < 2; ++grp)
      for (const Piece& pc : grp == 0 ? un.d : un.f)
        out.push_back(DualPiece{static_cast<int32_t>(u), static_cast<int32_t>(pc.call), pc.t0, pc.t1, grp + 1});
  }
  return out;
}

void staging_bytes(uint64_t* h2d, uint64_t* d2h) {
  if (h2d) *h2d = g_h2d_bytes.load(std::memory_order_relaxed);
  if (d2h) *d2h = g_d2h_bytes.load(std::memory_order_relaxed);
}

void gemm_async(Scalar alpha, const MatrixView& a, const MatrixView& b, Scalar beta, const MatrixView& c,
                const Config& cfg, void* stream, FlopCounter* fc) {
  if (ranges_overlap(c, a) || ranges_overlap(c, b)) throw Error("gemm: C must not alias A or B");
  const ExecutionPlan p = plan(alpha, a, b, beta, c, cfg);
  execute(p, cfg.numerics, stream, fc, cfg.splitk);
}

void gemm_batch(const std::vector<GemmCall>& calls, const Config& cfg, FlopCounter* fc) {
  run_batch(calls, cfg, cudaStreamLegacy, true, fc);
}

void gemm_batch_async(const std::vector<GemmCall>& calls, const Config& cfg, void* stream, FlopCounter* fc) {
  run_batch(calls, cfg, stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy, false, fc);
}

void gemm(Scalar alpha, const MatrixView& a, const MatrixView& b, Scalar beta, const MatrixView& c,
          const Config& cfg, FlopCounter* fc) {
  // A lone call on device operands: plan it and run it on the legacy stream,
  // then synchronise -- what the batch runner does for one such call, without
  // its copy streams, fork / join events and stream arenas (the same kernels
  // and workspace sizes, so the same bits).  MDGEMM_LONE_FASTPATH=0: always the
  // batch runner.
  static const bool fast = [] {
    const char* f = std::getenv("MDGEMM_LONE_FASTPATH");
    return !(f && std::atoi(f) == 0);
  }();
  auto on_device = [](const MatrixView& v) { return v.m == 0 || v.n == 0 || is_device_ptr(v.base); };
  if (fast && on_device(c) && on_device(a) && on_device(b)) {
    if (ranges_overlap(c, a) || ranges_overlap(c, b)) throw Error("gemm: C must not alias A or B");
    const ExecutionPlan p = plan(alpha, a, b, beta, c, cfg);
    execute(p, cfg.numerics, cudaStreamLegacy, fc, cfg.splitk);
    cuda_check(cudaStreamSynchronize(cudaStreamLegacy), "gemm synchronisation");
    return;
  }
  gemm_batch({GemmCall{alpha, a, b, beta, c}}, cfg, fc);
}

void reset_reservation() { reset_reservation_impl(); }

}  // namespace mdgemm
