// Multi-GPU gemm: C and B split into column panels, A
// broadcast once over NVLink / NVSwitch with NCCL, no reduction.  The
// reference parallelises only over CPU threads (gemm_core.cpp:133-144,
// 170-178); this is the B200 build's scale-out of the same call.
//
// Two entry points:
//  * gemm_sharded (one process per GPU, the torchrun layout): every rank holds
//    its own B and C column panels; the root's A is broadcast on the
//    communicator's stream while the rank packs its B panel, then A is packed
//    and the panel gemm runs.  A column panel of C is an ordinary gemm on
//    slice(B), slice(C) (dtypes.cpp:157-166): same plan, no reduction.
//  * gemm_multi (one process, several GPUs): the whole problem in the
//    caller's memory; panels are scattered to the devices, A is broadcast
//    from the first device, the panels run concurrently, C panels come back.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": the copy the process
// already mapped -- PyTorch's -- or the system one), so single-GPU users never
// need it; a multi-GPU call without it fails with an Error.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "driver.hpp"
#include "mdgemm_b200.h"

namespace mdgemm {

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string missing;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.missing = std::string("NCCL is not available (dlopen libnccl.so.2: ") + dlerror() + ")";
      return a;
    }
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p && a.missing.empty()) a.missing = std::string("NCCL symbol missing: ") + name;
      return p;
    };
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(sym("ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(sym("ncclCommInitRank"));
    a.comm_init_all = reinterpret_cast<decltype(a.comm_init_all)>(sym("ncclCommInitAll"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(sym("ncclCommDestroy"));
    a.broadcast = reinterpret_cast<decltype(a.broadcast)>(sym("ncclBroadcast"));
    a.group_start = reinterpret_cast<decltype(a.group_start)>(sym("ncclGroupStart"));
    a.group_end = reinterpret_cast<decltype(a.group_end)>(sym("ncclGroupEnd"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("ncclGetErrorString"));
    return a;
  }();
  if (!api.missing.empty()) throw Error(api.missing);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(std::string(what) + ": " + nccl().error_string(r));
}

// The byte window a strided view addresses (first to one past the last element).
size_t window_bytes(const MatrixView& v) {
  if (v.m <= 0 || v.n <= 0) return 0;
  return static_cast<size_t>((v.m - 1) * v.rs + (v.n - 1) * v.cs + 1) * dtype_size(v.dtype);
}

}  // namespace

// ------------------------------------------------------------- communicator
struct Communicator::Impl {
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0, device = 0;
  cudaStream_t stream = nullptr;  // broadcasts
  cudaEvent_t ready = nullptr;    // A arrived
  cudaEvent_t start = nullptr;    // the caller's stream reached the call
};

Communicator::Communicator(const CommId& id, int nranks, int rank) : impl_(std::make_unique<Impl>()) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw Error("Communicator: bad rank / size");
  cuda_check(cudaGetDevice(&impl_->device), "cudaGetDevice");
  ncclUniqueId uid;
  static_assert(sizeof(uid) == sizeof(id.bytes), "unique id size");
  std::memcpy(&uid, id.bytes, sizeof(uid));
  nccl_check(nccl().comm_init_rank(&impl_->comm, nranks, uid, rank), "ncclCommInitRank");
  impl_->nranks = nranks;
  impl_->rank = rank;
  cuda_check(cudaStreamCreateWithFlags(&impl_->stream, cudaStreamNonBlocking), "comm stream");
  cuda_check(cudaEventCreateWithFlags(&impl_->ready, cudaEventDisableTiming), "comm event");
  cuda_check(cudaEventCreateWithFlags(&impl_->start, cudaEventDisableTiming), "comm event");
}

Communicator::~Communicator() {
  if (!impl_) return;
  if (impl_->comm) nccl().comm_destroy(impl_->comm);
  if (impl_->stream) cudaStreamDestroy(impl_->stream);
  if (impl_->ready) cudaEventDestroy(impl_->ready);
  if (impl_->start) cudaEventDestroy(impl_->start);
}

CommId Communicator::unique_id() {
  ncclUniqueId uid;
  nccl_check(nccl().get_unique_id(&uid), "ncclGetUniqueId");
  CommId id;
  std::memcpy(id.bytes, &uid, sizeof(uid));
  return id;
}

int Communicator::size() const { return impl_->nranks; }
int Communicator::rank() const { return impl_->rank; }
int Communicator::device() const { return impl_->device; }

// ------------------------------------------------------------ gemm_sharded
void gemm_sharded(Communicator& comm, int root, Scalar alpha, const MatrixView& a, const MatrixView& b_panel,
                  Scalar beta, const MatrixView& c_panel, const Config& cfg, void* stream, FlopCounter* fc) {
  Communicator::Impl& cm = *comm.impl_;
  if (root < 0 || root >= cm.nranks) throw Error("gemm_sharded: bad root rank");
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  if (dev != cm.device) throw Error("gemm_sharded: the current device is not the communicator's");
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
  const bool is_root = cm.rank == root;

  // Every rank passes A's geometry (the root's view; non-root ranks may leave
  // base null and the library receives A into its own buffer).
  MatrixView av = a;
  const size_t bytes = window_bytes(av);
  void* recv = nullptr;
  if (!is_root && !a.base && bytes > 0)
    cuda_check(ws_alloc(&recv, bytes, st), "gemm_sharded: A receive buffer");
  if (recv) av.base = static_cast<std::byte*>(recv);
  const bool work = b_panel.n > 0 && c_panel.n > 0;
  ExecutionPlan p;
  try {  // policy and alias errors before any device work (dispatch.cpp:118-119)
    if (work) {
      if (ranges_overlap(c_panel, av) || ranges_overlap(c_panel, b_panel))
        throw Error("gemm: C must not alias A or B");
      p = plan(alpha, av, b_panel, beta, c_panel, cfg);
    }
  } catch (...) {
    if (recv) cudaFreeAsync(recv, st);
    throw;
  }

  // 1. A's byte window by broadcast on the communicator's stream, after the
  //    caller's stream reached the call
  cuda_check(cudaEventRecord(cm.start, st), "event");
  cuda_check(cudaStreamWaitEvent(cm.stream, cm.start, 0), "event");
  if (bytes > 0 && cm.nranks > 1)
    nccl_check(nccl().broadcast(av.base, av.base, bytes, ncclUint8, root, cm.comm, cm.stream), "ncclBroadcast(A)");
  cuda_check(cudaEventRecord(cm.ready, cm.stream), "event");

  // 2. the panel gemm: B packs under the broadcast, A after it
  if (work) {
    const OperandReady ready{cm.ready, p.logical_transpose};
    // a shard never takes split-K: its panels keep the rounding of the
    // unsharded call's whole-k grid (gpu.splitk = off makes that call
    // bitwise equal to the assembled panels)
    execute_scheduled(p, cfg.numerics, st, fc, false, nullptr, 0, nullptr, false, true, &ready);
  } else {
    cuda_check(cudaStreamWaitEvent(st, cm.ready, 0), "event");
  }
  if (recv) cuda_check(cudaFreeAsync(recv, st), "gemm_sharded: release");
}

// -------------------------------------------------------------- gemm_multi
namespace {

struct DeviceSet {
  std::vector<int> devices;
  std::vector<ncclComm_t> comms;
  std::vector<cudaStream_t> streams;
};

DeviceSet& device_set(const std::vector<int>& devices) {
  static std::mutex mu;
  static std::vector<std::unique_ptr<DeviceSet>> sets;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& s : sets)
    if (s->devices == devices) return *s;
  auto s = std::make_unique<DeviceSet>();
  s->devices = devices;
  s->comms.resize(devices.size());
  s->streams.resize(devices.size());
  if (devices.size() > 1)
    nccl_check(nccl().comm_init_all(s->comms.data(), static_cast<int>(devices.size()), devices.data()),
               "ncclCommInitAll");
  for (size_t i = 0; i < devices.size(); ++i) {
    cuda_check(cudaSetDevice(devices[i]), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&s->streams[i], cudaStreamNonBlocking), "stream");
  }
  sets.push_back(std::move(s));
  return *sets.back();
}

bool on_device(const MatrixView& v, int* dev) {
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, v.base) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (attr.type != cudaMemoryTypeDevice && attr.type != cudaMemoryTypeManaged) return false;
  *dev = attr.device;
  return true;
}

// A compact device copy of a column-major (rs == 1) or row-major (cs == 1)
// view, stream-ordered (2-D copies: only the view's own elements move).
struct Copy2D {
  size_t width, height, spitch, dpitch;
};
Copy2D copy_shape(const MatrixView& v, int64_t* ld) {
  const size_t esz = dtype_size(v.dtype);
  if (v.rs == 1) {
    *ld = std::max<int64_t>(v.m, 1);
    return Copy2D{static_cast<size_t>(v.m) * esz, static_cast<size_t>(v.n), static_cast<size_t>(v.cs) * esz,
                  static_cast<size_t>(*ld) * esz};
  }
  if (v.cs == 1) {
    *ld = std::max<int64_t>(v.n, 1);
    return Copy2D{static_cast<size_t>(v.n) * esz, static_cast<size_t>(v.m), static_cast<size_t>(v.rs) * esz,
                  static_cast<size_t>(*ld) * esz};
  }
  throw Error("gemm_multi: a panel that must move between devices needs a column- or row-major view");
}

MatrixView to_device(const MatrixView& v, cudaStream_t st, std::vector<std::pair<void*, cudaStream_t>>& owned) {
  MatrixView out = v;
  if (v.m <= 0 || v.n <= 0) return out;
  int64_t ld = 0;
  const Copy2D c = copy_shape(v, &ld);
  void* d = nullptr;
  cuda_check(ws_alloc(&d, c.dpitch * c.height, st), "gemm_multi: panel allocation");
  owned.emplace_back(d, st);
  cuda_check(cudaMemcpy2DAsync(d, c.dpitch, v.base, c.spitch, c.width, c.height, cudaMemcpyDefault, st),
             "gemm_multi: panel copy");
  out.base = static_cast<std::byte*>(d);
  if (v.rs == 1) out.cs = ld;
  else out.rs = ld;
  return out;
}

void from_device(const MatrixView& dst, const MatrixView& src, cudaStream_t st) {
  int64_t ld = 0;
  const Copy2D c = copy_shape(dst, &ld);
  cuda_check(cudaMemcpy2DAsync(dst.base, c.spitch, src.base, c.dpitch, c.width, c.height, cudaMemcpyDefault, st),
             "gemm_multi: C panel return");
}

MatrixView column_slice(const MatrixView& v, int64_t j0, int64_t nb) {
  MatrixView out = v;
  out.base = v.base + static_cast<size_t>(j0 * v.cs) * dtype_size(v.dtype);
  out.n = nb;
  return out;
}

}  // namespace

void shard_columns(int64_t n, int world, int rank, int64_t align, int64_t* j0, int64_t* nb) {
  if (world < 1 || rank < 0 || rank >= world || n < 0 || align < 1) throw Error("shard_columns: bad arguments");
  const int64_t per = (n + world - 1) / world;
  const int64_t chunk = (per + align - 1) / align * align;
  const int64_t lo = std::min<int64_t>(static_cast<int64_t>(rank) * chunk, n);
  *j0 = lo;
  *nb = std::min<int64_t>(chunk, n - lo);
}

void gemm_multi(Scalar alpha, const MatrixView& a, const MatrixView& b, Scalar beta, const MatrixView& c,
                const Config& cfg, const std::vector<int>& devices, FlopCounter* fc) {
  if (devices.empty()) throw Error("gemm_multi: no devices");
  int count = 0;
  cuda_check(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
  for (int d : devices)
    if (d < 0 || d >= count) throw Error("gemm_multi: device " + std::to_string(d) + " does not exist");
  if (ranges_overlap(c, a) || ranges_overlap(c, b)) throw Error("gemm: C must not alias A or B");
  int caller = 0;
  cuda_check(cudaGetDevice(&caller), "cudaGetDevice");
  plan(alpha, a, b, beta, c, cfg);  // policy errors before any device work (dispatch.cpp:118-119)
  DeviceSet& ds = device_set(devices);
  const int world = static_cast<int>(devices.size());
  std::vector<std::pair<void*, cudaStream_t>> owned;
  std::vector<MatrixView> cpan(world), cdev(world);
  std::vector<MatrixView> alocal(world);
  std::vector<FlopCounter> fcs(world);
  try {
    // A: the first device's copy (the caller's, when it is already there), broadcast to the rest
    int adev = -1;
    const bool a_on_first = on_device(a, &adev) && adev == devices[0];
    cuda_check(cudaSetDevice(devices[0]), "cudaSetDevice");
    alocal[0] = a_on_first ? a : to_device(a, ds.streams[0], owned);
    const size_t abytes = window_bytes(alocal[0]);
    for (int r = 1; r < world; ++r) {
      cuda_check(cudaSetDevice(devices[r]), "cudaSetDevice");
      alocal[r] = alocal[0];
      void* d = nullptr;
      if (abytes) {
        cuda_check(ws_alloc(&d, abytes, ds.streams[r]), "gemm_multi: A allocation");
        owned.emplace_back(d, ds.streams[r]);
      }
      alocal[r].base = static_cast<std::byte*>(d);
    }
    cuda_check(cudaStreamSynchronize(ds.streams[0]), "gemm_multi: A staging");
    if (world > 1 && abytes > 0) {
      nccl_check(nccl().group_start(), "ncclGroupStart");
      for (int r = 0; r < world; ++r)
        nccl_check(nccl().broadcast(alocal[r].base, alocal[r].base, abytes, ncclUint8, 0, ds.comms[r],
                                    ds.streams[r]),
                   "ncclBroadcast(A)");
      nccl_check(nccl().group_end(), "ncclGroupEnd");
    }
    // B / C column panels: the caller's memory when it is the device's own,
    // else a copy on the device (peer copies over NVLink, or host staging)
    for (int r = 0; r < world; ++r) {
      int64_t j0 = 0, nb = 0;
      shard_columns(c.n, world, r, 128, &j0, &nb);
      cpan[r] = column_slice(c, j0, nb);
      if (nb == 0) continue;
      cuda_check(cudaSetDevice(devices[r]), "cudaSetDevice");
      const MatrixView bpan = column_slice(b, j0, nb);
      int bd = -1, cd = -1;
      const MatrixView bl = on_device(bpan, &bd) && bd == devices[r] ? bpan : to_device(bpan, ds.streams[r], owned);
      cdev[r] = on_device(cpan[r], &cd) && cd == devices[r] ? cpan[r] : to_device(cpan[r], ds.streams[r], owned);
      const ExecutionPlan p = plan(alpha, alocal[r], bl, beta, cdev[r], cfg);
      execute_scheduled(p, cfg.numerics, ds.streams[r], &fcs[r], false, nullptr, 0, nullptr, false);
      if (cdev[r].base != cpan[r].base) from_device(cpan[r], cdev[r], ds.streams[r]);
    }
    for (int r = 0; r < world; ++r) {
      cuda_check(cudaSetDevice(devices[r]), "cudaSetDevice");
      for (auto& o : owned)
        if (o.second == ds.streams[r]) cuda_check(cudaFreeAsync(o.first, o.second), "gemm_multi: release");
      cuda_check(cudaStreamSynchronize(ds.streams[r]), "gemm_multi");
    }
  } catch (...) {
    cudaSetDevice(caller);
    throw;
  }
  cuda_check(cudaSetDevice(caller), "cudaSetDevice");
  if (fc)
    for (const FlopCounter& f : fcs) fc->add(f.value());
}

}  // namespace mdgemm
