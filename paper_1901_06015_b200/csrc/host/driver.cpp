// Execution half of gemm() on the GPU: replaces the reference's
// gemm_blocked + C_temp + write_back + beta_pass (dispatch.cpp:359-388,
// gemm_core.cpp:74-185).  Host C++ only: it sizes the packed panels, launches
// the pack kernels and one gemm kernel per call, and keeps the reference's
// FlopCounter accounting.
#include "driver.hpp"
#include "profile.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <vector>

namespace mdgemm {

namespace {

int device_sms_impl() {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  static std::mutex mu;
  static std::vector<int> cache;
  std::lock_guard<std::mutex> lock(mu);
  if (cache.size() <= static_cast<size_t>(dev)) cache.resize(dev + 1, 0);
  if (cache[dev] == 0) {
    int sms = 0;
    cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "SM count");
    // tests only (MDGEMM_SMS): schedule for fewer SMs than the device has, so
    // that small problems exercise the persistent, stream-K and multi-tile
    // paths (compute-sanitizer runs)
    if (const char* f = std::getenv("MDGEMM_SMS")) {
      const int cap = std::atoi(f);
      if (cap > 0 && cap < sms) sms = cap;
    }
    cache[dev] = sms;
  }
  return cache[dev];
}

}  // namespace

int device_sms() { return device_sms_impl(); }

// The library's own stream-ordered pool per device (workspace, staged host
// operands).  A private pool, not the device's default one: its "keep what
// you have" release threshold must not change how other users of the
// default pool in the same process (PyTorch, other libraries) get memory
// back, and trim_workspace() can hand it all back.
cudaMemPool_t workspace_pool() {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  static std::mutex mu;
  static std::vector<cudaMemPool_t> pools;
  std::lock_guard<std::mutex> lock(mu);
  if (pools.size() <= static_cast<size_t>(dev)) pools.resize(dev + 1, nullptr);
  if (!pools[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    cuda_check(cudaMemPoolCreate(&pool, &props), "cudaMemPoolCreate");
    // Keep stream-ordered workspace cached between calls (release with
    // trim_workspace / mdg_trim_workspace).
    uint64_t keep = ~0ULL;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    // Never let an allocation on one compute stream wait for a free on
    // another (the allocator would insert that dependency to reuse the
    // block, serialising the concurrent calls of a batch): grow instead.
    int no = 0;
    cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
    pools[dev] = pool;
    // Optional up-front reservation (MDGEMM_POOL_RESERVE_GB): growing the
    // pool maps new memory in the middle of a batch.
    if (const char* f = std::getenv("MDGEMM_POOL_RESERVE_GB")) {
      const double gb = std::atof(f);
      void* p = nullptr;
      if (gb > 0 && cudaMallocFromPoolAsync(&p, static_cast<size_t>(gb * (1ull << 30)), pool, cudaStreamLegacy) ==
                        cudaSuccess) {
        cudaFreeAsync(p, cudaStreamLegacy);
        cudaStreamSynchronize(cudaStreamLegacy);
      }
      cudaGetLastError();
    }
  }
  return pools[dev];
}

cudaError_t ws_alloc(void** p, size_t bytes, cudaStream_t st) {
  return cudaMallocFromPoolAsync(p, bytes, workspace_pool(), st);
}

void trim_workspace(size_t keep_bytes) {
  cuda_check(cudaDeviceSynchronize(), "trim_workspace: synchronize");
  cuda_check(cudaMemPoolTrimTo(workspace_pool(), keep_bytes), "cudaMemPoolTrimTo");
  reset_reservation();
  if (keep_bytes == 0) trim_host_staging();
}

namespace {

int32_t dt_code(Datatype t) {
  return (t.domain == Domain::Complex ? 2 : 0) + (t.precision == Precision::Double ? 1 : 0);
}

mdg::DBeta to_dbeta(const Scalar& b) {
  return mdg::DBeta{b.re, b.im, b.is_zero() ? 1 : 0, b.is_one() ? 1 : 0};
}

// Packed operand consumed by a kernel tile of `tile` real rows (left) or
// columns (right); a complex operand packed Standard counts complex rows.
struct Packed {
  mdg::PackDesc desc{};
  size_t bytes = 0;
};

// pitch: real elements between consecutive panel lines (0: the tile, the
// reference layout)
Packed prepare_pack(const MatrixView& src, Side side, PackFormat fmt, bool conj, const Scalar& scale,
                    Datatype target, int64_t tile, int64_t lpad, int64_t pitch = 0) {
  const bool halves = fmt == PackFormat::Standard && src.dtype.domain == Domain::Complex;
  Packed out;
  out.desc = make_pack_desc(src, side, fmt, conj, scale, target, halves ? tile / 2 : tile, lpad, &out.bytes,
                            halves ? pitch / 2 : pitch);
  return out;
}

// Algorithmic bytes of one pack: the source elements read plus the packed
// buffer written.
double pack_traffic(const MatrixView& src, size_t packed) {
  return static_cast<double>(src.m) * src.n * dtype_size(src.dtype) + static_cast<double>(packed);
}

// Real inner-dimension steps per source column of A (left) / row of B (right):
// 2 for the 1m formats (1e, 1r), 1 for Standard.
int64_t k_factor(PackFormat f) { return f == PackFormat::Standard ? 1 : 2; }

// The plan restricted to real inner steps [lo, hi): column slices of A's
// source view, row slices of B's.
ExecutionPlan k_slice(const ExecutionPlan& p, int64_t lo, int64_t hi, int64_t f_a, int64_t f_b) {
  ExecutionPlan q = p;
  q.k = hi - lo;
  q.a.base = p.a.base + static_cast<size_t>(lo / f_a * p.a.cs) * dtype_size(p.a.dtype);
  q.a.n = (hi - lo) / f_a;
  q.b.base = p.b.base + static_cast<size_t>(lo / f_b * p.b.rs) * dtype_size(p.b.dtype);
  q.b.m = (hi - lo) / f_b;
  return q;
}

bool onem_direct(const ExecutionPlan& p);

}  // namespace

// FAST per-KC-block structure of a plan without C_temp: 0 one combine after
// the full inner dimension, 1 one combine per KC block.  The reference's
// Temp / 1m-temp routes round each KC block's sum into C (gemm_core.cpp:
// 125-127); that changes the values only where C is stored at another
// precision than the computation's (each block meets C's rounding, or C's
// wider accumulation).  Where the two precisions agree, the block boundaries
// only reorder the sum in the computation precision -- within the bound FAST
// already meets -- and the call keeps one pass (and the dual kernel).  C_temp
// plans and the Direct paths accumulate continuously: one combine.  Odd KC
// blocks of a 1m image would split a complex element's real and imaginary
// steps; those plans keep one combine too.
int fast_block_mode(const ExecutionPlan& p, int64_t* f_a, int64_t* f_b) {
  if (p.ctemp || p.k <= p.params.kc || p.params.kc < 1) return 0;
  if (p.c.dtype.precision == p.comp_prec) return 0;
  const int64_t fa = k_factor(p.format_a), fb = k_factor(p.format_b);
  if (p.params.kc % fa || p.params.kc % fb) return 0;
  int mode = 0;
  const bool onem = p.ukr_path == UkrPath::OneMColumn || p.ukr_path == UkrPath::OneMRow;
  if (p.ukr_path == UkrPath::Temp) mode = 1;
  if (onem && !onem_direct(p)) mode = 1;  // C of another precision: virtual_ukr_temp per block
  if (f_a) *f_a = fa;
  if (f_b) *f_b = fb;
  return mode;
}

namespace {

bool onem_direct(const ExecutionPlan& p) {
  const FlattenAxis ax = p.ukr_path == UkrPath::OneMColumn ? FlattenAxis::Rows : FlattenAxis::Cols;
  return p.beta.im == 0.0 && p.c.dtype.precision == p.comp_prec && can_flatten(p.c, ax);
}

}  // namespace

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
}

mdg::DView to_dview(const MatrixView& v) {
  return mdg::DView{reinterpret_cast<char*>(v.base), v.m, v.n, v.rs, v.cs, dt_code(v.dtype), v.conj ? 1 : 0};
}

PackGeometry pack_geometry(const MatrixView& src, Side side, PackFormat format, Datatype target,
                           int64_t reg_block, int64_t panel_len, int64_t pitch) {
  if (reg_block < 1) throw Error("pack_block: reg_block must be at least 1");
  if (pitch != 0 && pitch < reg_block) throw Error("pack_block: line pitch below the panel dimension");
  const bool left = side == Side::Left;
  PackGeometry g;
  int64_t rows = 0, cols = 0;
  switch (format) {
    case PackFormat::Standard:
      if (target.domain != src.dtype.domain) throw Error("pack_block: Standard packing cannot change the domain");
      g.block_dtype = target;
      rows = src.m;
      cols = src.n;
      break;
    case PackFormat::OneE:
      if (src.dtype.domain != Domain::Complex) throw Error("pack_block: OneE requires a complex source");
      if (reg_block % 2) throw Error("pack_block: OneE requires an even reg_block");
      g.block_dtype = Datatype{Domain::Real, target.precision};
      rows = 2 * src.m;
      cols = 2 * src.n;
      break;
    case PackFormat::OneR:
      if (src.dtype.domain != Domain::Complex) throw Error("pack_block: OneR requires a complex source");
      g.block_dtype = Datatype{Domain::Real, target.precision};
      rows = left ? src.m : 2 * src.m;
      cols = left ? 2 * src.n : src.n;
      break;
  }
  const int64_t extent = left ? rows : cols;
  g.panels = (extent + reg_block - 1) / reg_block;
  g.len = left ? cols : rows;
  g.lpad = std::max(g.len, panel_len);
  g.pitch = pitch ? pitch : reg_block;
  g.bytes = static_cast<size_t>(g.panels * g.pitch * g.lpad) * dtype_size(g.block_dtype);
  return g;
}

uint64_t reference_flops(const ExecutionPlan& p) {
  if (p.m <= 0 || p.n <= 0 || p.k <= 0) return 0;
  const uint64_t MR = static_cast<uint64_t>(p.ukr.mr), NR = static_cast<uint64_t>(p.ukr.nr);
  const uint64_t tiles = static_cast<uint64_t>((p.m + p.ukr.mr - 1) / p.ukr.mr) *
                         static_cast<uint64_t>((p.n + p.ukr.nr - 1) / p.ukr.nr);
  uint64_t total = 2 * MR * NR * static_cast<uint64_t>(p.k) * tiles;
  // gemm_ukr adds mr*nr when called directly with beta not in {0,1}
  // (kernels.cpp:73-76): the Direct path and 1m-direct, first KC block only.
  bool direct_ukr = false;
  if (!p.ctemp) {
    if (p.ukr_path == UkrPath::Direct) direct_ukr = true;
    if ((p.ukr_path == UkrPath::OneMColumn || p.ukr_path == UkrPath::OneMRow) && onem_direct(p))
      direct_ukr = true;
  }
  if (direct_ukr && p.beta.re != 0.0 && p.beta.re != 1.0) total += MR * NR * tiles;
  return total;
}

void pack_block_device(void* dst, const MatrixView& src, Side side, PackFormat format, bool conj,
                       Scalar scale, Datatype target, std::int64_t reg_block, void* stream) {
  pack_block_device_padded(dst, src, side, format, conj, scale, target, reg_block, 0, stream);
}

mdg::PackDesc make_pack_desc(const MatrixView& src, Side side, PackFormat format, bool conj,
                             const Scalar& scale, Datatype target, int64_t reg_block, int64_t panel_len,
                             size_t* bytes, int64_t pitch) {
  if (scale.im != 0.0 && format == PackFormat::Standard)
    throw Error("pack_block: complex scale requires OneE or OneR format");
  const PackGeometry g = pack_geometry(src, side, format, target, reg_block, panel_len, pitch);
  mdg::PackDesc d{};
  d.src = to_dview(src);
  d.side = side == Side::Left ? MDG_SIDE_LEFT : MDG_SIDE_RIGHT;
  d.format = static_cast<int32_t>(format);
  d.do_conj = src.conj != conj;  // packing.cpp:140
  d.unit_scale = scale.is_one();
  d.sre = scale.re;
  d.sim = scale.im;
  d.target_single = target.precision == Precision::Single;
  d.out_complex = g.block_dtype.domain == Domain::Complex;
  d.pd = reg_block;
  d.pitch = static_cast<int32_t>(g.pitch);
  d.pd_shift = -1;
  if ((reg_block & (reg_block - 1)) == 0)
    for (int s = 0; s < 63; ++s)
      if ((int64_t{1} << s) == reg_block) d.pd_shift = s;
  d.panels = g.panels;
  d.len = g.len;
  d.lpad = g.lpad;
  // Source index space covered by the kernel, panel padding included.
  const int64_t src_units = format == PackFormat::OneE ? reg_block / 2 : reg_block;
  d.ext_i = side == Side::Left ? g.panels * src_units : src.m;
  d.ext_j = side == Side::Left ? src.n : g.panels * src_units;
  if (bytes) *bytes = g.bytes;
  return d;
}

void pack_block_device_padded(void* dst, const MatrixView& src, Side side, PackFormat format, bool conj,
                              Scalar scale, Datatype target, int64_t reg_block, int64_t panel_len,
                              void* stream) {
  size_t bytes = 0;
  const mdg::PackDesc d = make_pack_desc(src, side, format, conj, scale, target, reg_block, panel_len, &bytes);
  prof::Scope scope(MDG_KERNEL_PACK, static_cast<cudaStream_t>(stream), pack_traffic(src, bytes));
  cuda_check(mdg::launch_pack(d, dst, static_cast<cudaStream_t>(stream)), "pack kernel");
}

std::size_t packed_bytes(const MatrixView& src, Side side, PackFormat format, Datatype target,
                         std::int64_t reg_block) {
  return pack_geometry(src, side, format, target, reg_block, 0).bytes;
}

// C as a 2-D TMA tensor for the fused epilogue (common.cuh: fast_epilogue),
// boxes of (tile extent along C's contiguous dimension) x C_BOX_COLS lines.
// Returns the MDG_CMAP_* mode (0: none; the element-wise epilogue then):
//   COLS       column-major C: inner = rows x components, outer = columns;
//   ROWS       row-major C (a transposed plan): inner = columns x components,
//              outer = rows;
//   REAL_PART  a real view with rs == 2 (the real part of an interleaved
//              complex C, case 1c): inner = both halves of each row pair.
// All need 16-byte aligned base and line strides.
static int encode_c_map(mdg::DEpilogue& e, int bm, int bn) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<Encode>(nullptr);
    return reinterpret_cast<Encode>(fn);
  }();
  if (!encode) return mdg::MDG_CMAP_NONE;
  const bool single = e.out.dtype == MDG_DT_S || e.out.dtype == MDG_DT_C;
  const int nc = (e.out.dtype == MDG_DT_C || e.out.dtype == MDG_DT_Z) ? 2 : 1;
  const int esr = single ? 4 : 8, esz = esr * nc;
  const int orows = e.pair == MDG_PAIR_ROWS ? bm / 2 : bm, ocols = e.pair == MDG_PAIR_COLS ? bn / 2 : bn;
  const auto base = reinterpret_cast<uintptr_t>(e.out.base);
  if (e.out.m <= 0 || e.out.n <= 0 || base % 16) return mdg::MDG_CMAP_NONE;
  int mode = mdg::MDG_CMAP_NONE;
  cuuint64_t dims[2];
  cuuint64_t stride = 0;
  cuuint32_t inner = 0;
  if (e.out.rs == 1) {
    mode = mdg::MDG_CMAP_COLS;
    dims[0] = static_cast<cuuint64_t>(e.out.m * nc);
    dims[1] = static_cast<cuuint64_t>(e.out.n);
    stride = static_cast<cuuint64_t>(e.out.cs * esz);
    inner = static_cast<cuuint32_t>(orows * nc);
  } else if (e.out.cs == 1) {
    mode = mdg::MDG_CMAP_ROWS;
    dims[0] = static_cast<cuuint64_t>(e.out.n * nc);
    dims[1] = static_cast<cuuint64_t>(e.out.m);
    stride = static_cast<cuuint64_t>(e.out.rs * esz);
    inner = static_cast<cuuint32_t>(ocols * nc);
  } else if (e.out.rs == 2 && nc == 1) {
    mode = mdg::MDG_CMAP_REAL_PART;
    dims[0] = static_cast<cuuint64_t>(2 * e.out.m);
    dims[1] = static_cast<cuuint64_t>(e.out.n);
    stride = static_cast<cuuint64_t>(e.out.cs * esr);
    inner = static_cast<cuuint32_t>(2 * orows);
  } else {
    return mdg::MDG_CMAP_NONE;
  }
  if (stride % 16 || (inner * esr) % 16 || inner > 256) return mdg::MDG_CMAP_NONE;
  // the kernels pass box coordinates as 32-bit ints: a taller or wider C
  // takes the element-wise path
  if (dims[0] > 0x7fffffffull || dims[1] > 0x7fffffffull) return mdg::MDG_CMAP_NONE;
  const cuuint64_t strides[1] = {stride};
  const cuuint32_t box[2] = {inner, static_cast<cuuint32_t>(mdg::C_BOX_COLS)};
  const cuuint32_t estride[2] = {1, 1};
  const bool ok = encode(&e.cmap, single ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                         e.out.base, dims, strides, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  e.sw_ok = 0;
  if (ok && mode == mdg::MDG_CMAP_COLS && nc == 1) {  // swizzled 128-byte boxes (warp-specialised kernels)
    const cuuint32_t box_sw[2] = {static_cast<cuuint32_t>(128 / esr), static_cast<cuuint32_t>(mdg::C_BOX_COLS)};
    e.sw_ok = encode(&e.cmap_sw, single ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                     e.out.base, dims, strides, box_sw, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
                  ? 1
                  : 0;
    if (const char* f = std::getenv("MDGEMM_C_SWIZZLE"))  // tuning: 0 = plain boxes in the WS kernels
      if (std::atoi(f) == 0) e.sw_ok = 0;
  }
  return ok ? mode : mdg::MDG_CMAP_NONE;
}

// Resident CTAs per SM of a fast kernel (occupancy query, cached per
// tile shape x kernel x C datatype; the value is the same on every B200).
static int ctas_per_sm(const mdg::FastTile& t, bool single, int cdt) {
  static std::atomic<int> cache[3][2][4] = {};
  const int ti = t.bm == 128 ? 0 : (t.bn == 128 ? 1 : 2);
  std::atomic<int>& slot = cache[ti][single ? 1 : 0][cdt & 3];
  int v = slot.load(std::memory_order_relaxed);
  if (v == 0) {
    v = single ? mdg::ffma_ctas_per_sm(t, cdt) : mdg::dmma_ctas_per_sm(t, cdt);
    slot.store(v, std::memory_order_relaxed);
  }
  return v;
}

void execute(const ExecutionPlan& p, Numerics numerics, void* stream_ptr, FlopCounter* fc, bool allow_splitk) {
  execute_scheduled(p, numerics, stream_ptr, fc, false, nullptr, 0, nullptr, allow_splitk);
}

size_t workspace_bytes(const ExecutionPlan& p, Numerics numerics, bool shared, bool allow_splitk) {
  size_t n = 0;
  execute_scheduled(p, numerics, nullptr, nullptr, shared, nullptr, 0, &n, allow_splitk);
  return n;
}

void execute_scheduled(const ExecutionPlan& p, Numerics numerics, void* stream_ptr, FlopCounter* fc, bool shared,
                       void* arena, size_t arena_bytes, size_t* ws_needed, bool allow_splitk, bool block_split,
                       const OperandReady* ready) {
  cudaStream_t st = static_cast<cudaStream_t>(stream_ptr);
  if (ws_needed) *ws_needed = 0;
  if (p.m == 0 || p.n == 0) return;
  // Device-ordered entry points need device operands; a host pointer here
  // would fault inside a kernel and poison the context, so refuse it.
  auto require_device = [](const MatrixView& v, const char* what) {
    if (v.m == 0 || v.n == 0) return;
    cudaPointerAttributes attr{};
    const cudaError_t e = cudaPointerGetAttributes(&attr, v.base);
    if (e != cudaSuccess) cudaGetLastError();
    if (e != cudaSuccess || (attr.type != cudaMemoryTypeDevice && attr.type != cudaMemoryTypeManaged))
      throw Error(std::string("execute: operand ") + what +
                  " is not in device memory (use gemm()/gemm_batch() for host operands)");
  };
  if (!ws_needed) {  // (a workspace query may see host operands that are staged later)
    require_device(p.c, "C");
    if (p.k > 0) {
      require_device(p.a, "A");
      require_device(p.b, "B");
    }
  }
  if (p.k == 0) {
    if (ws_needed) return;
    if (!p.beta.is_one()) {
      prof::Scope scope(MDG_KERNEL_BETA, st, 2.0 * p.c.m * p.c.n * dtype_size(p.c.dtype));
      cuda_check(mdg::launch_beta_pass(to_dview(p.c), to_dbeta(p.beta), device_sms(), st), "beta pass");
    }
    return;
  }
  const bool single = p.comp_prec == Precision::Single;
  const bool exact = numerics == Numerics::Exact;
  const int sms = device_sms();

  // ctemp.enable = off (or auto with several threads) on a Temp-path plan with
  // C stored at another precision than the computation's: the reference
  // rounds each KC block's partial sum into C (gemm_core.cpp:125-127,
  // kernels.cpp:97-132).  FAST keeps that structure: one kernel pass per KC
  // block of the real inner dimension, beta on the first and 1 afterwards.
  if (!exact && block_split) {
    int64_t f_a = 1, f_b = 1;
    const int mode = fast_block_mode(p, &f_a, &f_b);
    if (mode != 0) {
      const int64_t kc = p.params.kc;
      if (ws_needed) {  // the first (largest) block's workspace
        ExecutionPlan q = k_slice(p, 0, std::min(kc, p.k), f_a, f_b);
        execute_scheduled(q, numerics, nullptr, nullptr, shared, nullptr, 0, ws_needed, allow_splitk, false);
        return;
      }
      for (int64_t pc = 0; pc < p.k;) {
        const int64_t hi = std::min(pc + kc, p.k);
        ExecutionPlan q = k_slice(p, pc, hi, f_a, f_b);
        if (pc > 0) q.beta = Scalar{1.0, 0.0, p.beta.dtype};
        execute_scheduled(q, numerics, stream_ptr, nullptr, shared, arena, arena_bytes, nullptr, allow_splitk, false,
                          ready);
        pc = hi;
      }
      if (fc) fc->add(reference_flops(p));
      return;
    }
  }

  mdg::FastTile tile{64, 64, 1};
  if (!exact) tile = single ? mdg::choose_ffma_tile(p.m, p.n, sms) : mdg::choose_dmma_tile(p.m, p.n, sms);
  // Warp-specialised persistent kernels (gemm_{dmma,ffma}_ws.cu): 128x128
  // tiles, one CTA per SM, the C traffic of one tile under the next tile's
  // mainloop.
  bool dmma_ws = false;  // (either computation precision)
  if (!exact) {
    int mode = 0;  // MDGEMM_{DMMA,FFMA}_WS: 1 force on (where it applies), -1 off, 0 auto
    if (const char* f = std::getenv(single ? "MDGEMM_FFMA_WS" : "MDGEMM_DMMA_WS")) mode = std::atoi(f);
    const int64_t t128 = ((p.m + 127) / 128) * ((p.n + 127) / 128);
    mdg::DEpilogue probe{};  // the kernel moves C only through a TMA tensor map
    probe.out = to_dview(p.c);
    probe.pair = static_cast<int32_t>(p.pair_axis);
    const bool complex_c = probe.out.dtype == MDG_DT_C || probe.out.dtype == MDG_DT_Z;
    const int cmode = encode_c_map(probe, 128, 128);
    // WS kernels: column-major C; the FFMA one also the real part of an
    // interleaved complex C (case 1c: cfg4 cdds)
    const bool c_ok = (cmode == mdg::MDG_CMAP_COLS && (!complex_c || probe.pair != MDG_PAIR_NONE)) ||
                      (single && cmode == mdg::MDG_CMAP_REAL_PART && probe.out.dtype == MDG_DT_S);
    // auto: real C (measured at the cfg2 sizes 2048-4096: DMMA +1..7 %,
    // FFMA +2..4 %, short k far more -- rank-64 ssss 19.6 -> 27.3 TFLOP/s;
    // complex C -1..2 %), one full wave of 128x128 tiles,
    // and the GPU to itself (a persistent grid inside a concurrent batch
    // would wait for slots the other calls hold; MDGEMM_DMMA_WS=2 allows it)
    const bool want = mode == 1 || (mode == 0 && !complex_c && !shared) || (mode == 2 && !complex_c);
    if (want && t128 >= sms && c_ok) {
      dmma_ws = true;
      tile = mdg::FastTile{128, 128, 16};
    }
  }
  const int64_t lpad = (p.k + tile.bk - 1) / tile.bk * tile.bk;

  Packed pa = prepare_pack(p.a, Side::Left, p.format_a, p.conj_a, p.pack_scale_a, p.target_dtype_a, tile.bm, lpad);
  Packed pb = prepare_pack(p.b, Side::Right, p.format_b, p.conj_b, p.pack_scale_b, p.target_dtype_b, tile.bn, lpad);

  // Split-K when the tile grid cannot fill the machine (deterministic: the
  // partial tiles are summed in split order by the reduce pass).
  const int64_t tiles = ((p.m + tile.bm - 1) / tile.bm) * ((p.n + tile.bn - 1) / tile.bn);
  const int per_sm = exact || dmma_ws ? 1 : ctas_per_sm(tile, single, to_dview(p.c).dtype);
  const int64_t nk = lpad / tile.bk;
  int splits = exact || dmma_ws || !allow_splitk ? 1 : mdg::choose_splits(tiles, nk, sms * per_sm);
  int kb_per_split = static_cast<int>(nk);
  if (splits > 1) {
    kb_per_split = static_cast<int>((nk + splits - 1) / splits);
    splits = static_cast<int>((nk + kb_per_split - 1) / kb_per_split);
  }
  // Stream-K tail for a call that has the GPU to itself, when the classic
  // grid's last wave would run mostly empty: whole-tile CTAs for all but the
  // last full wave, then one CTA per slot sharing the rest as k-block ranges
  // (common.cuh: make_sched); bitwise identical to the classic grid.
  // Measured on B200 over the cfg2 sizes 1792..4096: +2..11 % for the DMMA
  // and FFMA kernels whenever the tail wave is less than ~85 % full, neutral
  // above.  Inside a concurrent batch the classic grid stays: its
  // hardware-scheduled tiles interleave with the other calls' kernels.
  const int64_t slots = static_cast<int64_t>(sms) * per_sm;
  int sk_grid = 0;
  int ws_grid = 0;  // persistent grid of the warp-specialised kernel
  if (dmma_ws) {
    ws_grid = static_cast<int>(std::min<int64_t>(tiles, sms));
    int mode = 0;
    if (const char* f = std::getenv("MDGEMM_STREAMK")) mode = std::atoi(f);
    // stream-K tail: CTAs of this kernel progress in step (one per SM)
    if (mode >= 0 && tiles > sms && tiles % sms != 0 && nk >= 8) sk_grid = sms;
  } else if (!exact && splits == 1 && tiles > slots && tiles % slots != 0 && tile.bn == 128) {
    int mode = 0;  // tuning override MDGEMM_STREAMK: 0 auto, 1 force on, -1 off
    if (const char* f = std::getenv("MDGEMM_STREAMK")) mode = std::atoi(f);
    // Only where the tail matters (few waves) and tiles are mainloop-bound:
    // with a short k the epilogue dominates and the stream-K variant's
    // heavier epilogue costs more than the tail (cfg5 k=64: -43 %).
    const double tail = static_cast<double>(tiles % slots) / static_cast<double>(slots);
    const bool wins = tail < 0.85 && tiles < 8 * slots && nk >= 32;  // (13.8 waves: -2 %)
    if (mode == 1 || (mode == 0 && !shared && wins)) sk_grid = static_cast<int>(slots);
  }
  // The segment-loop kernel with one whole tile per CTA (sk_grid = tiles:
  // make_sched gives every CTA its own tile) is the classic schedule.  ptxas
  // compiles the FFMA 128x128 mainloop 4-6 % faster in that variant
  // (measured, cfg4: 61.2 -> 64.0 TFLOP/s), so it always runs there;
  // MDGEMM_STREAMK=2 forces it for every tile shape (experiments).
  {
    const char* f = std::getenv("MDGEMM_STREAMK");
    const bool force = f && std::atoi(f) == 2;
    if (!exact && !dmma_ws && splits == 1 && sk_grid == 0 && tiles > 0 &&
        ((single && tile.bm == 128 && tile.bn == 128) || (force && tile.bn == 128)))
      sk_grid = static_cast<int>(tiles);
  }
  // partial-tile slots and publish flags only where ranges split tiles
  const bool sk_ranges = sk_grid > 0 && tiles % sk_grid != 0;
  const size_t acc_size = single ? sizeof(float) : sizeof(double);
  const size_t off_b = (pa.bytes + 255) / 256 * 256;
  const size_t off_p = off_b + (pb.bytes + 255) / 256 * 256;
  const size_t part_bytes = splits > 1 ? static_cast<size_t>(splits * tiles * tile.bm * tile.bn) * acc_size
                            : sk_ranges ? static_cast<size_t>(sk_grid) * tile.bm * tile.bn * acc_size
                                        : 0;
  const size_t off_f = off_p + (part_bytes + 255) / 256 * 256;
  // publish flags + the start ticket (common.cuh: logical_cta)
  const size_t flag_bytes = sk_ranges ? static_cast<size_t>(sk_grid + 1) * sizeof(int) : 0;
  if (ws_needed) {
    *ws_needed = off_f + flag_bytes;
    return;
  }
  // The caller's arena (gemm_batch: one per compute stream, reused by the
  // stream's calls in stream order) or a stream-ordered pool allocation.
  void* ws = nullptr;
  const bool owned = !(arena && arena_bytes >= off_f + flag_bytes);
  if (owned) {
    cuda_check(ws_alloc(&ws, off_f + flag_bytes, st), "workspace allocation");
  } else {
    ws = arena;
  }
  char* wsa = static_cast<char*>(ws);
  cudaError_t err = flag_bytes > 0 ? cudaMemsetAsync(wsa + off_f, 0, flag_bytes, st) : cudaSuccess;
  cuda_check(err, "stream-K flags");
  if (ready && ready->event) {
    // one operand arrives on another stream (gemm_sharded: the broadcast of
    // A): pack the other one first, then wait for it and pack it
    const bool right_late = ready->right;
    const Packed& first = right_late ? pa : pb;
    const Packed& late = right_late ? pb : pa;
    const MatrixView& fv = right_late ? p.a : p.b;
    const MatrixView& lv = right_late ? p.b : p.a;
    char* fdst = right_late ? wsa : wsa + off_b;
    char* ldst = right_late ? wsa + off_b : wsa;
    {
      prof::Scope scope(MDG_KERNEL_PACK, st, pack_traffic(fv, first.bytes));
      err = mdg::launch_pack(first.desc, fdst, st);
    }
    if (err == cudaSuccess) err = cudaStreamWaitEvent(st, ready->event, 0);
    if (err == cudaSuccess) {
      prof::Scope scope(MDG_KERNEL_PACK, st, pack_traffic(lv, late.bytes));
      err = mdg::launch_pack(late.desc, ldst, st);
    }
  } else if (mdg::pack_pair_ok(pa.desc, pb.desc)) {  // both operands in one launch
    prof::Scope scope(MDG_KERNEL_PACK, st, pack_traffic(p.a, pa.bytes) + pack_traffic(p.b, pb.bytes));
    err = mdg::launch_pack_pair(pa.desc, wsa, pb.desc, wsa + off_b, st);
  } else {
    {
      prof::Scope scope(MDG_KERNEL_PACK, st, pack_traffic(p.a, pa.bytes));
      err = mdg::launch_pack(pa.desc, wsa, st);
    }
    if (err == cudaSuccess) {
      prof::Scope scope(MDG_KERNEL_PACK, st, pack_traffic(p.b, pb.bytes));
      err = mdg::launch_pack(pb.desc, wsa + off_b, st);
    }
  }

  mdg::GemmDesc g{};
  g.a = mdg::DPanels{wsa, tile.bm, lpad};
  g.b = mdg::DPanels{wsa + off_b, tile.bn, lpad};
  g.me = p.m;
  g.ne = p.n;
  g.ke = p.k;
  g.epi.out = to_dview(p.c);
  g.epi.pair = static_cast<int32_t>(p.pair_axis);
  g.epi.beta = to_dbeta(p.beta);
  g.epi.me = p.m;
  g.epi.ne = p.n;
  g.epi.cmap_ok = exact ? mdg::MDG_CMAP_NONE : encode_c_map(g.epi, tile.bm, tile.bn);
  if (const char* f = std::getenv("MDGEMM_C_TMA"))  // tuning: 0 = element-wise epilogue
    if (std::atoi(f) == 0) g.epi.cmap_ok = 0;
  g.kc = p.params.kc;
  g.seed_beta = p.beta.re;
  // Short inner dimension: C traffic dominates, walk whole tile-columns so the
  // concurrently written C stays within a few column panels (TLB reach).
  // Otherwise the resident wave should touch as few panel bytes as
  // possible: g tile-rows x slots/g tile-columns reads g A panels (bm rows)
  // and slots/g B panels (bn columns), minimal at g = sqrt(slots bn / bm)
  // (24 for the DMMA 64x128 pair, 30 for FFMA at three CTAs per SM).  Same
  // speed as 8-row groups (the mainloop is pipe-bound), ~15-30 % less DRAM
  // re-reading of the panels.
  {
    const int64_t tiles_m = (p.m + tile.bm - 1) / tile.bm;
    const int64_t sq = static_cast<int64_t>(std::lround(std::sqrt(static_cast<double>(sms) * per_sm * tile.bn / tile.bm)));
    g.group_rows = static_cast<int32_t>(p.k <= 512 ? tiles_m : std::max<int64_t>(1, std::min(sq, tiles_m)));
  }
  if (const char* force = std::getenv("MDGEMM_GROUP_ROWS")) g.group_rows = std::atoi(force);
  g.splits = splits;
  g.kb_per_split = kb_per_split;
  g.partials = splits > 1 ? wsa + off_p : nullptr;
  g.sk_grid = sk_grid;
  g.sk_partials = sk_ranges ? wsa + off_p : nullptr;
  g.sk_flags = sk_ranges ? reinterpret_cast<int*>(wsa + off_f) : nullptr;
  g.prefetch = 0;
  g.c_prefetch = nk <= 16 ? 1 : 0;  // short k: the epilogue's C traffic is the critical path
  if (const char* force = std::getenv("MDGEMM_C_PREFETCH")) g.c_prefetch = std::atoi(force);
  if (const char* force = std::getenv("MDGEMM_PREFETCH")) g.prefetch = std::atoi(force);

  if (err == cudaSuccess) {
    if (exact) {
      // Replay the reference's output path for this plan.
      g.exact_mode = mdg::EXACT_BLOCK_COMBINE;
      const bool onem = p.ukr_path == UkrPath::OneMColumn || p.ukr_path == UkrPath::OneMRow;
      const FlattenAxis ax = p.ukr_path == UkrPath::OneMColumn ? FlattenAxis::Rows : FlattenAxis::Cols;
      const bool onem_flat = onem && p.c.dtype.precision == p.comp_prec && can_flatten(p.c, ax);
      if (p.ctemp) {
        g.exact_mode = mdg::EXACT_FULL_THEN_COMBINE;
      } else if (p.ukr_path == UkrPath::Direct) {
        g.exact_mode = mdg::EXACT_DIRECT_SEEDED;
      } else if (onem_flat && p.beta.im == 0.0) {
        g.exact_mode = mdg::EXACT_DIRECT_SEEDED;
        g.epi.out = to_dview(real_flatten(p.c, ax));
        g.epi.pair = MDG_PAIR_NONE;
      } else if (onem_flat) {
        g.exact_mode = mdg::EXACT_ONEM_MIXED;
        g.flat = to_dview(real_flatten(p.c, ax));
      }
      prof::Scope scope(MDG_KERNEL_EXACT, st, 2.0 * p.m * p.n * p.k);
      err = mdg::launch_gemm_exact(g, single, sms, st);
    } else {
      const int kind = single ? MDG_KERNEL_FFMA : MDG_KERNEL_DMMA;
      const char* trace_path = std::getenv("MDGEMM_TRACE");  // tuning: per-CTA timeline of every gemm kernel
      const int64_t grid = dmma_ws ? ws_grid : sk_grid > 0 ? mdg::sk_launch_grid(tiles, sk_grid) : tiles * splits;
      if (trace_path && grid > 0 && err == cudaSuccess)
        err = ws_alloc(reinterpret_cast<void**>(&g.trace), grid * mdg::TRACE_WORDS * 8, st);
      {
        prof::Scope scope(kind, st, 2.0 * p.m * p.n * p.k);
        if (err == cudaSuccess)
          err = dmma_ws  ? (single ? mdg::launch_gemm_ffma_ws(g, ws_grid, st) : mdg::launch_gemm_dmma_ws(g, ws_grid, st))
                : single ? mdg::launch_gemm_ffma(g, tile, st)
                         : mdg::launch_gemm_dmma(g, tile, st);
      }
      if (g.trace) {
        std::vector<unsigned long long> h(static_cast<size_t>(grid) * mdg::TRACE_WORDS);
        if (err == cudaSuccess)
          err = cudaMemcpyAsync(h.data(), g.trace, h.size() * 8, cudaMemcpyDeviceToHost, st);
        if (err == cudaSuccess) err = cudaStreamSynchronize(st);
        cudaFreeAsync(g.trace, st);
        g.trace = nullptr;
        if (FILE* f = std::fopen(trace_path, "a")) {
          std::fprintf(f, "K %s %lld %lld %lld %d %d %d %lld\n", single ? "ffma" : "dmma", (long long)p.m,
                       (long long)p.n, (long long)p.k, tile.bm, tile.bn, splits, (long long)grid);
          for (int64_t b = 0; b < grid; ++b) {
            const unsigned long long* r = &h[static_cast<size_t>(b) * mdg::TRACE_WORDS];
            std::fprintf(f, "%llu %llu %llu %llu %llu %llu\n", r[0], r[1], r[2], r[3], r[4], r[5]);
          }
          std::fclose(f);
        }
      }
      if (err == cudaSuccess && splits > 1) {
        prof::Scope scope(kind, st, 0.0);  // same job: its time counts against the gemm's flops
        err = mdg::launch_splitk_reduce(g, tile, single, st);
      }
    }
  }
  const cudaError_t ferr = owned ? cudaFreeAsync(ws, st) : cudaSuccess;
  cuda_check(err, "gemm kernels");
  cuda_check(ferr, "workspace release");
  if (fc) fc->add(reference_flops(p));
}

// ---------------------------------------------------------------- dual-pipe jobs
bool dual_eligible(const ExecutionPlan& p, Numerics numerics) {
  if (numerics != Numerics::Fast || p.m <= 0 || p.n <= 0 || p.k <= 0) return false;
  if (fast_block_mode(p) != 0) return false;  // per-KC-block rounding into C: execute()
  if (p.c.dtype.domain == Domain::Complex && p.pair_axis == PairAxis::None) return false;
  const int64_t bm = p.comp_prec == Precision::Single ? mdg::DUAL_F_BM : mdg::DUAL_D_BM;
  const int64_t tiles = ((p.m + bm - 1) / bm) * ((p.n + mdg::DUAL_D_BN - 1) / mdg::DUAL_D_BN);
  return tiles < (int64_t{1} << 30);
}

DualPrep dual_prepare(const ExecutionPlan& p) {
  DualPrep d;
  d.single = p.comp_prec == Precision::Single;
  const int64_t bm = d.single ? mdg::DUAL_F_BM : mdg::DUAL_D_BM;
  const int64_t bn = d.single ? mdg::DUAL_F_BN : mdg::DUAL_D_BN;
  const int64_t bk = d.single ? mdg::DUAL_F_BK : mdg::DUAL_BK;
  d.lpad = (p.k + bk - 1) / bk * bk;
  // D jobs: panel lines at the dual kernel's conflict-free smem pitch, so a
  // stage stays one contiguous bulk copy per operand
  const int64_t pitch = d.single ? 0 : mdg::dual_d_pitch();
  const Packed pa =
      prepare_pack(p.a, Side::Left, p.format_a, p.conj_a, p.pack_scale_a, p.target_dtype_a, bm, d.lpad, pitch);
  const Packed pb =
      prepare_pack(p.b, Side::Right, p.format_b, p.conj_b, p.pack_scale_b, p.target_dtype_b, bn, d.lpad, pitch);
  d.pa = pa.desc;
  d.pb = pb.desc;
  d.bytes_a = pa.bytes;
  d.bytes_b = pb.bytes;
  d.off_b = (pa.bytes + 255) / 256 * 256;
  d.bytes = d.off_b + (pb.bytes + 255) / 256 * 256;
  d.tile_flops = 2.0 * static_cast<double>((p.m + bm - 1) / bm * bm) * static_cast<double>((p.n + bn - 1) / bn * bn) *
                 static_cast<double>(d.lpad);
  d.tiles = static_cast<int32_t>(((p.m + bm - 1) / bm) * ((p.n + bn - 1) / bn));
  return d;
}

void dual_describe(const ExecutionPlan& p, void* ws, mdg::DualJob* job, mdg::PackGroup* g, double* traffic) {
  const DualPrep d = dual_prepare(p);
  char* w = static_cast<char*>(ws);
  if (g->n + 2 > mdg::PACK_GROUP_MAX) throw Error("dual_describe: pack group full");
  g->d[g->n] = d.pa;
  g->dst[g->n++] = w;
  g->d[g->n] = d.pb;
  g->dst[g->n++] = w + d.off_b;
  if (traffic) *traffic += pack_traffic(p.a, d.bytes_a) + pack_traffic(p.b, d.bytes_b);
  const int64_t bm = d.single ? mdg::DUAL_F_BM : mdg::DUAL_D_BM;
  const int64_t bn = d.single ? mdg::DUAL_F_BN : mdg::DUAL_D_BN;
  *job = mdg::DualJob{};
  job->a = w;
  job->b = w + d.off_b;
  job->lpad = d.lpad;
  job->me = p.m;
  job->ne = p.n;
  job->out = to_dview(p.c);
  job->beta = to_dbeta(p.beta);
  job->pair = static_cast<int32_t>(p.pair_axis);
  job->tiles_m = static_cast<int32_t>((p.m + bm - 1) / bm);
  job->tiles_n = static_cast<int32_t>((p.n + bn - 1) / bn);
}

void dual_pack_group(mdg::PackGroup& g, double traffic, cudaStream_t st) {
  if (g.n == 0) return;
  prof::Scope scope(MDG_KERNEL_PACK, st, traffic);
  cuda_check(mdg::launch_pack_group(g, st), "pack kernel");
}

int dual_grid() {
  // One SM is left to the next launches' pack kernels: a dual CTA holds
  // every register of its SM, so without them those packs wait for the launch
  // to drain and the kernel stream idles while they run.  Measured on the cfg2
  // sweep (profiles/r02/dual_spare_sms.txt): 0 spare SMs -> 52,470 GFLOPS,
  // 1 -> 52,640, 2 -> 52,620, 4 -> 52,390 with two pack arenas; 2 spare SMs
  // with three arenas (staging.cpp: dual_arenas, the packs may run two
  // launches ahead) -> 52,710.  With the faster packs of the end of round 2
  // (vector / interior tiles) one spare SM is enough: 0 -> 53,280, 1 -> 53,520,
  // 2 -> 53,420, 3 -> 53,130 (profiles/r02/dual_spare_sms_vec.txt).
  // MDGEMM_DUAL_SPARE_SMS overrides.
  static const int spare = [] {
    const char* f = std::getenv("MDGEMM_DUAL_SPARE_SMS");
    return f ? std::max(0, std::atoi(f)) : 1;
  }();
  int dev_count = 0;
  const int sms = cudaGetDeviceCount(&dev_count) == cudaSuccess && dev_count > 0 ? device_sms() : 148;
  cudaGetLastError();
  return std::max(1, sms - spare);
}

void dual_launch(const mdg::DualDesc& desc, double flops_d, double flops_f, cudaStream_t st) {
  mdg::DualDesc& d = const_cast<mdg::DualDesc&>(desc);
  static const int prefetch = [] {  // tuning: MDGEMM_DUAL_PREFETCH = 0 turns the C L2 prefetch off
    const char* f = std::getenv("MDGEMM_DUAL_PREFETCH");
    return f ? std::atoi(f) : 1;
  }();
  d.prefetch_c = prefetch;
  static const int sleep_ns = [] {  // tuning: MDGEMM_DUAL_SLEEP = suspend hint in ns (0: spinning waits)
    const char* f = std::getenv("MDGEMM_DUAL_SLEEP");
    return f ? std::atoi(f) : 20000;
  }();
  d.sleep_ns = sleep_ns;
  prof::Scope scope(MDG_KERNEL_DUAL_D, st, flops_d, MDG_KERNEL_DUAL_F, flops_f);
  cuda_check(mdg::launch_gemm_dual(d, dual_grid(), st), "dual-pipe gemm kernel");
}

}  // namespace mdgemm
