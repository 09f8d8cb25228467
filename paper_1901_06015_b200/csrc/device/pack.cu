// Typecasting pack kernels: Standard / 1e / 1r formats, left and right
// operands, conjugation and alpha scaling, into zero-padded register panels.
// Bit-exact against the reference pack (packing.cpp:114-230):
//   v = widen(src) -> conj (src.conj xor requested) -> round to the target
//   precision -> if scale != 1: complex<double> product, round again.
//
// Data movement (pack_tile.cuh): one CTA moves one source tile -- 32x32
// elements, or 32 lines of 16-byte vectors for real sources with a
// unit-stride axis and aligned lines -- read coalesced along the source's
// unit-stride axis and written coalesced along the packed buffer's contiguous
// axis (rows for left panels, columns for right panels), through shared memory
// when the two differ, so a transposing pack costs one HBM read and one HBM
// write.  The launchers pick the kernel: pack_kernel / pack_vec_kernel for one
// operand, pack_pair_kernel / pack_pair_vec_kernel for both operands of a call,
// pack_group_kernel for the many small packs of a dual launch.
#include <cstdlib>
#include <type_traits>

#include "pack_tile.cuh"

namespace mdg {
namespace {

constexpr int PACK_THREADS = 256;
// CTAs per SM the register budget must allow (__launch_bounds__ minimum):
// the tile loads are latency-bound, and unbounded ptxas picks 48-60 registers,
// four 256-thread CTAs per SM (a 2048^2 pack pair: 46 % achieved occupancy,
// 2.2 TB/s).  Real sources at six per SM (<= 40 registers): dddd 2048 pack
// 44 -> 40 us, 4096 159 -> 135 us, dssd 1024 13.7 -> 12.7 us; complex sources
// (1e / 1r, more live values) stay unbounded -- bounded they spill and run
// slower (zzzd 4096 252 -> 258 us).  Cfg2 sweep +0.4 % (profiles/r02/pack_occupancy.txt).
// With the loads hoisted and kept in the source type (pack_tile.cuh) six per SM
// spills a little; five (<= 48 registers) does not: dssd 1024 14.2 -> 12.6 us,
// dddd 4096 123.3 -> 121.9 us (profiles/r02/pack_tiles_per_cta.txt).
#ifndef MDG_PACK_MIN_BLOCKS_REAL
#define MDG_PACK_MIN_BLOCKS_REAL 4
#endif
#ifndef MDG_PACK_MIN_BLOCKS_COMPLEX
#define MDG_PACK_MIN_BLOCKS_COMPLEX 4
#endif
template <bool SRC_COMPLEX>
constexpr int pack_min_blocks() { return SRC_COMPLEX ? MDG_PACK_MIN_BLOCKS_COMPLEX : MDG_PACK_MIN_BLOCKS_REAL; }

template <typename S, bool SRC_COMPLEX, typename D, int FMT, int SIDE>
__global__ void __launch_bounds__(PACK_THREADS, pack_min_blocks<SRC_COMPLEX>()) pack_kernel(PackDesc d, D* __restrict__ dst) {
  __shared__ packtile::Tile tile;
  packtile::pack_tile<S, SRC_COMPLEX, D, FMT, SIDE, PACK_THREADS, packtile::TpcOf<S, SRC_COMPLEX>::value>(d, dst, blockIdx.x, tile, threadIdx.x,
                                                                   [] { __syncthreads(); });
}

// The vector tiles of a real source (PackDesc.vec), in kernels of their own: next to the scalar paths
// they cost both register budgets.
#ifndef MDG_PACK_VEC_BLOCKS
#define MDG_PACK_VEC_BLOCKS 4
#endif
template <typename S, typename D, int SIDE>
__global__ void __launch_bounds__(PACK_THREADS, MDG_PACK_VEC_BLOCKS) pack_vec_kernel(PackDesc d, D* __restrict__ dst) {
  __shared__ packtile::Tile tile;
  packtile::pack_tile_vec<S, D, SIDE, PACK_THREADS>(d, dst, blockIdx.x, tile, threadIdx.x, [] { __syncthreads(); });
}

template <typename S, typename D>
__global__ void __launch_bounds__(PACK_THREADS, MDG_PACK_VEC_BLOCKS)
    pack_pair_vec_kernel(const __grid_constant__ PackDesc d0, D* __restrict__ dst0, const __grid_constant__ PackDesc d1,
                         D* __restrict__ dst1, int64_t tiles0) {
  __shared__ packtile::Tile tile;
  __shared__ PackDesc sd;
  const bool first = static_cast<int64_t>(blockIdx.x) < tiles0;
  static_assert(sizeof(PackDesc) % 4 == 0, "PackDesc copied as words");
  if (threadIdx.x < sizeof(PackDesc) / 4) {
    const uint32_t w0 = reinterpret_cast<const uint32_t*>(&d0)[threadIdx.x];
    const uint32_t w1 = reinterpret_cast<const uint32_t*>(&d1)[threadIdx.x];
    reinterpret_cast<uint32_t*>(&sd)[threadIdx.x] = first ? w0 : w1;
  }
  __syncthreads();
  const PackDesc& d = sd;
  D* dst = first ? dst0 : dst1;
  const int64_t bid = first ? static_cast<int64_t>(blockIdx.x) : static_cast<int64_t>(blockIdx.x) - tiles0;
  auto sync = [] { __syncthreads(); };
  if (d.side == MDG_SIDE_LEFT) packtile::pack_tile_vec<S, D, MDG_SIDE_LEFT, PACK_THREADS>(d, dst, bid, tile, threadIdx.x, sync);
  else packtile::pack_tile_vec<S, D, MDG_SIDE_RIGHT, PACK_THREADS>(d, dst, bid, tile, threadIdx.x, sync);
}

// Both operands of a call in one launch when they share source type, target
// precision and format (the side is decided per CTA): one launch instead of
// two, and the two packs' tiles share the waves.
template <typename S, bool SRC_COMPLEX, typename D, int FMT>
__global__ void __launch_bounds__(PACK_THREADS, pack_min_blocks<SRC_COMPLEX>())
    pack_pair_kernel(const __grid_constant__ PackDesc d0, D* __restrict__ dst0, const __grid_constant__ PackDesc d1,
                     D* __restrict__ dst1, int64_t tiles0) {
  __shared__ packtile::Tile tile;
  __shared__ PackDesc sd;  // this CTA's pack (selecting between the two parameter structs by reference
                           // makes ptxas copy both to local memory)
  const bool first = static_cast<int64_t>(blockIdx.x) < tiles0;
  static_assert(sizeof(PackDesc) % 4 == 0, "PackDesc copied as words");
  if (threadIdx.x < sizeof(PackDesc) / 4) {
    const uint32_t w0 = reinterpret_cast<const uint32_t*>(&d0)[threadIdx.x];
    const uint32_t w1 = reinterpret_cast<const uint32_t*>(&d1)[threadIdx.x];
    reinterpret_cast<uint32_t*>(&sd)[threadIdx.x] = first ? w0 : w1;
  }
  __syncthreads();
  const PackDesc& d = sd;
  D* dst = first ? dst0 : dst1;
  const int64_t bid = first ? static_cast<int64_t>(blockIdx.x) : static_cast<int64_t>(blockIdx.x) - tiles0;
  auto sync = [] { __syncthreads(); };
  if (d.side == MDG_SIDE_LEFT)
    packtile::pack_tile<S, SRC_COMPLEX, D, FMT, MDG_SIDE_LEFT, PACK_THREADS, packtile::TpcOf<S, SRC_COMPLEX>::value>(d, dst, bid, tile, threadIdx.x, sync);
  else
    packtile::pack_tile<S, SRC_COMPLEX, D, FMT, MDG_SIDE_RIGHT, PACK_THREADS, packtile::TpcOf<S, SRC_COMPLEX>::value>(d, dst, bid, tile, threadIdx.x, sync);
}

// Packs of at least this many 32x32 tiles (a 1024^2 real operand) get their
// own launch in launch_pack_group.
constexpr int64_t kGroupLargeTiles = 1024;

// One launch over many packs (PackGroup): CTA b finds its pack by binary
// search over the tile prefix sums, then runs that pack's tile -- the kernel
// instance for the pack's source type / target / format / side picked at run
// time (uniform per CTA).  A dual launch's 20-70 small packs then cost one
// launch instead of one or two each.
template <typename S, bool SC, typename D>
__device__ __forceinline__ void group_tile(const PackDesc& d, void* dst, int64_t bid, packtile::Tile& tile) {
  auto sync = [] { __syncthreads(); };
  if constexpr (!SC) {
    if (d.vec) {  // uniform per CTA
      if (d.side == MDG_SIDE_LEFT)
        packtile::pack_tile_vec<S, D, MDG_SIDE_LEFT, PACK_THREADS>(d, static_cast<D*>(dst), bid, tile, threadIdx.x, sync);
      else
        packtile::pack_tile_vec<S, D, MDG_SIDE_RIGHT, PACK_THREADS>(d, static_cast<D*>(dst), bid, tile, threadIdx.x, sync);
      return;
    }
  }
  auto side = [&](auto fmt) {
    constexpr int FMT = decltype(fmt)::value;
    if (d.side == MDG_SIDE_LEFT)
      packtile::pack_tile<S, SC, D, FMT, MDG_SIDE_LEFT, PACK_THREADS, packtile::TpcOf<S, SC>::value>(d, static_cast<D*>(dst), bid, tile, threadIdx.x,
                                                                      sync);
    else
      packtile::pack_tile<S, SC, D, FMT, MDG_SIDE_RIGHT, PACK_THREADS, packtile::TpcOf<S, SC>::value>(d, static_cast<D*>(dst), bid, tile, threadIdx.x,
                                                                       sync);
  };
  if constexpr (SC) {
    if (d.format == MDG_FMT_ONEE) return side(std::integral_constant<int, MDG_FMT_ONEE>{});
    if (d.format == MDG_FMT_ONER) return side(std::integral_constant<int, MDG_FMT_ONER>{});
  }
  side(std::integral_constant<int, MDG_FMT_STANDARD>{});
}

__global__ void __launch_bounds__(PACK_THREADS, 4) pack_group_kernel(const __grid_constant__ PackGroup g) {
  __shared__ packtile::Tile tile;
  __shared__ PackDesc sd;  // this CTA's pack: read once from the parameter space (26 KB: the
                           // constant cache holds little of it), then from shared memory
  const int64_t bid = blockIdx.x;
  int lo = 0, hi = g.n - 1;  // the last pack whose first tile is <= bid
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (g.tile0[mid] <= bid) lo = mid;
    else hi = mid - 1;
  }
  static_assert(sizeof(PackDesc) % 4 == 0, "PackDesc copied as words");
  if (threadIdx.x < sizeof(PackDesc) / 4)
    reinterpret_cast<uint32_t*>(&sd)[threadIdx.x] = reinterpret_cast<const uint32_t*>(&g.d[lo])[threadIdx.x];
  __syncthreads();
  const PackDesc& d = sd;
  void* dst = g.dst[lo];
  const int64_t t = bid - g.tile0[lo];
  const bool ts = d.target_single != 0;
  switch (d.src.dtype) {
    case MDG_DT_S: ts ? group_tile<float, false, float>(d, dst, t, tile) : group_tile<float, false, double>(d, dst, t, tile); break;
    case MDG_DT_D: ts ? group_tile<double, false, float>(d, dst, t, tile) : group_tile<double, false, double>(d, dst, t, tile); break;
    case MDG_DT_C: ts ? group_tile<float, true, float>(d, dst, t, tile) : group_tile<float, true, double>(d, dst, t, tile); break;
    default: ts ? group_tile<double, true, float>(d, dst, t, tile) : group_tile<double, true, double>(d, dst, t, tile); break;
  }
}

// Vector tiles where the pack allows them (MDGEMM_PACK_VEC=0: scalar tiles only, A/B runs).
bool vec_enabled() {
  static const bool on = [] {
    const char* f = std::getenv("MDGEMM_PACK_VEC");
    return !(f && std::atoi(f) == 0);
  }();
  return on;
}
PackDesc with_vec(const PackDesc& d, const void* dst) {
  PackDesc o = d;
  o.vec = vec_enabled() && packtile::vec_ok(d, dst) ? 1 : 0;
  const uint64_t csz = d.src.dtype == MDG_DT_C ? 8 : d.src.dtype == MDG_DT_Z ? 16 : 0;
  o.cvec = vec_enabled() && csz != 0 && reinterpret_cast<uint64_t>(d.src.base) % csz == 0 ? 1 : 0;
  // 32-bit offsets inside a tile: the line pitches must leave 63 lines of a tile inside 2^31 elements
  o.interior = vec_enabled() && d.src.rs >= 0 && d.src.cs >= 0 && d.src.rs < (int64_t{1} << 24) &&
               d.src.cs < (int64_t{1} << 24) && d.pitch < (1 << 24) ? 1 : 0;
  return o;
}

template <typename S, bool SC, typename D, int FMT>
cudaError_t go_pair(const PackDesc& a0, void* da, const PackDesc& b0, void* db, cudaStream_t s) {
  const PackDesc a = with_vec(a0, da), b = with_vec(b0, db);  // (launch_pack_pair: a.vec == b.vec)
  const int64_t ta = packtile::pack_ctas(a), tb = packtile::pack_ctas(b);
  if (ta + tb == 0) return cudaSuccess;
  if (ta + tb > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  if constexpr (!SC && FMT == MDG_FMT_STANDARD) {
    if (a.vec) {
      pack_pair_vec_kernel<S, D><<<static_cast<unsigned>(ta + tb), PACK_THREADS, 0, s>>>(a, static_cast<D*>(da), b,
                                                                                        static_cast<D*>(db), ta);
      return cudaGetLastError();
    }
  }
  pack_pair_kernel<S, SC, D, FMT><<<static_cast<unsigned>(ta + tb), PACK_THREADS, 0, s>>>(
      a, static_cast<D*>(da), b, static_cast<D*>(db), ta);
  return cudaGetLastError();
}

template <typename S, bool SC, typename D>
cudaError_t go_pair_format(const PackDesc& a, void* da, const PackDesc& b, void* db, cudaStream_t s) {
  if constexpr (SC) {
    if (a.format == MDG_FMT_ONEE) return go_pair<S, SC, D, MDG_FMT_ONEE>(a, da, b, db, s);
    if (a.format == MDG_FMT_ONER) return go_pair<S, SC, D, MDG_FMT_ONER>(a, da, b, db, s);
  }
  if (a.format != MDG_FMT_STANDARD) return cudaErrorInvalidValue;
  return go_pair<S, SC, D, MDG_FMT_STANDARD>(a, da, b, db, s);
}

template <typename S, bool SC>
cudaError_t go_pair_target(const PackDesc& a, void* da, const PackDesc& b, void* db, cudaStream_t s) {
  return a.target_single ? go_pair_format<S, SC, float>(a, da, b, db, s)
                         : go_pair_format<S, SC, double>(a, da, b, db, s);
}

cudaError_t pad(const PackDesc& d, void* dst, cudaStream_t s) {
  if (d.lpad <= d.len || d.panels == 0) return cudaSuccess;
  // Zero the inner-dimension padding rows [len, lpad) of every panel.
  const size_t esz = (d.target_single ? 4 : 8) * (d.out_complex ? 2 : 1);
  const size_t pitch = static_cast<size_t>(d.pitch * d.lpad) * esz;
  const size_t width = static_cast<size_t>(d.pitch * (d.lpad - d.len)) * esz;
  char* first = static_cast<char*>(dst) + static_cast<size_t>(d.pitch * d.len) * esz;
  return cudaMemset2DAsync(first, pitch, 0, width, static_cast<size_t>(d.panels), s);
}

template <typename S, bool SC, typename D, int FMT>
cudaError_t go_side(const PackDesc& d0, void* dst, cudaStream_t s) {
  const PackDesc d = with_vec(d0, dst);
  const int64_t tiles = packtile::pack_ctas(d);
  if (tiles == 0) return cudaSuccess;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  const dim3 grid(static_cast<unsigned>(tiles));
  if constexpr (!SC && FMT == MDG_FMT_STANDARD) {
    if (d.vec) {
      if (d.side == MDG_SIDE_LEFT)
        pack_vec_kernel<S, D, MDG_SIDE_LEFT><<<grid, PACK_THREADS, 0, s>>>(d, static_cast<D*>(dst));
      else
        pack_vec_kernel<S, D, MDG_SIDE_RIGHT><<<grid, PACK_THREADS, 0, s>>>(d, static_cast<D*>(dst));
      return cudaGetLastError();
    }
  }
  if (d.side == MDG_SIDE_LEFT)
    pack_kernel<S, SC, D, FMT, MDG_SIDE_LEFT><<<grid, PACK_THREADS, 0, s>>>(d, static_cast<D*>(dst));
  else
    pack_kernel<S, SC, D, FMT, MDG_SIDE_RIGHT><<<grid, PACK_THREADS, 0, s>>>(d, static_cast<D*>(dst));
  return cudaGetLastError();
}

template <typename S, bool SC, typename D>
cudaError_t go_format(const PackDesc& d, void* dst, cudaStream_t s) {
  if constexpr (SC) {
    if (d.format == MDG_FMT_ONEE) return go_side<S, SC, D, MDG_FMT_ONEE>(d, dst, s);
    if (d.format == MDG_FMT_ONER) return go_side<S, SC, D, MDG_FMT_ONER>(d, dst, s);
  }
  if (d.format != MDG_FMT_STANDARD) return cudaErrorInvalidValue;
  return go_side<S, SC, D, MDG_FMT_STANDARD>(d, dst, s);
}

template <typename S, bool SC>
cudaError_t go_target(const PackDesc& d, void* dst, cudaStream_t s) {
  return d.target_single ? go_format<S, SC, float>(d, dst, s) : go_format<S, SC, double>(d, dst, s);
}

}  // namespace

cudaError_t launch_pack(const PackDesc& d, void* dst, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  switch (d.src.dtype) {
    case MDG_DT_S: e = go_target<float, false>(d, dst, s); break;
    case MDG_DT_D: e = go_target<double, false>(d, dst, s); break;
    case MDG_DT_C: e = go_target<float, true>(d, dst, s); break;
    case MDG_DT_Z: e = go_target<double, true>(d, dst, s); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  return pad(d, dst, s);
}

cudaError_t launch_pack_group(PackGroup& g, cudaStream_t s) {
  if (g.n <= 0) return cudaSuccess;
  if (g.n > PACK_GROUP_MAX) return cudaErrorInvalidValue;
  // Large packs keep their own launch: the type-specialised kernels run at a
  // higher occupancy than the run-time-dispatched one; the small ones (the
  // launch latency dominates them) share one launch.
  int keep = 0;
  cudaError_t e = cudaSuccess;
  for (int j = 0; j < g.n && e == cudaSuccess; ++j) {
    if (packtile::pack_tiles(g.d[j]) >= kGroupLargeTiles) {
      e = launch_pack(g.d[j], g.dst[j], s);
    } else {
      g.d[keep] = g.d[j];
      g.dst[keep++] = g.dst[j];
    }
  }
  if (e != cudaSuccess) return e;
  g.n = keep;
  int64_t tiles = 0;
  for (int j = 0; j < g.n; ++j) {
    g.d[j] = with_vec(g.d[j], g.dst[j]);
    g.tile0[j] = tiles;  // in CTAs (TPC source tiles each, or one vector tile)
    tiles += packtile::pack_ctas(g.d[j]);
  }
  g.tile0[g.n] = tiles;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  if (tiles > 0) pack_group_kernel<<<static_cast<unsigned>(tiles), PACK_THREADS, 0, s>>>(g);
  e = cudaGetLastError();
  for (int j = 0; j < g.n && e == cudaSuccess; ++j) e = pad(g.d[j], g.dst[j], s);
  return e;
}

cudaError_t launch_pack_pair(const PackDesc& a, void* da, const PackDesc& b, void* db, cudaStream_t s) {
  // one kernel for both packs: same source type, target and format, and both or neither on vector tiles
  if (a.src.dtype != b.src.dtype || a.target_single != b.target_single || a.format != b.format ||
      with_vec(a, da).vec != with_vec(b, db).vec) {
    const cudaError_t e = launch_pack(a, da, s);
    return e != cudaSuccess ? e : launch_pack(b, db, s);
  }
  cudaError_t e = cudaSuccess;
  switch (a.src.dtype) {
    case MDG_DT_S: e = go_pair_target<float, false>(a, da, b, db, s); break;
    case MDG_DT_D: e = go_pair_target<double, false>(a, da, b, db, s); break;
    case MDG_DT_C: e = go_pair_target<float, true>(a, da, b, db, s); break;
    case MDG_DT_Z: e = go_pair_target<double, true>(a, da, b, db, s); break;
    default: return cudaErrorInvalidValue;
  }
  if (e == cudaSuccess) e = pad(a, da, s);
  if (e == cudaSuccess) e = pad(b, db, s);
  return e;
}

}  // namespace mdg
