// Typecasting pack kernels: Standard / 1e / 1r formats, left and right
// operands, conjugation and alpha scaling, into zero-padded register panels.
// Bit-exact against the reference pack (packing.cpp:114-230):
//   v = widen(src) -> conj (src.conj xor requested) -> round to the target
//   precision -> if scale != 1: complex<double> product, round again.
//
// Data movement: one CTA stages a 32x32 source tile in shared memory, read
// coalesced along the source's unit-stride axis and written coalesced along
// the packed buffer's contiguous axis (rows for left panels, columns for
// right panels), so a transposing pack costs one HBM read and one HBM write.
#include "common.cuh"

namespace mdg {
namespace {

constexpr int TILE = 32;
constexpr int PACK_THREADS = 256;

template <typename S, bool SRC_COMPLEX>
__device__ __forceinline__ double2 load_src(const DView& v, int64_t i, int64_t j) {
  const S* p = reinterpret_cast<const S*>(v.base) + (i * v.rs + j * v.cs) * (SRC_COMPLEX ? 2 : 1);
  if constexpr (SRC_COMPLEX) {
    return make_double2(static_cast<double>(p[0]), static_cast<double>(p[1]));
  } else {
    return make_double2(static_cast<double>(p[0]), 0.0);
  }
}

__device__ __forceinline__ double2 process(double2 v, const PackDesc& d) {
  if (d.do_conj) v.y = -v.y;
  const bool sp = d.target_single;
  double re = rnd(v.x, sp), im = rnd(v.y, sp);
  if (!d.unit_scale) {
    const double2 p = cmul(re, im, d.sre, d.sim);
    re = rnd(p.x, sp);
    im = rnd(p.y, sp);
  }
  return make_double2(re, im);
}

template <typename D>
struct Pair;
template <>
struct Pair<float> {
  using T = float2;
  static __device__ __forceinline__ T make(double a, double b) {
    return make_float2(static_cast<float>(a), static_cast<float>(b));
  }
};
template <>
struct Pair<double> {
  using T = double2;
  static __device__ __forceinline__ T make(double a, double b) { return make_double2(a, b); }
};

template <typename S, bool SRC_COMPLEX, typename D, int FMT, int SIDE>
__global__ void __launch_bounds__(PACK_THREADS) pack_kernel(PackDesc d, D* __restrict__ dst) {
  __shared__ double2 tile[TILE][TILE + 1];
  const int64_t tiles_i = (d.ext_i + TILE - 1) / TILE;
  const int64_t bid = blockIdx.x;
  const int64_t i0 = (bid % tiles_i) * TILE;
  const int64_t j0 = (bid / tiles_i) * TILE;
  const int t = threadIdx.x;
  const int lane = t & 31, row = t >> 5;

  // Load: coalesce along the source's unit-stride axis.
  const bool i_fast = d.src.rs <= d.src.cs;
#pragma unroll
  for (int r = 0; r < TILE / 8; ++r) {
    const int ii = i_fast ? lane : row + 8 * r;
    const int jj = i_fast ? row + 8 * r : lane;
    const int64_t i = i0 + ii, j = j0 + jj;
    double2 v = make_double2(0.0, 0.0);  // padded slots take literal zeros
    if (i < d.src.m && j < d.src.n) v = process(load_src<S, SRC_COMPLEX>(d.src, i, j), d);
    tile[jj][ii] = v;
  }
  __syncthreads();

  // Store: coalesce along the packed buffer's contiguous axis.
  const int64_t PD = d.pd, LP = d.lpad;
#pragma unroll
  for (int r = 0; r < TILE / 8; ++r) {
    const int ii = SIDE == MDG_SIDE_LEFT ? lane : row + 8 * r;
    const int jj = SIDE == MDG_SIDE_LEFT ? row + 8 * r : lane;
    const int64_t i = i0 + ii, j = j0 + jj;
    if (i >= d.ext_i || j >= d.ext_j) continue;
    const double2 v = tile[jj][ii];
    // offset of packed-logical (pr, pc) in block elements; power-of-two panel
    // dims (every kernel tile) avoid the 64-bit division per element
    const int sh = d.pd_shift;
    auto off = [&](int64_t pr, int64_t pc) -> int64_t {
      const int64_t x = SIDE == MDG_SIDE_LEFT ? pr : pc, y = SIDE == MDG_SIDE_LEFT ? pc : pr;
      if (sh >= 0) return ((x >> sh) * LP + y) * PD + (x & (PD - 1));
      return (x / PD) * PD * LP + y * PD + x % PD;
    };
    if constexpr (FMT == MDG_FMT_STANDARD) {
      if constexpr (SRC_COMPLEX) {
        reinterpret_cast<typename Pair<D>::T*>(dst)[off(i, j)] = Pair<D>::make(v.x, v.y);
      } else {
        dst[off(i, j)] = static_cast<D>(v.x);
      }
    } else if constexpr (FMT == MDG_FMT_ONEE) {
      using P = typename Pair<D>::T;
      if constexpr (SIDE == MDG_SIDE_LEFT) {
        // rows (2i, 2i+1) x cols (2j, 2j+1) = [[re, -im], [im, re]]
        *reinterpret_cast<P*>(dst + off(2 * i, 2 * j)) = Pair<D>::make(v.x, v.y);
        *reinterpret_cast<P*>(dst + off(2 * i, 2 * j + 1)) = Pair<D>::make(-v.y, v.x);
      } else {
        // rows (2i, 2i+1) x cols (2j, 2j+1) = [[re, im], [-im, re]]
        *reinterpret_cast<P*>(dst + off(2 * i, 2 * j)) = Pair<D>::make(v.x, v.y);
        *reinterpret_cast<P*>(dst + off(2 * i + 1, 2 * j)) = Pair<D>::make(-v.y, v.x);
      }
    } else {  // 1r
      if constexpr (SIDE == MDG_SIDE_LEFT) {
        dst[off(i, 2 * j)] = static_cast<D>(v.x);
        dst[off(i, 2 * j + 1)] = static_cast<D>(v.y);
      } else {
        dst[off(2 * i, j)] = static_cast<D>(v.x);
        dst[off(2 * i + 1, j)] = static_cast<D>(v.y);
      }
    }
  }
}

template <typename S, bool SC, typename D, int FMT>
cudaError_t go_side(const PackDesc& d, void* dst, cudaStream_t s) {
  const int64_t tiles = ((d.ext_i + TILE - 1) / TILE) * ((d.ext_j + TILE - 1) / TILE);
  if (tiles == 0) return cudaSuccess;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  const dim3 grid(static_cast<unsigned>(tiles));
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
  if (e != cudaSuccess || d.lpad <= d.len || d.panels == 0) return e;
  // Zero the inner-dimension padding rows [len, lpad) of every panel.
  const size_t esz = (d.target_single ? 4 : 8) * (d.out_complex ? 2 : 1);
  const size_t pitch = static_cast<size_t>(d.pd * d.lpad) * esz;
  const size_t width = static_cast<size_t>(d.pd * (d.lpad - d.len)) * esz;
  char* first = static_cast<char*>(dst) + static_cast<size_t>(d.pd * d.len) * esz;
  return cudaMemset2DAsync(first, pitch, 0, width, static_cast<size_t>(d.panels), s);
}

}  // namespace mdg
