// The tiles of a typecasting pack (Standard / 1e / 1r, left or right panels,
// conjugation, alpha scaling) -- the bodies of pack.cu's kernels.  Bit-exact
// against the reference pack (packing.cpp:114-230):
//   v = widen(src) -> conj (src.conj xor requested) -> round to the target
//   precision -> if scale != 1: complex<double> product, round again.
// Three bodies share that element pipeline (process_typed) and the panel
// layout (put_packed's offsets), so their packed bytes are identical:
//   pack_tile           a 32x32 source tile, any strides, any extents (bounds
//                       tests, padding, 64-bit index arithmetic);
//   pack_tile_interior  the same tile when it lies inside the source and its
//                       panel-axis indices share a panel: no tests, 32-bit
//                       offsets from one 64-bit origin per side;
//   pack_tile_vec       real sources with a unit-stride axis and 16-byte
//                       aligned lines: 32 lines x 32 V elements in 8- / 16-byte
//                       vectors.
// A tile is read coalesced along the source's unit-stride axis and written
// coalesced along the packed panels' contiguous axis, through shared memory
// when the two differ.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace mdg {
namespace packtile {

constexpr int TILE = 32;
using Tile = double2[TILE][TILE + 1];

// A source element as loaded (its own type: a thread keeps several loads in
// flight, and a float costs one register where the widened pair costs four).
template <typename S, bool SRC_COMPLEX>
struct Raw {
  S re, im;
};
template <typename S>
struct Raw<S, false> {
  S re;
};

template <typename S, bool SRC_COMPLEX>
__device__ __forceinline__ Raw<S, SRC_COMPLEX> load_raw(const DView& v, int64_t i, int64_t j, bool cvec) {
  const S* p = reinterpret_cast<const S*>(v.base) + (i * v.rs + j * v.cs) * (SRC_COMPLEX ? 2 : 1);
  if constexpr (SRC_COMPLEX) {
    if (cvec) {  // the base is aligned to the complex element (uniform per launch): one load
      using V = typename std::conditional<sizeof(S) == 4, float2, double2>::type;
      const V q = *reinterpret_cast<const V*>(p);
      return Raw<S, true>{q.x, q.y};
    }
    return Raw<S, true>{p[0], p[1]};  // a complex element is only guaranteed the alignment of its real type
  } else {
    return Raw<S, false>{p[0]};
  }
}

template <typename S, bool SRC_COMPLEX>
__device__ __forceinline__ double2 widen(const Raw<S, SRC_COMPLEX>& r) {
  if constexpr (SRC_COMPLEX) {
    return make_double2(static_cast<double>(r.re), static_cast<double>(r.im));
  } else {
    return make_double2(static_cast<double>(r.re), 0.0);
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

// The element pipeline on a loaded element, result in the target type.  With
// a unit scale the pipeline is widen -> conj -> round to the target: one
// conversion of the source value (none when the types agree) gives the same
// bits, and a float -> float pack no longer spends four F2F conversions per
// element on a round trip through double.
template <typename S, bool SRC_COMPLEX, typename D>
__device__ __forceinline__ typename Pair<D>::T process_typed(const Raw<S, SRC_COMPLEX>& r, const PackDesc& d) {
  if (d.unit_scale) {  // uniform per launch
    typename Pair<D>::T o;
    o.x = static_cast<D>(r.re);
    if constexpr (SRC_COMPLEX) {
      const D im = static_cast<D>(r.im);
      o.y = d.do_conj ? -im : im;
    } else {
      o.y = d.do_conj ? -D(0) : D(0);
    }
    return o;
  }
  const double2 v = process(widen<S, SRC_COMPLEX>(r), d);
  return Pair<D>::make(v.x, v.y);
}

// Store one processed source element (i, j) -- packed-logical row / column
// of the block -- in the panel layout of FMT / SIDE.
template <typename D, bool SRC_COMPLEX, int FMT, int SIDE>
__device__ __forceinline__ void put_packed(const PackDesc& d, D* __restrict__ dst, int64_t i, int64_t j,
                                           typename Pair<D>::T v) {
  const int64_t PD = d.pd, LP = d.lpad, PT = d.pitch;
  // offset of packed-logical (pr, pc) in block elements; power-of-two panel
  // dims (every kernel tile) avoid the 64-bit division per element
  const int sh = d.pd_shift;
  auto off = [&](int64_t pr, int64_t pc) -> int64_t {
    const int64_t x = SIDE == MDG_SIDE_LEFT ? pr : pc, y = SIDE == MDG_SIDE_LEFT ? pc : pr;
    const int64_t o = sh >= 0 ? ((x >> sh) * LP + y) * PT + (x & (PD - 1)) : (x / PD) * PT * LP + y * PT + x % PD;
    MDG_CHECK(o >= 0 && o < d.panels * LP * PT && y < LP, "packed offset outside the panels");
    return o;
  };
  if constexpr (FMT == MDG_FMT_STANDARD) {
    if constexpr (SRC_COMPLEX) {
      reinterpret_cast<typename Pair<D>::T*>(dst)[off(i, j)] = v;
    } else {
      dst[off(i, j)] = v.x;
    }
  } else if constexpr (FMT == MDG_FMT_ONEE) {
    using P = typename Pair<D>::T;
    if constexpr (SIDE == MDG_SIDE_LEFT) {
      // rows (2i, 2i+1) x cols (2j, 2j+1) = [[re, -im], [im, re]]
      *reinterpret_cast<P*>(dst + off(2 * i, 2 * j)) = v;
      *reinterpret_cast<P*>(dst + off(2 * i, 2 * j + 1)) = P{-v.y, v.x};
    } else {
      // rows (2i, 2i+1) x cols (2j, 2j+1) = [[re, im], [-im, re]]
      *reinterpret_cast<P*>(dst + off(2 * i, 2 * j)) = v;
      *reinterpret_cast<P*>(dst + off(2 * i + 1, 2 * j)) = P{-v.y, v.x};
    }
  } else {  // 1r
    if constexpr (SIDE == MDG_SIDE_LEFT) {
      dst[off(i, 2 * j)] = v.x;
      dst[off(i, 2 * j + 1)] = v.y;
    } else {
      dst[off(2 * i, j)] = v.x;
      dst[off(2 * i + 1, j)] = v.y;
    }
  }
}

// A scalar tile that lies inside the source (no padding, no edge) and whose 32 panel-axis indices fall
// into one panel: no bounds tests, one 64-bit tile origin per side and
// 32-bit offsets inside the tile.  (ncu of the c -> s pack pair of a 4096^2 call: ALU pipe 61 % busy, issue
// slots 65 %, DRAM 35 % -- the packs of 4- and 8-byte elements were bound by their index arithmetic.)
// Same loads, same element pipeline, same stores as pack_tile's general path.
template <typename S, bool SRC_COMPLEX, typename D, int FMT, int SIDE, int NT, class Sync>
__device__ __forceinline__ void pack_tile_interior(const PackDesc& d, D* __restrict__ dst, int64_t ti0, int64_t tj0,
                                                   Tile& tile, int t, Sync sync) {
  constexpr int ROWS = NT / 32, PER = TILE / ROWS;
  constexpr int NC = SRC_COMPLEX ? 2 : 1;
  constexpr int FX = FMT == MDG_FMT_ONEE ? 2 : 1;      // packed units per source index along the panel axis
  constexpr int FY = FMT == MDG_FMT_STANDARD ? 1 : 2;  // ... along the panel lines
  using P = typename Pair<D>::T;
  const int lane = t & 31, row = t >> 5;
  const bool i_fast = d.src.rs <= d.src.cs;
  const int64_t sc = i_fast ? d.src.rs : d.src.cs, sl = i_fast ? d.src.cs : d.src.rs;  // strides along the lanes / the lines
  const S* sp = reinterpret_cast<const S*>(d.src.base) + (ti0 * d.src.rs + tj0 * d.src.cs) * NC;
  const bool cvec = d.cvec != 0;
  Raw<S, SRC_COMPLEX> raw[PER];
#pragma unroll
  for (int r = 0; r < PER; ++r) {
    const S* p = sp + (lane * sc + (row + ROWS * r) * sl) * NC;
    if constexpr (SRC_COMPLEX) {
      if (cvec) {
        using V = typename std::conditional<sizeof(S) == 4, float2, double2>::type;
        const V q = *reinterpret_cast<const V*>(p);
        raw[r] = Raw<S, true>{q.x, q.y};
      } else {
        raw[r] = Raw<S, true>{p[0], p[1]};
      }
    } else {
      raw[r] = Raw<S, false>{p[0]};
    }
  }
  // packed origin of the tile: panel-axis index x0, line y0
  const int64_t x0 = FX * (SIDE == MDG_SIDE_LEFT ? ti0 : tj0), y0 = FY * (SIDE == MDG_SIDE_LEFT ? tj0 : ti0);
  const int PT = d.pitch;
  const int64_t tb = ((x0 >> d.pd_shift) * d.lpad + y0) * PT + (x0 & (d.pd - 1));
  MDG_CHECK(tb >= 0 && tb + (FY * TILE - 1) * static_cast<int64_t>(PT) + FX * TILE - 1 < d.panels * d.lpad * PT &&
                y0 + FY * TILE <= d.lpad,
            "packed tile outside the panels (interior tile)");
  // element (a, b) of the tile: a along the panel axis, b along the lines
  auto put = [&](int a, int b, P v) {
    const int loc = FY * b * PT + FX * a;
    if constexpr (FMT == MDG_FMT_STANDARD) {
      if constexpr (SRC_COMPLEX) reinterpret_cast<P*>(dst)[tb + loc] = v;
      else dst[tb + loc] = v.x;
    } else if constexpr (FMT == MDG_FMT_ONEE) {
      *reinterpret_cast<P*>(dst + tb + loc) = v;
      *reinterpret_cast<P*>(dst + tb + loc + PT) = P{-v.y, v.x};
    } else {
      dst[tb + loc] = v.x;
      dst[tb + loc + PT] = v.y;
    }
  };
  if (i_fast == (SIDE == MDG_SIDE_LEFT)) {  // the source's unit-stride axis is the panel axis
#pragma unroll
    for (int r = 0; r < PER; ++r) put(lane, row + ROWS * r, process_typed<S, SRC_COMPLEX, D>(raw[r], d));
    return;
  }
  P(*st)[TILE + 1] = reinterpret_cast<P(*)[TILE + 1]>(&tile[0][0]);
#pragma unroll
  for (int r = 0; r < PER; ++r) st[lane][row + ROWS * r] = process_typed<S, SRC_COMPLEX, D>(raw[r], d);
  sync();
#pragma unroll
  for (int r = 0; r < PER; ++r) put(lane, row + ROWS * r, st[row + ROWS * r][lane]);
}

// Source tiles TPC * bid .. TPC * bid + TPC - 1 (source tiles column-major over
// ext_i x ext_j) by NT threads (thread t of NT); sync() separates the staging
// from the stores.  The thread issues all its loads, kept in the source's own
// type, before it converts or stages anything (the transposing path used to
// convert and stage each element as it arrived: zzzd 4096 packs 252 -> 221 us,
// dddd 4096 135 -> 124 us).  When the
// source's unit-stride axis is the packed panels' contiguous axis (a left
// pack of a column-major A, a right pack of a row-major B) the tile needs no
// transpose: each element goes straight from its load to its store, both
// coalesced, with no shared-memory round trip or barrier.
template <typename S, bool SRC_COMPLEX, typename D, int FMT, int SIDE, int NT, int TPC, class Sync>
__device__ __forceinline__ void pack_tile(const PackDesc& d, D* __restrict__ dst, int64_t bid, Tile& tile, int t,
                                          Sync sync) {
  constexpr int ROWS = NT / 32;  // warps: tile rows per pass
  constexpr int PER = TILE / ROWS;
  const int64_t tiles_i = (d.ext_i + TILE - 1) / TILE;
  const int64_t tiles = tiles_i * ((d.ext_j + TILE - 1) / TILE);
  if constexpr (TPC == 1) {
    constexpr int FX = FMT == MDG_FMT_ONEE ? 2 : 1;
    const int64_t ti0 = (bid % tiles_i) * TILE, tj0 = (bid / tiles_i) * TILE;
    if (bid < tiles && ti0 + TILE <= d.src.m && tj0 + TILE <= d.src.n &&
        d.pd_shift >= 5 + (FX == 2 ? 1 : 0) && d.interior) {  // uniform per CTA
      pack_tile_interior<S, SRC_COMPLEX, D, FMT, SIDE, NT>(d, dst, ti0, tj0, tile, t, sync);
      return;
    }
  }
  const int lane = t & 31, row = t >> 5;
  const bool i_fast = d.src.rs <= d.src.cs;
  int64_t i0[TPC], j0[TPC];
#pragma unroll
  for (int u = 0; u < TPC; ++u) {
    const int64_t tb = bid * TPC + u;  // past the last tile: no element passes the extent tests below
    i0[u] = tb < tiles ? (tb % tiles_i) * TILE : d.ext_i;
    j0[u] = tb < tiles ? (tb / tiles_i) * TILE : d.ext_j;
  }
  // all of the thread's loads in flight before the first store (or staging)
  Raw<S, SRC_COMPLEX> raw[TPC][PER];
#pragma unroll
  for (int u = 0; u < TPC; ++u)
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const int ii = i_fast ? lane : row + ROWS * r;
      const int jj = i_fast ? row + ROWS * r : lane;
      const int64_t i = i0[u] + ii, j = j0[u] + jj;
      raw[u][r] = Raw<S, SRC_COMPLEX>{};
      if (i < d.src.m && j < d.src.n) raw[u][r] = load_raw<S, SRC_COMPLEX>(d.src, i, j, d.cvec != 0);
    }

  if (i_fast == (SIDE == MDG_SIDE_LEFT)) {  // no transpose (uniform per launch)
#pragma unroll
    for (int u = 0; u < TPC; ++u)
#pragma unroll
      for (int r = 0; r < PER; ++r) {
        const int ii = i_fast ? lane : row + ROWS * r;
        const int jj = i_fast ? row + ROWS * r : lane;
        const int64_t i = i0[u] + ii, j = j0[u] + jj;
        if (i >= d.ext_i || j >= d.ext_j) continue;
        // padded slots take literal zeros (not processed: the reference pads with +0 / -0 as stored)
        const typename Pair<D>::T v =
            (i < d.src.m && j < d.src.n) ? process_typed<S, SRC_COMPLEX, D>(raw[u][r], d) : typename Pair<D>::T{D(0), D(0)};
        put_packed<D, SRC_COMPLEX, FMT, SIDE>(d, dst, i, j, v);
      }
    return;
  }

  // the staging tile in the target type
  typename Pair<D>::T(*st)[TILE + 1] = reinterpret_cast<typename Pair<D>::T(*)[TILE + 1]>(&tile[0][0]);
#pragma unroll
  for (int u = 0; u < TPC; ++u) {
    if (bid * TPC + u >= tiles) break;  // uniform per CTA
    if (u > 0) sync();                  // the previous tile's stores have read the staging tile
    // Stage: the loads were coalesced along the source's unit-stride axis.
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const int ii = i_fast ? lane : row + ROWS * r;
      const int jj = i_fast ? row + ROWS * r : lane;
      const int64_t i = i0[u] + ii, j = j0[u] + jj;
      // padded slots take literal zeros
      st[jj][ii] = (i < d.src.m && j < d.src.n) ? process_typed<S, SRC_COMPLEX, D>(raw[u][r], d) : typename Pair<D>::T{D(0), D(0)};
    }
    sync();
    // Store: coalesce along the packed buffer's contiguous axis.
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const int ii = SIDE == MDG_SIDE_LEFT ? lane : row + ROWS * r;
      const int jj = SIDE == MDG_SIDE_LEFT ? row + ROWS * r : lane;
      const int64_t i = i0[u] + ii, j = j0[u] + jj;
      if (i >= d.ext_i || j >= d.ext_j) continue;
      put_packed<D, SRC_COMPLEX, FMT, SIDE>(d, dst, i, j, st[jj][ii]);
    }
  }
}

// ---------------------------------------------------------------- vector tiles
// Real sources with a unit-stride axis and 16-byte aligned lines (vec_ok) move
// in vectors: a tile is 32 lines of 32 V contiguous source elements (V = 16
// bytes / the wider of the source and target element), every thread loads
// four vectors before anything else and stores vectors of up to 16 bytes.
// Same element pipeline (process), so the packed bytes are those of pack_tile.
// Scalar tiles left a 2048^2 float pack pair at 1.9 TB/s: 4-byte loads, four
// per thread, are too few bytes in flight.
template <typename S, typename D>
struct VecGeom {
  static constexpr int V = 16 / (sizeof(S) > sizeof(D) ? sizeof(S) : sizeof(D));  // source elements per load
  static constexpr int W = 16 / sizeof(D);                                        // target elements per transposed store
  static constexpr int CW = TILE * V;                                             // tile width along the contiguous axis
};

template <int BYTES>
struct VecWord;
template <>
struct VecWord<16> {
  using T = uint4;
};
template <>
struct VecWord<8> {
  using T = uint2;
};

// Host and device: can the pack use vector tiles?  (dst: the packed block.)
__host__ __device__ inline bool vec_ok(const PackDesc& d, const void* dst) {
  if (d.src.dtype != MDG_DT_S && d.src.dtype != MDG_DT_D) return false;
  if (d.format != MDG_FMT_STANDARD || d.out_complex || d.pd_shift < 2) return false;
  const int ssz = d.src.dtype == MDG_DT_S ? 4 : 8, dsz = d.target_single ? 4 : 8;
  const int64_t ld = d.src.rs == 1 ? d.src.cs : d.src.rs;
  if (d.src.rs != 1 && d.src.cs != 1) return false;
  if (d.src.rs == 1 && d.src.cs == 1) return false;
  if (ld < 0 || (ld * ssz) % 16 != 0) return false;
  if (reinterpret_cast<uint64_t>(d.src.base) % 16 != 0 || reinterpret_cast<uint64_t>(dst) % 16 != 0) return false;
  if ((static_cast<int64_t>(d.pitch) * dsz) % 16 != 0) return false;
  return true;
}

template <typename S, typename D>
__host__ __device__ inline int64_t vec_tiles(const PackDesc& d) {
  constexpr int CW = VecGeom<S, D>::CW;
  const bool i_fast = d.src.rs == 1;
  const int64_t ext_c = i_fast ? d.ext_i : d.ext_j, ext_l = i_fast ? d.ext_j : d.ext_i;
  return ((ext_c + CW - 1) / CW) * ((ext_l + TILE - 1) / TILE);
}

// INSIDE: the tile lies inside the source (no edge, no padding): no bounds tests.
template <bool INSIDE, typename S, typename D, int SIDE, int NT, class Sync>
__device__ __forceinline__ void pack_tile_vec_body(const PackDesc& d, D* __restrict__ dst, int64_t c0, int64_t l0,
                                                   Tile& tile_mem, int t, Sync sync) {
  using G = VecGeom<S, D>;
  constexpr int V = G::V, W = G::W, CW = G::CW;
  constexpr int ROWS = NT / 32, PER = TILE / ROWS;
  static_assert(sizeof(Tile) >= sizeof(D) * CW * (TILE + 1), "staging tile");
  const bool i_fast = d.src.rs == 1;  // the source's contiguous axis c is i (else j); l is the other axis
  const int64_t ext_c = i_fast ? d.ext_i : d.ext_j, ext_l = i_fast ? d.ext_j : d.ext_i;
  const int64_t src_c = i_fast ? d.src.m : d.src.n, src_l = i_fast ? d.src.n : d.src.m;
  const int64_t ld = i_fast ? d.src.cs : d.src.rs;
  const int lane = t & 31, row = t >> 5;
  const int64_t LP = d.lpad, PT = d.pitch;
  const int sh = d.pd_shift;
  // packed offset of (x, y): x along the panel axis, y the line; xpart(x) + y * PT
  auto xpart = [&](int64_t x) -> int64_t { return (x >> sh) * LP * PT + (x & (d.pd - 1)); };
  auto checked = [&](int64_t o, int64_t y) -> int64_t {
    MDG_CHECK(o >= 0 && o < d.panels * LP * PT && y < LP, "packed offset outside the panels (vector tile)");
    return o;
  };

  // all loads first: vector (c, l) = source elements c .. c + V - 1 of line l
  using LW = typename VecWord<V * sizeof(S)>::T;
  union RawVec {
    LW w;
    S e[V];
  };
  RawVec raw[PER];
  const int64_t c = c0 + lane * V;
  const S* colp = reinterpret_cast<const S*>(d.src.base) + c + (l0 + row) * ld;
#pragma unroll
  for (int r = 0; r < PER; ++r) {
    const S* p = colp + static_cast<int64_t>(ROWS * r) * ld;
    if constexpr (INSIDE) {
      raw[r].w = *reinterpret_cast<const LW*>(p);
    } else {
      const int64_t l = l0 + row + ROWS * r;
#pragma unroll
      for (int v = 0; v < V; ++v) raw[r].e[v] = S(0);
      if (l < src_l && c < src_c) {
        if (c + V <= src_c) {
          raw[r].w = *reinterpret_cast<const LW*>(p);
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v)
            if (c + v < src_c) raw[r].e[v] = p[v];
        }
      }
    }
  }
  // element (c + v, l) of the source index space: processed inside the source, a literal zero in the padding
  auto value = [&](int r, int v) -> D {
    if constexpr (!INSIDE) {
      const int64_t l = l0 + row + ROWS * r;
      if (!(l < src_l && c + v < src_c)) return D(0);
    }
    return process_typed<S, false, D>(Raw<S, false>{raw[r].e[v]}, d).x;
  };

  if (i_fast == (SIDE == MDG_SIDE_LEFT)) {  // c is the panel axis: vector in, vector out
    using OW = typename VecWord<V * sizeof(D)>::T;
    union OutVec {
      OW w;
      D e[V];
    };
    const int64_t cb = xpart(c) + (l0 + row) * PT;
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const int64_t l = l0 + row + ROWS * r;
      if constexpr (!INSIDE)
        if (c >= ext_c || l >= ext_l) continue;  // ext_c is a multiple of the panel dim: whole vectors
      OutVec o;
#pragma unroll
      for (int v = 0; v < V; ++v) o.e[v] = value(r, v);
      *reinterpret_cast<OW*>(dst + checked(cb + static_cast<int64_t>(ROWS * r) * PT, l)) = o.w;
    }
    return;
  }

  // c is the panels' line axis, l the panel axis: stage [c][l] (row lane + 32 v holds c = lane V + v:
  // conflict-free scalar writes), then each thread gathers W consecutive l of one c and stores 16 bytes
  constexpr int P = TILE + 1;
  D* st = reinterpret_cast<D*>(&tile_mem[0][0]);
#pragma unroll
  for (int r = 0; r < PER; ++r)
#pragma unroll
    for (int v = 0; v < V; ++v) st[(v * 32 + lane) * P + row + ROWS * r] = value(r, v);
  sync();
  using SW = typename VecWord<W * sizeof(D)>::T;
  union StVec {
    SW w;
    D e[W];
  };
  constexpr int VPR = TILE / W;   // store vectors per staged row
  constexpr int NVEC = CW * VPR;  // per tile
  static_assert(NVEC % NT == 0 && NT % VPR == 0, "whole passes, one l-vector per thread");
  const int lv = t % VPR;  // the thread's l-vector is the same in every pass
  const int64_t x = l0 + lv * W;
  if constexpr (!INSIDE)
    if (x >= ext_l) return;  // ext_l is a multiple of the panel dim: whole vectors
  const int64_t xb = xpart(x) + c0 * PT;
#pragma unroll
  for (int q = 0; q < NVEC / NT; ++q) {
    const int srow = t / VPR + (NT / VPR) * q;  // staged row srow = v * 32 + lane'
    const int cc = (srow & 31) * V + (srow >> 5);
    if constexpr (!INSIDE)
      if (c0 + cc >= ext_c) continue;
    StVec o;
#pragma unroll
    for (int w = 0; w < W; ++w) o.e[w] = st[srow * P + lv * W + w];
    *reinterpret_cast<SW*>(dst + checked(xb + static_cast<int64_t>(cc) * PT, c0 + cc)) = o.w;
  }
}

template <typename S, typename D, int SIDE, int NT, class Sync>
__device__ __forceinline__ void pack_tile_vec(const PackDesc& d, D* __restrict__ dst, int64_t bid, Tile& tile_mem, int t,
                                              Sync sync) {
  constexpr int CW = VecGeom<S, D>::CW;
  const bool i_fast = d.src.rs == 1;
  const int64_t ext_c = i_fast ? d.ext_i : d.ext_j;
  const int64_t src_c = i_fast ? d.src.m : d.src.n, src_l = i_fast ? d.src.n : d.src.m;
  const int64_t tiles_c = (ext_c + CW - 1) / CW;
  const int64_t c0 = (bid % tiles_c) * CW, l0 = (bid / tiles_c) * TILE;
  if (c0 + CW <= src_c && l0 + TILE <= src_l)  // uniform per CTA
    pack_tile_vec_body<true, S, D, SIDE, NT>(d, dst, c0, l0, tile_mem, t, sync);
  else
    pack_tile_vec_body<false, S, D, SIDE, NT>(d, dst, c0, l0, tile_mem, t, sync);
}

// Source tiles of a pack (the grid of pack.cu's kernels).
__host__ __device__ inline int64_t pack_tiles(const PackDesc& d) {
  return ((d.ext_i + TILE - 1) / TILE) * ((d.ext_j + TILE - 1) / TILE);
}

// Source tiles per CTA, and the CTAs of a pack.  Measured on B200
// (profiles/r02/pack_tiles_per_cta.txt): one tile per CTA with its loads
// hoisted beats two or four -- a fat CTA's staging / store phases no longer
// overlap other CTAs' loads, and its index state spills at the six-CTA
// register bound (dddd 4096 pack pair 124 / 148 / 154 us at 1 / 2 / 4).
#ifndef MDG_PACK_TPC
#define MDG_PACK_TPC 1
#endif
#ifndef MDG_PACK_TPC_C
#define MDG_PACK_TPC_C 1
#endif
// per source type: complex single sources (8-byte elements) may take their own count
template <typename S, bool SRC_COMPLEX>
struct TpcOf {
  static constexpr int value = SRC_COMPLEX && sizeof(S) == 4 ? MDG_PACK_TPC_C : MDG_PACK_TPC;
};
__host__ __device__ inline int64_t pack_ctas(const PackDesc& d) {
  if (d.vec) {
    const bool ss = d.src.dtype == MDG_DT_S, ts = d.target_single != 0;
    return ss ? (ts ? vec_tiles<float, float>(d) : vec_tiles<float, double>(d))
              : (ts ? vec_tiles<double, float>(d) : vec_tiles<double, double>(d));
  }
  const int tpc = d.src.dtype == MDG_DT_C ? MDG_PACK_TPC_C : MDG_PACK_TPC;
  return (pack_tiles(d) + tpc - 1) / tpc;
}

}  // namespace packtile
}  // namespace mdg
