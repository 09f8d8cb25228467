// FAST numerics, computation precision double: warp-specialised persistent
// variant of the DMMA kernel (gemm_dmma.cu), one CTA per SM.
//
//   warps 0-7  MMA: one 128x128 tile cooperatively (64x32 warp tiles of
//              DMMA.8x8x4), two warps per SM sub-partition (one warp per
//              sub-partition reaches only ~65 % of the DMMA rate, measured
//              by `tools/peaks 10 occ`);
//   warp  8    producer: one lane streams 16-deep A/B slabs with TMA bulk
//              copies into a STAGES-deep ring;
//   warp  9    C mover: one lane moves C through a tile-sized buffer in C's
//              storage precision with 2-D TMA tensor copies -- it loads the
//              NEXT tile's C while the MMA warps run that tile's mainloop,
//              and stores each finished tile.
//
// After its mainloop the MMA warps combine their accumulators with the C
// tile already in shared memory (accumulate_element, kernels.cpp:79-95, via
// combine_typed -- the same arithmetic as the classic epilogue) and write the
// result in place; the C mover stores it and immediately loads the next C.
// So the C traffic of a tile overlaps the next tile's mainloop, and the MMA
// warps' epilogue is a pass over shared memory.  mbarriers: c_full (C tile
// landed, or nothing to load when beta = 0) and res_full (results written).
//
// Each CTA walks tiles blockIdx + w * gridDim (wave-major, so concurrently
// running CTAs share panels in L2); with d.sk_grid the partial last wave is
// shared as stream-K ranges whose split tiles are finished by SEEDING the
// next CTA's accumulators (common.cuh), so every element's rounding sequence
// -- and the result, bitwise -- is the classic kernel's.  One CTA per SM
// also means no co-resident CTA competes for issue slots: CTAs progress in
// step and the static schedule stays balanced.  Requires a column-major,
// 16-byte aligned C (a TMA tensor map, d.epi.cmap_ok); the driver keeps the
// classic kernel otherwise.
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace mdg {
namespace {

constexpr int WS_BM = 128, WS_BN = 128, WS_BK = 16;
constexpr int WS_WM = 2, WS_WN = 4;  // 8 MMA warps, 64x32 warp tiles
constexpr int WS_MMA_WARPS = WS_WM * WS_WN;
constexpr int WS_MMA_THREADS = WS_MMA_WARPS * 32;
constexpr int WS_PROD_WARP = WS_MMA_WARPS;
constexpr int WS_CMOV_WARP = WS_MMA_WARPS + 1;
constexpr int WS_THREADS = (WS_MMA_WARPS + 2) * 32;
constexpr int WS_MT = 8, WS_NT = 4;
constexpr int WS_STAGE_A = WS_BK * WS_BM, WS_STAGE_B = WS_BK * WS_BN;  // doubles

template <int CDT>
struct WsCfg {
  using O = OutType<CDT>;
  static constexpr int ESZR = O::kSingle ? 4 : 8;                   // bytes per real element of C
  static constexpr size_t CTILE = size_t(WS_BM) * WS_BN * ESZR;     // 64 / 128 KB
  static constexpr int STAGES = O::kSingle ? 4 : 3;                 // 128 / 96 KB ring
  static constexpr size_t RING = size_t(STAGES) * (WS_STAGE_A + WS_STAGE_B) * sizeof(double);
  static constexpr size_t SMEM = RING + CTILE + (2 * STAGES + 2) * sizeof(uint64_t);
};

// Persistent schedule of CTA b out of G: whole tiles b + w G (w < dpw), then
// (stream-K) the CTA's k-block range of the last G + tiles % G tiles.
struct WsSched {
  int nk, nseg, dpw, G;
  int b;                     // logical CTA number (logical_cta)
  int start_tile, start_k1;  // SEG_START (start_k1 == 0: none)
  int full0, full1;          // whole tiles of the range
  int end_tile, end_k0;      // SEG_END (end_k0 == 0: none)
};

__device__ __forceinline__ WsSched ws_sched(int64_t tiles, int nk, bool sk, int cta) {
  WsSched s{};
  s.nk = nk;
  s.G = static_cast<int>(gridDim.x);
  const int64_t G = gridDim.x, b = cta;
  s.b = cta;
  const int64_t R = tiles % G;
  if (!sk || R == 0) {
    s.dpw = static_cast<int>((tiles - b + G - 1) / G);
    s.nseg = s.dpw;
    return s;
  }
  const int64_t dp = (tiles / G - 1) * G;
  s.dpw = static_cast<int>(dp / G);
  const int64_t U = (tiles - dp) * nk;
  const int64_t u0 = dp * nk + b * U / G, u1 = dp * nk + (b + 1) * U / G;
  s.start_tile = static_cast<int>(u1 / nk);
  s.start_k1 = static_cast<int>(u1 % nk);
  s.end_tile = static_cast<int>(u0 / nk);
  s.end_k0 = static_cast<int>(u0 % nk);
  s.full0 = static_cast<int>((u0 + nk - 1) / nk);
  s.full1 = s.start_tile;
  s.nseg = (s.start_k1 != 0) + s.dpw + (s.full1 - s.full0) + (s.end_k0 != 0);
  return s;
}

// Order: the whole-tile waves first, so every CTA runs them in step (the
// wave's CTAs then share each A/B slab in L2 -- a START segment of varying
// length up front would offset them by up to a tile), then SEG_START, the
// range's whole tiles, SEG_END last.  CTA b+1 reaches its SEG_END no earlier
// than CTA b finishes its SEG_START, since every range is >= one tile long.
__device__ __forceinline__ Seg ws_seg(const WsSched& s, int idx) {
  if (idx < s.dpw) return Seg{s.b + idx * s.G, 0, s.nk, SEG_FULL};
  idx -= s.dpw;
  if (s.start_k1 != 0) {
    if (idx == 0) return Seg{s.start_tile, 0, s.start_k1, SEG_START};
    --idx;
  }
  if (idx < s.full1 - s.full0) return Seg{s.full0 + idx, 0, s.nk, SEG_FULL};
  return Seg{s.end_tile, s.end_k0, s.nk, SEG_END};
}

// Byte offset of element (r, c) of the 128x128 C tile when it is held as
// SWIZZLE_128B boxes of 128 bytes (128/ESZ rows) x 16 columns, column-chunk
// major: inside a box, column cc is one 128-byte line whose 16-byte chunks are
// permuted by XOR with cc % 8 (the TMA 128B swizzle of a 1 KB-aligned box).
// accumulate_element for real C in its storage precision (combine_typed's real path)
__device__ __forceinline__ float ws_add(float x, float y) { return __fadd_rn(x, y); }
__device__ __forceinline__ double ws_add(double x, double y) { return __dadd_rn(x, y); }
__device__ __forceinline__ float ws_mul(float x, float y) { return __fmul_rn(x, y); }
__device__ __forceinline__ double ws_mul(double x, double y) { return __dmul_rn(x, y); }

template <int ESZ>
__device__ __forceinline__ uint32_t ws_swz_off(int r, int c) {
  constexpr int RB = 128 / ESZ, NRB = 128 / RB;
  const int cb = c >> 4, cc = c & 15, rb = r / RB, rr = r % RB;
  const uint32_t byte = static_cast<uint32_t>(rr * ESZ);
  return static_cast<uint32_t>((cb * NRB + rb) * 2048 + cc * 128) + ((((byte >> 4) ^ (cc & 7)) << 4) | (byte & 15));
}

__device__ __forceinline__ void dmma884_ws(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int CDT>
__global__ void __launch_bounds__(WS_THREADS, 1) gemm_dmma_ws_kernel(const __grid_constant__ GemmDesc d) {
  using W = WsCfg<CDT>;
  using O = OutType<CDT>;
  using R = typename O::R;
  constexpr int NC = O::NC;
  extern __shared__ __align__(128) unsigned char smem[];
  double* sA = reinterpret_cast<double*>(smem);
  double* sB = sA + W::STAGES * WS_STAGE_A;
  unsigned char* ctile = smem + W::RING;
  uint64_t* full = reinterpret_cast<uint64_t*>(ctile + W::CTILE);
  uint64_t* empty = full + W::STAGES;
  uint64_t* c_full = empty + W::STAGES;  // C mover -> MMA warps: this tile's C is in ctile
  uint64_t* res_full = c_full + 1;       // MMA warps -> C mover: results written (one arrive per warp)

  const int tiles_m = static_cast<int>((d.me + WS_BM - 1) / WS_BM);
  const int tiles_n = static_cast<int>((d.ne + WS_BN - 1) / WS_BN);
  const int64_t tiles = static_cast<int64_t>(tiles_m) * tiles_n;
  const int64_t lpad = d.a.lpad;
  const WsSched sc = ws_sched(tiles, static_cast<int>(lpad / WS_BK), d.sk_grid > 0, logical_cta(sk_ticket(d)));

  const DEpilogue& e = d.epi;
  const bool prow = e.pair == MDG_PAIR_ROWS, pcol = e.pair == MDG_PAIR_COLS;
  const int orows = prow ? WS_BM / 2 : WS_BM, ocols = pcol ? WS_BN / 2 : WS_BN;
  const bool reads_c = !e.beta.is_zero;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == WS_PROD_WARP) {  // ------------------------------------------ producer
    if (lane == 0) {
      for (int s = 0; s < W::STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], WS_MMA_WARPS);
      }
      mbar_init(c_full, 1);
      mbar_init(res_full, WS_MMA_WARPS);
      mbar_fence_init();
    }
    __syncwarp();
    named_arrive(2, WS_THREADS);
    if (lane != 0) return;
    int it = 0;
    for (int si = 0; si < sc.nseg; ++si) {
      const Seg sg = ws_seg(sc, si);
      int tm, tn;
      tile_coords(sg.tile, tiles_m, tiles_n, d.group_rows, tm, tn);
      MDG_CHECK(tm >= 0 && tm < tiles_m && tn >= 0 && tn < tiles_n && sg.k0 >= 0 && sg.k0 <= sg.k1 &&
                    static_cast<int64_t>(sg.k1) * WS_BK <= lpad,
                "producer tile / k-block range");
      const double* Ag = static_cast<const double*>(d.a.data) + static_cast<int64_t>(tm) * WS_BM * lpad;
      const double* Bg = static_cast<const double*>(d.b.data) + static_cast<int64_t>(tn) * WS_BN * lpad;
      for (int kb = sg.k0; kb < sg.k1; ++kb, ++it) {
        const int s = it % W::STAGES;
        if (it >= W::STAGES) mbar_wait(&empty[s], ((it / W::STAGES) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], (WS_STAGE_A + WS_STAGE_B) * sizeof(double));
        bulk_g2s(sA + s * WS_STAGE_A, Ag + static_cast<int64_t>(kb) * WS_STAGE_A, WS_STAGE_A * sizeof(double),
                 &full[s]);
        bulk_g2s(sB + s * WS_STAGE_B, Bg + static_cast<int64_t>(kb) * WS_STAGE_B, WS_STAGE_B * sizeof(double),
                 &full[s]);
      }
    }
    return;
  }
  named_sync(2, WS_THREADS);  // barriers initialised

  if (warp == WS_CMOV_WARP) {  // ------------------------------------------ C mover
    if (lane != 0) return;
    const uint32_t col_bytes = orows * O::ESZ;
    const uint32_t tile_bytes = static_cast<uint32_t>(ocols) * col_bytes;
    auto coords = [&](const Seg& sg, int& x0, int& y0) {
      int tm, tn;
      tile_coords(sg.tile, tiles_m, tiles_n, d.group_rows, tm, tn);
      x0 = (prow ? tm * (WS_BM / 2) : tm * WS_BM) * NC;
      y0 = pcol ? tn * (WS_BN / 2) : tn * WS_BN;
    };
    // swizzled layout (e.sw_ok, real C): 128-byte x 16-column boxes, column
    // chunk major, SWIZZLE_128B (ws_swz_off); else one box per 16 columns
    const bool swz = NC == 1 && e.sw_ok && (smem_u32(ctile) & 1023) == 0;  // the swizzle atom is 1 KB
    constexpr int RB = 128 / O::ESZ, NRB = WS_BM / RB;
    auto load = [&](const Seg& sg) {  // C of the tile the MMA warps finish next
      if (!reads_c) {
        mbar_arrive(c_full);
        return;
      }
      int x0, y0;
      coords(sg, x0, y0);
      mbar_arrive_expect_tx(c_full, tile_bytes);
      if (swz) {
        for (int b = 0; b < WS_BN / C_BOX_COLS; ++b)
          for (int rb = 0; rb < NRB; ++rb)
            tensor_load_2d(ctile + static_cast<size_t>(b * NRB + rb) * 2048, &e.cmap_sw, x0 + rb * RB,
                           y0 + b * C_BOX_COLS, c_full);
        return;
      }
      for (int b = 0; b < ocols; b += C_BOX_COLS)
        tensor_load_2d(ctile + static_cast<size_t>(b) * col_bytes, &e.cmap, x0, y0 + b, c_full);
    };
    auto store = [&](int x0, int y0) {
      if (swz) {
        for (int b = 0; b < WS_BN / C_BOX_COLS; ++b)
          for (int rb = 0; rb < NRB; ++rb)
            tensor_store_2d(&e.cmap_sw, x0 + rb * RB, y0 + b * C_BOX_COLS,
                            ctile + static_cast<size_t>(b * NRB + rb) * 2048);
        return;
      }
      for (int b = 0; b < ocols; b += C_BOX_COLS)
        tensor_store_2d(&e.cmap, x0, y0 + b, ctile + static_cast<size_t>(b) * col_bytes);
    };
    int epis = 0, pending = -1;  // pending: segment whose C is loaded and whose results are awaited
    for (int si = 0; si < sc.nseg; ++si) {
      const Seg sg = ws_seg(sc, si);
      if (sg.kind == SEG_START) continue;
      if (pending >= 0) {  // store the previous tile, then reuse the buffer for this one
        mbar_wait(res_full, epis & 1);
        int x0, y0;
        coords(ws_seg(sc, pending), x0, y0);
        store(x0, y0);
        bulk_commit();
        bulk_wait_read();
        ++epis;
      }
      fence_proxy_async();
      load(sg);
      pending = si;
    }
    if (pending >= 0) {
      mbar_wait(res_full, epis & 1);
      int x0, y0;
      coords(ws_seg(sc, pending), x0, y0);
      store(x0, y0);
      bulk_commit();
      bulk_wait_read();  // the smem must outlive the store's reads
    }
    return;
  }

  // ---------------------------------------------------------------- MMA warps
  const int tid = threadIdx.x;
  const int wm = warp % WS_WM, wn = warp / WS_WM;
  const int g = lane >> 2, tig = lane & 3;
  const uint32_t full_u = smem_u32(full), empty_u = smem_u32(empty);
  const double* a_base = sA + wm * 64 + g + tig * WS_BM;
  const double* b_base = sB + wn * 32 + g + tig * WS_BN;
  int it = 0, epis = 0;
  for (int si = 0; si < sc.nseg; ++si) {
    const Seg sg = ws_seg(sc, si);
    double acc[WS_MT][WS_NT][2];
    if (sg.kind == SEG_END) {  // continue CTA b-1's accumulation of this tile
      check_sk_slot(sc.b - 1, d.sk_grid);
      if (tid == 0) flag_acquire_wait(d.sk_flags + sc.b - 1);
      named_sync(1, WS_MMA_THREADS);
      const double* slot =
          static_cast<const double*>(d.sk_partials) + static_cast<int64_t>(sc.b - 1) * (WS_BM * WS_BN);
#pragma unroll
      for (int i = 0; i < WS_MT; ++i)
#pragma unroll
        for (int j = 0; j < WS_NT; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            acc[i][j][h] = __ldcg(slot + ((i * WS_NT + j) * 2 + h) * WS_MMA_THREADS + tid);
    } else {
#pragma unroll
      for (int i = 0; i < WS_MT; ++i)
#pragma unroll
        for (int j = 0; j < WS_NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    }
    for (int kb = sg.k0; kb < sg.k1; ++kb, ++it) {
      const int s = it % W::STAGES;
      mbar_wait_u32(full_u + 8 * s, (it / W::STAGES) & 1);
      const double* a = a_base + s * WS_STAGE_A;
      const double* b = b_base + s * WS_STAGE_B;
#pragma unroll
      for (int kk = 0; kk < WS_BK; kk += 4) {
        double af[WS_MT], bf[WS_NT];
#pragma unroll
        for (int i = 0; i < WS_MT; ++i) af[i] = a[kk * WS_BM + i * 8];
#pragma unroll
        for (int j = 0; j < WS_NT; ++j) bf[j] = b[kk * WS_BN + j * 8];
#pragma unroll
        for (int i = 0; i < WS_MT; ++i)
#pragma unroll
          for (int j = 0; j < WS_NT; ++j) dmma884_ws(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
      fence_proxy_async();  // generic reads of the stage before its TMA refill
      __syncwarp();
      if (lane == 0) mbar_arrive_u32(empty_u + 8 * s);
    }
    if (sg.kind == SEG_START) {  // publish the first k-blocks of the tile for CTA b+1
      double* slot = static_cast<double*>(d.sk_partials) + static_cast<int64_t>(sc.b) * (WS_BM * WS_BN);
#pragma unroll
      for (int i = 0; i < WS_MT; ++i)
#pragma unroll
        for (int j = 0; j < WS_NT; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) __stcg(slot + ((i * WS_NT + j) * 2 + h) * WS_MMA_THREADS + tid, acc[i][j][h]);
      __threadfence();
      named_sync(1, WS_MMA_THREADS);
      check_sk_slot(sc.b, d.sk_grid);
      if (tid == 0) flag_release(d.sk_flags + sc.b);
      continue;
    }
    // combine with this tile's C (already in ctile) in place.  The epilogue
    // parameters are re-read here through an opaque pointer: hoisted above
    // the segment loop they would stay live through the mainloop, which runs
    // at the register cap (168).
    mbar_wait(c_full, epis & 1);
    const DEpilogue* ep = &d.epi;
    asm volatile("" : "+l"(ep));
    const bool eprow = ep->pair == MDG_PAIR_ROWS, epcol = ep->pair == MDG_PAIR_COLS;
    const int eorows = eprow ? WS_BM / 2 : WS_BM;
    const DBeta eb = ep->beta;  // one copy in registers, not a parameter-space load per element
    const bool ereads = !eb.is_zero, econj = ep->out.conj != 0;
    const bool eswz = NC == 1 && ep->sw_ok && (smem_u32(smem + W::RING) & 1023) == 0;
    R* const ect = reinterpret_cast<R*>(smem + W::RING);
    if constexpr (NC == 1) {
      // real C: accumulate_element (combine_typed) with the beta case and the
      // tile layout resolved once per tile, not per element
      const R rb = static_cast<R>(eb.re);
      auto pass = [&](auto mode, auto swz) {
#pragma unroll
        for (int i = 0; i < WS_MT; ++i)
#pragma unroll
          for (int j = 0; j < WS_NT; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int r = wm * 64 + i * 8 + g, c = wn * 32 + j * 8 + 2 * tig + h;
              R* p = decltype(swz)::value ? reinterpret_cast<R*>(smem + W::RING + ws_swz_off<O::ESZ>(r, c))
                                          : ect + c * eorows + r;
              const R tv = static_cast<R>(acc[i][j][h]);
              if constexpr (decltype(mode)::value == 0) {
                *p = tv;
              } else if constexpr (decltype(mode)::value == 1) {
                *p = ws_add(*p, tv);
              } else {
                *p = ws_add(ws_mul(rb, *p), tv);
              }
            }
      };
      using Z = std::integral_constant<int, 0>;
      using One = std::integral_constant<int, 1>;
      using Gen = std::integral_constant<int, 2>;
      if (eswz) {
        if (eb.is_zero) pass(Z{}, std::true_type{});
        else if (eb.is_one) pass(One{}, std::true_type{});
        else pass(Gen{}, std::true_type{});
      } else {
        if (eb.is_zero) pass(Z{}, std::false_type{});
        else if (eb.is_one) pass(One{}, std::false_type{});
        else pass(Gen{}, std::false_type{});
      }
    } else {
#pragma unroll
    for (int i = 0; i < WS_MT; ++i)
#pragma unroll
      for (int j = 0; j < WS_NT; ++j) {
        const int r = wm * 64 + i * 8 + g, c = wn * 32 + j * 8 + 2 * tig;
        const double a0 = acc[i][j][0], a1 = acc[i][j][1];  // (r, c), (r, c + 1)
        {
          // complex C: a column pair (pcol: re, im of element (r, c/2)) or a
          // row pair held by lanes g and g^1 (prow: element (r/2, c) for even
          // g, (r/2, c+1) for odd g after one exchange)
          R tv[2];
          R* p;
          if (epcol) {
            tv[0] = static_cast<R>(a0);
            tv[1] = static_cast<R>(a1);
            p = ect + ((c >> 1) * eorows + r) * 2;
          } else {
            const double other = __shfl_xor_sync(0xffffffffu, (g & 1) ? a0 : a1, 4);
            const bool odd = g & 1;
            tv[0] = static_cast<R>(odd ? other : a0);
            tv[1] = static_cast<R>(odd ? a1 : other);
            p = ect + ((odd ? c + 1 : c) * eorows + (r >> 1)) * 2;
          }
          R cv[2] = {R(0), R(0)};
          if (ereads) {
            cv[0] = p[0];
            cv[1] = p[1];
          }
          combine_typed<CDT>(eb, econj, cv, tv);
          p[0] = cv[0];
          p[1] = cv[1];
        }
      }
    }
    fence_proxy_async();  // generic writes of ctile before the C mover's TMA store reads them
    __syncwarp();
    if (lane == 0) mbar_arrive(res_full);
    ++epis;
  }
}

// ------------------------------------------------------------------------
// Variant with epilogue warps (real single-precision C, swizzled C tile):
// the MMA warps only round their accumulators to C's precision and dump them
// into a stage buffer laid out like the C tile, then start the next tile's
// mainloop; six epilogue warps combine stage and C tile (accumulate_element,
// 16-byte vectors, conflict-free) while the MMA warps compute.  For short k
// (cfg5: k = 64 is 4 k-blocks per tile) the combine pass otherwise runs
// between two mainloops with the DMMA pipe idle.
//   warps 0-7   MMA (setmaxnreg 168)
//   warp  8     producer lane;  warp 9: C mover lane
//   warps 10-15 epilogue (warpgroups 2-3: setmaxnreg 88)
constexpr int WE_THREADS = 512;
constexpr int WE_EPI_WARP0 = 10, WE_EPI_WARPS = 6;
constexpr int WE_STAGES = 3;
constexpr size_t WE_RING = size_t(WE_STAGES) * (WS_STAGE_A + WS_STAGE_B) * sizeof(double);  // 96 KB
constexpr size_t WE_CTILE = size_t(WS_BM) * WS_BN * sizeof(float);                         // 64 KB
constexpr size_t WE_SMEM = WE_RING + 2 * WE_CTILE + (2 * WE_STAGES + 4) * sizeof(uint64_t);

__global__ void __launch_bounds__(WE_THREADS, 1) gemm_dmma_ws_epi_kernel(const __grid_constant__ GemmDesc d) {
  extern __shared__ __align__(1024) unsigned char smem[];
  double* sA = reinterpret_cast<double*>(smem);
  double* sB = sA + WE_STAGES * WS_STAGE_A;
  unsigned char* ctile = smem + WE_RING;              // C (TMA, swizzled boxes)
  unsigned char* stage = ctile + WE_CTILE;            // rounded results, same layout
  uint64_t* full = reinterpret_cast<uint64_t*>(stage + WE_CTILE);
  uint64_t* empty = full + WE_STAGES;
  uint64_t* c_full = empty + WE_STAGES;  // mover -> epilogue: this tile's C is in ctile
  uint64_t* staged = c_full + 1;         // MMA warps -> epilogue: results in stage (8 arrivals)
  uint64_t* stage_free = staged + 1;     // epilogue -> MMA warps: stage read (6 arrivals)
  uint64_t* res_full = stage_free + 1;   // epilogue -> mover: ctile combined (6 arrivals)

  const int tiles_m = static_cast<int>((d.me + WS_BM - 1) / WS_BM);
  const int tiles_n = static_cast<int>((d.ne + WS_BN - 1) / WS_BN);
  const int64_t tiles = static_cast<int64_t>(tiles_m) * tiles_n;
  const int64_t lpad = d.a.lpad;
  const WsSched sc = ws_sched(tiles, static_cast<int>(lpad / WS_BK), d.sk_grid > 0, logical_cta(sk_ticket(d)));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (smem_u32(ctile) & 1023) __trap();  // the 128-byte swizzle needs 1 KB-aligned boxes
  if (threadIdx.x == 0) {
    for (int s = 0; s < WE_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], WS_MMA_WARPS);
    }
    mbar_init(c_full, 1);
    mbar_init(staged, WS_MMA_WARPS);
    mbar_init(stage_free, WE_EPI_WARPS);
    mbar_init(res_full, WE_EPI_WARPS);
    mbar_fence_init();
  }
  __syncthreads();

  if (warp >= WS_MMA_WARPS) {  // ---------------------------- producer, mover, epilogue
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;\n");
    const DEpilogue& e = d.epi;
    const bool reads_c = !e.beta.is_zero;
    constexpr int RB = 32, NRB = WS_BM / RB;  // 128-byte box lines of floats
    auto coords = [&](const Seg& sg, int& x0, int& y0) {
      int tm, tn;
      tile_coords(sg.tile, tiles_m, tiles_n, d.group_rows, tm, tn);
      x0 = tm * WS_BM;
      y0 = tn * WS_BN;
    };
    if (warp == WS_PROD_WARP) {
      if (lane != 0) return;
      int it = 0;
      for (int si = 0; si < sc.nseg; ++si) {
        const Seg sg = ws_seg(sc, si);
        int tm, tn;
        tile_coords(sg.tile, tiles_m, tiles_n, d.group_rows, tm, tn);
        MDG_CHECK(tm >= 0 && tm < tiles_m && tn >= 0 && tn < tiles_n && sg.k0 >= 0 && sg.k0 <= sg.k1 &&
                      static_cast<int64_t>(sg.k1) * WS_BK <= lpad,
                  "producer tile / k-block range");
        const double* Ag = static_cast<const double*>(d.a.data) + static_cast<int64_t>(tm) * WS_BM * lpad;
        const double* Bg = static_cast<const double*>(d.b.data) + static_cast<int64_t>(tn) * WS_BN * lpad;
        for (int kb = sg.k0; kb < sg.k1; ++kb, ++it) {
          const int s = it % WE_STAGES;
          if (it >= WE_STAGES) mbar_wait(&empty[s], ((it / WE_STAGES) - 1) & 1);
          mbar_arrive_expect_tx(&full[s], (WS_STAGE_A + WS_STAGE_B) * sizeof(double));
          bulk_g2s(sA + s * WS_STAGE_A, Ag + static_cast<int64_t>(kb) * WS_STAGE_A, WS_STAGE_A * sizeof(double),
                   &full[s]);
          bulk_g2s(sB + s * WS_STAGE_B, Bg + static_cast<int64_t>(kb) * WS_STAGE_B, WS_STAGE_B * sizeof(double),
                   &full[s]);
        }
      }
      return;
    }
    if (warp == WS_CMOV_WARP) {
      if (lane != 0) return;
      auto boxes = [&](int x0, int y0, bool load) {
        for (int b = 0; b < WS_BN / C_BOX_COLS; ++b)
          for (int rb = 0; rb < NRB; ++rb) {
            unsigned char* box = ctile + static_cast<size_t>(b * NRB + rb) * 2048;
            if (load)
              tensor_load_2d(box, &e.cmap_sw, x0 + rb * RB, y0 + b * C_BOX_COLS, c_full);
            else
              tensor_store_2d(&e.cmap_sw, x0 + rb * RB, y0 + b * C_BOX_COLS, box);
          }
      };
      int epis = 0, pending = -1;
      for (int si = 0; si < sc.nseg; ++si) {
        const Seg sg = ws_seg(sc, si);
        if (sg.kind == SEG_START) continue;
        if (pending >= 0) {  // store the previous tile, then reuse the buffer for this one
          mbar_wait(res_full, epis & 1);
          int x0, y0;
          coords(ws_seg(sc, pending), x0, y0);
          boxes(x0, y0, false);
          bulk_commit();
          bulk_wait_read();
          ++epis;
        }
        fence_proxy_async();
        if (reads_c) {
          int x0, y0;
          coords(sg, x0, y0);
          mbar_arrive_expect_tx(c_full, static_cast<uint32_t>(WE_CTILE));
          boxes(x0, y0, true);
        } else {
          mbar_arrive(c_full);
        }
        pending = si;
      }
      if (pending >= 0) {
        mbar_wait(res_full, epis & 1);
        int x0, y0;
        coords(ws_seg(sc, pending), x0, y0);
        boxes(x0, y0, false);
        bulk_commit();
        bulk_wait_read();
      }
      return;
    }
    // epilogue warps: stage (+) C, in place in ctile, 16-byte vectors
    if (warp < WE_EPI_WARP0) return;
    const int et = threadIdx.x - WE_EPI_WARP0 * 32;
    const float rb = static_cast<float>(e.beta.re);
    const int mode = e.beta.is_zero ? 0 : (e.beta.is_one ? 1 : 2);
    int epis = 0;
    for (int si = 0; si < sc.nseg; ++si) {
      if (ws_seg(sc, si).kind == SEG_START) continue;
      mbar_wait(staged, epis & 1);
      mbar_wait(c_full, epis & 1);
      const float4* sv = reinterpret_cast<const float4*>(stage);
      float4* cv = reinterpret_cast<float4*>(ctile);
      constexpr int NV = static_cast<int>(WE_CTILE / 16);
      for (int v = et; v < NV; v += WE_EPI_WARPS * 32) {
        const float4 t = sv[v];
        float4 c = cv[v];
        if (mode == 0) {
          c = t;
        } else if (mode == 1) {
          c.x = __fadd_rn(c.x, t.x);
          c.y = __fadd_rn(c.y, t.y);
          c.z = __fadd_rn(c.z, t.z);
          c.w = __fadd_rn(c.w, t.w);
        } else {
          c.x = __fadd_rn(__fmul_rn(rb, c.x), t.x);
          c.y = __fadd_rn(__fmul_rn(rb, c.y), t.y);
          c.z = __fadd_rn(__fmul_rn(rb, c.z), t.z);
          c.w = __fadd_rn(__fmul_rn(rb, c.w), t.w);
        }
        cv[v] = c;
      }
      fence_proxy_async();  // generic writes of ctile before the mover's TMA store reads them
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(stage_free);
        mbar_arrive(res_full);
      }
      ++epis;
    }
    return;
  }

  // ---------------------------------------------------------------- MMA warps
  asm volatile("setmaxnreg.inc.sync.aligned.u32 168;\n");
  const int tid = threadIdx.x;
  const int wm = warp % WS_WM, wn = warp / WS_WM;
  const int g = lane >> 2, tig = lane & 3;
  const uint32_t full_u = smem_u32(full), empty_u = smem_u32(empty);
  const double* a_base = sA + wm * 64 + g + tig * WS_BM;
  const double* b_base = sB + wn * 32 + g + tig * WS_BN;
  int it = 0, epis = 0;
  for (int si = 0; si < sc.nseg; ++si) {
    const Seg sg = ws_seg(sc, si);
    double acc[WS_MT][WS_NT][2];
    if (sg.kind == SEG_END) {  // continue CTA b-1's accumulation of this tile
      check_sk_slot(sc.b - 1, d.sk_grid);
      if (tid == 0) flag_acquire_wait(d.sk_flags + sc.b - 1);
      named_sync(1, WS_MMA_THREADS);
      const double* slot =
          static_cast<const double*>(d.sk_partials) + static_cast<int64_t>(sc.b - 1) * (WS_BM * WS_BN);
#pragma unroll
      for (int i = 0; i < WS_MT; ++i)
#pragma unroll
        for (int j = 0; j < WS_NT; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            acc[i][j][h] = __ldcg(slot + ((i * WS_NT + j) * 2 + h) * WS_MMA_THREADS + tid);
    } else {
#pragma unroll
      for (int i = 0; i < WS_MT; ++i)
#pragma unroll
        for (int j = 0; j < WS_NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    }
    for (int kb = sg.k0; kb < sg.k1; ++kb, ++it) {
      const int s = it % WE_STAGES;
      mbar_wait_u32(full_u + 8 * s, (it / WE_STAGES) & 1);
      const double* a = a_base + s * WS_STAGE_A;
      const double* b = b_base + s * WS_STAGE_B;
#pragma unroll
      for (int kk = 0; kk < WS_BK; kk += 4) {
        double af[WS_MT], bf[WS_NT];
#pragma unroll
        for (int i = 0; i < WS_MT; ++i) af[i] = a[kk * WS_BM + i * 8];
#pragma unroll
        for (int j = 0; j < WS_NT; ++j) bf[j] = b[kk * WS_BN + j * 8];
#pragma unroll
        for (int i = 0; i < WS_MT; ++i)
#pragma unroll
          for (int j = 0; j < WS_NT; ++j) dmma884_ws(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive_u32(empty_u + 8 * s);
    }
    if (sg.kind == SEG_START) {  // publish the first k-blocks of the tile for CTA b+1
      double* slot = static_cast<double*>(d.sk_partials) + static_cast<int64_t>(sc.b) * (WS_BM * WS_BN);
#pragma unroll
      for (int i = 0; i < WS_MT; ++i)
#pragma unroll
        for (int j = 0; j < WS_NT; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) __stcg(slot + ((i * WS_NT + j) * 2 + h) * WS_MMA_THREADS + tid, acc[i][j][h]);
      __threadfence();
      named_sync(1, WS_MMA_THREADS);
      check_sk_slot(sc.b, d.sk_grid);
      if (tid == 0) flag_release(d.sk_flags + sc.b);
      continue;
    }
    // round to C's precision (accumulate_element's tc) into the stage buffer
    if (epis > 0) mbar_wait(stage_free, (epis - 1) & 1);
#pragma unroll
    for (int i = 0; i < WS_MT; ++i)
#pragma unroll
      for (int j = 0; j < WS_NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = wm * 64 + i * 8 + g, c = wn * 32 + j * 8 + 2 * tig + h;
          *reinterpret_cast<float*>(stage + ws_swz_off<4>(r, c)) = static_cast<float>(acc[i][j][h]);
        }
    __syncwarp();
    if (lane == 0) mbar_arrive(staged);
    ++epis;
  }
}

}  // namespace

size_t dmma_ws_smem(int cdt) {
  size_t s = 0;
  MDG_DISPATCH_CDT(cdt, CDT, { s = WsCfg<CDT>::SMEM; });
  return s;
}

cudaError_t launch_gemm_dmma_ws(const GemmDesc& d, int grid, cudaStream_t s) {
  if (grid <= 0) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  // real single-precision C in swizzled boxes: the epilogue-warp variant
  static const bool epi_warps = [] {
    const char* f = std::getenv("MDGEMM_WS_EPI_WARPS");  // tuning: 0 = always the plain WS kernel
    return f ? std::atoi(f) != 0 : true;
  }();
  if (epi_warps && d.epi.out.dtype == MDG_DT_S && d.epi.sw_ok && d.epi.pair == MDG_PAIR_NONE) {
    e = cudaFuncSetAttribute(gemm_dmma_ws_epi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(WE_SMEM));
    if (e != cudaSuccess) return e;
    gemm_dmma_ws_epi_kernel<<<static_cast<unsigned>(grid), WE_THREADS, WE_SMEM, s>>>(d);
    return cudaGetLastError();
  }
  MDG_DISPATCH_CDT(d.epi.out.dtype, CDT, {
    auto kern = gemm_dmma_ws_kernel<CDT>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(WsCfg<CDT>::SMEM));
    if (e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>(grid), WS_THREADS, WsCfg<CDT>::SMEM, s>>>(d);
  });
  return cudaGetLastError();
}

}  // namespace mdg
