// FAST numerics, computation precision single: warp-specialised persistent
// variant of the FFMA2 kernel (gemm_ffma.cu), one CTA per SM -- the same
// structure as gemm_dmma_ws.cu:
//
//   warps 0-7  MMA: one 128x128 tile, each thread an 8x8 register tile in
//              two 4x4 quadrants updated with paired FP32 FMAs (FFMA2),
//              two warps per SM sub-partition;
//   warp  8    producer: TMA bulk copies of 16-deep A/B slabs into the ring;
//   warp  9    C mover: 2-D TMA tensor loads of the NEXT tile's C into a
//              tile buffer in C's storage precision, tensor stores of each
//              finished tile.
//
// After the mainloop the MMA warps combine their accumulators with the C
// tile in shared memory (combine_typed: accumulate_element, kernels.cpp:
// 79-95) in place.  The register tile keeps both halves of a complex pair in
// one thread (rows 4i..4i+3 / columns 4j..4j+3 are consecutive), so pairing
// needs no exchange.  Stream-K tail with seeded continuation as in the DMMA
// kernel: bitwise identical to the classic FFMA kernel.
#include <cstdlib>

#include "common.cuh"

namespace mdg {
namespace {

constexpr int FW_BM = 128, FW_BN = 128, FW_BK = 16;
constexpr int FW_TYM = FW_BM / 8, FW_TXN = FW_BN / 8;  // 16 x 16 threads
constexpr int FW_MMA_THREADS = FW_TYM * FW_TXN;          // 256
constexpr int FW_MMA_WARPS = FW_MMA_THREADS / 32;
constexpr int FW_PROD_WARP = FW_MMA_WARPS;
constexpr int FW_CMOV_WARP = FW_MMA_WARPS + 1;
constexpr int FW_THREADS = (FW_MMA_WARPS + 2) * 32;
constexpr int FW_STAGE_A = FW_BK * FW_BM, FW_STAGE_B = FW_BK * FW_BN;  // floats

template <int CDT>
struct FwCfg {
  using O = OutType<CDT>;
  static constexpr int ESZR = O::kSingle ? 4 : 8;
  // 128 KB: double C, or single C held as the real part of an interleaved
  // complex C (the imaginary halves ride along unchanged)
  static constexpr size_t CTILE = size_t(FW_BM) * FW_BN * 8;
  static constexpr int STAGES = O::kSingle ? 6 : 4;              // 96 / 64 KB ring
  static constexpr size_t RING = size_t(STAGES) * (FW_STAGE_A + FW_STAGE_B) * sizeof(float);
  static constexpr size_t SMEM = RING + CTILE + (2 * STAGES + 2) * sizeof(uint64_t);
};

struct FwSched {
  int nk, nseg, dpw, G;
  int b;                     // logical CTA number (logical_cta)
  int start_tile, start_k1;
  int full0, full1;
  int end_tile, end_k0;
};

__device__ __forceinline__ FwSched fw_sched(int64_t tiles, int nk, bool sk, int cta) {
  FwSched s{};
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

// whole-tile waves first (in step across CTAs), then the stream-K range
// (see gemm_dmma_ws.cu: ws_seg)
__device__ __forceinline__ Seg fw_seg(const FwSched& s, int idx) {
  if (idx < s.dpw) return Seg{s.b + idx * s.G, 0, s.nk, SEG_FULL};
  idx -= s.dpw;
  if (s.start_k1 != 0) {
    if (idx == 0) return Seg{s.start_tile, 0, s.start_k1, SEG_START};
    --idx;
  }
  if (idx < s.full1 - s.full0) return Seg{s.full0 + idx, 0, s.nk, SEG_FULL};
  return Seg{s.end_tile, s.end_k0, s.nk, SEG_END};
}

template <int CDT>
__global__ void __launch_bounds__(FW_THREADS, 1) gemm_ffma_ws_kernel(const __grid_constant__ GemmDesc d) {
  using W = FwCfg<CDT>;
  using O = OutType<CDT>;
  using R = typename O::R;
  constexpr int NC = O::NC;
  extern __shared__ __align__(128) unsigned char smem[];
  float* sA = reinterpret_cast<float*>(smem);
  float* sB = sA + W::STAGES * FW_STAGE_A;
  unsigned char* ctile = smem + W::RING;
  uint64_t* full = reinterpret_cast<uint64_t*>(ctile + W::CTILE);
  uint64_t* empty = full + W::STAGES;
  uint64_t* c_full = empty + W::STAGES;
  uint64_t* res_full = c_full + 1;

  const int tiles_m = static_cast<int>((d.me + FW_BM - 1) / FW_BM);
  const int tiles_n = static_cast<int>((d.ne + FW_BN - 1) / FW_BN);
  const int64_t tiles = static_cast<int64_t>(tiles_m) * tiles_n;
  const int64_t lpad = d.a.lpad;
  const FwSched sc = fw_sched(tiles, static_cast<int>(lpad / FW_BK), d.sk_grid > 0, logical_cta(sk_ticket(d)));

  const DEpilogue& e = d.epi;
  const bool prow = e.pair == MDG_PAIR_ROWS, pcol = e.pair == MDG_PAIR_COLS;
  const int orows = prow ? FW_BM / 2 : FW_BM, ocols = pcol ? FW_BN / 2 : FW_BN;
  const bool reads_c = !e.beta.is_zero;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == FW_PROD_WARP) {  // ------------------------------------------ producer
    if (lane == 0) {
      for (int s = 0; s < W::STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], FW_MMA_WARPS);
      }
      mbar_init(c_full, 1);
      mbar_init(res_full, FW_MMA_WARPS);
      mbar_fence_init();
    }
    __syncwarp();
    named_arrive(2, FW_THREADS);
    if (lane != 0) return;
    int it = 0;
    for (int si = 0; si < sc.nseg; ++si) {
      const Seg sg = fw_seg(sc, si);
      int tm, tn;
      tile_coords(sg.tile, tiles_m, tiles_n, d.group_rows, tm, tn);
      MDG_CHECK(tm >= 0 && tm < tiles_m && tn >= 0 && tn < tiles_n && sg.k0 >= 0 && sg.k0 <= sg.k1 &&
                    static_cast<int64_t>(sg.k1) * FW_BK <= lpad,
                "producer tile / k-block range");
      const float* Ag = static_cast<const float*>(d.a.data) + static_cast<int64_t>(tm) * FW_BM * lpad;
      const float* Bg = static_cast<const float*>(d.b.data) + static_cast<int64_t>(tn) * FW_BN * lpad;
      for (int kb = sg.k0; kb < sg.k1; ++kb, ++it) {
        const int s = it % W::STAGES;
        if (it >= W::STAGES) mbar_wait(&empty[s], ((it / W::STAGES) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], (FW_STAGE_A + FW_STAGE_B) * sizeof(float));
        bulk_g2s(sA + s * FW_STAGE_A, Ag + static_cast<int64_t>(kb) * FW_STAGE_A, FW_STAGE_A * sizeof(float),
                 &full[s]);
        bulk_g2s(sB + s * FW_STAGE_B, Bg + static_cast<int64_t>(kb) * FW_STAGE_B, FW_STAGE_B * sizeof(float),
                 &full[s]);
      }
    }
    return;
  }
  named_sync(2, FW_THREADS);

  if (warp == FW_CMOV_WARP) {  // ------------------------------------------ C mover
    if (lane != 0) return;
    const bool halfc = NC == 1 && e.cmap_ok == MDG_CMAP_REAL_PART;  // real part of interleaved complex C
    const uint32_t col_bytes = (halfc ? 2 : 1) * orows * O::ESZ;
    const uint32_t tile_bytes = static_cast<uint32_t>(ocols) * col_bytes;
    auto coords = [&](const Seg& sg, int& x0, int& y0) {
      int tm, tn;
      tile_coords(sg.tile, tiles_m, tiles_n, d.group_rows, tm, tn);
      x0 = (prow ? tm * (FW_BM / 2) : tm * FW_BM) * (halfc ? 2 : NC);
      y0 = pcol ? tn * (FW_BN / 2) : tn * FW_BN;
    };
    auto store = [&](int seg_idx) {
      int x0, y0;
      coords(fw_seg(sc, seg_idx), x0, y0);
      for (int b = 0; b < ocols; b += C_BOX_COLS)
        tensor_store_2d(&e.cmap, x0, y0 + b, ctile + static_cast<size_t>(b) * col_bytes);
      bulk_commit();
      bulk_wait_read();
    };
    int epis = 0, pending = -1;
    for (int si = 0; si < sc.nseg; ++si) {
      const Seg sg = fw_seg(sc, si);
      if (sg.kind == SEG_START) continue;
      if (pending >= 0) {
        mbar_wait(res_full, epis & 1);
        store(pending);
        ++epis;
      }
      fence_proxy_async();
      if (reads_c || halfc) {  // a real part always needs the imaginary halves it writes back
        int x0, y0;
        coords(sg, x0, y0);
        mbar_arrive_expect_tx(c_full, tile_bytes);
        for (int b = 0; b < ocols; b += C_BOX_COLS)
          tensor_load_2d(ctile + static_cast<size_t>(b) * col_bytes, &e.cmap, x0, y0 + b, c_full);
      } else {
        mbar_arrive(c_full);
      }
      pending = si;
    }
    if (pending >= 0) {
      mbar_wait(res_full, epis & 1);
      store(pending);
    }
    return;
  }

  // ---------------------------------------------------------------- MMA warps
  const int tid = threadIdx.x;
  const int tx = tid % FW_TXN, ty = tid / FW_TXN;
  const bool conj = e.out.conj != 0;
  const uint32_t full_u = smem_u32(full), empty_u = smem_u32(empty);
  const float* a_base = sA + ty * 4;
  const float* b_base = sB + tx * 4;
  R* const ct = reinterpret_cast<R*>(ctile);
  int it = 0, epis = 0;
  for (int si = 0; si < sc.nseg; ++si) {
    const Seg sg = fw_seg(sc, si);
    uint64_t acc[8][4];
    if (sg.kind == SEG_END) {  // continue CTA b-1's accumulation of this tile
      check_sk_slot(sc.b - 1, d.sk_grid);
      if (tid == 0) flag_acquire_wait(d.sk_flags + sc.b - 1);
      named_sync(1, FW_MMA_THREADS);
      const uint64_t* slot =
          static_cast<const uint64_t*>(d.sk_partials) + static_cast<int64_t>(sc.b - 1) * (FW_BM * FW_BN / 2);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int p = 0; p < 4; ++p) acc[i][p] = __ldcg(slot + (i * 4 + p) * FW_MMA_THREADS + tid);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int p = 0; p < 4; ++p) acc[i][p] = 0ull;
    }
    for (int kb = sg.k0; kb < sg.k1; ++kb, ++it) {
      const int s = it % W::STAGES;
      mbar_wait_u32(full_u + 8 * s, (it / W::STAGES) & 1);
      const float* a = a_base + s * FW_STAGE_A;
      const float* b = b_base + s * FW_STAGE_B;
#pragma unroll
      for (int kk = 0; kk < FW_BK; ++kk) {
        const float4 a0 = *reinterpret_cast<const float4*>(a + kk * FW_BM);
        const float4 a1 = *reinterpret_cast<const float4*>(a + kk * FW_BM + FW_BM / 2);
        const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(b + kk * FW_BN);
        const ulonglong2 b1 = *reinterpret_cast<const ulonglong2*>(b + kk * FW_BN + FW_BN / 2);
        const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const uint64_t bp[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          uint64_t ai;
          asm("mov.b64 %0, {%1, %1};" : "=l"(ai) : "f"(av[i]));
#pragma unroll
          for (int p = 0; p < 4; ++p) asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i][p]) : "l"(ai), "l"(bp[p]));
        }
      }
      fence_proxy_async();  // generic reads of the stage before its TMA refill
      __syncwarp();
      if (lane == 0) mbar_arrive_u32(empty_u + 8 * s);
    }
    if (sg.kind == SEG_START) {  // publish the first k-blocks of the tile for CTA b+1
      uint64_t* slot =
          static_cast<uint64_t*>(d.sk_partials) + static_cast<int64_t>(sc.b) * (FW_BM * FW_BN / 2);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int p = 0; p < 4; ++p) __stcg(slot + (i * 4 + p) * FW_MMA_THREADS + tid, acc[i][p]);
      __threadfence();
      named_sync(1, FW_MMA_THREADS);
      check_sk_slot(sc.b, d.sk_grid);
      if (tid == 0) flag_release(d.sk_flags + sc.b);
      continue;
    }
    // combine with this tile's C (already in ctile) in place
    mbar_wait(c_full, epis & 1);
    const bool e_half = NC == 1 && e.cmap_ok == MDG_CMAP_REAL_PART;
    auto val = [&](int i, int j) -> float {
      const uint64_t v = acc[i][j >> 1];
      return __uint_as_float(static_cast<uint32_t>((j & 1) ? (v >> 32) : v));
    };
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = i < 4 ? ty * 4 + i : FW_BM / 2 + ty * 4 + (i - 4);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = j < 4 ? tx * 4 + j : FW_BN / 2 + tx * 4 + (j - 4);
        if constexpr (NC == 1) {
          R* p = e_half ? ct + (c * orows + r) * 2 : ct + c * orows + r;
          R cv = reads_c ? *p : R(0);
          const R tv = static_cast<R>(val(i, j));
          combine_typed<CDT>(e.beta, conj, &cv, &tv);
          *p = cv;
        } else {
          // complex C: the element's two parts are (r, c) and (r, c+1)
          // (pcol) or (r, c) and (r+1, c) (prow), both in this thread
          const bool lead = pcol ? (j & 1) == 0 : (i & 1) == 0;
          if (!lead) continue;
          R tv[2];
          R* p;
          if (pcol) {
            tv[0] = static_cast<R>(val(i, j));
            tv[1] = static_cast<R>(val(i, j + 1));
            p = ct + ((c >> 1) * orows + r) * 2;
          } else {
            tv[0] = static_cast<R>(val(i, j));
            tv[1] = static_cast<R>(val(i + 1, j));
            p = ct + (c * orows + (r >> 1)) * 2;
          }
          R cv[2] = {R(0), R(0)};
          if (reads_c) {
            cv[0] = p[0];
            cv[1] = p[1];
          }
          combine_typed<CDT>(e.beta, conj, cv, tv);
          p[0] = cv[0];
          p[1] = cv[1];
        }
      }
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(res_full);
    ++epis;
  }
}

}  // namespace

size_t ffma_ws_smem(int cdt) {
  size_t s = 0;
  MDG_DISPATCH_CDT(cdt, CDT, { s = FwCfg<CDT>::SMEM; });
  return s;
}

cudaError_t launch_gemm_ffma_ws(const GemmDesc& d, int grid, cudaStream_t s) {
  if (grid <= 0) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  MDG_DISPATCH_CDT(d.epi.out.dtype, CDT, {
    auto kern = gemm_ffma_ws_kernel<CDT>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(FwCfg<CDT>::SMEM));
    if (e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>(grid), FW_THREADS, FwCfg<CDT>::SMEM, s>>>(d);
  });
  return cudaGetLastError();
}

}  // namespace mdg
