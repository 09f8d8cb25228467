// FAST numerics, computation precision single: the reference's float
// microkernel (ukr_impl<float>, kernels.cpp:7-40) as an FP32 SIMT CTA tile.
// No TF32: tensor cores would not reproduce fp32 products.
//
// Same feed as the DMMA kernel: a producer warp streams BK x BM / BK x BN
// slabs of the packed panels into a STAGES-deep shared-memory ring with one
// TMA bulk copy per operand per stage (mbarrier completion).  Each compute
// thread owns an 8x8 register tile split into two 4x4 quadrants
// ({ty*4, BM/2+ty*4} x {tx*4, BN/2+tx*4}) so every fragment is one
// conflict-free LDS.128, and updates it with Blackwell's paired FP32 FMA
// (fma.rn.f32x2 -> SASS FFMA2, A's element broadcast into both lanes), which
// halves the issue slots of the outer product.  The fused typecast-accumulate
// epilogue (fast_epilogue) follows; the kernel is instantiated per C
// storage datatype.  A CTA works through the segment list of common.cuh
// (one tile, a split-K slice, or a stream-K range).
#include <cstdlib>

#include "common.cuh"

namespace mdg {
namespace {

template <int BM_, int BN_, int STAGES_, int MINB_, int EPI_ESZ = 8>
struct FfmaCfg {
  static constexpr int BM = BM_, BN = BN_, STAGES = STAGES_, MINB = MINB_;
  static constexpr int BK = 16;
  static constexpr int TYM = BM / 8, TXN = BN / 8;
  static constexpr int NCT = TYM * TXN;  // compute threads
  static constexpr int NCW = NCT / 32;
  static constexpr int THREADS = NCT + 32;
  static constexpr int STAGE_A = BK * BM, STAGE_B = BK * BN;  // floats
  static constexpr size_t RING_BYTES = size_t(STAGES) * (STAGE_A + STAGE_B) * sizeof(float);
  // epilogue: the staged accumulator tile (EPI_ESZ = bytes per real element
  // of C's storage) plus a C chunk buffer of at least 16 columns
  static constexpr size_t EPI_BYTES = size_t(BM) * BN * EPI_ESZ + size_t(BM) * EPI_ESZ * 16;
  static constexpr size_t REGION = RING_BYTES > EPI_BYTES ? RING_BYTES : EPI_BYTES;
  // full[STAGES], empty[STAGES], C-chunk barrier, segment-done barrier
  static constexpr size_t SMEM = REGION + (2 * STAGES + 2) * sizeof(uint64_t);
  static_assert(NCT % 32 == 0, "compute threads must be whole warps");
};

template <class C, int CDT, bool SK>
__global__ void __launch_bounds__(C::THREADS, C::MINB) gemm_ffma_kernel(const __grid_constant__ GemmDesc d) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* sA = reinterpret_cast<float*>(smem);
  float* sB = sA + C::STAGES * C::STAGE_A;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::REGION);
  uint64_t* empty = full + C::STAGES;
  uint64_t* cbar = empty + C::STAGES;  // C-chunk load completion
  uint64_t* segdone = cbar + 1;        // consumers finished an epilogue: the ring may be refilled

  const int tiles_m = static_cast<int>((d.me + C::BM - 1) / C::BM);
  const int tiles_n = static_cast<int>((d.ne + C::BN - 1) / C::BN);
  const int64_t tiles = static_cast<int64_t>(tiles_m) * tiles_n;
  const int64_t lpad = d.a.lpad;
  const Sched sc = make_sched<SK>(d, tiles, static_cast<int>(lpad / C::BK), SK ? logical_cta(sk_ticket(d)) : 0);

  const int tid = threadIdx.x;
  const unsigned long long t_start = d.trace ? globaltimer() : 0;
  unsigned long long t_first = 0, t_loop = 0;
  // The producer sets up the barriers and starts streaming without waiting
  // for the consumers (a CTA that starts next to busy ones gets few issue
  // slots; the first TMA copies should not queue behind its whole prologue).
  if (tid >= C::NCT) {  // ---------------- producer warp
    if (tid == C::NCT) {
      for (int s = 0; s < C::STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], C::NCW);
      }
      mbar_init(cbar, 1);
      mbar_init(segdone, 1);
      mbar_fence_init();
    }
    __syncwarp();
    named_arrive(2, C::THREADS);
    if (tid == C::NCT) {
      int it = 0, epis = 0;
      bool after_epilogue = false;
      for (int si = 0; si < sc.nseg; ++si) {
        const Seg sg = sched_seg<SK>(sc, d, si);
        if (after_epilogue) mbar_wait(segdone, (epis++) & 1);  // the epilogue reused the ring's memory
        int tm, tn;
        tile_coords(sg.tile, tiles_m, tiles_n, d.group_rows, tm, tn);
        MDG_CHECK(tm >= 0 && tm < tiles_m && tn >= 0 && tn < tiles_n && sg.k0 >= 0 && sg.k0 <= sg.k1 &&
                      static_cast<int64_t>(sg.k1) * C::BK <= lpad,
                  "producer tile / k-block range");
        const float* Ag = static_cast<const float*>(d.a.data) + static_cast<int64_t>(tm) * C::BM * lpad;
        const float* Bg = static_cast<const float*>(d.b.data) + static_cast<int64_t>(tn) * C::BN * lpad;
        for (int kb = sg.k0; kb < sg.k1; ++kb, ++it) {
          const int s = it % C::STAGES;
          if (d.prefetch > 0 && kb + d.prefetch < sg.k1) {
            const int64_t pk = static_cast<int64_t>(kb + d.prefetch);
            bulk_prefetch_l2(Ag + pk * C::STAGE_A, C::STAGE_A * sizeof(float));
            bulk_prefetch_l2(Bg + pk * C::STAGE_B, C::STAGE_B * sizeof(float));
          }
          if (it >= C::STAGES) mbar_wait(&empty[s], ((it / C::STAGES) - 1) & 1);
          if (d.trace && it == 0) d.trace[static_cast<size_t>(blockIdx.x) * TRACE_WORDS + 5] = globaltimer();
          mbar_arrive_expect_tx(&full[s], (C::STAGE_A + C::STAGE_B) * sizeof(float));
          bulk_g2s(sA + s * C::STAGE_A, Ag + static_cast<int64_t>(kb) * C::STAGE_A, C::STAGE_A * sizeof(float),
                   &full[s]);
          bulk_g2s(sB + s * C::STAGE_B, Bg + static_cast<int64_t>(kb) * C::STAGE_B, C::STAGE_B * sizeof(float),
                   &full[s]);
        }
        after_epilogue = sg.kind == SEG_FULL || sg.kind == SEG_END;
        if (d.c_prefetch && after_epilogue)
          prefetch_c_tile<CDT>(d.epi, static_cast<int64_t>(tm) * C::BM, static_cast<int64_t>(tn) * C::BN, C::BM, C::BN);
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  named_sync(2, C::THREADS);  // the producer has initialised the barriers
  // acc[i][p] holds the column pair (2p, 2p+1) of register-tile row i; one
  // FFMA2 updates a pair with A's element broadcast, so the 64 multiply-adds
  // per inner step cost 32 issue slots.
  const int tx = tid % C::TXN, ty = tid / C::TXN;
  const int lane = tid & 31;
  const uint32_t full_u = smem_u32(full), empty_u = smem_u32(empty);
  const float* a_base = sA + ty * 4;
  const float* b_base = sB + tx * 4;
  uint32_t cphase = 0;
  int it = 0;
  for (int si = 0; si < sc.nseg; ++si) {
    const Seg sg = sched_seg<SK>(sc, d, si);
    uint64_t acc[8][4];
    if (SK && sg.kind == SEG_END) {  // continue CTA b-1's accumulation of this tile
      const int prev = sc.sk - 1;
      check_sk_slot(prev, d.sk_grid);
      if (tid == 0) flag_acquire_wait(d.sk_flags + prev);
      named_sync(1, C::NCT);
      const uint64_t* slot =
          static_cast<const uint64_t*>(d.sk_partials) + static_cast<int64_t>(prev) * (C::BM * C::BN / 2);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int p = 0; p < 4; ++p) acc[i][p] = __ldcg(slot + (i * 4 + p) * C::NCT + tid);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int p = 0; p < 4; ++p) acc[i][p] = 0ull;
    }

    for (int kb = sg.k0; kb < sg.k1; ++kb, ++it) {
      const int s = it % C::STAGES;
      mbar_wait_u32(full_u + 8 * s, (it / C::STAGES) & 1);
      if (d.trace && it == 0) t_first = globaltimer();
      const float* a = a_base + s * C::STAGE_A;
      const float* b = b_base + s * C::STAGE_B;
#pragma unroll
      for (int kk = 0; kk < C::BK; ++kk) {
        const float4 a0 = *reinterpret_cast<const float4*>(a + kk * C::BM);
        const float4 a1 = *reinterpret_cast<const float4*>(a + kk * C::BM + C::BM / 2);
        const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(b + kk * C::BN);
        const ulonglong2 b1 = *reinterpret_cast<const ulonglong2*>(b + kk * C::BN + C::BN / 2);
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
      // The stage was read through the generic proxy (LDS); the producer's next
      // TMA write into it goes through the async proxy.  Order the two before
      // releasing the slot (without this fence the refill can land before the
      // reads complete: a cross-proxy WAR race).
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive_u32(empty_u + 8 * s);
    }
    if (d.trace) t_loop = globaltimer();

    if (SK && sg.kind == SEG_START) {  // publish the first k-blocks of the tile for CTA b+1
      const int self = sc.sk;
      check_sk_slot(self, d.sk_grid);
      uint64_t* slot = static_cast<uint64_t*>(d.sk_partials) + static_cast<int64_t>(self) * (C::BM * C::BN / 2);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int p = 0; p < 4; ++p) __stcg(slot + (i * 4 + p) * C::NCT + tid, acc[i][p]);
      __threadfence();
      named_sync(1, C::NCT);
      if (tid == 0) flag_release(d.sk_flags + self);
      continue;
    }
    int tm, tn;
    tile_coords(sg.tile, tiles_m, tiles_n, d.group_rows, tm, tn);
    if (!SK && sg.kind == SEG_SPLIT) {  // split-K: this CTA's partial tile, column-major, for the reduce pass
      const int split = static_cast<int>(blockIdx.x / tiles);
      float* part = static_cast<float*>(d.partials) + (split * tiles + sg.tile) * (C::BM * C::BN);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = j < 4 ? tx * 4 + j : C::BN / 2 + tx * 4 + (j - 4);
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          v[i] = __uint_as_float(static_cast<uint32_t>((j & 1) ? (acc[i][j >> 1] >> 32) : acc[i][j >> 1]));
        *reinterpret_cast<float4*>(&part[c * C::BM + ty * 4]) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4*>(&part[c * C::BM + C::BM / 2 + ty * 4]) = make_float4(v[4], v[5], v[6], v[7]);
      }
      continue;
    }
    named_sync(1, C::NCT);  // every consumer is done with the ring
    // Stream-K: epilogue parameters through an opaque pointer (no hoisting
    // out of the segment loop, see gemm_dmma.cu).
    const DEpilogue* ep = &d.epi;
    if (SK) asm volatile("" : "+l"(ep));
    fast_epilogue<CDT>(smem, static_cast<uint32_t>(C::REGION), cbar, *ep, static_cast<int64_t>(tm) * C::BM,
                       static_cast<int64_t>(tn) * C::BN, C::BM, C::BN, tid, C::NCT, cphase, [&](auto&& put) {
#pragma unroll
                         for (int i = 0; i < 8; ++i) {
                           const int r = i < 4 ? ty * 4 + i : C::BM / 2 + ty * 4 + (i - 4);
#pragma unroll
                           for (int j = 0; j < 8; ++j) {
                             const int c = j < 4 ? tx * 4 + j : C::BN / 2 + tx * 4 + (j - 4);
                             const uint64_t v = acc[i][j >> 1];
                             put(r, c, __uint_as_float(static_cast<uint32_t>((j & 1) ? (v >> 32) : v)));
                           }
                         }
                       });
    if (SK && si + 1 < sc.nseg) {  // hand the shared memory back to the producer
      fence_proxy_async();
      named_sync(1, C::NCT);
      if (tid == 0) mbar_arrive(segdone);
    }
  }
  if (d.trace && tid == 0) trace_stamp(d.trace, t_start, t_first, t_loop);
}

using Big = FfmaCfg<128, 128, 8, 1>;
using Pair = FfmaCfg<64, 128, 8, 2>;  // two CTAs per SM: epilogues overlap mainloops
// Three CTAs per SM (72 KB each): a 6-stage ring, and an epilogue that stages
// the tile in C's storage precision with a C chunk buffer of >= 16 columns.
using Pair3 = FfmaCfg<64, 128, 6, 3, 4>;   // single-precision C
using Pair3d = FfmaCfg<64, 128, 6, 3, 8>;  // double-precision C
using Small = FfmaCfg<64, 64, 6, 4>;

// The configuration a tile shape runs with for C's storage datatype.
template <class C, int CDT>
using CfgFor = typename std::conditional<
    (C::BM == 64 && C::BN == 128),
    typename std::conditional<(CDT == MDG_DT_S || CDT == MDG_DT_C), Pair3, Pair3d>::type, C>::type;

template <class C>
cudaError_t run(const GemmDesc& d, cudaStream_t s) {
  const int64_t tiles = ((d.me + C::BM - 1) / C::BM) * ((d.ne + C::BN - 1) / C::BN);
  if (tiles == 0) return cudaSuccess;
  const int64_t grid =
      d.sk_grid > 0 ? sk_launch_grid(tiles, d.sk_grid) : tiles * (d.splits > 1 ? d.splits : 1);
  cudaError_t e = cudaSuccess;
  MDG_DISPATCH_CDT(d.epi.out.dtype, CDT, {
    using K = CfgFor<C, CDT>;
    auto kern = d.sk_grid > 0 ? gemm_ffma_kernel<K, CDT, true> : gemm_ffma_kernel<K, CDT, false>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(K::SMEM));
    if (e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>(grid), K::THREADS, K::SMEM, s>>>(d);
  });
  return cudaGetLastError();
}

template <class C>
int ctas_per_sm(int cdt) {
  int n = 0;
  MDG_DISPATCH_CDT(cdt, CDT, {
    using K = CfgFor<C, CDT>;
    if (cudaFuncSetAttribute(gemm_ffma_kernel<K, CDT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(K::SMEM)) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, gemm_ffma_kernel<K, CDT, false>, K::THREADS, K::SMEM) !=
            cudaSuccess)
      n = 1;
  });
  return n > 0 ? n : 1;
}

}  // namespace

int ffma_ctas_per_sm(const FastTile& t, int cdt) {
  if (t.bm == 128 && t.bn == 128) return ctas_per_sm<Big>(cdt);
  if (t.bm == 64 && t.bn == 128) return ctas_per_sm<Pair>(cdt);
  return ctas_per_sm<Small>(cdt);
}

FastTile choose_ffma_tile(int64_t me, int64_t ne, int sms) {
  if (const char* force = std::getenv("MDGEMM_FFMA_TILE")) {  // tuning override: 64 | 128 | 64128
    const int t = std::atoi(force);
    if (t == 64 || t == 128) return FastTile{t, t, 16};
    if (t == 64128) return FastTile{64, 128, 16};
  }
  // 64x128 (two CTAs per SM, epilogue of one under the other's mainloop) up
  // to 8192^2 outputs; beyond that the 128x128 tile's lower operand traffic
  // per flop wins (measured: +2 % at 4096, -2 % at 16384).
  const int64_t pair = ((me + 63) / 64) * ((ne + 127) / 128);
  if (pair >= 4LL * sms && me * ne > 8192LL * 8192) return FastTile{128, 128, 16};
  if (pair >= 2LL * sms) return FastTile{64, 128, 16};
  return FastTile{64, 64, 16};
}

cudaError_t launch_gemm_ffma(const GemmDesc& d, const FastTile& t, cudaStream_t s) {
  if (t.bm == 128 && t.bn == 128) return run<Big>(d, s);
  if (t.bm == 64 && t.bn == 128) return run<Pair>(d, s);
  if (t.bm == 64 && t.bn == 64) return run<Small>(d, s);
  return cudaErrorInvalidValue;
}

}  // namespace mdg
