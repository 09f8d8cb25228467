// FAST numerics, computation precision double: the real microkernel of the
// reference (ukr_impl<double>, kernels.cpp:7-40) as an sm_100a CTA tile on
// the FP64 tensor pipe.  tcgen05 has no f64 kind, so the MMA is warp-level
// DMMA (mma.sync m8n8k4 .f64 -> SASS DMMA.8x8x4).
//
// Layout: the pack kernels write Ã / B̃ as panels of BM rows (BN columns)
// with one contiguous BM-vector (BN-vector) per inner step, so the BK x BM
// slab a stage needs is ONE contiguous block: a single cp.async.bulk (TMA
// bulk copy) per operand per stage, completing on an mbarrier.
//
// Warp roles: warp NCW (last) is the producer (one elected lane issues the
// bulk copies into a STAGES-deep ring); warps 0..NCW-1 consume.  After the
// k loop the ring is reused for the fused typecast-accumulate epilogue
// (fast_epilogue: accumulate_element semantics, kernels.cpp:79-95), which
// moves C through shared memory with TMA bulk copies.  The kernel is
// instantiated per C storage datatype (CDT) so the epilogue stays small.  A
// CTA works through the segment list of common.cuh (one tile, a split-K
// slice, or a stream-K range).
#include <cstdlib>

#include "common.cuh"

namespace mdg {
namespace {

template <int BM_, int BN_, int WM_, int WN_, int STAGES_, int MINB_ = 1>
struct DmmaCfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, STAGES = STAGES_, MINB = MINB_;
  static constexpr int BK = 16;
  static constexpr int NCW = WM * WN;
  static constexpr int NCT = NCW * 32;
  static constexpr int THREADS = (NCW + 1) * 32;
  static constexpr int WTM = BM / WM, WTN = BN / WN;
  static constexpr int MT = WTM / 8, NT = WTN / 8;
  static constexpr int STAGE_A = BK * BM, STAGE_B = BK * BN;  // doubles
  static constexpr size_t RING_BYTES = size_t(STAGES) * (STAGE_A + STAGE_B) * sizeof(double);
  // epilogue: the staged accumulator tile (<= 8 bytes per real element) plus
  // C chunks of at least half the tile
  static constexpr size_t EPI_BYTES = size_t(BM) * BN * sizeof(double) * 3 / 2;
  static constexpr size_t REGION = RING_BYTES > EPI_BYTES ? RING_BYTES : EPI_BYTES;
  // full[STAGES], empty[STAGES], C-chunk barrier, segment-done barrier
  static constexpr size_t SMEM = REGION + (2 * STAGES + 2) * sizeof(uint64_t);
  static_assert(WTM % 8 == 0 && WTN % 8 == 0, "warp tile must be a multiple of 8x8");
};

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <class C, int CDT, bool SK>
__global__ void __launch_bounds__(C::THREADS, C::MINB) gemm_dmma_kernel(const __grid_constant__ GemmDesc d) {
  extern __shared__ __align__(128) unsigned char smem[];
  double* sA = reinterpret_cast<double*>(smem);
  double* sB = sA + C::STAGES * C::STAGE_A;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::REGION);
  uint64_t* empty = full + C::STAGES;
  uint64_t* cbar = empty + C::STAGES;  // C-chunk load completion
  uint64_t* segdone = cbar + 1;        // consumers finished an epilogue: the ring may be refilled

  const int tiles_m = static_cast<int>((d.me + C::BM - 1) / C::BM);
  const int tiles_n = static_cast<int>((d.ne + C::BN - 1) / C::BN);
  const int64_t tiles = static_cast<int64_t>(tiles_m) * tiles_n;
  const int64_t lpad = d.a.lpad;
  const Sched sc = make_sched<SK>(d, tiles, static_cast<int>(lpad / C::BK), SK ? logical_cta(sk_ticket(d)) : 0);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned long long t_start = d.trace ? globaltimer() : 0;
  unsigned long long t_first = 0, t_loop = 0;
  // The producer sets up the barriers and starts streaming without waiting
  // for the consumers (see gemm_ffma.cu).
  if (warp == C::NCW) {  // ---------------- producer
    if (lane == 0) {
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
    if (lane == 0) {
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
        const double* Ag = static_cast<const double*>(d.a.data) + static_cast<int64_t>(tm) * C::BM * lpad;
        const double* Bg = static_cast<const double*>(d.b.data) + static_cast<int64_t>(tn) * C::BN * lpad;
        for (int kb = sg.k0; kb < sg.k1; ++kb, ++it) {
          const int s = it % C::STAGES;
          if (d.prefetch > 0 && kb + d.prefetch < sg.k1) {
            const int64_t pk = static_cast<int64_t>(kb + d.prefetch);
            bulk_prefetch_l2(Ag + pk * C::STAGE_A, C::STAGE_A * sizeof(double));
            bulk_prefetch_l2(Bg + pk * C::STAGE_B, C::STAGE_B * sizeof(double));
          }
          if (it >= C::STAGES) mbar_wait(&empty[s], ((it / C::STAGES) - 1) & 1);
          if (d.trace && it == 0) d.trace[static_cast<size_t>(blockIdx.x) * TRACE_WORDS + 5] = globaltimer();
          mbar_arrive_expect_tx(&full[s], (C::STAGE_A + C::STAGE_B) * sizeof(double));
          bulk_g2s(sA + s * C::STAGE_A, Ag + static_cast<int64_t>(kb) * C::STAGE_A, C::STAGE_A * sizeof(double),
                   &full[s]);
          bulk_g2s(sB + s * C::STAGE_B, Bg + static_cast<int64_t>(kb) * C::STAGE_B, C::STAGE_B * sizeof(double),
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
  const int wm = warp % C::WM, wn = warp / C::WM;
  const int g = lane >> 2, tig = lane & 3;
  const int tid = threadIdx.x;
  // (Register-double-buffered fragments do not fit: 10 warps per SM leave
  // 168 registers per thread and the 64x32 warp tile's accumulators take 128.)
  const uint32_t full_u = smem_u32(full), empty_u = smem_u32(empty);
  const double* a_base = sA + wm * C::WTM + g + tig * C::BM;
  const double* b_base = sB + wn * C::WTN + g + tig * C::BN;
  uint32_t cphase = 0;
  int it = 0;
  for (int si = 0; si < sc.nseg; ++si) {
    const Seg sg = sched_seg<SK>(sc, d, si);
    double acc[C::MT][C::NT][2];
    if (SK && sg.kind == SEG_END) {  // continue CTA b-1's accumulation of this tile
      const int prev = sc.sk - 1;
      check_sk_slot(prev, d.sk_grid);
      if (tid == 0) flag_acquire_wait(d.sk_flags + prev);
      named_sync(1, C::NCT);
      const double* slot = static_cast<const double*>(d.sk_partials) + static_cast<int64_t>(prev) * (C::BM * C::BN);
#pragma unroll
      for (int i = 0; i < C::MT; ++i)
#pragma unroll
        for (int j = 0; j < C::NT; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) acc[i][j][h] = __ldcg(slot + ((i * C::NT + j) * 2 + h) * C::NCT + tid);
    } else {
#pragma unroll
      for (int i = 0; i < C::MT; ++i)
#pragma unroll
        for (int j = 0; j < C::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    }

    for (int kb = sg.k0; kb < sg.k1; ++kb, ++it) {
      const int s = it % C::STAGES;
      mbar_wait_u32(full_u + 8 * s, (it / C::STAGES) & 1);
      if (d.trace && it == 0) t_first = globaltimer();
      const double* a = a_base + s * C::STAGE_A;
      const double* b = b_base + s * C::STAGE_B;
#pragma unroll
      for (int kk = 0; kk < C::BK; kk += 4) {
        double af[C::MT], bf[C::NT];
#pragma unroll
        for (int i = 0; i < C::MT; ++i) af[i] = a[kk * C::BM + i * 8];
#pragma unroll
        for (int j = 0; j < C::NT; ++j) bf[j] = b[kk * C::BN + j * 8];
#pragma unroll
        for (int i = 0; i < C::MT; ++i)
#pragma unroll
          for (int j = 0; j < C::NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
      // generic-proxy reads of the stage before its async-proxy (TMA) refill
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive_u32(empty_u + 8 * s);
    }
    if (d.trace) t_loop = globaltimer();

    if (SK && sg.kind == SEG_START) {  // publish the first k-blocks of the tile for CTA b+1
      const int self = sc.sk;
      check_sk_slot(self, d.sk_grid);
      double* slot = static_cast<double*>(d.sk_partials) + static_cast<int64_t>(self) * (C::BM * C::BN);
#pragma unroll
      for (int i = 0; i < C::MT; ++i)
#pragma unroll
        for (int j = 0; j < C::NT; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) __stcg(slot + ((i * C::NT + j) * 2 + h) * C::NCT + tid, acc[i][j][h]);
      __threadfence();
      named_sync(1, C::NCT);
      if (tid == 0) flag_release(d.sk_flags + self);
      continue;
    }
    int tm, tn;
    tile_coords(sg.tile, tiles_m, tiles_n, d.group_rows, tm, tn);
    if (!SK && sg.kind == SEG_SPLIT) {  // split-K: this CTA's partial tile, column-major, for the reduce pass
      const int split = static_cast<int>(blockIdx.x / tiles);
      double* part = static_cast<double*>(d.partials) + (split * tiles + sg.tile) * (C::BM * C::BN);
#pragma unroll
      for (int i = 0; i < C::MT; ++i)
#pragma unroll
        for (int j = 0; j < C::NT; ++j) {
          const int r = wm * C::WTM + i * 8 + g;
          const int c = wn * C::WTN + j * 8 + 2 * tig;
          part[c * C::BM + r] = acc[i][j][0];
          part[(c + 1) * C::BM + r] = acc[i][j][1];
        }
      continue;
    }
    named_sync(1, C::NCT);  // every consumer is done with the ring
    // Stream-K: read the epilogue parameters through an opaque pointer so the
    // compiler cannot hoist them out of the segment loop (they would stay
    // live through the mainloop and push it into spills).
    const DEpilogue* ep = &d.epi;
    if (SK) asm volatile("" : "+l"(ep));
    fast_epilogue<CDT>(smem, static_cast<uint32_t>(C::REGION), cbar, *ep, static_cast<int64_t>(tm) * C::BM,
                       static_cast<int64_t>(tn) * C::BN, C::BM, C::BN, tid, C::NCT, cphase, [&](auto&& put) {
#pragma unroll
                         for (int i = 0; i < C::MT; ++i)
#pragma unroll
                           for (int j = 0; j < C::NT; ++j) {
                             const int r = wm * C::WTM + i * 8 + g;
                             const int c = wn * C::WTN + j * 8 + 2 * tig;
                             put(r, c, acc[i][j][0]);
                             put(r, c + 1, acc[i][j][1]);
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

template <class C>
cudaError_t run(const GemmDesc& d, cudaStream_t s) {
  const int64_t tiles = ((d.me + C::BM - 1) / C::BM) * ((d.ne + C::BN - 1) / C::BN);
  if (tiles == 0) return cudaSuccess;
  const int64_t grid =
      d.sk_grid > 0 ? sk_launch_grid(tiles, d.sk_grid) : tiles * (d.splits > 1 ? d.splits : 1);
  cudaError_t e = cudaSuccess;
  MDG_DISPATCH_CDT(d.epi.out.dtype, CDT, {
    auto kern = d.sk_grid > 0 ? gemm_dmma_kernel<C, CDT, true> : gemm_dmma_kernel<C, CDT, false>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::SMEM));
    if (e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>(grid), C::THREADS, C::SMEM, s>>>(d);
  });
  return cudaGetLastError();
}

using Big = DmmaCfg<128, 128, 2, 4, 4>;
// Two CTAs per SM (4 DMMA warps each, same 64x32 warp tiles): one CTA's
// epilogue overlaps the other's mainloop.
using Pair = DmmaCfg<64, 128, 1, 4, 4, 2>;
using Small = DmmaCfg<64, 64, 2, 2, 4, 3>;  // three per SM

template <class C>
int ctas_per_sm(int cdt) {
  int n = 0;
  MDG_DISPATCH_CDT(cdt, CDT, {
    if (cudaFuncSetAttribute(gemm_dmma_kernel<C, CDT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(C::SMEM)) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, gemm_dmma_kernel<C, CDT, false>, C::THREADS, C::SMEM) !=
            cudaSuccess)
      n = 1;
  });
  return n > 0 ? n : 1;
}

}  // namespace

int dmma_ctas_per_sm(const FastTile& t, int cdt) {
  if (t.bm == 128 && t.bn == 128) return ctas_per_sm<Big>(cdt);
  if (t.bm == 64 && t.bn == 128) return ctas_per_sm<Pair>(cdt);
  return ctas_per_sm<Small>(cdt);
}

FastTile choose_dmma_tile(int64_t me, int64_t ne, int sms) {
  if (const char* force = std::getenv("MDGEMM_DMMA_TILE")) {  // tuning override: 64 | 128 | 64128
    const int t = std::atoi(force);
    if (t == 64 || t == 128) return FastTile{t, t, 16};
    if (t == 64128) return FastTile{64, 128, 16};
  }
  // 64x128 tiles, two CTAs per SM (measured better than 128x128 at every
  // BASELINE shape), once they fill one wave (the driver runs a partial last
  // wave as stream-K); 64x64 (three per SM) for small problems.
  const int64_t pair = ((me + 63) / 64) * ((ne + 127) / 128);
  return pair >= 2LL * sms ? FastTile{64, 128, 16} : FastTile{64, 64, 16};
}

cudaError_t launch_gemm_dmma(const GemmDesc& d, const FastTile& t, cudaStream_t s) {
  if (t.bm == 128 && t.bn == 128) return run<Big>(d, s);
  if (t.bm == 64 && t.bn == 128) return run<Pair>(d, s);
  if (t.bm == 64 && t.bn == 64) return run<Small>(d, s);
  return cudaErrorInvalidValue;
}

}  // namespace mdg
