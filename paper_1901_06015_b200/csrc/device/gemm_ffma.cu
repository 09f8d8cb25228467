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
// storage datatype.
#include <cstdlib>

#include "common.cuh"

namespace mdg {
namespace {

template <int BM_, int BN_, int STAGES_, int MINB_>
struct FfmaCfg {
  static constexpr int BM = BM_, BN = BN_, STAGES = STAGES_, MINB = MINB_;
  static constexpr int BK = 16;
  static constexpr int TYM = BM / 8, TXN = BN / 8;
  static constexpr int NCT = TYM * TXN;  // compute threads
  static constexpr int NCW = NCT / 32;
  static constexpr int THREADS = NCT + 32;
  static constexpr int STAGE_A = BK * BM, STAGE_B = BK * BN;  // floats
  static constexpr size_t RING_BYTES = size_t(STAGES) * (STAGE_A + STAGE_B) * sizeof(float);
  // epilogue: the staged accumulator tile (<= 8 bytes per real element) plus
  // C chunks of at least half the tile
  static constexpr size_t EPI_BYTES = size_t(BM) * BN * sizeof(double) * 3 / 2;
  static constexpr size_t REGION = RING_BYTES > EPI_BYTES ? RING_BYTES : EPI_BYTES;
  static constexpr size_t SMEM = REGION + (2 * STAGES + 1) * sizeof(uint64_t);
  static_assert(NCT % 32 == 0, "compute threads must be whole warps");
};

template <class C, int CDT>
__global__ void __launch_bounds__(C::THREADS, C::MINB) gemm_ffma_kernel(GemmDesc d) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* sA = reinterpret_cast<float*>(smem);
  float* sB = sA + C::STAGES * C::STAGE_A;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::REGION);
  uint64_t* empty = full + C::STAGES;
  uint64_t* cbar = empty + C::STAGES;  // C-chunk load completion

  const int tiles_m = static_cast<int>((d.me + C::BM - 1) / C::BM);
  const int tiles_n = static_cast<int>((d.ne + C::BN - 1) / C::BN);
  const int64_t tiles = static_cast<int64_t>(tiles_m) * tiles_n;
  const int split = static_cast<int>(blockIdx.x / tiles);  // split-K slice of this CTA
  const int64_t tile_id = blockIdx.x % tiles;
  int tm, tn;
  tile_coords(tile_id, tiles_m, tiles_n, d.group_rows, tm, tn);
  const int64_t lpad = d.a.lpad;
  const int nk_all = static_cast<int>(lpad / C::BK);
  const int kb0 = d.splits > 1 ? split * d.kb_per_split : 0;
  const int nk = d.splits > 1 ? min(nk_all - kb0, d.kb_per_split) : nk_all;
  const float* Ag = static_cast<const float*>(d.a.data) + static_cast<int64_t>(tm) * C::BM * lpad +
                    static_cast<int64_t>(kb0) * C::STAGE_A;
  const float* Bg = static_cast<const float*>(d.b.data) + static_cast<int64_t>(tn) * C::BN * lpad +
                    static_cast<int64_t>(kb0) * C::STAGE_B;

  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NCW);
    }
    mbar_init(cbar, 1);
    mbar_fence_init();
  }
  __syncthreads();

  if (tid >= C::NCT) {  // ---------------- producer warp
    if (tid == C::NCT) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::STAGES;
        if (d.prefetch > 0 && kb + d.prefetch < nk) {
          const int64_t pk = static_cast<int64_t>(kb + d.prefetch);
          bulk_prefetch_l2(Ag + pk * C::STAGE_A, C::STAGE_A * sizeof(float));
          bulk_prefetch_l2(Bg + pk * C::STAGE_B, C::STAGE_B * sizeof(float));
        }
        if (kb >= C::STAGES) mbar_wait(&empty[s], ((kb / C::STAGES) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], (C::STAGE_A + C::STAGE_B) * sizeof(float));
        bulk_g2s(sA + s * C::STAGE_A, Ag + static_cast<int64_t>(kb) * C::STAGE_A,
                 C::STAGE_A * sizeof(float), &full[s]);
        bulk_g2s(sB + s * C::STAGE_B, Bg + static_cast<int64_t>(kb) * C::STAGE_B,
                 C::STAGE_B * sizeof(float), &full[s]);
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  // acc[i][p] holds the column pair (2p, 2p+1) of register-tile row i; one
  // FFMA2 updates a pair with A's element broadcast, so the 64 multiply-adds
  // per inner step cost 32 issue slots.
  const int tx = tid % C::TXN, ty = tid / C::TXN;
  const int lane = tid & 31;
  uint64_t acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int p = 0; p < 4; ++p) acc[i][p] = 0ull;

  const uint32_t full_u = smem_u32(full), empty_u = smem_u32(empty);
  const float* a_base = sA + ty * 4;
  const float* b_base = sB + tx * 4;
  for (int kb = 0; kb < nk; ++kb) {
    const int s = kb % C::STAGES;
    mbar_wait_u32(full_u + 8 * s, (kb / C::STAGES) & 1);
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

  // ------------------------------------------------------------ epilogue
  if (d.splits > 1) {  // split-K: this CTA's partial tile, column-major, for the reduce pass
    float* part = static_cast<float*>(d.partials) + (split * tiles + tile_id) * (C::BM * C::BN);
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
    return;
  }
  named_sync(1, C::NCT);  // every consumer is done with the ring
  fast_epilogue<CDT>(smem, static_cast<uint32_t>(C::REGION), cbar, d.epi, static_cast<int64_t>(tm) * C::BM,
                     static_cast<int64_t>(tn) * C::BN, C::BM, C::BN, tid, C::NCT, [&](auto&& put) {
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
}

template <class C>
cudaError_t run(const GemmDesc& d, cudaStream_t s) {
  const int64_t tiles = ((d.me + C::BM - 1) / C::BM) * ((d.ne + C::BN - 1) / C::BN);
  if (tiles == 0) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  MDG_DISPATCH_CDT(d.epi.out.dtype, CDT, {
    e = cudaFuncSetAttribute(gemm_ffma_kernel<C, CDT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(C::SMEM));
    if (e != cudaSuccess) return e;
    gemm_ffma_kernel<C, CDT><<<static_cast<unsigned>(tiles * (d.splits > 1 ? d.splits : 1)), C::THREADS, C::SMEM,
                               s>>>(d);
  });
  return cudaGetLastError();
}

using Big = FfmaCfg<128, 128, 8, 1>;
using Pair = FfmaCfg<64, 128, 8, 2>;  // two CTAs per SM: epilogues overlap mainloops
using Small = FfmaCfg<64, 64, 6, 4>;

}  // namespace

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
