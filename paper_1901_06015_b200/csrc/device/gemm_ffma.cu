// FAST numerics, computation precision single: the reference's float
// microkernel (ukr_impl<float>, kernels.cpp:7-40) as an FP32 FFMA SIMT CTA
// tile.  No TF32: tensor cores would not reproduce fp32 products.
//
// Same feed as the DMMA kernel: a producer warp streams BK x BM / BK x BN
// slabs of the packed panels into a STAGES-deep shared-memory ring with one
// TMA bulk copy per operand per stage (mbarrier completion); the compute
// threads each own an 8x8 register tile split into two 4x4 quadrants
// ({ty*4, BM/2+ty*4} x {tx*4, BN/2+tx*4}) so every fragment is one
// conflict-free LDS.128.  The fused typecast-accumulate epilogue follows.
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
  static constexpr size_t SMEM = RING_BYTES + 2 * STAGES * sizeof(uint64_t);
  static_assert(NCT % 32 == 0, "compute threads must be whole warps");
  static_assert(size_t(BM) * BN * sizeof(float) <= RING_BYTES, "epilogue tile must fit the ring");
};

template <class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB) gemm_ffma_kernel(GemmDesc d) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* sA = reinterpret_cast<float*>(smem);
  float* sB = sA + C::STAGES * C::STAGE_A;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::RING_BYTES);
  uint64_t* empty = full + C::STAGES;

  const int tiles_m = static_cast<int>((d.me + C::BM - 1) / C::BM);
  const int tiles_n = static_cast<int>((d.ne + C::BN - 1) / C::BN);
  int tm, tn;
  tile_coords(blockIdx.x, tiles_m, tiles_n, tm, tn);
  const int64_t lpad = d.a.lpad;
  const int nk = static_cast<int>(lpad / C::BK);
  const float* Ag = static_cast<const float*>(d.a.data) + static_cast<int64_t>(tm) * C::BM * lpad;
  const float* Bg = static_cast<const float*>(d.b.data) + static_cast<int64_t>(tn) * C::BN * lpad;

  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NCW);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (tid >= C::NCT) {  // ---------------- producer warp
    if (tid == C::NCT) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::STAGES;
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
  // FFMA2 (fma.rn.f32x2) updates a pair with A's element broadcast, so the
  // 64 multiply-adds per inner step cost 32 issue slots.
  const int tx = tid % C::TXN, ty = tid / C::TXN;
  const int lane = tid & 31;
  uint64_t acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int p = 0; p < 4; ++p) acc[i][p] = 0ull;

  for (int kb = 0; kb < nk; ++kb) {
    const int s = kb % C::STAGES;
    mbar_wait(&full[s], (kb / C::STAGES) & 1);
    const float* a = sA + s * C::STAGE_A + ty * 4;
    const float* b = sB + s * C::STAGE_B + tx * 4;
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
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ------------------------------------------------------------ epilogue
  named_sync(1, C::NCT);
  float* T = reinterpret_cast<float*>(smem);  // BM x BN, column-major
  auto lo = [](uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v)); };
  auto hi = [](uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v >> 32)); };
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int c = (j < 4 ? tx * 4 + j : C::BN / 2 + tx * 4 + (j - 4));
    const int p = j >> 1;
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = (j & 1) ? hi(acc[i][p]) : lo(acc[i][p]);
    *reinterpret_cast<float4*>(&T[c * C::BM + ty * 4]) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(&T[c * C::BM + C::BM / 2 + ty * 4]) = make_float4(v[4], v[5], v[6], v[7]);
  }
  named_sync(1, C::NCT);
  tile_epilogue(T, C::BM, C::BM, C::BN, static_cast<int64_t>(tm) * C::BM,
                static_cast<int64_t>(tn) * C::BN, d.epi, tid, C::NCT);
}

template <class C>
cudaError_t run(const GemmDesc& d, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(gemm_ffma_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(C::SMEM));
  if (e != cudaSuccess) return e;
  const int64_t tiles = ((d.me + C::BM - 1) / C::BM) * ((d.ne + C::BN - 1) / C::BN);
  if (tiles == 0) return cudaSuccess;
  gemm_ffma_kernel<C><<<static_cast<unsigned>(tiles), C::THREADS, C::SMEM, s>>>(d);
  return cudaGetLastError();
}

using Big = FfmaCfg<128, 128, 4, 1>;
using Big2 = FfmaCfg<128, 128, 4, 2>;  // 2 CTAs/SM (register-capped)
using Small = FfmaCfg<64, 64, 4, 4>;

int big_variant() {
  static const int v = [] {
    const char* e = std::getenv("MDGEMM_FFMA_VARIANT");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

}  // namespace

FastTile choose_ffma_tile(int64_t me, int64_t ne, int sms) {
  const int64_t big = ((me + 127) / 128) * ((ne + 127) / 128);
  if (big >= 2LL * sms) return FastTile{128, 128, 16};
  return FastTile{64, 64, 16};
}

cudaError_t launch_gemm_ffma(const GemmDesc& d, const FastTile& t, cudaStream_t s) {
  if (t.bm == 128 && t.bn == 128) return big_variant() == 2 ? run<Big2>(d, s) : run<Big>(d, s);
  if (t.bm == 64 && t.bn == 64) return run<Small>(d, s);
  return cudaErrorInvalidValue;
}

}  // namespace mdg
