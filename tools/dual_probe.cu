// Dual-pipe probe: the REAL mainloops of the DMMA kernel (TMA bulk ring +
// LDS fragments + DMMA.8x8x4) and of the FFMA2 kernel (TMA ring + LDS.128 +
// FFMA2 8x8 register tiles) running side by side in one persistent CTA per
// SM, each warp group on its own tile stream with its own producer lane and
// ring.  No epilogue (accumulators are folded into a sink).  Answers: how
// much of the serialized FP64 + FP32 time does co-residency on one SM save
// with real operand traffic, not register-only loops (tools/peaks mix)?
//
//   dual_probe            -> one line per configuration:
//   cfg  D-only TF/s  F-only TF/s  dual: D TF/s, F TF/s, serialized-equivalent speed-up
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

#include "../paper_1901_06015_b200/csrc/device/common.cuh"

using namespace mdg;

namespace {

constexpr int BK = 16;

template <int ND, int DWM, int NF, int DSTAGES, int FSTAGES, int RD, int RF, int RP>
struct Cfg {
  static constexpr int D_WN = 4, D_WM = ND / D_WN;  // warps: D_WM x 4, warp tile DWM x 32
  static constexpr int BM_D = DWM * (D_WM > 0 ? D_WM : 1), BN_D = 128;
  static constexpr int BM_F = NF * 16, BN_F = 128;  // NF*32 threads as (NF*2) x 16, 8x8 each
  static constexpr int SA_D = BK * BM_D, SB_D = BK * BN_D;  // doubles per stage
  static constexpr int SA_F = BK * BM_F, SB_F = BK * BN_F;  // floats per stage
  static constexpr size_t RING_D = size_t(DSTAGES) * (SA_D + SB_D) * 8;
  static constexpr size_t RING_F = size_t(FSTAGES) * (SA_F + SB_F) * 4;
  static constexpr int WG_D = (ND + 3) / 4, WG_F = (NF + 3) / 4;
  static constexpr int WARPS = 4 * (WG_D + WG_F + 1);  // + one producer warpgroup
  static constexpr int THREADS = WARPS * 32;
  static constexpr size_t SMEM = RING_D + RING_F + (2 * DSTAGES + 2 * FSTAGES) * 8;
};

struct Prob {
  const void* a;
  const void* b;
  int tiles_m, tiles_n, nk;  // lpad = nk * BK
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int ND, int DWM, int NF, int DSTAGES, int FSTAGES, int RD, int RF, int RP>
__global__ void __launch_bounds__(Cfg<ND, DWM, NF, DSTAGES, FSTAGES, RD, RF, RP>::THREADS, 1)
    dual_kernel(Prob pd, Prob pf, double* sink, unsigned long long* t_end) {
  using C = Cfg<ND, DWM, NF, DSTAGES, FSTAGES, RD, RF, RP>;
  extern __shared__ __align__(128) unsigned char smem[];
  double* dA = reinterpret_cast<double*>(smem);
  double* dB = dA + DSTAGES * C::SA_D;
  float* fA = reinterpret_cast<float*>(smem + C::RING_D);
  float* fB = fA + FSTAGES * C::SA_F;
  uint64_t* dfull = reinterpret_cast<uint64_t*>(smem + C::RING_D + C::RING_F);
  uint64_t* dempty = dfull + DSTAGES;
  uint64_t* ffull = dempty + DSTAGES;
  uint64_t* fempty = ffull + FSTAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wg = warp >> 2;
  const int G = gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < DSTAGES; ++s) {
      mbar_init(&dfull[s], 1);
      mbar_init(&dempty[s], ND > 0 ? ND : 1);
    }
    for (int s = 0; s < FSTAGES; ++s) {
      mbar_init(&ffull[s], 1);
      mbar_init(&fempty[s], NF > 0 ? NF : 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int tiles_d = pd.tiles_m * pd.tiles_n, tiles_f = pf.tiles_m * pf.tiles_n;

  if (wg == C::WG_D + C::WG_F) {  // ------------------------------------ producers
    if constexpr (RP > 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(RP));
    if (warp == 4 * (C::WG_D + C::WG_F) && lane == 0 && ND > 0) {
      int it = 0;
      for (int t = blockIdx.x; t < tiles_d; t += G) {
        const int tm = t % pd.tiles_m, tn = t / pd.tiles_m;
        const int64_t lpad = int64_t(pd.nk) * BK;
        const double* Ag = static_cast<const double*>(pd.a) + int64_t(tm) * C::BM_D * lpad;
        const double* Bg = static_cast<const double*>(pd.b) + int64_t(tn) * C::BN_D * lpad;
        for (int kb = 0; kb < pd.nk; ++kb, ++it) {
          const int s = it % DSTAGES;
          if (it >= DSTAGES) mbar_wait(&dempty[s], ((it / DSTAGES) - 1) & 1);
          mbar_arrive_expect_tx(&dfull[s], (C::SA_D + C::SB_D) * 8);
          bulk_g2s(dA + s * C::SA_D, Ag + int64_t(kb) * C::SA_D, C::SA_D * 8, &dfull[s]);
          bulk_g2s(dB + s * C::SB_D, Bg + int64_t(kb) * C::SB_D, C::SB_D * 8, &dfull[s]);
        }
      }
    }
    if (warp == 4 * (C::WG_D + C::WG_F) + 1 && lane == 0 && NF > 0) {
      int it = 0;
      for (int t = blockIdx.x; t < tiles_f; t += G) {
        const int tm = t % pf.tiles_m, tn = t / pf.tiles_m;
        const int64_t lpad = int64_t(pf.nk) * BK;
        const float* Ag = static_cast<const float*>(pf.a) + int64_t(tm) * C::BM_F * lpad;
        const float* Bg = static_cast<const float*>(pf.b) + int64_t(tn) * C::BN_F * lpad;
        for (int kb = 0; kb < pf.nk; ++kb, ++it) {
          const int s = it % FSTAGES;
          if (it >= FSTAGES) mbar_wait(&fempty[s], ((it / FSTAGES) - 1) & 1);
          mbar_arrive_expect_tx(&ffull[s], (C::SA_F + C::SB_F) * 4);
          bulk_g2s(fA + s * C::SA_F, Ag + int64_t(kb) * C::SA_F, C::SA_F * 4, &ffull[s]);
          bulk_g2s(fB + s * C::SB_F, Bg + int64_t(kb) * C::SB_F, C::SB_F * 4, &ffull[s]);
        }
      }
    }
    return;
  }

  if (wg < C::WG_D) {  // ------------------------------------------------ DMMA warps
    if constexpr (RD > 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(RD));
    if constexpr (ND > 0) {
      if (warp >= ND) return;
      constexpr int MT = DWM / 8, NT = 4;
      const int wm = warp % C::D_WM, wn = warp / C::D_WM;
      const int g = lane >> 2, tig = lane & 3;
      const double* a_base = dA + wm * DWM + g + tig * C::BM_D;
      const double* b_base = dB + wn * 32 + g + tig * C::BN_D;
      const uint32_t full_u = smem_u32(dfull), empty_u = smem_u32(dempty);
      double keep = 0.0;
      int it = 0;
      for (int t = blockIdx.x; t < tiles_d; t += G) {
        double acc[MT][NT][2];
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        for (int kb = 0; kb < pd.nk; ++kb, ++it) {
          const int s = it % DSTAGES;
          mbar_wait_u32(full_u + 8 * s, (it / DSTAGES) & 1);
          const double* a = a_base + s * C::SA_D;
          const double* b = b_base + s * C::SB_D;
#pragma unroll
          for (int kk = 0; kk < BK; kk += 4) {
            double af[MT], bf[NT];
#pragma unroll
            for (int i = 0; i < MT; ++i) af[i] = a[kk * C::BM_D + i * 8];
#pragma unroll
            for (int j = 0; j < NT; ++j) bf[j] = b[kk * C::BN_D + j * 8];
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
              for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive_u32(empty_u + 8 * s);
        }
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) keep += acc[i][j][0] + acc[i][j][1];
      }
      if (keep == 12345.678) sink[threadIdx.x] = keep;
      __syncwarp();
      if (lane == 0) atomicMax(&t_end[0], globaltimer());
    }
    return;
  }

  // ------------------------------------------------------------------ FFMA warps
  if constexpr (RF > 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(RF));
  if constexpr (NF > 0) {
    const int ft = threadIdx.x - 128 * C::WG_D;
    if (ft >= NF * 32) return;
    const int tx = ft % 16, ty = ft / 16;
    const float* a_base = fA + ty * 4;
    const float* b_base = fB + tx * 4;
    const uint32_t full_u = smem_u32(ffull), empty_u = smem_u32(fempty);
    float keep = 0.f;
    int it = 0;
    for (int t = blockIdx.x; t < tiles_f; t += G) {
      uint64_t acc[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int p = 0; p < 4; ++p) acc[i][p] = 0ull;
      for (int kb = 0; kb < pf.nk; ++kb, ++it) {
        const int s = it % FSTAGES;
        mbar_wait_u32(full_u + 8 * s, (it / FSTAGES) & 1);
        const float* a = a_base + s * C::SA_F;
        const float* b = b_base + s * C::SB_F;
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
          const float4 a0 = *reinterpret_cast<const float4*>(a + kk * C::BM_F);
          const float4 a1 = *reinterpret_cast<const float4*>(a + kk * C::BM_F + C::BM_F / 2);
          const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(b + kk * C::BN_F);
          const ulonglong2 b1 = *reinterpret_cast<const ulonglong2*>(b + kk * C::BN_F + C::BN_F / 2);
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
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(empty_u + 8 * s);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int p = 0; p < 4; ++p) keep += __uint_as_float(static_cast<uint32_t>(acc[i][p]));
    }
    if (keep == 12345.678f) sink[threadIdx.x] = keep;
    __syncwarp();
    if (lane == 0) atomicMax(&t_end[1], globaltimer());
  }
}

struct Result {
  float ms;
  double d_tf, f_tf;
};

template <int ND, int DWM, int NF, int DSTAGES, int FSTAGES, int RD, int RF, int RP>
Result run(int sms, const Prob& pd, const Prob& pf, double* sink, unsigned long long* t_end) {
  using C = Cfg<ND, DWM, NF, DSTAGES, FSTAGES, RD, RF, RP>;
  auto k = dual_kernel<ND, DWM, NF, DSTAGES, FSTAGES, RD, RF, RP>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  unsigned long long t0h;
  float best = 1e30f;
  unsigned long long best_end[2] = {0, 0}, best_start = 0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaMemset(t_end, 0, 3 * sizeof(unsigned long long));
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    k<<<sms, C::THREADS, C::SMEM>>>(pd, pf, sink, t_end);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (cudaGetLastError() != cudaSuccess) {
      printf("launch failed\n");
      exit(1);
    }
    if (ms < best) {
      best = ms;
      cudaMemcpy(best_end, t_end, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    }
  }
  (void)t0h;
  (void)best_start;
  const double fd = 2.0 * pd.tiles_m * C::BM_D * double(pd.tiles_n) * C::BN_D * pd.nk * BK;
  const double ff = 2.0 * pf.tiles_m * C::BM_F * double(pf.tiles_n) * C::BN_F * pf.nk * BK;
  // group end times relative to the earlier group's end: rates over the kernel time for the
  // group finishing last, and scaled for the earlier one
  Result r{best, 0, 0};
  const double dt = (double(best_end[0]) - double(best_end[1])) * 1e-6;  // ms, D end - F end
  double td = best, tf = best;
  if (ND > 0 && NF > 0) {
    if (dt > 0) tf = best - dt;
    else td = best + dt;
  }
  r.d_tf = ND > 0 ? fd / (td * 1e-3) / 1e12 : 0;
  r.f_tf = NF > 0 ? ff / (tf * 1e-3) / 1e12 : 0;
  return r;
}

template <int ND, int DWM, int NF, int DSTAGES, int FSTAGES, int RD, int RF, int RP>
void config(const char* name, int sms, void* bufd_a, void* bufd_b, void* buff_a, void* buff_b, double* sink,
            unsigned long long* t_end, int nk, int waves_d, int waves_f) {
  using C = Cfg<ND, DWM, NF, DSTAGES, FSTAGES, RD, RF, RP>;
  Prob pd{bufd_a, bufd_b, sms, waves_d, nk};  // tiles_m = sms: every CTA one tile per wave
  Prob pf{buff_a, buff_b, sms, waves_f, nk};
  Prob none{bufd_a, bufd_b, 0, 0, nk};
  const Result rd = run<ND, DWM, NF, DSTAGES, FSTAGES, RD, RF, RP>(sms, pd, none, sink, t_end);
  const Result rf = run<ND, DWM, NF, DSTAGES, FSTAGES, RD, RF, RP>(sms, none, pf, sink, t_end);
  const Result rb = run<ND, DWM, NF, DSTAGES, FSTAGES, RD, RF, RP>(sms, pd, pf, sink, t_end);
  // serialized time at the solo rates of this kernel, and at the measured pipe peaks
  const double serial = rd.ms + rf.ms;
  const double fd = 2.0 * sms * C::BM_D * double(waves_d) * C::BN_D * nk * BK;
  const double ff = 2.0 * sms * C::BM_F * double(waves_f) * C::BN_F * nk * BK;
  const double ideal_serial_ms = (fd / 37.0e12 + ff / 72.0e12) * 1e3;
  printf("%-28s threads %4d smem %6zu | D-only %6.2f TF/s  F-only %6.2f TF/s | dual %7.3f ms: D %6.2f F %6.2f TF/s"
         " | serial(solo) %7.3f ms -> x%.3f | serial(peaks) %7.3f ms -> x%.3f\n",
         name, C::THREADS, C::SMEM, rd.d_tf, rf.f_tf, rb.ms, rb.d_tf, rb.f_tf, serial, serial / rb.ms,
         ideal_serial_ms, ideal_serial_ms / rb.ms);
  fflush(stdout);
}

}  // namespace

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nk = argc > 1 ? atoi(argv[1]) : 256;  // k = 4096
  // operand panels: tiles_m = sms tiles of up to 128 rows (A), up to 8 waves x 128 columns (B)
  const size_t lpad = size_t(nk) * BK;
  const size_t a_elems = size_t(sms) * 128 * lpad, b_elems = size_t(8) * 128 * lpad;
  void *da, *db, *fa, *fb;
  cudaMalloc(&da, a_elems * 8);
  cudaMalloc(&db, b_elems * 8);
  cudaMalloc(&fa, a_elems * 4);
  cudaMalloc(&fb, b_elems * 4);
  cudaMemset(da, 0, a_elems * 8);
  cudaMemset(db, 0, b_elems * 8);
  cudaMemset(fa, 0, a_elems * 4);
  cudaMemset(fb, 0, b_elems * 4);
  double* sink;
  unsigned long long* t_end;
  cudaMalloc(&sink, 4096 * 8);
  cudaMalloc(&t_end, 4 * 8);
  printf("dual-pipe probe: %d SMs, k = %zu, one persistent CTA per SM; D = DMMA 64x128 tiles (DWM x 32 warp tiles),"
         " F = FFMA2 (NF*16)x128 tiles\n", sms, lpad);
  // name, ND, DWM, NF, DSTAGES, FSTAGES, RD, RF, RP ; waves chosen so D and F take similar time
  // (F flops per tile-wave = BM_F/BM_D x D's, at ~2x the rate)
  config<8, 64, 4, 3, 6, 168, 0, 40>("d8(64x32) f4 smr168/-/40", sms, da, db, fa, fb, sink, t_end, nk, 2, 4);
  config<12, 32, 4, 3, 6, 104, 144, 24>("d12(32x32) f4 smr104/144/24", sms, da, db, fa, fb, sink, t_end, nk, 3, 4);
  config<12, 32, 4, 3, 6, 104, 144, 24>("d12(32x32) f4 F2x", sms, da, db, fa, fb, sink, t_end, nk, 3, 8);
  return 0;
}
