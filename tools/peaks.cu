// Peak-throughput microbenchmarks for the arithmetic pipes the mixed-datatype
// gemm uses on sm_100a: FP64 DFMA (SIMT), FP64 DMMA (mma.sync .f64, several
// shapes), FP32 FFMA (SIMT).  Every kernel runs independent dependency chains
// so the pipe, not latency, is the limit.  Prints one JSON object.
#include <cstdio>
#include <string>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void k_dfma(double* out, double s) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], s, 0.5);
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += a[i];
  if (r == 1234.5) out[0] = r;
}

__global__ void k_ffma(float* out, float s) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s, 0.5f);
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) r += a[i];
  if (r == 1234.5f) out[0] = r;
}

// Paired fp32 FMA (sm_100 fma.rn.f32x2 -> SASS FFMA2), 3-register form with a
// broadcast scalar operand, as the FFMA gemm mainloop issues it.
__global__ void k_ffma2(float* out, float s) {
  unsigned long long acc[8], x[8];
  float bv[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float v = threadIdx.x * 1e-3f + i;
    asm("mov.b64 %0, {%1, %2};" : "=l"(acc[i]) : "f"(v), "f"(v + 1.0f));
    asm("mov.b64 %0, {%1, %2};" : "=l"(x[i]) : "f"(v * 0.5f), "f"(v * 0.25f));
    bv[i] = s + i;
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      unsigned long long b;
      asm("mov.b64 %0, {%1, %1};" : "=l"(b) : "f"(bv[i]));
      asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i]) : "l"(b), "l"(x[i]));
    }
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += __uint_as_float(static_cast<unsigned>(acc[i]));
  if (r == 1234.5f) out[0] = r;
}

// m8n8k4: A 1 f64, B 1 f64, C 2 f64 per thread.
__global__ void k_dmma_884(double* out) {
  double a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3 + i; b[i] = 0.5 + i; }
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a[i]), "d"(b[i]));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += c[i][0] + c[i][1];
  if (r == 1234.5) out[0] = r;
}

// m16n8k4: A 2, B 1, C 4.
__global__ void k_dmma_1684(double* out) {
  double a0[4], a1[4], b[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) { a0[i] = threadIdx.x * 1e-3 + i; a1[i] = 0.25 * i; b[i] = 0.5 + i; }
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0[i]), "d"(a1[i]), "d"(b[i]));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) r += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (r == 1234.5) out[0] = r;
}


template <typename F>
static float time_it(F launch, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch(); launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

// Co-residency probe: warps [0, dw) run the DMMA loop, the rest the FFMA2
// loop, in one CTA -- do the FP64 tensor pipe and the FP32 FMA pipe overlap?
__global__ void k_mix(double* dout, float* fout, int dw, int dit, int fit) {
  const int warp = threadIdx.x >> 5;
  if (warp < dw) {
    double a[8], b[8], c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3 + i; b[i] = 0.5 + i; c[i][0] = c[i][1] = 0; }
    for (int it = 0; it < dit; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a[i]), "d"(b[i]));
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += c[i][0] + c[i][1];
    if (r == 1234.5) dout[0] = r;
  } else {
    unsigned long long acc[8], x[8];
    float bv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float v = threadIdx.x * 1e-3f + i;
      asm("mov.b64 %0, {%1, %2};" : "=l"(acc[i]) : "f"(v), "f"(v + 1.0f));
      asm("mov.b64 %0, {%1, %2};" : "=l"(x[i]) : "f"(v * 0.5f), "f"(v * 0.25f));
      bv[i] = 0.999f + i;
    }
    for (int it = 0; it < fit; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        unsigned long long b;
        asm("mov.b64 %0, {%1, %1};" : "=l"(b) : "f"(bv[i]));
        asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i]) : "l"(b), "l"(x[i]));
      }
    }
    float r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += __uint_as_float(static_cast<unsigned>(acc[i]));
    if (r == 1234.5f) fout[0] = r;
  }
}


// Steady-state co-issue probe: warps [0, dw) loop on DMMA.8x8x4, the rest on
// FFMA2 with NCH independent accumulator chains (fewer chains = a throttled
// FP32 group), ALL until a common deadline; each group counts its iterations.
// Unlike k_mix (fixed work per warp, one group finishing first) this gives the
// rates while BOTH groups run: the frontier the dual-pipe kernel works against.
template <int NCH>
__global__ void k_steady(unsigned long long* counts, int dw, unsigned long long dur_ns) {
  const int warp = threadIdx.x >> 5;
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned long long iters = 0;
  if (warp < dw) {
    double a[8], b[8], c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3 + i; b[i] = 0.5 + i; c[i][0] = c[i][1] = 0; }
    do {
      for (int it = 0; it < 64; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a[i]), "d"(b[i]));
      }
      iters += 64;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < dur_ns);
    double r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += c[i][0] + c[i][1];
    if (r == 1234.5) counts[2] = 1;
    if ((threadIdx.x & 31) == 0) atomicAdd(&counts[0], iters * 8);  // DMMAs of this warp
  } else {
    unsigned long long acc[NCH], x[NCH];
    float bv[NCH];
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      const float v = threadIdx.x * 1e-3f + i;
      asm("mov.b64 %0, {%1, %2};" : "=l"(acc[i]) : "f"(v), "f"(v + 1.0f));
      asm("mov.b64 %0, {%1, %2};" : "=l"(x[i]) : "f"(v * 0.5f), "f"(v * 0.25f));
      bv[i] = 0.999f + i;
    }
    do {
      for (int it = 0; it < 256; ++it) {
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
          unsigned long long b;
          asm("mov.b64 %0, {%1, %1};" : "=l"(b) : "f"(bv[i]));
          asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i]) : "l"(b), "l"(x[i]));
        }
      }
      iters += 256;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < dur_ns);
    float r = 0;
#pragma unroll
    for (int i = 0; i < NCH; ++i) r += __uint_as_float(static_cast<unsigned>(acc[i]));
    if (r == 1234.5f) counts[2] = 1;
    if ((threadIdx.x & 31) == 0) atomicAdd(&counts[1], iters * NCH);  // warp-wide FFMA2s of this warp
  }
}

template <int NCH>
static void run_steady(unsigned long long* counts, int sms, int dw, int fw, bool first) {
  const unsigned long long dur = 2000000ull;  // 2 ms
  unsigned long long h[3] = {0, 0, 0};
  cudaMemset(counts, 0, 24);
  k_steady<NCH><<<sms, 32 * (dw + fw)>>>(counts, dw, dur);  // warm-up
  cudaDeviceSynchronize();
  cudaMemset(counts, 0, 24);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_steady<NCH><<<sms, 32 * (dw + fw)>>>(counts, dw, dur);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaMemcpy(h, counts, 24, cudaMemcpyDeviceToHost);
  const double dt = double(h[0]) * (8 * 8 * 4 * 2) / (ms * 1e-3) / 1e12;
  const double ft = double(h[1]) * 32 * 4 / (ms * 1e-3) / 1e12;
  printf("%s\"d%d_f%d_ch%d\": [%.2f, %.2f, %.3f]", first ? "" : ", ", dw, fw, NCH, dt, ft, dt / 37.0 + ft / 72.0);
}

int main(int argc, char** argv) {
  int sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  double* dout; float* fout;
  CK(cudaMalloc(&dout, 64)); CK(cudaMalloc(&fout, 64));
  int reps = argc > 1 ? atoi(argv[1]) : 20;
  if (argc > 2 && std::string(argv[2]) == "mix") {  // DMMA and FFMA2 warps side by side
    printf("{\"sms\": %d", sms);
    // 8 DMMA warps + 8 FFMA2 warps per SM; iteration counts chosen so each
    // alone would take about the same time at its peak
    const int dit = 2048, fit = 8192;
    // (DMMA warps, FFMA warps) per SM
    const int cfgs[][2] = {{8, 0}, {0, 8}, {8, 8}, {4, 0}, {0, 4}, {4, 4}, {8, 4}, {4, 8}, {4, 12}};
    for (auto& c : cfgs) {
      const int dw = c[0], fw = c[1];
      dim3 grid(sms), block(32 * (dw + fw));
      float ms = time_it([&] { k_mix<<<grid, block>>>(dout, fout, dw, dit, fit); }, reps);
      const double dfl = double(sms) * dw * dit * 8 * (8 * 8 * 4 * 2);
      const double ffl = double(sms) * fw * 32 * fit * 8 * 4;
      const double dt = dfl / (ms * 1e-3) / 1e12, ft = ffl / (ms * 1e-3) / 1e12;
      printf(", \"d%d_f%d\": [%.2f, %.2f, %.3f]", dw, fw, dt, ft, dt / 37.0 + ft / 72.0);
    }
    printf("}\n");
    return 0;
  }
  if (argc > 2 && std::string(argv[2]) == "steady") {  // both groups until a common deadline
    unsigned long long* counts;
    CK(cudaMalloc(&counts, 24));
    printf("{\"what\": \"[DMMA TF/s, FFMA2 TF/s, sum of fractions of 37 / 72] while both groups run (2 ms, register-only loops); dD_fF_chN = D DMMA warps + F FFMA2 warps per SM, N independent FFMA2 chains per thread\", ");
    bool first = true;
    for (int dw : {8, 12})
      for (int fw : {0, 4, 8}) {
        run_steady<8>(counts, sms, dw, fw, first); first = false;
        if (fw) { run_steady<4>(counts, sms, dw, fw, false); run_steady<2>(counts, sms, dw, fw, false); run_steady<1>(counts, sms, dw, fw, false); }
      }
    run_steady<8>(counts, sms, 0, 4, false);
    run_steady<8>(counts, sms, 0, 8, false);
    run_steady<8>(counts, sms, 4, 4, false);
    run_steady<8>(counts, sms, 4, 8, false);
    run_steady<8>(counts, sms, 4, 12, false);
    printf("}\n");
    CK(cudaGetLastError());
    return 0;
  }
  if (argc > 2 && std::string(argv[2]) == "occ") {  // pipe rate vs resident warps per SM
    printf("{\"sms\": %d", sms);
    const int cfgs[][2] = {{1, 4}, {1, 8}, {2, 4}, {1, 12}, {3, 4}, {1, 16}};
    for (auto& c : cfgs) {
      dim3 grid(sms * c[0]), block(32 * c[1]);
      double nwarps = double(grid.x) * c[1];
      float ms = time_it([&] { k_dmma_884<<<grid, block>>>(dout); }, reps);
      printf(", \"dmma884_%dcta_%dw_tflops\": %.3f", c[0], c[1],
             nwarps * (ITERS / 4) * 8 * (8 * 8 * 4 * 2) / (ms * 1e-3) / 1e12);
      double nthr = double(grid.x) * block.x;
      ms = time_it([&] { k_ffma2<<<grid, block>>>(fout, 0.999f); }, reps);
      printf(", \"ffma2_%dcta_%dw_tflops\": %.3f", c[0], c[1], nthr * ITERS * 8 * 4 / (ms * 1e-3) / 1e12);
    }
    printf("}\n");
    return 0;
  }
  printf("{\"sms\": %d, \"clock_khz_attr\": %d", sms, clk);
  for (int wpb : {4, 8, 16}) {
    dim3 grid(sms * 4), block(32 * wpb);
    double nthr = double(grid.x) * block.x;
    float ms = time_it([&] { k_dfma<<<grid, block>>>(dout, 0.999); }, reps);
    printf(", \"dfma_w%d_tflops\": %.3f", wpb, nthr * ITERS * 8 * 2 / (ms * 1e-3) / 1e12);
    ms = time_it([&] { k_ffma<<<grid, block>>>(fout, 0.999f); }, reps);
    printf(", \"ffma_w%d_tflops\": %.3f", wpb, nthr * ITERS * 16 * 2 / (ms * 1e-3) / 1e12);
    ms = time_it([&] { k_ffma2<<<grid, block>>>(fout, 0.999f); }, reps);
    printf(", \"ffma2_w%d_tflops\": %.3f", wpb, nthr * ITERS * 8 * 4 / (ms * 1e-3) / 1e12);
    double nwarps = double(grid.x) * wpb;
    ms = time_it([&] { k_dmma_884<<<grid, block>>>(dout); }, reps);
    printf(", \"dmma884_w%d_tflops\": %.3f", wpb, nwarps * (ITERS / 4) * 8 * (8 * 8 * 4 * 2) / (ms * 1e-3) / 1e12);
    ms = time_it([&] { k_dmma_1684<<<grid, block>>>(dout); }, reps);
    printf(", \"dmma1684_w%d_tflops\": %.3f", wpb, nwarps * (ITERS / 4) * 4 * (16 * 8 * 4 * 2) / (ms * 1e-3) / 1e12);
  }
  CK(cudaGetLastError());
  printf("}\n");
  return 0;
}
