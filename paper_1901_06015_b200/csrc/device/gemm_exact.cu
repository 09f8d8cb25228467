// EXACT numerics: replays the reference engine's rounding sequence per output
// element so the device result is bitwise identical to the CPU reference for
// the same Config.  The reference accumulates each C element in the
// computation precision T with separate multiply and add, inner index
// ascending (ukr_impl, kernels.cpp:26-35), and the plan decides how the sum
// meets C:
//   FULL_THEN_COMBINE  C_temp engaged (dispatch.cpp:366-385): the sum runs
//                      from zero over all k, then one accumulate_element.
//   DIRECT_SEEDED      Direct / 1m-direct path: accumulators seeded with
//                      beta*c in T (kernels.cpp:13-24), continued across KC
//                      blocks exactly, stored in T.
//   BLOCK_COMBINE      Temp path without C_temp (kernels.cpp:97-132,
//                      gemm_core.cpp:125-127): one accumulate_element per KC
//                      block, beta on the first block and 1 afterwards.
//   ONEM_MIXED         1m with a complex beta and a flattenable C of the
//                      computation precision: virtual_ukr_onem takes the temp
//                      tile for the first KC block only (kernels.cpp:141-150);
//                      later blocks (beta = 1) continue in T on real_flatten(C).
// This is a SIMT kernel with one output element per thread; it is the
// bit-reproducibility mode, not the throughput path.
#include "common.cuh"

namespace mdg {
namespace {

__device__ __forceinline__ float tmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float tadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double tmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double tadd(double a, double b) { return __dadd_rn(a, b); }

template <typename T>
__global__ void __launch_bounds__(256) gemm_exact_kernel(GemmDesc d) {
  const DEpilogue& e = d.epi;
  const bool prow = e.pair == MDG_PAIR_ROWS, pcol = e.pair == MDG_PAIR_COLS;
  const bool two = prow || pcol;
  const int64_t orows = prow ? e.me / 2 : e.me;
  const int64_t ocols = pcol ? e.ne / 2 : e.ne;
  const T* A = static_cast<const T*>(d.a.data);
  const T* B = static_cast<const T*>(d.b.data);
  const int64_t pda = d.a.pd, lpa = d.a.lpad, pdb = d.b.pd, lpb = d.b.lpad;

  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < orows * ocols;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t oi = idx % orows, oj = idx / orows;
    const int64_t r0 = prow ? 2 * oi : oi, c0 = pcol ? 2 * oj : oj;
    const int64_t r1 = prow ? r0 + 1 : r0, c1 = pcol ? c0 + 1 : c0;
    const T* a0 = A + (r0 / pda) * pda * lpa + r0 % pda;
    const T* a1 = A + (r1 / pda) * pda * lpa + r1 % pda;
    const T* b0 = B + (c0 / pdb) * pdb * lpb + c0 % pdb;
    const T* b1 = B + (c1 / pdb) * pdb * lpb + c1 % pdb;

    auto run = [&](T s0, T s1, int64_t lo, int64_t hi, T& o0, T& o1) {
      for (int64_t l = lo; l < hi; ++l) {
        s0 = tadd(s0, tmul(a0[l * pda], b0[l * pdb]));
        if (two) s1 = tadd(s1, tmul(a1[l * pda], b1[l * pdb]));
      }
      o0 = s0;
      o1 = s1;
    };

    if (d.exact_mode == EXACT_DIRECT_SEEDED) {
      // Real output view in storage precision == T; seed as gemm_ukr does.
      T* cp = reinterpret_cast<T*>(elem_addr(e.out, oi, oj));
      const T bt = static_cast<T>(d.seed_beta);
      T seed = T(0);
      if (bt != T(0)) seed = bt == T(1) ? *cp : tmul(bt, *cp);
      T s0, s1;
      run(seed, T(0), 0, d.ke, s0, s1);
      *cp = s0;
    } else if (d.exact_mode == EXACT_FULL_THEN_COMBINE) {
      T s0, s1;
      run(T(0), T(0), 0, d.ke, s0, s1);
      combine_element(e.out, oi, oj, e.beta, static_cast<double>(s0),
                      two ? static_cast<double>(s1) : 0.0);
    } else if (d.exact_mode == EXACT_ONEM_MIXED) {
      const int64_t hi = d.kc < d.ke ? d.kc : d.ke;
      T s0, s1;
      run(T(0), T(0), 0, hi, s0, s1);
      combine_element(e.out, oi, oj, e.beta, static_cast<double>(s0), static_cast<double>(s1));
      if (hi < d.ke) {
        // raw stored components continue accumulating in T (beta = 1, direct)
        T* q0 = reinterpret_cast<T*>(elem_addr(d.flat, prow ? r0 : oi, prow ? oj : c0));
        T* q1 = reinterpret_cast<T*>(elem_addr(d.flat, prow ? r1 : oi, prow ? oj : c1));
        T t0, t1;
        run(*q0, *q1, hi, d.ke, t0, t1);
        *q0 = t0;
        *q1 = t1;
      }
    } else {
      const DBeta unit{1.0, 0.0, 0, 1};
      for (int64_t pc = 0; pc < d.ke; pc += d.kc) {
        const int64_t hi = pc + d.kc < d.ke ? pc + d.kc : d.ke;
        T s0, s1;
        run(T(0), T(0), pc, hi, s0, s1);
        combine_element(e.out, oi, oj, pc == 0 ? e.beta : unit, static_cast<double>(s0),
                        two ? static_cast<double>(s1) : 0.0);
      }
    }
  }
}

}  // namespace

cudaError_t launch_gemm_exact(const GemmDesc& d, bool single, int sms, cudaStream_t s) {
  const bool prow = d.epi.pair == MDG_PAIR_ROWS, pcol = d.epi.pair == MDG_PAIR_COLS;
  const int64_t total = (prow ? d.me / 2 : d.me) * (pcol ? d.ne / 2 : d.ne);
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  if (blocks > int64_t{sms} * 64) blocks = int64_t{sms} * 64;
  if (single)
    gemm_exact_kernel<float><<<static_cast<unsigned>(blocks), 256, 0, s>>>(d);
  else
    gemm_exact_kernel<double><<<static_cast<unsigned>(blocks), 256, 0, s>>>(d);
  return cudaGetLastError();
}

}  // namespace mdg
