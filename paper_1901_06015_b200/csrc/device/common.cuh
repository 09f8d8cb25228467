// Shared device code for the sm_100a mixed-datatype gemm.
//
// * DView / ld_elem / st_elem     -- strided typed element access (the device
//                                    twin of load_elem/store_elem,
//                                    dtypes.cpp:176-213).
// * cmul                          -- complex<double> product exactly as the
//                                    reference's x86-64 build evaluates it:
//                                    separate multiplies and adds, with the
//                                    C99 Annex G recovery when both parts are
//                                    NaN (what GCC's __muldc3 does).
// * combine_element               -- accumulate_element (kernels.cpp:79-95):
//                                    typecast-on-accumulate into C's storage
//                                    precision, beta applied in double.
// * mbarrier / cp.async.bulk      -- the TMA bulk-copy feed of the mainloops.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "desc.h"

namespace mdg {

__device__ __forceinline__ double rnd(double v, bool single) {
  return single ? static_cast<double>(__double2float_rn(v)) : v;
}

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ double unit_copysign(bool cond, double s) {
  return copysign(cond ? 1.0 : 0.0, s);
}

// (a + bi)(c + di)
__device__ __forceinline__ double2 cmul(double a, double b, double c, double d) {
  const double ac = dmul(a, c), bd = dmul(b, d), ad = dmul(a, d), bc = dmul(b, c);
  double x = dsub(ac, bd), y = dadd(ad, bc);
  if (isnan(x) && isnan(y)) {
    bool recalc = false;
    if (isinf(a) || isinf(b)) {
      a = unit_copysign(isinf(a), a);
      b = unit_copysign(isinf(b), b);
      if (isnan(c)) c = copysign(0.0, c);
      if (isnan(d)) d = copysign(0.0, d);
      recalc = true;
    }
    if (isinf(c) || isinf(d)) {
      c = unit_copysign(isinf(c), c);
      d = unit_copysign(isinf(d), d);
      if (isnan(a)) a = copysign(0.0, a);
      if (isnan(b)) b = copysign(0.0, b);
      recalc = true;
    }
    if (!recalc && (isinf(ac) || isinf(bd) || isinf(ad) || isinf(bc))) {
      if (isnan(a)) a = copysign(0.0, a);
      if (isnan(b)) b = copysign(0.0, b);
      if (isnan(c)) c = copysign(0.0, c);
      if (isnan(d)) d = copysign(0.0, d);
      recalc = true;
    }
    if (recalc) {
      x = dmul(__longlong_as_double(0x7ff0000000000000LL), dsub(dmul(a, c), dmul(b, d)));
      y = dmul(__longlong_as_double(0x7ff0000000000000LL), dadd(dmul(a, d), dmul(b, c)));
    }
  }
  return make_double2(x, y);
}

__device__ __forceinline__ bool dt_single(int dt) { return dt == MDG_DT_S || dt == MDG_DT_C; }
__device__ __forceinline__ bool dt_complex(int dt) { return dt == MDG_DT_C || dt == MDG_DT_Z; }

__device__ __forceinline__ char* elem_addr(const DView& v, int64_t i, int64_t j) {
  const int64_t esz = (dt_single(v.dtype) ? 4 : 8) * (dt_complex(v.dtype) ? 2 : 1);
  return v.base + (i * v.rs + j * v.cs) * esz;
}

// Widened (re, im) of element (i, j), honouring the view's conj flag.
__device__ __forceinline__ double2 ld_elem(const DView& v, int64_t i, int64_t j) {
  const char* p = elem_addr(v, i, j);
  double re, im = 0.0;
  switch (v.dtype) {
    case MDG_DT_S: re = *reinterpret_cast<const float*>(p); break;
    case MDG_DT_D: re = *reinterpret_cast<const double*>(p); break;
    case MDG_DT_C: {
      const float2 f = *reinterpret_cast<const float2*>(p);
      re = f.x;
      im = f.y;
      break;
    }
    default: {
      const double2 f = *reinterpret_cast<const double2*>(p);
      re = f.x;
      im = f.y;
      break;
    }
  }
  if (v.conj) im = -im;
  return make_double2(re, im);
}

__device__ __forceinline__ void st_elem(const DView& v, int64_t i, int64_t j, double re, double im) {
  char* p = elem_addr(v, i, j);
  switch (v.dtype) {
    case MDG_DT_S: *reinterpret_cast<float*>(p) = __double2float_rn(re); break;
    case MDG_DT_D: *reinterpret_cast<double*>(p) = re; break;
    case MDG_DT_C: *reinterpret_cast<float2*>(p) = make_float2(__double2float_rn(re), __double2float_rn(im)); break;
    default: *reinterpret_cast<double2*>(p) = make_double2(re, im); break;
  }
}

// c(i,j) := beta (*) c(i,j) + typecast(t)   -- kernels.cpp:79-95.
__device__ __forceinline__ void combine_element(const DView& out, int64_t i, int64_t j,
                                                const DBeta& beta, double tre, double tim) {
  const bool sp = dt_single(out.dtype);
  const double cre = rnd(tre, sp), cim = rnd(tim, sp);
  double rre, rim;
  if (beta.is_zero) {
    rre = cre;
    rim = cim;
  } else {
    const double2 c = ld_elem(out, i, j);
    if (beta.is_one) {
      rre = rnd(dadd(c.x, cre), sp);
      rim = rnd(dadd(c.y, cim), sp);
    } else {
      const double2 bc = cmul(beta.re, beta.im, c.x, c.y);
      rre = rnd(dadd(rnd(bc.x, sp), cre), sp);
      rim = rnd(dadd(rnd(bc.y, sp), cim), sp);
    }
  }
  if (!dt_complex(out.dtype)) rim = 0.0;
  st_elem(out, i, j, rre, rim);
}

// ------------------------------------------------------------ async copies
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// One TMA bulk copy global -> shared, completing on `bar` (tx bytes).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Named barrier over the compute warps only (the producer warp skips it).
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// Real-image tile epilogue shared by the fast kernels: `T` holds the
// BM x BN accumulator tile column-major (leading dim ldt) in shared memory;
// each thread combines output elements, pairing rows/columns into complex
// values when the plan asks (virtual_ukr_temp's pairing, kernels.cpp:122-131).
template <typename Acc>
__device__ __forceinline__ void tile_epilogue(const Acc* T, int ldt, int BM, int BN, int64_t r0,
                                              int64_t c0, const DEpilogue& e, int tid, int nthr) {
  const bool prow = e.pair == MDG_PAIR_ROWS, pcol = e.pair == MDG_PAIR_COLS;
  const int orows = prow ? BM / 2 : BM;
  const int ocols = pcol ? BN / 2 : BN;
  const int total = orows * ocols;
  for (int idx = tid; idx < total; idx += nthr) {
    const int oi = idx % orows, oj = idx / orows;
    const int r = prow ? 2 * oi : oi, c = pcol ? 2 * oj : oj;
    const int64_t gr = r0 + r, gc = c0 + c;
    if (gr >= e.me || gc >= e.ne) continue;
    const double tre = static_cast<double>(T[c * ldt + r]);
    double tim = 0.0;
    if (prow) tim = static_cast<double>(T[c * ldt + r + 1]);
    if (pcol) tim = static_cast<double>(T[(c + 1) * ldt + r]);
    combine_element(e.out, prow ? gr / 2 : gr, pcol ? gc / 2 : gc, e.beta, tre, tim);
  }
}

// Grouped tile raster: walks GROUP tile-rows at a time so concurrently
// running CTAs share A panels and B panels in L2.
__device__ __forceinline__ void tile_coords(int64_t id, int tiles_m, int tiles_n, int& tm, int& tn) {
  constexpr int GROUP = 8;
  const int64_t per_group = static_cast<int64_t>(GROUP) * tiles_n;
  const int group = static_cast<int>(id / per_group);
  const int first = group * GROUP;
  const int gsize = min(tiles_m - first, GROUP);
  const int64_t in = id % per_group;
  tm = first + static_cast<int>(in % gsize);
  tn = static_cast<int>(in / gsize);
}

}  // namespace mdg
