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
// * combine_value/combine_element -- accumulate_element (kernels.cpp:79-95):
//                                    typecast-on-accumulate into C's storage
//                                    precision, beta applied in double.
// * mbarrier / cp.async.bulk      -- the TMA bulk-copy feed of the mainloops.
// * fast_epilogue                 -- the fused typecast-accumulate epilogue
//                                    of the DMMA / FFMA kernels.
#pragma once

#include <cstdint>
#include <type_traits>

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

// Annex G recovery of an (a+bi)(c+di) that came out NaN + NaN i; cold path,
// kept out of line so the hot epilogues stay small.
static __device__ __noinline__ double2 cmul_recover(double a, double b, double c, double d, double ac, double bd,
                                             double ad, double bc, double x, double y) {
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
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    x = dmul(inf, dsub(dmul(a, c), dmul(b, d)));
    y = dmul(inf, dadd(dmul(a, d), dmul(b, c)));
  }
  return make_double2(x, y);
}

// (a + bi)(c + di)
__device__ __forceinline__ double2 cmul(double a, double b, double c, double d) {
  const double ac = dmul(a, c), bd = dmul(b, d), ad = dmul(a, d), bc = dmul(b, c);
  const double x = dsub(ac, bd), y = dadd(ad, bc);
  if (isnan(x) && isnan(y)) return cmul_recover(a, b, c, d, ac, bd, ad, bc, x, y);
  return make_double2(x, y);
}

__host__ __device__ __forceinline__ bool dt_single(int dt) { return dt == MDG_DT_S || dt == MDG_DT_C; }
__host__ __device__ __forceinline__ bool dt_complex(int dt) { return dt == MDG_DT_C || dt == MDG_DT_Z; }

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

// The arithmetic of accumulate_element once c(i,j) is in hand (c ignored when
// beta == 0); returns the value to store.  kernels.cpp:79-95.
__device__ __forceinline__ double2 combine_value(int out_dtype, const DBeta& beta, double2 c, double tre,
                                                 double tim) {
  const bool sp = dt_single(out_dtype);
  const double cre = rnd(tre, sp), cim = rnd(tim, sp);
  double rre, rim;
  if (beta.is_zero) {
    rre = cre;
    rim = cim;
  } else if (beta.is_one) {
    rre = rnd(dadd(c.x, cre), sp);
    rim = rnd(dadd(c.y, cim), sp);
  } else {
    const double2 bc = cmul(beta.re, beta.im, c.x, c.y);
    rre = rnd(dadd(rnd(bc.x, sp), cre), sp);
    rim = rnd(dadd(rnd(bc.y, sp), cim), sp);
  }
  if (!dt_complex(out_dtype)) rim = 0.0;
  return make_double2(rre, rim);
}

// c(i,j) := beta (*) c(i,j) + typecast(t) on a strided view.
__device__ __forceinline__ void combine_element(const DView& out, int64_t i, int64_t j, const DBeta& beta,
                                                double tre, double tim) {
  const double2 c = beta.is_zero ? make_double2(0.0, 0.0) : ld_elem(out, i, j);
  const double2 v = combine_value(out.dtype, beta, c, tre, tim);
  st_elem(out, i, j, v.x, v.y);
}

// Compile-time view of C's storage datatype.
template <int CDT>
struct OutType {
  static constexpr bool kComplex = CDT == MDG_DT_C || CDT == MDG_DT_Z;
  static constexpr bool kSingle = CDT == MDG_DT_S || CDT == MDG_DT_C;
  static constexpr int NC = kComplex ? 2 : 1;
  using R = typename std::conditional<kSingle, float, double>::type;
  static constexpr int ESZ = NC * static_cast<int>(sizeof(R));
};

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

// One TMA bulk copy shared -> global (bulk-group completion).
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
// Generic-proxy shared-memory writes become visible to the async (TMA) proxy.
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// Named barrier over the compute warps only (the producer warp skips it).
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// --------------------------------------------------------- fused epilogue
// The accumulator tile (BM x BN real-image values held in registers) meets C
// here: element (r, c) of the real image maps to output element (r, c), or
// to a component of complex element (r/2, c) / (r, c/2) when the plan pairs
// rows / columns (virtual_ukr_temp's pairing, kernels.cpp:122-131).
//
// The tile is processed in column chunks.  For each chunk the threads stage
// their accumulators in shared memory, already rounded to C's storage
// precision and laid out like C (the first step of accumulate_element
// rounds t to storage precision anyway, so this is exact).  When the C
// chunk is column-contiguous (rs == 1, full tile, 16-byte aligned columns)
// it is moved with TMA bulk copies -- one per column, all in flight at once
// -- and combined in place by a rolled loop; otherwise the loop reads and
// writes C directly.  `emit(put)` must call put(r, c, value) for every
// accumulator the calling thread holds.  Code size matters here: this runs
// once per tile after a long mainloop, so it is a compact rolled loop over a
// chunk rather than an unrolled per-register sequence.
template <int CDT, class Emit>
__device__ __forceinline__ void fast_epilogue(unsigned char* smem, uint32_t region, uint64_t* cbar,
                                              const DEpilogue& e, int64_t r0, int64_t c0, int BM, int BN, int tid,
                                              int nthr, Emit emit) {
  using O = OutType<CDT>;
  using R = typename O::R;
  constexpr int NC = O::NC;
  const bool prow = e.pair == MDG_PAIR_ROWS, pcol = e.pair == MDG_PAIR_COLS;
  const int orows = prow ? BM / 2 : BM, ocols = pcol ? BN / 2 : BN;
  const int64_t oi0 = prow ? r0 / 2 : r0, oj0 = pcol ? c0 / 2 : c0;
  const int64_t om = prow ? e.me / 2 : e.me, on = pcol ? e.ne / 2 : e.ne;  // output extent
  const bool reads_c = !e.beta.is_zero;
  const uint32_t col_bytes = orows * O::ESZ;
  R* const out = reinterpret_cast<R*>(e.out.base);
  const uint64_t first = reinterpret_cast<uint64_t>(out + (oi0 * e.out.rs + oj0 * e.out.cs) * NC);
  const bool tma = e.out.rs == 1 && oi0 + orows <= om && oj0 + ocols <= on && (first & 15) == 0 &&
                   (col_bytes & 15) == 0 && ((e.out.cs * O::ESZ) & 15) == 0;
  // The whole accumulator tile is staged first (so no accumulator stays live
  // past this point); C then streams through the rest of the region.
  unsigned char* tbuf = smem;
  unsigned char* cbuf = smem + ocols * col_bytes;
  const int CH = tma ? min(ocols, static_cast<int>((region - ocols * col_bytes) / col_bytes)) : ocols;
  if (tma && reads_c && tid == 0) fence_proxy_async();
  emit([&](int r, int c, double v) {
    const int oi = prow ? r >> 1 : r, oj = pcol ? c >> 1 : c;
    const int comp = prow ? (r & 1) : (pcol ? (c & 1) : 0);
    reinterpret_cast<R*>(tbuf)[(oj * orows + oi) * NC + comp] = static_cast<R>(v);
  });
  uint32_t phase = 0;

  for (int j0 = 0; j0 < ocols; j0 += CH) {
    const int ch = min(CH, ocols - j0);
    if (tma && reads_c && tid == 0) {
      mbar_arrive_expect_tx(cbar, ch * col_bytes);
      for (int j = 0; j < ch; ++j)
        bulk_g2s(cbuf + j * col_bytes, out + (oi0 + (oj0 + j0 + j) * e.out.cs) * NC, col_bytes, cbar);
    }
    named_sync(1, nthr);
    const int n = ch * orows;
    if (tma) {
      if (reads_c) {
        mbar_wait(cbar, phase);
        phase ^= 1;
      }
      for (int idx = tid; idx < n; idx += nthr) {
        R* cp = reinterpret_cast<R*>(cbuf) + idx * NC;
        const R* tp = reinterpret_cast<const R*>(tbuf) + (j0 * orows + idx) * NC;
        double2 c = make_double2(0.0, 0.0);
        if (reads_c) {
          c.x = cp[0];
          if (NC == 2) c.y = e.out.conj ? -static_cast<double>(cp[1]) : static_cast<double>(cp[1]);
        }
        const double2 v = combine_value(CDT, e.beta, c, tp[0], NC == 2 ? static_cast<double>(tp[NC - 1]) : 0.0);
        cp[0] = static_cast<R>(v.x);
        if (NC == 2) cp[NC - 1] = static_cast<R>(v.y);
      }
      fence_proxy_async();
      named_sync(1, nthr);
      if (tid == 0) {
        for (int j = 0; j < ch; ++j)
          bulk_s2g(out + (oi0 + (oj0 + j0 + j) * e.out.cs) * NC, cbuf + j * col_bytes, col_bytes);
        bulk_commit();
        bulk_wait_read();
      }
    } else {
      for (int idx = tid; idx < n; idx += nthr) {
        const int oi = idx % orows, oj = idx / orows;
        const int64_t gi = oi0 + oi, gj = oj0 + j0 + oj;
        if (gi >= om || gj >= on) continue;
        R* cp = out + (gi * e.out.rs + gj * e.out.cs) * NC;
        const R* tp = reinterpret_cast<const R*>(tbuf) + (j0 * orows + idx) * NC;
        double2 c = make_double2(0.0, 0.0);
        if (reads_c) {
          c.x = cp[0];
          if (NC == 2) c.y = e.out.conj ? -static_cast<double>(cp[1]) : static_cast<double>(cp[1]);
        }
        const double2 v = combine_value(CDT, e.beta, c, tp[0], NC == 2 ? static_cast<double>(tp[NC - 1]) : 0.0);
        cp[0] = static_cast<R>(v.x);
        if (NC == 2) cp[NC - 1] = static_cast<R>(v.y);
      }
    }
    named_sync(1, nthr);  // chunk buffers are free again
  }
  if (tma && tid == 0) bulk_wait_all();
}

// Grouped tile raster: walks `group` tile-rows at a time.  A short group
// (8) makes concurrently running CTAs share A and B panels in L2 (long k);
// a group spanning all tile-rows keeps the concurrent C tiles inside a few
// column panels (short k, where C traffic dominates).
__device__ __forceinline__ void tile_coords(int64_t id, int tiles_m, int tiles_n, int group_rows, int& tm,
                                            int& tn) {
  const int GROUP = group_rows > 0 ? group_rows : 8;
  const int64_t per_group = static_cast<int64_t>(GROUP) * tiles_n;
  const int group = static_cast<int>(id / per_group);
  const int first = group * GROUP;
  const int gsize = min(tiles_m - first, GROUP);
  const int64_t in = id % per_group;
  tm = first + static_cast<int>(in % gsize);
  tn = static_cast<int>(in / gsize);
}

// Launch helper: instantiate a kernel template for C's storage datatype.
#define MDG_DISPATCH_CDT(dtype, CDT_NAME, ...)         \
  switch (dtype) {                                     \
    case MDG_DT_S: {                                   \
      constexpr int CDT_NAME = MDG_DT_S;               \
      __VA_ARGS__;                                     \
    } break;                                           \
    case MDG_DT_D: {                                   \
      constexpr int CDT_NAME = MDG_DT_D;               \
      __VA_ARGS__;                                     \
    } break;                                           \
    case MDG_DT_C: {                                   \
      constexpr int CDT_NAME = MDG_DT_C;               \
      __VA_ARGS__;                                     \
    } break;                                           \
    default: {                                         \
      constexpr int CDT_NAME = MDG_DT_Z;               \
      __VA_ARGS__;                                     \
    } break;                                           \
  }

}  // namespace mdg
