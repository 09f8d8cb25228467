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

// Device-side checks of the checked build (make -C paper_1901_06015_b200/csrc
// checked -> libmdgemm_b200_checked.so, loaded with MDGEMM_LIBRARY=checked):
// every index the kernels derive -- tile and k-block of a TMA source, shared
// memory destination of a bulk copy, stream-K slot, packed-buffer offset, C
// element of the element-wise epilogues -- is checked against its bound, and
// a violation traps with a message.  The release build compiles them out.
#ifdef MDG_DEVICE_CHECKS
#include <cstdio>
#define MDG_CHECK(cond, what)                                                                                  \
  do {                                                                                                        \
    if (!(cond)) {                                                                                            \
      printf("mdgemm device check failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__,         \
             static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));                                    \
      __trap();                                                                                               \
    }                                                                                                         \
  } while (0)
#else
#define MDG_CHECK(cond, what) \
  do {                        \
  } while (0)
#endif

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

// accumulate_element on values already in C's storage precision R (t rounded
// to R, c as stored).  Where the result provably equals the double-precision
// formulation it is computed in R: for binary32, the exact sum or product of
// two floats fits in a binary64, so rounding it once to float is the same as
// rounding it to double and then to float.  That covers beta = 0, beta = 1
// and a real beta on real C.  A general beta on complex C keeps the
// complex<double> product of the reference (combine_value).
template <int CDT>
__device__ __forceinline__ void combine_typed(const DBeta& beta, bool conj, typename OutType<CDT>::R* c,
                                              const typename OutType<CDT>::R* t) {
  using R = typename OutType<CDT>::R;
  constexpr bool cplx = OutType<CDT>::kComplex;
  auto add = [](R x, R y) -> R {
    if constexpr (sizeof(R) == 4) return __fadd_rn(x, y);
    else return __dadd_rn(x, y);
  };
  auto mul = [](R x, R y) -> R {
    if constexpr (sizeof(R) == 4) return __fmul_rn(x, y);
    else return __dmul_rn(x, y);
  };
  if (beta.is_zero) {
    c[0] = t[0];
    if constexpr (cplx) c[1] = t[1];
  } else if (beta.is_one) {
    c[0] = add(c[0], t[0]);
    if constexpr (cplx) c[1] = add(conj ? -c[1] : c[1], t[1]);
  } else if constexpr (!cplx) {
    c[0] = add(mul(static_cast<R>(beta.re), c[0]), t[0]);
  } else {
    const double2 v = combine_value(CDT, beta, make_double2(c[0], conj ? -static_cast<double>(c[1]) : c[1]),
                                    t[0], t[1]);
    c[0] = static_cast<R>(v.x);
    c[1] = static_cast<R>(v.y);
  }
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

// Producer / mover / epilogue-side waits: suspend instead of spinning (see
// mbar_wait_sleep_u32); the math warps' stage waits keep spinning
// (mbar_wait_u32).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "n"(20000)
      : "memory");
}

// Same, on a precomputed shared-window address: keeps the generic->shared
// conversion (S2R SR_CgaCtaId + LEA) out of the consumers' k loop.
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// Wait with a suspend-time hint: a thread whose phase is not complete is
// suspended (woken when the phase completes, or after `ns`) instead of
// spinning try_wait / branch / yield.  For waiters that share SM
// sub-partitions with math warps (the dual kernel's producer lanes spun on
// their empty barriers for a third of one sub-partition's issue slots).
__device__ __forceinline__ void mbar_wait_sleep_u32(uint32_t bar, uint32_t parity, uint32_t ns) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity), "r"(ns)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_u32(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}

// One TMA bulk copy global -> shared, completing on `bar` (tx bytes).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
#ifdef MDG_DEVICE_CHECKS
  {
    extern __shared__ __align__(128) unsigned char mdg_dyn_smem[];
    uint32_t dyn;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    const uint32_t lo = smem_u32(mdg_dyn_smem), d = smem_u32(dst);
    MDG_CHECK(d >= lo && d + bytes <= lo + dyn, "bulk copy destination outside the dynamic shared memory");
    MDG_CHECK((d & 15) == 0 && (bytes & 15) == 0 && (reinterpret_cast<uint64_t>(src) & 15) == 0,
              "bulk copy not 16-byte aligned");
  }
#endif
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}

// Tuning trace: one record of TRACE_WORDS per CTA (desc.h).
__device__ __forceinline__ void trace_stamp(unsigned long long* trace, unsigned long long t_start,
                                            unsigned long long t_first, unsigned long long t_loop) {
  unsigned long long* r = trace + static_cast<size_t>(blockIdx.x) * TRACE_WORDS;
  r[0] = smid();
  r[1] = t_start;
  r[2] = t_first;
  r[3] = t_loop;
  r[4] = globaltimer();
}

// 2-D TMA tensor copies of one box (coordinates in elements of the map).
__device__ __forceinline__ void tensor_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tensor_prefetch_2d(const CUtensorMap* map, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void tensor_store_2d(const CUtensorMap* map, int x, int y, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}

// Warm L2 with a global range ahead of the TMA ring (no shared memory, no
// completion): hides DRAM latency that a STAGES-deep ring cannot.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
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
// Arrive on a named barrier without waiting (the producer warp's half of a
// start-up handshake the consumers complete with named_sync).
__device__ __forceinline__ void named_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// --------------------------------------------------------- fused epilogue
// The accumulator tile (BM x BN real-image values held in registers) meets C
// here: element (r, c) of the real image maps to output element (r, c), or
// to a component of complex element (r/2, c) / (r, c/2) when the plan pairs
// rows / columns (virtual_ukr_temp's pairing, kernels.cpp:122-131).
//
// The tile is processed in column chunks.  The threads first stage all their
// accumulators in shared memory, already rounded to C's storage precision and
// laid out like C (accumulate_element rounds t to storage precision first,
// so this is exact).  When C is column-contiguous (rs == 1, full tile,
// 16-byte aligned columns) each chunk of C arrives by TMA bulk copies -- one
// per column segment, all in flight at once, issued before the staging so
// they overlap it -- and a rolled loop combines 16-byte vectors in C's own
// precision (combine_typed) and writes them straight to global memory.
// Otherwise a rolled scalar loop reads and writes C through its strides.
// `emit(put)` must call put(r, c, value) for every accumulator the calling
// thread holds.  Code size matters: this runs once per tile after a long
// mainloop, so it stays a compact rolled loop.
// Short inner dimension: the producer warms L2 with the C tile the epilogue
// will read (same geometry as fast_epilogue's TMA path), so the epilogue's C
// chunk loads hit L2 instead of waiting on DRAM.
template <int CDT>
__device__ __forceinline__ void prefetch_c_tile(const DEpilogue& e, int64_t r0, int64_t c0, int BM, int BN) {
  using O = OutType<CDT>;
  using R = typename O::R;
  if (e.beta.is_zero) return;
  const bool prow = e.pair == MDG_PAIR_ROWS, pcol = e.pair == MDG_PAIR_COLS;
  const int orows = prow ? BM / 2 : BM, ocols = pcol ? BN / 2 : BN;
  const int64_t oi0 = prow ? r0 / 2 : r0, oj0 = pcol ? c0 / 2 : c0;
  const int64_t om = prow ? e.me / 2 : e.me, on = pcol ? e.ne / 2 : e.ne;
  if (e.out.rs != 1 || oi0 >= om || oj0 >= on) return;
  const int rows = static_cast<int>(om - oi0 < orows ? om - oi0 : orows);
  const int cols = static_cast<int>(on - oj0 < ocols ? on - oj0 : ocols);
  const uint32_t bytes = static_cast<uint32_t>(rows * O::ESZ) & ~15u;
  if (bytes == 0) return;
  const R* out = reinterpret_cast<const R*>(e.out.base);
  for (int j = 0; j < cols; ++j) {
    const R* p = out + (oi0 + (oj0 + j) * e.out.cs) * O::NC;
    if ((reinterpret_cast<uint64_t>(p) & 15) == 0) bulk_prefetch_l2(p, bytes);
  }
}

template <int CDT, class Emit>
__device__ __forceinline__ void fast_epilogue(unsigned char* smem, uint32_t region, uint64_t* cbar,
                                              const DEpilogue& e, int64_t r0, int64_t c0, int BM, int BN, int tid,
                                              int nthr, uint32_t& phase, Emit emit) {
  using O = OutType<CDT>;
  using R = typename O::R;
  constexpr int NC = O::NC;
  constexpr int VEC = 16 / O::ESZ;  // output elements per 16-byte vector
  const bool prow = e.pair == MDG_PAIR_ROWS, pcol = e.pair == MDG_PAIR_COLS;
  const int orows = prow ? BM / 2 : BM, ocols = pcol ? BN / 2 : BN;
  const int64_t oi0 = prow ? r0 / 2 : r0, oj0 = pcol ? c0 / 2 : c0;
  const int64_t om = prow ? e.me / 2 : e.me, on = pcol ? e.ne / 2 : e.ne;  // output extent
  const bool reads_c = !e.beta.is_zero;
  const bool conj = e.out.conj != 0;
  R* const out = reinterpret_cast<R*>(e.out.base);
  // The tile is staged in "lines" along C's contiguous dimension: columns for
  // a column-major C (cmap_ok 1, and 3 = the real part of an interleaved
  // complex C), rows for a row-major one (2: a transposed plan).  With a TMA
  // tensor map, C moves as boxes of C_BOX_COLS lines (loads into cbuf, stores
  // from tbuf -- or from cbuf for a real part, whose imaginary halves go back
  // unchanged); the map clips edge tiles.  Chunks are whole boxes that fit
  // beside the staged tile.
  const int cmode = e.cmap_ok;
  const bool rowm = cmode == MDG_CMAP_ROWS;
  const bool halfc = cmode == MDG_CMAP_REAL_PART;
  const int nlines = rowm ? orows : ocols, llen = rowm ? ocols : orows;
  const uint32_t line_bytes = llen * O::ESZ;
  const uint32_t cline_bytes = halfc ? 2 * line_bytes : line_bytes;
  auto sidx = [&](int oi, int oj) { return rowm ? oi * ocols + oj : oj * orows + oi; };
  unsigned char* tbuf = smem;
  unsigned char* cbuf = smem + nlines * line_bytes;
  const int CH_FIT = static_cast<int>((region - nlines * line_bytes) / cline_bytes) / C_BOX_COLS * C_BOX_COLS;
  const bool tma = cmode != 0 && CH_FIT >= C_BOX_COLS;
  const bool loads = tma && (reads_c || halfc);  // a real part always needs the imaginary halves
  const int CH = tma ? min(nlines, CH_FIT) : nlines;
  const CUtensorMap* map = &e.cmap;
  const int x0 = static_cast<int>(rowm ? oj0 * NC : (halfc ? 2 * oi0 : oi0 * NC));
  const int64_t line0 = rowm ? oi0 : oj0;
  auto load_chunk = [&](int l0) {
    const int nb = (min(CH, nlines - l0) + C_BOX_COLS - 1) / C_BOX_COLS;
    fence_proxy_async();
    mbar_arrive_expect_tx(cbar, nb * C_BOX_COLS * cline_bytes);
    for (int b = 0; b < nb; ++b)
      tensor_load_2d(cbuf + b * C_BOX_COLS * cline_bytes, map, x0, static_cast<int>(line0 + l0 + b * C_BOX_COLS), cbar);
  };
  if (loads && tid == 0) load_chunk(0);
  emit([&](int r, int c, double v) {
    const int oi = prow ? r >> 1 : r, oj = pcol ? c >> 1 : c;
    const int comp = prow ? (r & 1) : (pcol ? (c & 1) : 0);
    reinterpret_cast<R*>(tbuf)[sidx(oi, oj) * NC + comp] = static_cast<R>(v);
  });
  named_sync(1, nthr);

  if (!tma) {  // element-wise through C's strides
    const int n = orows * ocols;
    for (int idx = tid; idx < n; idx += nthr) {
      const int oi = idx % orows, oj = idx / orows;
      const int64_t gi = oi0 + oi, gj = oj0 + oj;
      if (gi >= om || gj >= on) continue;
      MDG_CHECK(gi >= 0 && gj >= 0 && gi < e.out.m && gj < e.out.n, "epilogue element outside C");
      R* cp = out + (gi * e.out.rs + gj * e.out.cs) * NC;
      R cv[NC];
      const R* tp = reinterpret_cast<const R*>(tbuf) + static_cast<size_t>(sidx(oi, oj)) * NC;
#pragma unroll
      for (int u = 0; u < NC; ++u) cv[u] = reads_c ? cp[u] : R(0);
      combine_typed<CDT>(e.beta, conj, cv, tp);
#pragma unroll
      for (int u = 0; u < NC; ++u) cp[u] = cv[u];
    }
    return;
  }
  for (int l0 = 0; l0 < nlines; l0 += CH) {
    const int ch = min(CH, nlines - l0);
    if (loads) {
      mbar_wait(cbar, phase);
      phase ^= 1;
    }
    if (!halfc) {
      const int nv = ch * llen / VEC;
      for (int v = tid; v < nv; v += nthr) {
        const int idx = v * VEC;  // element within the chunk, line-major
        union {
          uint4 u;
          R x[VEC * NC];
        } cv, tv;
        uint4* tp = reinterpret_cast<uint4*>(tbuf + (static_cast<size_t>(l0) * llen + idx) * O::ESZ);
        tv.u = *tp;
        cv.u = reads_c ? *reinterpret_cast<const uint4*>(cbuf + static_cast<size_t>(idx) * O::ESZ) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < VEC; ++u) combine_typed<CDT>(e.beta, conj, &cv.x[u * NC], &tv.x[u * NC]);
        *tp = cv.u;
      }
    } else {  // real part: combine into the even slots of the interleaved chunk
      const int n = ch * llen;
      R* cb = reinterpret_cast<R*>(cbuf);
      const R* tb = reinterpret_cast<const R*>(tbuf) + static_cast<size_t>(l0) * llen;
      for (int idx = tid; idx < n; idx += nthr) {
        R cv = reads_c ? cb[2 * idx] : R(0);
        combine_typed<CDT>(e.beta, conj, &cv, &tb[idx]);
        cb[2 * idx] = cv;
      }
    }
    fence_proxy_async();  // generic writes before the async-proxy store reads them
    named_sync(1, nthr);  // ... and every thread is done with this chunk
    if (tid == 0) {
      for (int b = 0; b < ch; b += C_BOX_COLS) {
        const unsigned char* src = halfc ? cbuf + static_cast<size_t>(b) * cline_bytes
                                         : tbuf + static_cast<size_t>(l0 + b) * line_bytes;
        tensor_store_2d(map, x0, static_cast<int>(line0 + l0 + b), src);
      }
      bulk_commit();
      if (l0 + ch < nlines) {
        if (halfc) bulk_wait_read();  // the next chunk lands where this one is being stored from
        if (loads) load_chunk(l0 + ch);
      }
    }
  }
  if (tid == 0) bulk_wait_read();  // the stores have read the smem: it may be reused / released
}

// Grouped tile raster: walks `group` tile-rows at a time.  A short group
// (8) makes concurrently running CTAs share A and B panels in L2 (long k);
// a group spanning all tile-rows keeps the concurrent C tiles inside a few
// column panels (short k, where C traffic dominates).
// 32-bit unsigned arithmetic (a launch has < 2^31 tiles): it runs in every
// CTA's prologue, where a 64-bit division costs ~100 instructions.
__device__ __forceinline__ void tile_coords(int64_t id64, int tiles_m, int tiles_n, int group_rows, int& tm,
                                            int& tn) {
  const unsigned id = static_cast<unsigned>(id64);
  const unsigned GROUP = static_cast<unsigned>(group_rows > 0 ? min(group_rows, tiles_m) : min(8, tiles_m));
  const unsigned per_group = GROUP * static_cast<unsigned>(tiles_n);
  const unsigned group = id / per_group;
  const unsigned first = group * GROUP;
  const unsigned gsize = min(static_cast<unsigned>(tiles_m) - first, GROUP);
  const unsigned in = id - group * per_group;
  tn = static_cast<int>(in / gsize);
  tm = static_cast<int>(first + (in - static_cast<unsigned>(tn) * gsize));
}

// ---- work schedule of one CTA of the fast kernels ------------------------
//
// Classic grid: one segment, the whole k range of tile blockIdx % tiles (or
// split-K slice blockIdx / tiles of it).
//
// Stream-K hybrid grid (d.sk_grid = G, the resident CTA slots): with
// R = tiles % G > 0, the first dp = (tiles / G - 1) G CTAs take one whole tile
// each (hardware-scheduled waves, as in the classic grid) and the last G CTAs
// cut the remaining G + R tiles x nk k-blocks into G equal contiguous ranges,
// CTA b owning [b U/G, (b+1) U/G) of them.  A range is at least one tile
// long, so it ends inside a tile at most once on each side, giving up to
// three kinds of segment:
//   SEG_START  the first k-blocks of the tile the range ends in: accumulated
//              from zero and published to partial slot b (run FIRST, so the
//              next CTA never waits long);
//   SEG_FULL   whole tiles;
//   SEG_END    the rest of the tile the range starts in: the accumulators are
//              SEEDED with CTA b-1's published partial and the k loop simply
//              continues (run LAST).
// Continuing the accumulation instead of adding two partial sums keeps every
// element's rounding sequence identical to the single-CTA k loop, so the
// result is bitwise the same as the classic grid (and as any column shard).
enum SegKind : int { SEG_FULL = 0, SEG_START = 1, SEG_END = 2, SEG_SPLIT = 3 };

struct Seg {
  int tile;
  int k0, k1;  // k-block range
  int kind;
};

// 32-bit fields: the schedule stays live through the mainloop of a
// register-bound kernel (tiles and k-blocks per launch are < 2^31).
struct Sched {
  int tiles, nk, nseg;
  int sk;                    // stream-K slot of this CTA (-1: a whole-tile CTA)
  int start_tile, start_k1;  // SEG_START (start_k1 == 0: none)
  int full0;                 // first SEG_FULL tile (its range: [full0, start_tile))
  int end_tile, end_k0;      // SEG_END (end_k0 == 0: none)
};

// Stream-K CTAs wait for their predecessor's published partial tile, so the
// order of the CTA numbers must be an order in which CTAs START: a CTA takes
// its logical number from a ticket counter (zeroed with the publish flags)
// when it begins, so CTA b-1 is already running -- and finishes its first
// segment without waiting on anyone -- before CTA b can wait for it, however
// the hardware dispatches the grid or shares the SMs with other kernels.
// No ticket (no range splits a tile): the block index.
__device__ __forceinline__ int logical_cta(int* ticket) {
  __shared__ int cta;
  if (threadIdx.x == 0) cta = ticket ? atomicAdd(ticket, 1) : static_cast<int>(blockIdx.x);
  __syncthreads();
  return cta;
}
__device__ __forceinline__ int* sk_ticket(const GemmDesc& d) { return d.sk_flags ? d.sk_flags + d.sk_grid : nullptr; }

// SK is a template flag so the classic kernels compile to one straight
// segment (the segment loop costs registers).  cta: the logical CTA number
// (logical_cta) of a stream-K launch.
template <bool SK>
__device__ __forceinline__ Sched make_sched(const GemmDesc& d, int64_t tiles, int nk, int cta) {
  Sched s{};
  s.tiles = static_cast<int>(tiles);
  s.nk = nk;
  s.sk = -1;
  s.nseg = 1;
  if (!SK) return s;
  const int64_t G = d.sk_grid, dp = sk_dp_tiles(tiles, G);
  const int64_t b = static_cast<int64_t>(cta) - dp;
  if (b < 0) {  // a whole tile
    s.full0 = cta;
    s.start_tile = s.full0 + 1;
    return s;
  }
  s.sk = static_cast<int>(b);
  const int64_t U = (tiles - dp) * nk;
  const int64_t u0 = dp * nk + b * U / G, u1 = dp * nk + (b + 1) * U / G;
  s.start_tile = static_cast<int>(u1 / nk);
  s.start_k1 = static_cast<int>(u1 % nk);
  s.end_tile = static_cast<int>(u0 / nk);
  s.end_k0 = static_cast<int>(u0 % nk);
  s.full0 = static_cast<int>((u0 + nk - 1) / nk);
  s.nseg = (s.start_k1 != 0) + (s.start_tile - s.full0) + (s.end_k0 != 0);
  return s;
}

template <bool SK>
__device__ __forceinline__ Seg sched_seg(const Sched& s, const GemmDesc& d, int idx) {
  if (!SK) {
    const int tile = static_cast<int>(blockIdx.x % s.tiles);
    if (d.splits > 1) {
      const int k0 = static_cast<int>(blockIdx.x / s.tiles) * d.kb_per_split;
      return Seg{tile, k0, min(s.nk, k0 + d.kb_per_split), SEG_SPLIT};
    }
    return Seg{tile, 0, s.nk, SEG_FULL};
  }
  if (s.start_k1 != 0) {
    if (idx == 0) return Seg{s.start_tile, 0, s.start_k1, SEG_START};
    --idx;
  }
  if (idx < s.start_tile - s.full0) return Seg{s.full0 + idx, 0, s.nk, SEG_FULL};
  return Seg{s.end_tile, s.end_k0, s.nk, SEG_END};
}

// Stream-K partial slot / publish flag b of a grid with G slots.
__device__ __forceinline__ void check_sk_slot(int b, int64_t G) {
  MDG_CHECK(b >= 0 && b < G, "stream-K slot out of range");
}

__device__ __forceinline__ void flag_release(int* f) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(f), "r"(1) : "memory");
}
__device__ __forceinline__ void flag_acquire_wait(const int* f) {
  uint32_t v;
  while (true) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(f) : "memory");
    if (v) break;
    __nanosleep(64);
  }
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
