// FAST numerics: the FP64 DMMA pipe and the FP32 FMA pipe of every SM busy
// AT THE SAME TIME.  One persistent CTA per SM runs two independent warp
// groups, each on its own list of gemm jobs (calls of a gemm_batch that touch
// disjoint memory):
//
//   warps 0-7   D group: computation precision double, 128x128 tiles, 64x32
//               warp tiles of DMMA.8x8x4 (the DMMA kernels' mainloop), two
//               warps per SM sub-partition; setmaxnreg 168;
//   warps 8-11  F group: computation precision single, 64x128 tiles, 8x8
//               register tiles updated with paired FP32 FMAs (FFMA2, the
//               FFMA kernels' mainloop); setmaxnreg 144;
//   warp 12     D producer lane: TMA bulk copies of 16-deep slabs into the
//               D ring (3 x 32 KB);
//   warp 13     F producer lane: 32-deep slabs into the F ring (4 x 24 KB;
//               32-deep halves the per-stage barrier / proxy-fence cost
//               that a single FFMA2 warp per sub-partition cannot hide);
//   warps 14-15 idle (the producer warpgroup gives its registers away:
//               setmaxnreg 32; 256 x 168 + 128 x 144 + 128 x 32 = 64 K).
//
// Why: the DMMA and FFMA2 pipes are separate.  tools/dual_probe runs the
// real TMA/LDS mainloops side by side: 8 DMMA + 4 FFMA2 warps per SM give
// 28.7 + 34.9 TFLOP/s at once (0.78 + 0.48 of the measured pipe peaks), and
// the D group alone still runs at 35.8 (0.97).  4 DMMA + 8 FFMA2 warps give
// 21.1 + 48.2 but only 29.4 for DMMA alone; the cfg2 sweep has equal FP64 and
// FP32 flops, so the DMMA-heavy split wins.  The classic kernels cannot
// share an SM that way: two DMMA CTAs already fill its register file.
//
// Each group walks its jobs' tiles as one virtual index space (jobs sorted by
// k on the host, longest first), CTA b taking one tile per round of G in
// boustrophedon order (b, 2G-1-b, 2G+b, ...);
// the two groups never synchronise with each other.  The epilogue combines
// the accumulators straight into C through its strides (accumulate_element
// via combine_typed, the classic kernels' arithmetic), so results are bitwise
// identical to the classic DMMA / FFMA kernels: same k order, same DMMA/FFMA2
// rounding, same combine.  While one group runs its epilogue the other
// group's mainloop keeps the SM busy.
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace mdg {
namespace {

constexpr int DU_BK = DUAL_BK;      // D group k-block
constexpr int DF_BK = DUAL_F_BK;    // F group k-block
constexpr int DD_BM = 128, DD_BN = 128;  // D tile; 8 warps (2 x 4) of 64x32
constexpr int DF_BM = 64, DF_BN = 128;   // F tile; 128 threads (8 x 16) of 8x8
// D stages hold each 128-double k-line at a pitch of 132: a DMMA fragment
// load (lane g + 4 tig reads line kk + tig, element 8i + g) then covers all
// 32 banks of a half-warp once.  With the packed pitch of 128 the four tig
// lines of a half-warp fall on the same banks (4-way conflicts; ncu: 48 % of
// the shared-load wavefronts of the step were conflicts).
static_assert(DD_BM == DD_BN, "one line pitch for both D operands");
template <int PAD>
struct DPitch {
  static constexpr int P = DD_BM + PAD;           // smem line pitch (doubles)
  static constexpr int SA = DU_BK * P, SB = DU_BK * P;  // doubles per stage
};
constexpr int DF_SA = DF_BK * DF_BM, DF_SB = DF_BK * DF_BN;  // floats per stage
constexpr int DD_WARPS = 8, DF_WARPS = 4;
template <int DD_STAGES, int DF_STAGES, int PAD = 4>
struct DuRings {
  static constexpr size_t DD_RING = size_t(DD_STAGES) * (DPitch<PAD>::SA + DPitch<PAD>::SB) * sizeof(double);
  static constexpr size_t DF_RING = size_t(DF_STAGES) * (DF_SA + DF_SB) * sizeof(float);
  static constexpr size_t SMEM =
      DD_RING + DF_RING + (2 * DD_STAGES + 2 * DF_STAGES) * sizeof(uint64_t) + (DD_STAGES + DF_STAGES + DD_WARPS + DF_WARPS) * sizeof(int);
};
constexpr int DU_THREADS = 512;
constexpr int DD_PROD_WARP = 12, DF_PROD_WARP = 13;

// %laneid == 0, read where it is needed (ptxas otherwise keeps `lane` live
// through the mainloops and spills it at the groups' register caps)
__device__ __forceinline__ bool lane0() {
  uint32_t l;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
  return l == 0;
}

__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ void dmma884_du(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Virtual tile of CTA blockIdx.x in round r: boustrophedon order, so with the
// tiles sorted longest-k first every CTA gets a similar total (round-robin
// would hand the longest tile of every round to the same low CTA numbers).
__device__ __forceinline__ int snake_tile(int r, int G) {
  return r * G + ((r & 1) ? G - 1 - static_cast<int>(blockIdx.x) : static_cast<int>(blockIdx.x));
}

// Job of virtual tile v in a group's list (jobs' tile ranges are contiguous).
__device__ __forceinline__ int job_of(const DualJob* jobs, int njobs, int v) {
  int j = 0;
  while (j + 1 < njobs && jobs[j + 1].tile0 <= v) ++j;
  return j;
}

// Address of output element (oi, oj) in C's storage type R.
template <int CDT>
__device__ __forceinline__ typename OutType<CDT>::R* c_ptr(const DView& o, int64_t oi, int64_t oj) {
  using O = OutType<CDT>;
  MDG_CHECK(oi >= 0 && oj >= 0 && oi < o.m && oj < o.n, "dual epilogue element outside C");
  return reinterpret_cast<typename O::R*>(o.base) + (oi * o.rs + oj * o.cs) * O::NC;
}

// The epilogue goes straight to global memory through C's strides, in groups
// of N output elements: all N loads of C are issued before the first store
// (a store may alias any later load, so a load-combine-store sequence per
// element would wait one memory latency per element), then accumulate_element
// (combine_typed) and the stores.  ok[u] masks elements outside C.
template <int CDT, int N>
__device__ __forceinline__ void put_group(const DualJob& jb, typename OutType<CDT>::R* const (&p)[N],
                                          const bool (&ok)[N], const double (&t)[N][2]) {
  using O = OutType<CDT>;
  using R = typename O::R;
  constexpr int NC = O::NC;
  R cv[N][NC];
#pragma unroll
  for (int u = 0; u < N; ++u)
#pragma unroll
    for (int c = 0; c < NC; ++c) cv[u][c] = (ok[u] && !jb.beta.is_zero) ? p[u][c] : R(0);
  const bool conj = jb.out.conj != 0;
#pragma unroll
  for (int u = 0; u < N; ++u) {
    R tv[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) tv[c] = static_cast<R>(t[u][c]);
    combine_typed<CDT>(jb.beta, conj, cv[u], tv);
    if (ok[u]) {
#pragma unroll
      for (int c = 0; c < NC; ++c) p[u][c] = cv[u][c];
    }
  }
}

// D group epilogue: lane (g, tig) of warp (wm, wn) holds rows wm*64 + 8i + g,
// columns wn*32 + 8j + 2tig (+1) of the tile; one group per i.
template <int CDT>
__device__ __forceinline__ void epilogue_d(const DualJob& jb, int tm, int tn, int wm, int wn, int lane,
                                           double (&acc)[8][4][2]) {
  using R = typename OutType<CDT>::R;
  constexpr bool cplx = OutType<CDT>::kComplex;
  const int g = lane >> 2, tig = lane & 3;
  const int64_t r0 = static_cast<int64_t>(tm) * DD_BM + wm * 64, c0 = static_cast<int64_t>(tn) * DD_BN + wn * 32;
  const R* dummy = reinterpret_cast<const R*>(jb.out.base);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t R0 = r0 + i * 8 + g;
    if constexpr (!cplx) {
      R* p[8];
      bool ok[8];
      double t[8][2];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int u = 2 * j + h;
          const int64_t C = c0 + j * 8 + 2 * tig + h;
          ok[u] = R0 < jb.me && C < jb.ne;
          p[u] = ok[u] ? c_ptr<CDT>(jb.out, R0, C) : const_cast<R*>(dummy);
          t[u][0] = acc[i][j][h];
          t[u][1] = 0.0;
        }
      put_group<CDT, 8>(jb, p, ok, t);
    } else {
      R* p[4];
      bool ok[4];
      double t[4][2];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t C0 = c0 + j * 8 + 2 * tig;
        const double a0 = acc[i][j][0], a1 = acc[i][j][1];
        if (jb.pair == MDG_PAIR_COLS) {  // (re, im) = columns (C0, C0 + 1)
          ok[j] = R0 < jb.me && C0 < jb.ne;
          p[j] = ok[j] ? c_ptr<CDT>(jb.out, R0, C0 >> 1) : const_cast<R*>(dummy);
          t[j][0] = a0;
          t[j][1] = a1;
        } else {  // rows (2i, 2i + 1) held by lanes g, g ^ 1
          const double other = __shfl_xor_sync(0xffffffffu, (g & 1) ? a0 : a1, 4);
          const bool odd = g & 1;
          const int64_t col = odd ? C0 + 1 : C0;
          ok[j] = R0 < jb.me && col < jb.ne;
          p[j] = ok[j] ? c_ptr<CDT>(jb.out, R0 >> 1, col) : const_cast<R*>(dummy);
          t[j][0] = odd ? other : a0;
          t[j][1] = odd ? a1 : other;
        }
      }
      put_group<CDT, 4>(jb, p, ok, t);
    }
  }
}

// F group epilogue: thread (ty, tx) holds rows {4ty..4ty+3, 32+4ty..} x
// columns {4tx..4tx+3, 64+4tx..}; both parts of a complex pair are its own.
template <int CDT>
__device__ __forceinline__ void epilogue_f(const DualJob& jb, int tm, int tn, int ty, int tx, uint64_t (&acc)[8][4]) {
  using R = typename OutType<CDT>::R;
  constexpr bool cplx = OutType<CDT>::kComplex;
  auto val = [&](int i, int j) -> double {
    const uint64_t v = acc[i][j >> 1];
    return __uint_as_float(static_cast<uint32_t>((j & 1) ? (v >> 32) : v));
  };
  auto row = [&](int i) -> int64_t {
    return static_cast<int64_t>(tm) * DF_BM + (i < 4 ? ty * 4 + i : DF_BM / 2 + ty * 4 + (i - 4));
  };
  auto col = [&](int j) -> int64_t {
    return static_cast<int64_t>(tn) * DF_BN + (j < 4 ? tx * 4 + j : DF_BN / 2 + tx * 4 + (j - 4));
  };
  const R* dummy = reinterpret_cast<const R*>(jb.out.base);
  if constexpr (!cplx) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      R* p[8];
      bool ok[8];
      double t[8][2];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        ok[j] = row(i) < jb.me && col(j) < jb.ne;
        p[j] = ok[j] ? c_ptr<CDT>(jb.out, row(i), col(j)) : const_cast<R*>(dummy);
        t[j][0] = val(i, j);
        t[j][1] = 0.0;
      }
      put_group<CDT, 8>(jb, p, ok, t);
    }
  } else if (jb.pair == MDG_PAIR_COLS) {  // (re, im) = columns (j, j + 1), j even
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      R* p[4];
      bool ok[4];
      double t[4][2];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = 2 * q;
        ok[q] = row(i) < jb.me && col(j) < jb.ne;
        p[q] = ok[q] ? c_ptr<CDT>(jb.out, row(i), col(j) >> 1) : const_cast<R*>(dummy);
        t[q][0] = val(i, j);
        t[q][1] = val(i, j + 1);
      }
      put_group<CDT, 4>(jb, p, ok, t);
    }
  } else {  // (re, im) = rows (i, i + 1), i even
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      R* p[8];
      bool ok[8];
      double t[8][2];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        ok[j] = row(i) < jb.me && col(j) < jb.ne;
        p[j] = ok[j] ? c_ptr<CDT>(jb.out, row(i) >> 1, col(j)) : const_cast<R*>(dummy);
        t[j][0] = val(i, j);
        t[j][1] = val(i + 1, j);
      }
      put_group<CDT, 8>(jb, p, ok, t);
    }
  }
}

// The producer lane warms L2 with a tile's C (read by the epilogue after the
// mainloop) when it starts the tile: one bulk prefetch per output column
// segment when C's columns are contiguous (rs == 1).
__device__ __forceinline__ void prefetch_c(const DualJob& jb, int tm, int tn, int BM, int BN) {
  if (jb.beta.is_zero || jb.out.rs != 1) return;
  const bool prow = jb.pair == MDG_PAIR_ROWS, pcol = jb.pair == MDG_PAIR_COLS;
  const int64_t r0 = static_cast<int64_t>(tm) * BM, c0 = static_cast<int64_t>(tn) * BN;
  const int64_t oi0 = prow ? r0 / 2 : r0, oj0 = pcol ? c0 / 2 : c0;
  const int64_t om = prow ? jb.me / 2 : jb.me, on = pcol ? jb.ne / 2 : jb.ne;
  if (oi0 >= om || oj0 >= on) return;
  const int esz = (dt_single(jb.out.dtype) ? 4 : 8) * (dt_complex(jb.out.dtype) ? 2 : 1);
  const int64_t rows = min(om - oi0, static_cast<int64_t>(prow ? BM / 2 : BM));
  const int64_t cols = min(on - oj0, static_cast<int64_t>(pcol ? BN / 2 : BN));
  const uint32_t bytes = static_cast<uint32_t>(rows * esz) & ~15u;
  if (bytes == 0) return;
  for (int64_t j = 0; j < cols; ++j) {
    const char* q = jb.out.base + (oi0 + (oj0 + j) * jb.out.cs) * esz;
    if ((reinterpret_cast<uint64_t>(q) & 15) == 0) bulk_prefetch_l2(q, bytes);
  }
}

// Register split per warp group (setmaxnreg): RP producers, RD DMMA warps,
// RF FFMA2 warps; RP*128 + RD*256 + RF*128 = the CTA's launch allocation.
template <int DD_STAGES, int DF_STAGES, int PAD, int RP, int RD, int RF>
__device__ __forceinline__ void dual_body(const DualDesc& d) {
  constexpr size_t DD_RING = DuRings<DD_STAGES, DF_STAGES, PAD>::DD_RING;
  constexpr size_t DF_RING = DuRings<DD_STAGES, DF_STAGES, PAD>::DF_RING;
  constexpr int DD_P = DPitch<PAD>::P, DD_SA = DPitch<PAD>::SA, DD_SB = DPitch<PAD>::SB;
  const uint32_t sleep_ns = static_cast<uint32_t>(d.sleep_ns);  // producers' empty-slot waits (0: spin)
  extern __shared__ __align__(128) unsigned char smem[];
  double* dA = reinterpret_cast<double*>(smem);
  double* dB = dA + DD_STAGES * DD_SA;
  float* fA = reinterpret_cast<float*>(smem + DD_RING);
  float* fB = fA + DF_STAGES * DF_SA;
  uint64_t* dfull = reinterpret_cast<uint64_t*>(smem + DD_RING + DF_RING);
  uint64_t* dempty = dfull + DD_STAGES;
  uint64_t* ffull = dempty + DD_STAGES;
  uint64_t* fempty = ffull + DF_STAGES;
  int* dslot = reinterpret_cast<int*>(fempty + DF_STAGES);  // tile of each stage's first k-block
  int* fslot = dslot + DD_STAGES;
  int* dtile = fslot + DF_STAGES;  // D warps: the tile of the running mainloop
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = static_cast<int>(gridDim.x);
  if (threadIdx.x == 0) {
    for (int s = 0; s < DD_STAGES; ++s) {
      mbar_init(&dfull[s], 1);
      mbar_init(&dempty[s], DD_WARPS);
    }
    for (int s = 0; s < DF_STAGES; ++s) {
      mbar_init(&ffull[s], 1);
      mbar_init(&fempty[s], DF_WARPS);
    }
    mbar_fence_init();
    if (d.timing) atomicMax(&d.timing[0], ~globaltimer());  // ~start: zero-initialised like the ends
  }
  __syncthreads();

  if (warp >= DD_PROD_WARP) {  // ------------------------------------------ producers
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(RP));
    if (lane != 0) return;
    // Tile order: CTA b starts with tile b; with d.counters every further tile
    // comes from the group's atomic counter (the tiles are sorted longest-k
    // first, so CTAs that finish early take the next longest: balanced tails),
    // else the static boustrophedon rounds.  The producer hands the tile to
    // its consumers in the first stage's slot; -1 ends the list.
    // A stage is BK panel lines of the packed operands (SA / BK and SB / BK
    // elements each: the panel dimension, or the D group's padded pitch), one
    // contiguous bulk copy per operand
    auto run_producer = [&](auto* A, auto* B, uint64_t* full, uint64_t* empty, int* slot, const DualJob* jobs,
                            int njobs, int tiles, int* counter, int STAGES, int BM, int BN, int SA, int SB, int BK,
                            int esz) {
      using T = typename std::remove_pointer<decltype(A)>::type;
      int it = 0;
      auto next = [&](int r) -> int {
        if (counter) return r == 0 ? static_cast<int>(blockIdx.x) : atomicAdd(counter, 1) + G;
        int v;
        do {
          v = snake_tile(r, G);
          if (v < tiles) return v;
          ++r;
        } while ((r - 1) * G < tiles);
        return tiles;
      };
      for (int r = 0;; ++r) {
        const int v = next(r);
        if (v >= tiles) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait_sleep_u32(smem_u32(&empty[s]), ((it / STAGES) - 1) & 1, sleep_ns);
          slot[s] = -1;
          mbar_arrive(&full[s]);
          return;
        }
        const DualJob& jb = jobs[job_of(jobs, njobs, v)];
        int tm, tn;
        tile_coords(jb.tile_begin + v - jb.tile0, jb.tiles_m, jb.tiles_n, 0, tm, tn);
        MDG_CHECK(v >= jb.tile0 && tm >= 0 && tm < jb.tiles_m && tn >= 0 && tn < jb.tiles_n && jb.lpad % BK == 0,
                  "dual producer job / tile");
        if (d.prefetch_c) prefetch_c(jb, tm, tn, BM, BN);
        // panels of SA / BK (SB / BK) elements per line
        const T* Ag = static_cast<const T*>(jb.a) + static_cast<int64_t>(tm) * (SA / BK) * jb.lpad;
        const T* Bg = static_cast<const T*>(jb.b) + static_cast<int64_t>(tn) * (SB / BK) * jb.lpad;
        const int nk = static_cast<int>(jb.lpad / BK);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait_sleep_u32(smem_u32(&empty[s]), ((it / STAGES) - 1) & 1, sleep_ns);
          // stage word: the tile (2v) on its first k-block, bit 0 on its last
          slot[s] = (kb == 0 ? 2 * v : 0) | (kb == nk - 1 ? 1 : 0);
          mbar_arrive_expect_tx(&full[s], (SA + SB) * esz);
          bulk_g2s(A + s * SA, Ag + static_cast<int64_t>(kb) * SA, SA * esz, &full[s]);
          bulk_g2s(B + s * SB, Bg + static_cast<int64_t>(kb) * SB, SB * esz, &full[s]);
        }
        if (!counter && (r + 1) * G >= tiles) {  // static order: done after the last round
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait_sleep_u32(smem_u32(&empty[s]), ((it / STAGES) - 1) & 1, sleep_ns);
          slot[s] = -1;
          mbar_arrive(&full[s]);
          return;
        }
      }
    };
    if (warp == DD_PROD_WARP)
      run_producer(dA, dB, dfull, dempty, dslot, d.d, d.nd, d.tiles_d, d.counters ? d.counters : nullptr, DD_STAGES,
                   DD_BM, DD_BN, DD_SA, DD_SB, DU_BK, static_cast<int>(sizeof(double)));
    else if (warp == DF_PROD_WARP)
      run_producer(fA, fB, ffull, fempty, fslot, d.f, d.nf, d.tiles_f, d.counters ? d.counters + 1 : nullptr,
                   DF_STAGES, DF_BM, DF_BN, DF_SA, DF_SB, DF_BK, static_cast<int>(sizeof(float)));
    return;
  }

  if (warp < DD_WARPS) {  // ----------------------------------------------- D group
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(RD));
    const int wm = warp % 2, wn = warp / 2;
    const int g = lane >> 2, tig = lane & 3;
    const double* a_base = dA + wm * 64 + g + tig * DD_P;
    const double* b_base = dB + wn * 32 + g + tig * DD_P;
    const uint32_t full_u = smem_u32(dfull), empty_u = smem_u32(dempty);
    const uint32_t a_u = smem_u32(a_base), b_u = smem_u32(b_base);
    // Ring position in one register: stage in bits 0-1, phase in bit 2; the
    // k-block count runs down.  The loop state the D group keeps live at its
    // register cap is the accumulators, the fragments, this word, the count
    // and two shared addresses (the tile index waits in shared memory).
    uint32_t ring = 0;
    for (;;) {
      // the producer names the next tile in its first stage's slot
      mbar_wait_u32(full_u + 8 * (ring & 3), ring >> 2);
      const int w0 = *reinterpret_cast<volatile int*>(&dslot[ring & 3]);
      if (w0 < 0) break;
      if (lane == 0) dtile[warp] = w0 >> 1;  // read back for the epilogue
      double acc[8][4][2];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      bool first = true, last;
      do {
        const uint32_t s = ring & 3;
        if (!first) mbar_wait_u32(full_u + 8 * s, ring >> 2);
        first = false;
        last = *reinterpret_cast<volatile int*>(&dslot[s]) & 1;  // the producer marks the tile's last k-block
        const uint32_t a = a_u + s * (DD_SA * 8), b = b_u + s * (DD_SB * 8);
#pragma unroll
        for (int kk = 0; kk < DU_BK; kk += 4) {
          double af[8], bf[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) bf[j] = lds_f64(b + (kk * DD_P + j * 8) * 8);
#pragma unroll
          for (int i = 0; i < 8; ++i) af[i] = lds_f64(a + (kk * DD_P + i * 8) * 8);
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma884_du(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        fence_proxy_async();  // generic reads of the stage before its TMA refill
        __syncwarp();
        if (lane0()) mbar_arrive_u32(empty_u + 8 * s);
        ring = s + 1 == DD_STAGES ? (ring & 4) ^ 4 : ring + 1;
      } while (!last);
      __syncwarp();
      const int vt = *reinterpret_cast<volatile int*>(&dtile[warp]);
      const int jx = job_of(d.d, d.nd, vt);
      const DualJob* jp = &d.d[jx];
      int tm, tn;
      tile_coords(jp->tile_begin + vt - jp->tile0, jp->tiles_m, jp->tiles_n, 0, tm, tn);
      MDG_DISPATCH_CDT(jp->out.dtype, CDT, { epilogue_d<CDT>(*jp, tm, tn, warp % 2, warp / 2, lane, acc); });
    }
    if (d.timing && lane == 0) atomicMax(&d.timing[1], globaltimer());
    return;
  }

  // ------------------------------------------------------------------- F group
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(RF));
  const int ft = threadIdx.x - DD_WARPS * 32;
  const int tx = ft % 16, ty = ft / 16;
  const float* a_base = fA + ty * 4;
  const float* b_base = fB + tx * 4;
  const uint32_t full_u = smem_u32(ffull), empty_u = smem_u32(fempty);
  int* ftile = dtile + DD_WARPS;  // F warps: the tile of the running mainloop
  const int fw = warp - DD_WARPS;
  uint32_t ring = 0;  // stage in bits 0-2, phase in bit 3
  for (;;) {
    mbar_wait_u32(full_u + 8 * (ring & 7), ring >> 3);
    const int w0 = *reinterpret_cast<volatile int*>(&fslot[ring & 7]);
    if (w0 < 0) break;
    if (lane0()) ftile[fw] = w0 >> 1;  // read back for the epilogue
    uint64_t acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int p = 0; p < 4; ++p) acc[i][p] = 0ull;
    bool first = true, last;
    do {
      const uint32_t s = ring & 7;
      if (!first) mbar_wait_u32(full_u + 8 * s, ring >> 3);
      first = false;
      last = *reinterpret_cast<volatile int*>(&fslot[s]) & 1;  // the producer marks the tile's last k-block
      const float* a = a_base + s * DF_SA;
      const float* b = b_base + s * DF_SB;
#pragma unroll
      for (int kk = 0; kk < DF_BK; ++kk) {
        const float4 a0 = *reinterpret_cast<const float4*>(a + kk * DF_BM);
        const float4 a1 = *reinterpret_cast<const float4*>(a + kk * DF_BM + DF_BM / 2);
        const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(b + kk * DF_BN);
        const ulonglong2 b1 = *reinterpret_cast<const ulonglong2*>(b + kk * DF_BN + DF_BN / 2);
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
      if (lane0()) mbar_arrive_u32(empty_u + 8 * s);
      ring = s + 1 == DF_STAGES ? (ring & 8) ^ 8 : ring + 1;
    } while (!last);
    __syncwarp();
    const int v = *reinterpret_cast<volatile int*>(&ftile[fw]);
    const DualJob* jp = &d.f[job_of(d.f, d.nf, v)];
    int tm, tn;
    tile_coords(jp->tile_begin + v - jp->tile0, jp->tiles_m, jp->tiles_n, 0, tm, tn);
    MDG_DISPATCH_CDT(jp->out.dtype, CDT, { epilogue_f<CDT>(*jp, tm, tn, ty, tx, acc); });
  }
  if (d.timing && lane == 0) atomicMax(&d.timing[2], globaltimer());
}

// The whole register file (128 per thread at launch: 256 x 168 + 128 x 144 +
// 128 x 32 = 64 K).
template <int DD_STAGES, int DF_STAGES, int PAD>
__global__ void __launch_bounds__(DU_THREADS, 1) gemm_dual_kernel(const __grid_constant__ DualDesc d) {
  dual_body<DD_STAGES, DF_STAGES, PAD, 32, 168, 144>(d);
}

template <int DS, int FS, int PAD>
cudaError_t launch_stages(const DualDesc& d, int grid, cudaStream_t s) {
  constexpr size_t smem = DuRings<DS, FS, PAD>::SMEM;
  auto kern = gemm_dual_kernel<DS, FS, PAD>;
  cudaError_t attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (attr != cudaSuccess) return attr;
  kern<<<static_cast<unsigned>(grid), DU_THREADS, smem, s>>>(d);
  return cudaGetLastError();
}

}  // namespace

size_t dual_smem() { return DuRings<3, 4>::SMEM; }

static int dual_pad() {  // tuning: MDGEMM_DUAL_PAD = 0 packed D line pitch (4-way bank conflicts)
  static const int pad = [] {
    const char* f = std::getenv("MDGEMM_DUAL_PAD");
    return f && std::atoi(f) == 0 ? 0 : 4;
  }();
  return pad;
}

int dual_d_pitch() { return DD_BM + dual_pad(); }

cudaError_t launch_gemm_dual(const DualDesc& d, int grid, cudaStream_t s) {
  if (grid <= 0 || (d.tiles_d == 0 && d.tiles_f == 0)) return cudaSuccess;
  static const int variant = [] {  // tuning: MDGEMM_DUAL_STAGES = 0 (3 D / 4 F), 1 (3 / 5)
    const char* f = std::getenv("MDGEMM_DUAL_STAGES");
    return f ? std::atoi(f) : 0;
  }();
  if (dual_pad() == 0) return launch_stages<3, 4, 0>(d, grid, s);
  if (variant == 1) return launch_stages<3, 5, 4>(d, grid, s);
  return launch_stages<3, 4, 4>(d, grid, s);
}

}  // namespace mdg
