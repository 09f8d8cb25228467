// Plain descriptors passed by value from the host driver to the kernels,
// plus the host-callable launchers.  No CUDA runtime types in the
// signatures beyond cudaStream_t.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda.h>  // CUtensorMap (types only; the encoder is fetched at run time)
#include <cuda_runtime.h>

#include "mdgemm_b200.h"

namespace mdg {

// A strided typed view in device memory (MatrixView minus planner metadata).
struct DView {
  char* base;
  int64_t m, n, rs, cs;
  int32_t dtype;
  int32_t conj;
};

// Resolved beta of the plan (already rounded to C's storage precision).
struct DBeta {
  double re, im;
  int32_t is_zero, is_one;
};

// Where accumulated real-image values go: element (r, c) of the me x ne real
// computation maps onto `out` directly (pair NONE), or pairs rows (2i,2i+1)
// / columns (2j,2j+1) into one complex element.
struct DEpilogue {
  // C as a 2-D tiled tensor (inner dimension: rows x components in C's real
  // type, outer: columns) for TMA tensor loads/stores of C_BOX_COLS-column
  // boxes; valid when cmap_ok (column-major C with 16-byte aligned columns).
  CUtensorMap cmap;
  // The same C as SWIZZLE_128B boxes of 128 bytes x C_BOX_COLS lines (real
  // column-major C only, sw_ok): the warp-specialised kernels' tile buffer then
  // has no shared-memory bank conflicts in the combine pass.
  CUtensorMap cmap_sw;
  DView out;
  int32_t pair;
  int32_t cmap_ok;
  DBeta beta;
  int64_t me, ne;
  int32_t sw_ok;
  int32_t pad_sw;
};
constexpr int C_BOX_COLS = 16;  // lines (columns, or rows for MDG_CMAP_ROWS) per TMA box
// DEpilogue::cmap_ok: how the tensor map covers C
enum : int32_t {
  MDG_CMAP_NONE = 0,       // no map: element-wise epilogue
  MDG_CMAP_COLS = 1,       // column-major C (rs == 1)
  MDG_CMAP_ROWS = 2,       // row-major C (cs == 1): a transposed plan
  MDG_CMAP_REAL_PART = 3,  // real view with rs == 2 (real part of an interleaved complex C); the map
                           // covers both halves and the other half is written back unchanged
};

// Panel geometry of one packed operand, in real elements of the computation
// precision: panels of `pd` rows (left) / columns (right), `lpad` inner-
// dimension steps each, contiguous pd-vectors per step.
struct DPanels {
  const void* data;
  int64_t pd;
  int64_t lpad;
};

struct PackDesc {
  DView src;
  int32_t side, format;
  int32_t do_conj, unit_scale;
  double sre, sim;
  int32_t target_single;   // target precision is single
  int32_t out_complex;     // Standard pack of a complex source: complex elements
  int64_t pd;              // panel dim in packed-logical units (reg_block)
  int64_t panels;
  int64_t len;             // logical panel length
  int64_t lpad;            // allocated panel length (>= len), zero-filled
  int64_t ext_i, ext_j;    // source index space incl. panel padding
  int32_t pd_shift;        // log2(pd) when pd is a power of two, else -1
  int32_t pitch;           // elements between consecutive panel lines (= pd: the reference layout;
                           // wider: padded lines, the dual kernel's conflict-free D stages)
  int32_t vec;             // set by the pack launchers: 16-byte vector tiles (pack_tile.cuh: vec_ok)
  int32_t cvec;            // set by the pack launchers: complex source elements aligned to their own size
                           // (one 8- / 16-byte load per element instead of two)
  int32_t interior;        // set by the pack launchers: tiles inside the source take the 32-bit index path
  int32_t pad_;
};

// Exact (reference-replaying) gemm modes.
enum ExactMode : int32_t {
  EXACT_FULL_THEN_COMBINE = 0,  // C_temp: sum from zero over all k, one combine
  EXACT_DIRECT_SEEDED = 1,      // Direct: accumulators seeded with beta*c in T
  EXACT_BLOCK_COMBINE = 2,      // Temp without C_temp: combine per KC block
  EXACT_ONEM_MIXED = 3,         // 1m with complex beta: first KC block through the
                                // temp tile, later blocks continue in T on the
                                // flattened C (virtual_ukr_onem re-decides per block)
};

struct GemmDesc {
  DPanels a, b;
  int64_t me, ne, ke;
  DEpilogue epi;
  int32_t exact_mode;
  int32_t sk_grid;     // fast kernels: > 0 = stream-K grid of that many CTAs (common.cuh: make_sched)
  int64_t kc;          // EXACT_BLOCK_COMBINE block length (real inner steps)
  double seed_beta;    // EXACT_DIRECT_SEEDED: beta as passed to gemm_ukr
  DView flat;          // EXACT_ONEM_MIXED: real_flatten(C) of the 1m variant
  int32_t group_rows;  // tile raster group height (0 = default 8)
  int32_t splits;      // split-K factor of the fast kernels (1 = none)
  int32_t kb_per_split;  // 16-deep k-blocks per split
  int32_t prefetch;    // fast kernels: L2 prefetch distance in k-blocks ahead of the ring (0 = off)
  void* partials;      // splits > 1: per (tile, split) accumulator tiles, comp precision
  unsigned long long* trace;  // tuning only (MDGEMM_TRACE): TRACE_WORDS stamps per CTA
  void* sk_partials;   // stream-K: sk_grid partial tiles in thread-fragment order, comp precision
  int* sk_flags;       // stream-K: sk_grid publish flags + the start ticket, zeroed before the launch
  int32_t c_prefetch;  // producer warms L2 with the C tile after its loads (short k)
  int32_t pad0;
};

// Stream-K hybrid grid (common.cuh: make_sched): dp whole-tile CTAs, then G
// CTAs sharing the last G + tiles % G tiles as k-block ranges.
inline __host__ __device__ int64_t sk_dp_tiles(int64_t tiles, int64_t G) {
  return tiles % G == 0 ? tiles : (tiles / G - 1) * G;
}
inline __host__ __device__ int64_t sk_launch_grid(int64_t tiles, int64_t G) {
  return sk_dp_tiles(tiles, G) + (tiles % G == 0 ? 0 : G);
}

// Per-CTA timeline for the tuning trace: {smid, start, first stage ready,
// mainloop end, end} (%globaltimer nanoseconds).
// Word 5: the producer's first bulk-copy issue.
constexpr int TRACE_WORDS = 6;

// One job of the dual-pipe kernel (gemm_dual.cu): a FAST gemm whose operands
// are already packed with the group's tile as panel dimension (D group:
// 128-row A panels, 128-column B panels, doubles; F group: 64 / 128, floats)
// and panel length lpad (a multiple of the group's k-block: 16 / 32).
struct DualJob {
  const void* a;
  const void* b;
  int64_t lpad;
  int64_t me, ne;
  DView out;
  DBeta beta;
  int32_t pair;
  int32_t tiles_m, tiles_n;
  int32_t tile0;       // first virtual tile of the job in its group's list
  int32_t tile_begin;  // the job's first tile (raster order) in this launch
  int32_t pad0;
};
constexpr int DUAL_MAX_JOBS = 80;  // per group and launch (kernel parameter space)
struct DualDesc {
  int32_t nd, nf;            // jobs per group
  int32_t tiles_d, tiles_f;  // virtual tiles per group
  int32_t prefetch_c;        // producers warm L2 with each tile's C
  int32_t sleep_ns;          // suspend-time hint of the producers' empty-slot waits (0: spin)
  unsigned long long* timing;  // tuning only: {~first start, D end, F end} (%globaltimer ns, max-reduced) or null
  int* counters;               // {D, F} tile counters, zero before the launch (dynamic tiles), or null
  DualJob d[DUAL_MAX_JOBS];
  DualJob f[DUAL_MAX_JOBS];
};
// passed by value as a __grid_constant__ kernel parameter (limit 32764 bytes)
static_assert(sizeof(DualDesc) <= 32000, "DualDesc exceeds the kernel parameter space");
constexpr int DUAL_D_BM = 128, DUAL_D_BN = 128, DUAL_F_BM = 64, DUAL_F_BN = 128, DUAL_BK = 16, DUAL_F_BK = 32;

// Many packs in one launch (pack.cu: pack_group_kernel): the packs of a dual
// launch's FP64 or FP32 jobs -- up to both operands of DUAL_MAX_JOBS calls,
// any mix of source type, target, format and side; CTA b packs tile b -
// tile0[j] of pack j (tile0: prefix sums of the packs' tile counts).
constexpr int PACK_GROUP_MAX = 2 * DUAL_MAX_JOBS;
struct PackGroup {
  int32_t n;
  int32_t pad0;
  int64_t tile0[PACK_GROUP_MAX + 1];
  void* dst[PACK_GROUP_MAX];
  PackDesc d[PACK_GROUP_MAX];
};
static_assert(sizeof(PackGroup) <= 32000, "PackGroup exceeds the kernel parameter space");

// ---- host launchers (defined in the .cu files) ----
cudaError_t launch_pack(const PackDesc& d, void* dst, cudaStream_t s);
// g.n packs in one launch (fills g.tile0[g.n]); their panel padding rows too.
cudaError_t launch_pack_group(PackGroup& g, cudaStream_t s);
// Both packs of a call in one launch; valid when pack_pair_ok (same source
// type, target precision and format), else it falls back to two launches.
cudaError_t launch_pack_pair(const PackDesc& a, void* da, const PackDesc& b, void* db, cudaStream_t s);
inline bool pack_pair_ok(const PackDesc& a, const PackDesc& b) {
  return a.src.dtype == b.src.dtype && a.target_single == b.target_single && a.format == b.format;
}
// (sms: the SM count the grid-stride grids are sized for)
cudaError_t launch_beta_pass(const DView& out, const DBeta& beta, int sms, cudaStream_t s);
cudaError_t launch_fill_uniform(const DView& v, uint64_t state, int sms, cudaStream_t s);
cudaError_t launch_fill_normal(const DView& v, uint64_t state, int sms, cudaStream_t s);
cudaError_t launch_gemm_exact(const GemmDesc& d, bool single, int sms, cudaStream_t s);

// Fast kernels: tile shape chosen by the driver.
struct FastTile {
  int bm, bn, bk;
};
FastTile choose_dmma_tile(int64_t me, int64_t ne, int sms);
FastTile choose_ffma_tile(int64_t me, int64_t ne, int sms);
cudaError_t launch_gemm_dmma(const GemmDesc& d, const FastTile& t, cudaStream_t s);
cudaError_t launch_gemm_ffma(const GemmDesc& d, const FastTile& t, cudaStream_t s);
// Warp-specialised persistent DMMA kernel (gemm_dmma_ws.cu): 128x128 tiles,
// `grid` CTAs (one per SM); d.sk_grid = grid turns on the stream-K tail.
size_t dmma_ws_smem(int cdt);
cudaError_t launch_gemm_dmma_ws(const GemmDesc& d, int grid, cudaStream_t s);
size_t ffma_ws_smem(int cdt);
cudaError_t launch_gemm_ffma_ws(const GemmDesc& d, int grid, cudaStream_t s);
// Resident CTAs per SM of the kernel a tile shape / C datatype launches
// (occupancy query; sizes the split-K and stream-K grids).
int dmma_ctas_per_sm(const FastTile& t, int cdt);
int ffma_ctas_per_sm(const FastTile& t, int cdt);
// Dual-pipe kernel: one CTA per SM (grid), D and F groups on their job lists.
size_t dual_smem();
// Line pitch (doubles) of the D jobs' packed panels: the D group's smem
// stage pitch (MDGEMM_DUAL_PAD tuning: 128 + pad).
int dual_d_pitch();
cudaError_t launch_gemm_dual(const DualDesc& d, int grid, cudaStream_t s);
// Split-K: sum the `splits` partial tiles in split order and run the fused
// epilogue (one CTA per tile).
cudaError_t launch_splitk_reduce(const GemmDesc& d, const FastTile& t, bool single, cudaStream_t s);
// Split factor for a problem of `tiles` CTA tiles and `nk` k-blocks (1 = none).
int choose_splits(int64_t tiles, int64_t nk, int slots);

}  // namespace mdg
