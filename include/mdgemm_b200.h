/*
 * mdgemm_b200.h -- C ABI of the B200 (sm_100a) mixed-datatype gemm.
 *
 * This is the drop-in boundary.  The reference engine (arXiv 1901.06015,
 * "mdgemm", /root/reference/proj) runs   C := beta*C + alpha*A*B   for every
 * combination of real/complex x single/double storage of A, B, C plus a
 * separate computation precision read from C (128 "cabx" labels).  Its public
 * C++ entry point is
 *
 *     void mdgemm::gemm(Scalar alpha, const MatrixView& a, const MatrixView& b,
 *                       Scalar beta, const MatrixView& c, const Config& cfg,
 *                       FlopCounter* fc)                 (dispatch.hpp:89-91)
 *
 * and its execution half (everything after plan(), dispatch.cpp:359-388:
 * gemm_blocked, the C_temp buffer + write_back, beta_pass) is what this
 * library replaces with CUDA kernels.  Every struct below is plain old data
 * with fixed-width fields; no CUDA or C++ types cross the boundary.
 *
 * Error behaviour mirrors the reference's exceptions: MDG_ERR <-> mdgemm::Error,
 * MDG_ERR_SCALAR_POLICY <-> mdgemm::ScalarPolicyError (dtypes.hpp:14-20).
 * CUDA failures map to MDG_ERR_CUDA.  mdg_last_error() returns the message of
 * the most recent failure on the calling thread.
 */
#ifndef MDGEMM_B200_H
#define MDGEMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MDG_ABI_VERSION 2

/* ---- enumerations (values follow the reference enums' declaration order) -- */

/* Datatype s/d/c/z  (dtypes.hpp:44-47) */
enum { MDG_DT_S = 0, MDG_DT_D = 1, MDG_DT_C = 2, MDG_DT_Z = 3 };
/* Precision (dtypes.hpp:23) */
enum { MDG_PREC_SINGLE = 0, MDG_PREC_DOUBLE = 1 };
/* CaseId (dtypes.hpp:63) */
enum {
  MDG_CASE_0 = 0, MDG_CASE_1A, MDG_CASE_1B, MDG_CASE_1C,
  MDG_CASE_2AB, MDG_CASE_2AC, MDG_CASE_2BC, MDG_CASE_3
};
/* Side / PackFormat (packing.hpp:24-26) */
enum { MDG_SIDE_LEFT = 0, MDG_SIDE_RIGHT = 1 };
enum { MDG_FMT_STANDARD = 0, MDG_FMT_ONEE = 1, MDG_FMT_ONER = 2 };
/* Preference, PairAxis (kernels.hpp:13-17) */
enum { MDG_PREF_COLUMN = 0, MDG_PREF_ROW = 1 };
enum { MDG_PAIR_NONE = 0, MDG_PAIR_ROWS = 1, MDG_PAIR_COLS = 2 };
/* UkrPath, MacroMode (dispatch.hpp:32-33) */
enum { MDG_PATH_DIRECT = 0, MDG_PATH_TEMP = 1, MDG_PATH_ONEM_COLUMN = 2, MDG_PATH_ONEM_ROW = 3 };
enum { MDG_MACRO_STANDARD = 0, MDG_MACRO_ACCUMULATE_TYPECAST = 1 };
/* CTempMode (config.hpp:22), CTempDescriptor::Mode (dispatch.hpp:44) */
enum { MDG_CTEMP_AUTO = 0, MDG_CTEMP_ON = 1, MDG_CTEMP_OFF = 2 };
enum { MDG_CTEMP_COPY_BACK = 0, MDG_CTEMP_ACCUMULATE_BACK = 1 };

/* Device numerics (B200 extension, config key "gpu.numerics"):
 *  FAST  - DMMA (fp64) / FFMA (fp32) tensor/SIMT mainloops; C within the
 *          reference's error bound.
 *  EXACT - replays the reference's per-element rounding sequence (separate
 *          multiply and add, ascending inner index, beta seeding and per-KC
 *          block combine exactly as gemm_blocked does): bitwise identical to
 *          the reference CPU engine for the same Config. */
enum { MDG_NUMERICS_FAST = 0, MDG_NUMERICS_EXACT = 1 };
/* mdg_execute: OR into `numerics` to forbid split-K for this call */
enum { MDG_EXEC_NO_SPLITK = 0x100 };

/* Status codes */
enum { MDG_OK = 0, MDG_ERR = 1, MDG_ERR_SCALAR_POLICY = 2, MDG_ERR_CUDA = 3 };

/* ---- plain data mirrors of the reference types ---------------------------- */

/* MatrixView (dtypes.hpp:102-131).  Strides in elements of `dtype`. */
typedef struct mdg_view {
  void* base;
  int64_t m, n, rs, cs;
  int32_t dtype;
  int32_t conj;
  int32_t comp_prec;
  int32_t target_dtype;
} mdg_view_t;

/* Scalar (dtypes.hpp:70-83): payload held in double, rounded to dtype. */
typedef struct mdg_scalar {
  double re, im;
  int32_t dtype;
  int32_t reserved;
} mdg_scalar_t;

/* BlockingParams (config.hpp:13-20) */
typedef struct mdg_blocking {
  int64_t mc, nc, kc;
  int32_t mr, nr;
} mdg_blocking_t;

/* Config (config.hpp:38-72) + device numerics */
typedef struct mdg_config {
  mdg_blocking_t single_params;
  mdg_blocking_t double_params;
  int32_t threads;
  int32_t preference;
  int32_t ctemp;
  int32_t numerics;
  int32_t splitk;    /* gpu.splitk: 1 auto (default), 0 off */
  int32_t reserved;
} mdg_config_t;

/* ExecutionPlan (dispatch.hpp:52-80) */
typedef struct mdg_plan {
  int32_t case_id;
  int32_t logical_transpose;
  int32_t comp_prec;
  int32_t reserved0;
  int64_t m, n, k;
  mdg_view_t a, b, c;
  int32_t format_a, format_b;
  int32_t conj_a, conj_b;
  int32_t target_dtype_a, target_dtype_b;
  int64_t reg_block_a, reg_block_b;
  mdg_scalar_t alpha, beta, pack_scale_a, pack_scale_b;
  int32_t macro_mode, ukr_path, pair_axis;
  int32_t has_ctemp;
  int64_t ctemp_rows, ctemp_cols;
  int32_t ctemp_precision, ctemp_mode;
  mdg_blocking_t params;
  int32_t threads;
  int32_t ukr_precision, ukr_mr, ukr_nr, ukr_preference;
  int32_t reserved1;
} mdg_plan_t;

/* ---- entry points --------------------------------------------------------- */

int mdg_abi_version(void);
const char* mdg_last_error(void);

/* Config::defaults / Config::set / Config::load / Config::validate
 * (config.hpp:45-57, config.cpp:51-156).  Extra key: gpu.numerics=fast|exact. */
int mdg_config_defaults(mdg_config_t* out);
int mdg_config_set(mdg_config_t* cfg, const char* key, const char* value);
int mdg_config_load(mdg_config_t* out, const char* path_or_null, int apply_env);
int mdg_config_validate(const mdg_config_t* cfg);

/* MatrixView::make (dtypes.cpp:82-111): validates dims/strides. */
int mdg_view_make(void* base, int64_t m, int64_t n, int64_t rs, int64_t cs,
                  int32_t dtype, mdg_view_t* out);

/* classify_case / flops_of_case / apply_scalar_policy (dispatch.cpp:11-85). */
int32_t mdg_classify_case(int32_t c_domain_complex, int32_t a_domain_complex,
                          int32_t b_domain_complex);
uint64_t mdg_flops_of_case(int32_t case_id, int64_t m, int64_t n, int64_t k);
int mdg_apply_scalar_policy(mdg_scalar_t alpha, mdg_scalar_t beta, int32_t case_id,
                            int32_t comp_prec, int32_t c_storage_prec,
                            mdg_scalar_t* alpha_out, mdg_scalar_t* beta_out);

/* plan() (dispatch.cpp:106-305): host-only, no device work. */
int mdg_plan(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b,
             mdg_scalar_t beta, const mdg_view_t* c, const mdg_config_t* cfg,
             mdg_plan_t* out);

/* Executes a plan whose views hold DEVICE pointers, stream-ordered on
 * `stream` (a cudaStream_t, NULL = legacy default stream); does not
 * synchronise.  Replaces dispatch.cpp:359-388.  *flops_out (optional)
 * receives the reference FlopCounter value (kernels.cpp:73-76). */
int mdg_execute(const mdg_plan_t* p, int32_t numerics, void* stream,
                uint64_t* flops_out);

/* Whole gemm() (dispatch.cpp:350-389): alias check, plan, execute.
 * Views may hold host or device pointers (host operands are staged through
 * device memory).  Synchronous, like the reference. */
int mdg_gemm(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b,
             mdg_scalar_t beta, const mdg_view_t* c, const mdg_config_t* cfg,
             uint64_t* flops_out);

/* A batch of gemm() calls, equivalent to mdg_gemm on each in order.  Each
 * distinct host operand window crosses PCIe once per batch (it stays
 * resident in HBM while later calls read or update it; a host C is copied
 * back once, after its last writer); copies overlap neighbouring calls'
 * kernels and calls touching disjoint memory run concurrently.  Synchronous. */
typedef struct mdg_gemm_call {
  mdg_scalar_t alpha;
  mdg_view_t a, b;
  mdg_scalar_t beta;
  mdg_view_t c;
} mdg_gemm_call_t;

int mdg_gemm_batch(int32_t count, const mdg_gemm_call_t* calls, const mdg_config_t* cfg,
                   uint64_t* flops_out);

/* Same, forked from and joined back into `stream` without synchronising
 * (independent calls run concurrently on the library's compute streams). */
int mdg_gemm_batch_async(int32_t count, const mdg_gemm_call_t* calls, const mdg_config_t* cfg,
                         void* stream, uint64_t* flops_out);

/* The launch schedule mdg_gemm_batch would use on the dual-pipe kernel, computed
 * on the host without touching a device (tests / tooling): *npieces entries of
 * five int32 {launch, call, tile begin, tile end, group} (group 1 = FP64 job,
 * 2 = FP32 job, 0 = the call runs through mdg_execute in that launch slot),
 * at most `capacity` written; call_tiles[i] = the tiles of call i (0 if not a
 * dual job).  *npieces = 0 when the batch would not take the dual path. */
int mdg_dual_schedule(int32_t count, const mdg_gemm_call_t* calls, const mdg_config_t* cfg, int32_t capacity,
                      int32_t* pieces, int32_t* npieces, int32_t* call_tiles);

/* Same with device pointers only, stream-ordered, no synchronisation. */
int mdg_gemm_async(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b,
                   mdg_scalar_t beta, const mdg_view_t* c, const mdg_config_t* cfg,
                   void* stream, uint64_t* flops_out);

/* packed_bytes (packing.cpp:107-112); panel_len >= the logical panel length
 * pads every panel with zero rows (0 = no padding, the reference layout). */
size_t mdg_packed_bytes(const mdg_view_t* src, int32_t side, int32_t format,
                        int32_t target_dtype, int64_t reg_block, int64_t panel_len);

/* pack_block_into (packing.cpp:232-237) on the device: src and dst are device
 * pointers.  Byte-identical to the reference pack when panel_len == 0. */
int mdg_pack_operand(const mdg_view_t* src, int32_t side, int32_t format, int32_t conj,
                     mdg_scalar_t scale, int32_t target_dtype, int64_t reg_block,
                     int64_t panel_len, void* dst, void* stream);

/* fill_uniform (rng.hpp:49-56) on the device: the counter-based splitmix64
 * stream with state `rng_state`, so device inputs equal the reference's
 * seeded host inputs bit for bit. */
int mdg_fill_uniform(const mdg_view_t* v, uint64_t rng_state, void* stream);
/* normal(0,1) entries from the same stream (BASELINE configs[4]; the
 * reference has no normal generator): Box-Muller, real component t from draws
 * 2t and 2t+1: u1 = (1 - d0)/2, u2 = (1 + d1)/2, z = sqrt(-2 ln u1) cos(2 pi u2). */
int mdg_fill_normal(const mdg_view_t* v, uint64_t rng_state, void* stream);

/* Rng::split(tag) / Rng::split(salt) (rng.hpp:34-41) on a raw state. */
uint64_t mdg_rng_split_tag(uint64_t state, const char* tag);
uint64_t mdg_rng_split_salt(uint64_t state, uint64_t salt);

/* Column-panel sharding for the multi-GPU split (C and B split by columns,
 * A replicated): rank r of `world` gets columns [*j0, *j0 + *nb).  Panels
 * are multiples of `align` columns except the last. */
int mdg_shard_columns(int64_t n, int32_t world, int32_t rank, int64_t align,
                      int64_t* j0, int64_t* nb);

/* ---- multi-GPU: C and B column panels, A broadcast over
 * NVLink / NVSwitch with NCCL (loaded at run time), no reduction ---------
 * mdg_comm_*: one process per GPU.  Rank 0 gets an id (mdg_comm_unique_id),
 * the caller shares the 128 bytes with the other ranks (any out-of-band
 * channel), and every rank calls mdg_comm_init on its own device.
 * mdg_gemm_sharded: this rank's panel of C := beta*C + alpha*A*B; `a` is A on
 * the root (other ranks: the same geometry, base null = library-owned
 * receive buffer); b_panel / c_panel are this rank's device panels
 * (mdg_shard_columns).  Stream-ordered, no host synchronisation.
 * mdg_gemm_multi: the whole call over `ndev` GPUs of this process
 * (operands in host or device memory), synchronous. */
typedef struct mdg_comm* mdg_comm_t;
enum { MDG_COMM_ID_BYTES = 128 };
int mdg_comm_unique_id(uint8_t* id /* [MDG_COMM_ID_BYTES] */);
int mdg_comm_init(const uint8_t* id, int32_t nranks, int32_t rank, mdg_comm_t* out);
int mdg_comm_destroy(mdg_comm_t comm);
int mdg_gemm_sharded(mdg_comm_t comm, int32_t root, mdg_scalar_t alpha, const mdg_view_t* a,
                     const mdg_view_t* b_panel, mdg_scalar_t beta, const mdg_view_t* c_panel,
                     const mdg_config_t* cfg, void* stream, uint64_t* flops_out);
int mdg_gemm_multi(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b, mdg_scalar_t beta,
                   const mdg_view_t* c, const mdg_config_t* cfg, int32_t ndev, const int32_t* devices,
                   uint64_t* flops_out);

/* ---- instrumentation (the reference's FlopCounter, extended per kernel) ---
 * Every kernel the library launches bumps a process-wide counter.  Between
 * mdg_profile_begin() and mdg_profile_end() the calling thread also brackets
 * each launch with CUDA events on its stream (no synchronisation until
 * _end), and _end reports per kernel kind: launches, summed device time and
 * the algorithmic work (flops for gemm kernels, bytes read + written for
 * pack / beta kernels). */
enum {
  MDG_KERNEL_PACK = 0, MDG_KERNEL_DMMA = 1, MDG_KERNEL_FFMA = 2, MDG_KERNEL_EXACT = 3,
  MDG_KERNEL_BETA = 4, MDG_KERNEL_FILL = 5,
  /* the dual-pipe kernel (gemm_batch): each launch is recorded under both
   * kinds with the same device time, its work split by pipe (FP64 DMMA flops
   * under DUAL_D, FP32 FFMA flops under DUAL_F; DUAL_F counts no launch) */
  MDG_KERNEL_DUAL_D = 6, MDG_KERNEL_DUAL_F = 7, MDG_KERNEL_KINDS = 8
};

typedef struct mdg_kernel_stats {
  uint64_t launches;
  double total_ms;
  double work;
} mdg_kernel_stats_t;

/* Workspace: the library allocates packed panels, staged host operands and
 * C_temp-style scratch from its own stream-ordered pool per device, which
 * keeps what it has between calls (no mapping inside a batch).  This
 * synchronises the current device and returns the pool's memory above
 * keep_bytes to the system. */
int mdg_trim_workspace(uint64_t keep_bytes);

uint64_t mdg_launch_count(void);
/* Bytes the batch runner has staged host->device / device->host so far. */
void mdg_staging_bytes(uint64_t* h2d, uint64_t* d2h);
int mdg_profile_begin(void);
int mdg_profile_end(mdg_kernel_stats_t* out /* [MDG_KERNEL_KINDS] */);

#ifdef __cplusplus
}
#endif

#endif /* MDGEMM_B200_H */
