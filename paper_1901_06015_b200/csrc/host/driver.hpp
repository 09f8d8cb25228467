// Internal host-side declarations shared by the driver and the C ABI.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../device/desc.h"
#include "mdgemm/mdgemm.hpp"

namespace mdgemm {

// CUDA runtime failure, surfaced across the C ABI as MDG_ERR_CUDA.
struct CudaFailure : Error {
  explicit CudaFailure(const std::string& what) : Error(what) {}
};

void cuda_check(cudaError_t e, const char* what);

// SMs the kernels are scheduled for (the device's count, or MDGEMM_SMS when
// a test caps it).
int device_sms();
// The library's private stream-ordered pool on the current device, and a
// stream-ordered allocation from it (free with cudaFreeAsync).
cudaMemPool_t workspace_pool();
cudaError_t ws_alloc(void** p, size_t bytes, cudaStream_t st);
// Synchronise the device and return the pool's cached memory above
// keep_bytes to the system (mdg_trim_workspace).
void trim_workspace(size_t keep_bytes);
// Forget the batch reservation (the pool was trimmed).
void reset_reservation();

// Operand copies between HBM and host memory (hostcopy.cpp): pageable host
// memory goes through the library's pinned chunk ring (d2h_copy then returns
// once the bytes are in place), pinned memory takes a plain async copy.
bool host_pageable(const void* p);
void h2d_copy(void* dst, const void* src, size_t n, cudaStream_t st);
void d2h_copy(void* dst, const void* src, size_t n, cudaStream_t st);
void trim_host_staging();

mdg::DView to_dview(const MatrixView& v);

// resolve_geometry (packing.cpp:27-67) plus an optional padded panel length.
struct PackGeometry {
  Datatype block_dtype = dt_d;
  int64_t panels = 0;
  int64_t len = 0;   // logical panel length
  int64_t lpad = 0;  // allocated panel length
  int64_t pitch = 0; // elements between consecutive panel lines (>= reg_block)
  size_t bytes = 0;
};
PackGeometry pack_geometry(const MatrixView& src, Side side, PackFormat format, Datatype target,
                           int64_t reg_block, int64_t panel_len, int64_t pitch = 0);

mdg::PackDesc make_pack_desc(const MatrixView& src, Side side, PackFormat format, bool conj,
                             const Scalar& scale, Datatype target, int64_t reg_block, int64_t panel_len,
                             size_t* bytes, int64_t pitch = 0);

void pack_block_device_padded(void* dst, const MatrixView& src, Side side, PackFormat format, bool conj,
                              Scalar scale, Datatype target, int64_t reg_block, int64_t panel_len,
                              void* stream);

// An operand of a call that becomes ready on another stream (gemm_sharded:
// A arrives by broadcast): execute_scheduled packs the other operand first and
// makes the stream wait on `event` before packing this one.  `right`: the
// operand is the plan's right (B-side) operand (a transposed plan).
struct OperandReady {
  cudaEvent_t event = nullptr;
  bool right = false;
};

// execute() with the scheduling hint of the batch runner: `shared` = other
// calls of the same batch may run concurrently on the device, so the kernel
// keeps the hardware-scheduled classic grid (whose waves interleave with the
// neighbours') instead of a stream-K tail sized for an idle GPU.
// `arena` (optional): device workspace of `arena_bytes` the call may use in
// stream order instead of allocating (gemm_batch keeps one per compute
// stream).  `ws_needed` (optional): only report the workspace bytes the call
// would use, launching nothing.
void execute_scheduled(const ExecutionPlan& p, Numerics numerics, void* stream, FlopCounter* fc, bool shared,
                       void* arena = nullptr, size_t arena_bytes = 0, size_t* ws_needed = nullptr,
                       bool allow_splitk = true, bool block_split = true, const struct OperandReady* ready = nullptr);
size_t workspace_bytes(const ExecutionPlan& p, Numerics numerics, bool shared, bool allow_splitk = true);

// ---- the dual-pipe kernel (gemm_dual.cu), used by gemm_batch -------------
// FAST plans it can run: k > 0, non-empty, complex C paired.
bool dual_eligible(const ExecutionPlan& p, Numerics numerics);
// Packed operands of a dual job: A panels of the group's tile rows, B panels
// of its tile columns, k padded to 16; `bytes` of workspace, B at `off_b`.
struct DualPrep {
  mdg::PackDesc pa{}, pb{};
  size_t bytes_a = 0, bytes_b = 0;
  size_t off_b = 0, bytes = 0;
  int64_t lpad = 0;
  bool single = false;
  double tile_flops = 0.0;  // flops of the padded tile grid (2 tiles*BM*BN*lpad)
  int32_t tiles = 0;        // tiles of the group's tile shape
};
DualPrep dual_prepare(const ExecutionPlan& p);
// Describe the job of p with its packed operands at ws and append the two
// packs to g (p's views must be the device views the pack kernels read);
// traffic += the packs' algorithmic bytes.  dual_pack_group launches g.
void dual_describe(const ExecutionPlan& p, void* ws, mdg::DualJob* job, mdg::PackGroup* g, double* traffic);
void dual_pack_group(mdg::PackGroup& g, double traffic, cudaStream_t st);
// CTAs of a dual launch: the SMs less the ones left to the packs (148 B200
// SMs when no device is visible: the host-only schedule).
int dual_grid();
// One dual launch over d's job lists (grid = dual_grid()); flops per group for
// the profiling hook.
void dual_launch(const mdg::DualDesc& d, double flops_d, double flops_f, cudaStream_t st);

// The dual-pipe batch schedule of gemm_batch (host only, no device work): one
// entry per launch piece -- launch, call, tile range, group (1 FP64, 2 FP32;
// 0 = the call runs through execute() in that slot).  Empty when the batch
// would not take the dual path.  call_tiles: tiles of each dual call.
struct DualPiece {
  int32_t unit, call, t0, t1, group;
};
std::vector<DualPiece> dual_schedule_pieces(const std::vector<GemmCall>& calls, const Config& cfg,
                                            std::vector<int32_t>* call_tiles);

// FAST numerics of a plan without C_temp whose Temp / 1m route rounds into a
// C of another precision per KC block: 0 one combine, 1 per KC block (see
// driver.cpp); f_a / f_b receive the real inner steps per source column / row.
int fast_block_mode(const ExecutionPlan& p, int64_t* f_a = nullptr, int64_t* f_b = nullptr);

// The value the reference's FlopCounter reaches for this plan.
uint64_t reference_flops(const ExecutionPlan& p);

}  // namespace mdgemm
