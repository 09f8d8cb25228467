// Kernel launch accounting (see mdg_profile_begin in mdgemm_b200.h).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "mdgemm_b200.h"

namespace mdgemm::prof {

// RAII bracket around one kernel launch on `stream`.
class Scope {
 public:
  Scope(int kind, cudaStream_t stream, double work);
  ~Scope();
  Scope(const Scope&) = delete;
  Scope& operator=(const Scope&) = delete;

 private:
  int kind_;
  cudaStream_t stream_;
  double work_;
  cudaEvent_t start_ = nullptr;
};

uint64_t launches();
void begin();
void end(mdg_kernel_stats_t* out);

}  // namespace mdgemm::prof
