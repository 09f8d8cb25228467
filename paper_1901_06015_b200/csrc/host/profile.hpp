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
  // one launch whose time also counts under kind2 with work2 (no extra launch)
  Scope(int kind, cudaStream_t stream, double work, int kind2, double work2);
  ~Scope();
  Scope(const Scope&) = delete;
  Scope& operator=(const Scope&) = delete;

 private:
  int kind_;
  cudaStream_t stream_;
  double work_;
  int kind2_ = -1;
  double work2_ = 0.0;
  cudaEvent_t start_ = nullptr;
};

uint64_t launches();
void begin();
void end(mdg_kernel_stats_t* out);

}  // namespace mdgemm::prof
