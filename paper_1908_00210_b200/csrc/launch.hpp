// Host-side kernel selection and launch helpers (internal to libgdi).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace gdi {

struct GraphStats {
  int32_t n = 0;
  int64_t m = 0;
  int32_t max_degree = 0;
  bool unit = true;
  long long max_abs_field = 0;  // max_i sum_j |w_ij|
};

struct ExactPlan {
  const void* fn = nullptr;
  int group = 32;  // lanes per replica
  int block = 128;
  int grid = 1;
  int n_pad = 0;
  int smem = 0;
  const char* name = "";
};

// Returns 0, or -1 when no K1 variant fits (capacity).
int exact_plan(const GraphStats& st, int32_t replicas, ExactPlan* plan);
cudaError_t exact_launch(const ExactPlan& plan, const ExactArgs& args, cudaStream_t stream);

// K3 fused exact evaluation: {cut, sum} per replica into a zeroed buffer.
cudaError_t eval_launch(const EvalArgs& args, bool weighted, cudaStream_t stream);

}  // namespace gdi
