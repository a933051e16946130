// batched.h — K8: many small FRAM solves (n ≤ 64), one CTA per instance.
#pragma once
#include <cuda_runtime.h>
#include <string>
#include "../../include/fram.h"

namespace fram {

struct BatchedWs {
  void* inst_stats = nullptr;   // device int32[batch][4]: outer, passes, converged, status
  size_t inst_bytes = 0;
  void* staging = nullptr;      // host-input staging (A, B, K, X0 contiguous)
  size_t staging_bytes = 0;
  void* out_staging = nullptr;  // device X_out / perm / status when caller passes host memory
  size_t out_bytes = 0;
};

void batched_release(BatchedWs& ws);

fram_status batched_solve(BatchedWs& ws, long n, double lambda, const fram_schedule& sched, long batch, int dt,
                          const void* A, const void* B, const void* K, const double* X0, int prec,
                          cudaStream_t st, double* X_out, int32_t* perm_out, int32_t* status_out,
                          fram_stats* stats, int num_sms, std::string* err);

}  // namespace fram
