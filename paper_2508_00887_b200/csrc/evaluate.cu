// evaluate.cu — K9: quality of a discrete matching M (M[i, p(i)] = 1), the evaluation quantities of the
// paper (not on the solve's hot path):
//   Eq.(1) P:65   Φ(M) = ½⟨MᵀAM, Ã⟩ + λ⟨MᵀF, F̃⟩ = ½ Σ_ij A_ij Ã_{p(i)p(j)} + λ Σ_i ⟨F_i, F̃_{p(i)}⟩
//   P:379         matching error ½‖A − MÃMᵀ‖_F + ‖F − MF̃‖_F,  (MÃMᵀ)_ij = Ã_{p(i)p(j)}, (MF̃)_i = F̃_{p(i)}
// K9a: one CTA per row i accumulates, in FP64, Σ_j (A_ij − Ã_{p(i)p(j)})², Σ_j A_ij Ã_{p(i)p(j)},
// Σ_k (F_ik − F̃_{p(i)k})² and Σ_k F_ik F̃_{p(i)k} (block tree, fixed order) → part[i][4];
// K9b: one CTA sums the rows in a fixed order → out[4].  Deterministic; out-of-range p(i) sets *bad.
#include "common.cuh"
#include "internal.h"

namespace fram {
namespace {

constexpr int kEvT = 256;

__device__ __forceinline__ double ld_any(const void* p, int dt, long idx) {
  if (dt == 0) return reinterpret_cast<const double*>(p)[idx];
  if (dt == 1) return (double)reinterpret_cast<const float*>(p)[idx];
  return (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[idx]);
}

__device__ __forceinline__ double block_sum(double v, double* sw) {
  v = warp_sum_d(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sw[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kEvT / 32; ++w) s += sw[w];
  return s;                                            // valid in thread 0
}

__global__ void __launch_bounds__(kEvT) eval_rows_kernel(const void* A, const void* B, const void* F, const void* Ft,
                                                         int dt, long n, long d, const int32_t* perm, double* part,
                                                         int* bad) {
  __shared__ double sw[kEvT / 32];
  const long i = blockIdx.x;
  const int pi = perm[i];
  if (pi < 0 || pi >= n) {                             // invalid matching: flag, contribute nothing
    if (threadIdx.x == 0) { *bad = 1; part[i * 4] = part[i * 4 + 1] = part[i * 4 + 2] = part[i * 4 + 3] = 0.0; }
    return;
  }
  double e2 = 0.0, ab = 0.0, f2 = 0.0, ff = 0.0;
  for (long j = threadIdx.x; j < n; j += kEvT) {
    const int pj = perm[j];
    if (pj < 0 || pj >= n) { *bad = 1; continue; }
    const double a = ld_any(A, dt, i * n + j), bt = ld_any(B, dt, (long)pi * n + pj);
    const double df = a - bt;
    e2 += df * df;
    ab += a * bt;
  }
  if (F)
    for (long k = threadIdx.x; k < d; k += kEvT) {
      const double f = ld_any(F, dt, i * d + k), g = ld_any(Ft, dt, (long)pi * d + k);
      f2 += (f - g) * (f - g);
      ff += f * g;
    }
  const double s0 = block_sum(e2, sw), s1 = block_sum(f2, sw), s2 = block_sum(ab, sw), s3 = block_sum(ff, sw);
  if (threadIdx.x == 0) { part[i * 4] = s0; part[i * 4 + 1] = s1; part[i * 4 + 2] = s2; part[i * 4 + 3] = s3; }
}

__global__ void __launch_bounds__(kEvT) eval_sum_kernel(const double* part, long n, double* out) {
  __shared__ double sw[kEvT / 32];
  for (int c = 0; c < 4; ++c) {
    double v = 0.0;
    for (long i = threadIdx.x; i < n; i += kEvT) v += part[i * 4 + c];   // fixed order per thread
    const double s = block_sum(v, sw);
    if (threadIdx.x == 0) out[c] = s;
  }
}

}  // namespace

cudaError_t launch_evaluate(const void* A, const void* B, const void* F, const void* Ft, int dt, long n, long d,
                            const int32_t* perm, double* part, double* out, int* bad, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  eval_rows_kernel<<<(unsigned)n, kEvT, 0, st>>>(A, B, F, Ft, dt, n, d, perm, part, bad);
  eval_sum_kernel<<<1, kEvT, 0, st>>>(part, n, out);
  return cudaGetLastError();
}

}  // namespace fram
