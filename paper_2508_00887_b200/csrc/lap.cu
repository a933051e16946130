// lap.cu — K7: discretisation M = argmax_P ⟨P, N⟩ (Eq.(2); Alg.1 step 10 P:337; Hungarian
// P:316), the deterministic shortest-augmenting-path Kuhn–Munkres of reading R17, bit-exact with
// the oracle's LAP given the same N:
//   * rows inserted in order 1..n; potentials u, v; C = −N; every float op is an FP64 add/sub in
//     the oracle's association order ((C − u[i0]) − v[j]), so no FMA contraction can occur;
//   * each Dijkstra step's argmin over free columns is a block reduction on (minv[j], j) with ties
//     to the lowest j — the sequential strict-< scan's choice.
// One CTA (1024 threads); the row loop is sequential, the column scans are parallel.  Work arrays
// live in SMEM when they fit (n ≤ ~6000), else in the handle's global workspace.
#include <math_constants.h>
#include "common.cuh"
#include "internal.h"

namespace fram {
namespace {

constexpr int LAP_THREADS = 1024;
constexpr int LAP_WARPS = LAP_THREADS / 32;

__device__ __forceinline__ void argmin_merge(double& v, int& j, double ov, int oj) {
  if (ov < v || (ov == v && oj < j)) { v = ov; j = oj; }
}

__global__ void __launch_bounds__(LAP_THREADS, 1) lap_kernel(const double* __restrict__ N, long n, long ld,
                                                             int32_t* perm, void* gwork, int use_smem) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ double s_v[LAP_WARPS];
  __shared__ int s_j[LAP_WARPS];
  __shared__ double s_delta;
  __shared__ int s_j0, s_j1;
  unsigned char* base = use_smem ? dsm : reinterpret_cast<unsigned char*>(gwork);
  const long m = n + 1;
  double* u = reinterpret_cast<double*>(base);
  double* v = u + m;
  double* minv = v + m;
  int* p = reinterpret_cast<int*>(minv + m);
  int* way = p + m;
  unsigned char* used = reinterpret_cast<unsigned char*>(way + m);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (long j = tid; j < m; j += LAP_THREADS) { u[j] = 0.0; v[j] = 0.0; p[j] = 0; way[j] = 0; }
  __syncthreads();
  for (int i = 1; i <= (int)n; ++i) {
    for (long j = tid; j < m; j += LAP_THREADS) { minv[j] = CUDART_INF; used[j] = 0; }   // +inf
    if (tid == 0) { p[0] = i; s_j0 = 0; }
    __syncthreads();
    while (true) {
      const int j0 = s_j0;
      if (tid == 0) used[j0] = 1;
      const int i0 = p[j0];
      __syncthreads();
      const double* crow = N + (long)(i0 - 1) * ld;
      const double ui0 = u[i0];
      double best = CUDART_INF;
      int bj = 0x7fffffff;
      for (int j = tid + 1; j <= (int)n; j += LAP_THREADS) {
        if (!used[j]) {
          const double cur = __dsub_rn(__dsub_rn(-crow[j - 1], ui0), v[j]);
          double mv = minv[j];
          if (cur < mv) { mv = cur; minv[j] = cur; way[j] = j0; }
          if (mv < best) { best = mv; bj = j; }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
        argmin_merge(best, bj, ov, oj);
      }
      if (lane == 0) { s_v[warp] = best; s_j[warp] = bj; }
      __syncthreads();
      if (warp == 0) {
        best = s_v[lane];
        bj = s_j[lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, best, o);
          const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
          argmin_merge(best, bj, ov, oj);
        }
        if (lane == 0) { s_delta = best; s_j1 = bj; }
      }
      __syncthreads();
      const double delta = s_delta;
      const int j1 = s_j1;
      for (long j = tid; j < m; j += LAP_THREADS) {
        if (used[j]) {
          u[p[j]] = __dadd_rn(u[p[j]], delta);
          v[j] = __dsub_rn(v[j], delta);
        } else {
          minv[j] = __dsub_rn(minv[j], delta);
        }
      }
      __syncthreads();
      if (tid == 0) s_j0 = j1;
      const bool done = (p[j1] == 0);
      __syncthreads();
      if (done) break;
    }
    if (tid == 0) {                                    // augment along way[]
      int j0 = s_j0;
      do {
        const int j1 = way[j0];
        p[j0] = p[j1];
        j0 = j1;
      } while (j0 != 0);
    }
    __syncthreads();
  }
  for (long j = tid + 1; j < m; j += LAP_THREADS) perm[p[j] - 1] = (int32_t)(j - 1);
}

}  // namespace

size_t lap_work_bytes(long n) { return (size_t)(n + 1) * (3 * sizeof(double) + 2 * sizeof(int) + 1) + 64; }

cudaError_t launch_lap(const double* N, long n, long ld, int32_t* perm, void* work, cudaStream_t st) {
  const size_t bytes = lap_work_bytes(n);
  const bool smem = bytes <= 200 * 1024;
  if (smem) {
    cudaError_t e = cudaFuncSetAttribute(lap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
  }
  lap_kernel<<<1, LAP_THREADS, smem ? bytes : 0, st>>>(N, n, ld, perm, work, smem ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace fram
