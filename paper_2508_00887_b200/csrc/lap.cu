// lap.cu — K7: discretisation M = argmax_P ⟨P, N⟩ (Eq.(2); Alg.1 step 10 P:337; Hungarian
// P:316), the deterministic shortest-augmenting-path Kuhn–Munkres of reading R17, bit-exact with
// the oracle's LAP given the same N:
//   * rows inserted in order 1..n; potentials u, v; C = −N; every float op is an FP64 add/sub in
//     the oracle's association order ((C − u[i0]) − v[j]), so no FMA contraction can occur;
//   * each Dijkstra step's argmin over free columns is a block reduction on (minv[j], j) with ties
//     to the lowest j — the sequential strict-< scan's choice.
// One CTA.  Column j is owned by thread (j−1) mod THREADS for the whole solve: its minv[j], v[j]
// and used[j] live in that thread's REGISTERS, so a Dijkstra step is one coalesced read of row i0
// of N, a register scan, a warp-shuffle argmin and two __syncthreads.  Row potentials u[], the
// assignment p[] and way[] live in shared memory (global workspace when n is too large).
#include <math_constants.h>
#include "common.cuh"
#include "internal.h"

namespace fram {
namespace {

__device__ __forceinline__ void argmin_merge(double& v, int& j, double ov, int oj) {
  if (ov < v || (ov == v && oj < j)) { v = ov; j = oj; }
}

template <int THREADS, int CPT>
__global__ void __launch_bounds__(THREADS, 1) lap_kernel(const double* __restrict__ N, int n, long ld,
                                                         int32_t* perm, void* gwork, int use_smem) {
  constexpr int WARPS = THREADS / 32;
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ double s_v[WARPS];
  __shared__ int s_j[WARPS];
  unsigned char* base = use_smem ? dsm : reinterpret_cast<unsigned char*>(gwork);
  const int m = n + 1;
  double* u = reinterpret_cast<double*>(base);
  int* p = reinterpret_cast<int*>(u + m);
  int* way = p + m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  double minv[CPT], v[CPT];
#pragma unroll
  for (int k = 0; k < CPT; ++k) v[k] = 0.0;
  for (int j = tid; j < m; j += THREADS) { u[j] = 0.0; p[j] = 0; way[j] = 0; }
  __syncthreads();

  for (int i = 1; i <= n; ++i) {
    uint64_t used = 0;
#pragma unroll
    for (int k = 0; k < CPT; ++k) minv[k] = CUDART_INF;
    if (tid == 0) p[0] = i;
    int j0 = 0, i0 = i;
    __syncthreads();
    while (true) {
      if (j0 > 0 && ((j0 - 1) % THREADS) == tid) used |= 1ull << ((j0 - 1) / THREADS);   // used[j0] = true
      const double ui0 = u[i0];
      const double* crow = N + (long)(i0 - 1) * ld;
      double best = CUDART_INF;
      int bj = 0x7fffffff;
      double cv[CPT];                                   // issue every load of row i0 up front
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const int j = 1 + tid + k * THREADS;
        cv[k] = (j <= n) ? __ldcg(crow + (j - 1)) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const int j = 1 + tid + k * THREADS;
        if (j <= n && !((used >> k) & 1ull)) {
          const double cur = __dsub_rn(__dsub_rn(-cv[k], ui0), v[k]);
          if (cur < minv[k]) { minv[k] = cur; way[j] = j0; }
          if (minv[k] < best) { best = minv[k]; bj = j; }
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
      double delta = s_v[0];
      int j1 = s_j[0];
#pragma unroll
      for (int w = 1; w < WARPS; ++w) argmin_merge(delta, j1, s_v[w], s_j[w]);
      // potentials: used columns (incl. virtual column 0 ⇒ row p[0] = i) and free minv
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const int j = 1 + tid + k * THREADS;
        if (j <= n) {
          if ((used >> k) & 1ull) {
            const int r = p[j];
            u[r] = __dadd_rn(u[r], delta);
            v[k] = __dsub_rn(v[k], delta);
          } else {
            minv[k] = __dsub_rn(minv[k], delta);
          }
        }
      }
      if (tid == 0) u[i] = __dadd_rn(u[i], delta);
      __syncthreads();
      j0 = j1;
      i0 = p[j1];
      if (i0 == 0) break;
    }
    if (tid == 0) {                                    // augment along way[]
      int jj = j0;
      do {
        const int jw = way[jj];
        p[jj] = p[jw];
        jj = jw;
      } while (jj != 0);
    }
    __syncthreads();
  }
  for (int j = tid + 1; j < m; j += THREADS) perm[p[j] - 1] = (int32_t)(j - 1);
}

template <int THREADS, int CPT>
cudaError_t launch_t(const double* N, long n, long ld, int32_t* perm, void* work, cudaStream_t st) {
  const size_t bytes = lap_work_bytes(n);
  const bool smem = bytes <= 200 * 1024;
  auto fn = lap_kernel<THREADS, CPT>;
  if (smem) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
  }
  fn<<<1, THREADS, smem ? bytes : 0, st>>>(N, (int)n, ld, perm, work, smem ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace

size_t lap_work_bytes(long n) { return (size_t)(n + 1) * (sizeof(double) + 2 * sizeof(int)) + 64; }

cudaError_t launch_lap(const double* N, long n, long ld, int32_t* perm, void* work, cudaStream_t st) {
  if (n <= 256) return launch_t<256, 1>(N, n, ld, perm, work, st);
  if (n <= 512) return launch_t<256, 2>(N, n, ld, perm, work, st);
  if (n <= 1024) return launch_t<256, 4>(N, n, ld, perm, work, st);
  if (n <= 2048) return launch_t<256, 8>(N, n, ld, perm, work, st);
  if (n <= 4096) return launch_t<256, 16>(N, n, ld, perm, work, st);
  if (n <= 8192) return launch_t<1024, 8>(N, n, ld, perm, work, st);
  if (n <= 16384) return launch_t<1024, 16>(N, n, ld, perm, work, st);
  if (n <= 65536) return launch_t<1024, 64>(N, n, ld, perm, work, st);
  return cudaErrorInvalidValue;
}

}  // namespace fram
