// lap.cu — K7: discretisation M = argmax_P ⟨P, N⟩ (Eq.(2); Alg.1 step 10 P:337; Hungarian
// P:316), the deterministic shortest-augmenting-path Kuhn–Munkres of reading R17, bit-exact with
// the oracle's LAP given the same N:
//   * rows inserted in order 1..n; potentials u, v; C = −N; every float op is an FP64 add/sub in
//     the oracle's association order ((C − u[i0]) − v[j]), so no FMA contraction can occur;
//   * each Dijkstra step's argmin over free columns is a block reduction on (minv[j], j) with ties
//     to the lowest j — the sequential strict-< scan's choice.
// One CTA of up to 1024 threads.  Column j is owned by thread (j−1) mod THREADS for the whole solve:
// its minv[j], v[j], used[j] and (once used) p[j] live in that thread's REGISTERS, so a Dijkstra
// step is one coalesced read of row i0 of N, a register scan, a warp-shuffle argmin, ONE
// __syncthreads (per-warp candidates double-buffered by step parity; every warp then reduces the
// candidates itself) and register/shared potential updates.  Row potentials u[], the assignment
// p[] and way[] live in shared memory (global workspace when n is too large).  u[i0] can be read
// without a second barrier because the row about to enter the tree is never updated in the step
// that selects it.
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
  __shared__ double s_v[2][WARPS];                    // per-warp argmin candidates, double-buffered
  __shared__ int s_j[2][WARPS];                       // by step parity (one barrier per step)
  unsigned char* base = use_smem ? dsm : reinterpret_cast<unsigned char*>(gwork);
  const int m = n + 1;
  double* u = reinterpret_cast<double*>(base);        // row potentials u[0..n]
  int* p = reinterpret_cast<int*>(u + m);             // p[j]: row owning column j (0 = free)
  int* way = p + m;                                   // predecessor column on the search tree
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // column j = 1 + tid + k·THREADS lives in this thread's registers
  double minv[CPT], v[CPT];
  int prow[CPT];                                      // row owning a USED column (fixed during a search)
#pragma unroll
  for (int k = 0; k < CPT; ++k) { v[k] = 0.0; prow[k] = 0; }
  for (int j = tid; j < m; j += THREADS) { u[j] = 0.0; p[j] = 0; way[j] = 0; }
  __syncthreads();

  int par = 0;
  for (int i = 1; i <= n; ++i) {
    uint64_t used = 0;
#pragma unroll
    for (int k = 0; k < CPT; ++k) minv[k] = CUDART_INF;
    if (tid == 0) p[0] = i;                           // read only by thread 0's augmentation
    int j0 = 0, i0 = i;
    while (true) {
      // used[j0] = true (the owner remembers p[j0] = i0 for the potential updates)
      if (j0 > 0 && ((j0 - 1) % THREADS) == tid) {
        const int kk = (j0 - 1) / THREADS;
        used |= 1ull << kk;
#pragma unroll
        for (int k = 0; k < CPT; ++k)
          if (k == kk) prow[k] = i0;
      }
      const double ui0 = u[i0];                       // not written during this step (i0 ∉ tree)
      const double* crow = N + (long)(i0 - 1) * ld;
      double cv[CPT];
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const int j = 1 + tid + k * THREADS;
        cv[k] = (j <= n) ? __ldcg(crow + (j - 1)) : 0.0;
      }
      double best = CUDART_INF;
      int bj = 0x7fffffff;
#pragma unroll
      for (int k = 0; k < CPT; ++k) {                 // k ascending ⇒ j ascending: strict < keeps lowest j
        const int j = 1 + tid + k * THREADS;
        if (j <= n && !((used >> k) & 1ull)) {
          const double cur = __dsub_rn(__dsub_rn(-cv[k], ui0), v[k]);   // (C[i0][j] − u[i0]) − v[j]
          if (cur < minv[k]) { minv[k] = cur; way[j] = j0; }
          if (minv[k] < best) { best = minv[k]; bj = j; }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
        argmin_merge(best, bj, __shfl_xor_sync(0xffffffffu, best, o), __shfl_xor_sync(0xffffffffu, bj, o));
      if (lane == 0) { s_v[par][warp] = best; s_j[par][warp] = bj; }
      __syncthreads();
      // every warp reduces the WARPS candidates itself (no second barrier)
      double delta = (lane < WARPS) ? s_v[par][lane] : CUDART_INF;
      int j1 = (lane < WARPS) ? s_j[par][lane] : 0x7fffffff;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)                // lanes ≥ WARPS hold +inf: all lanes converge
        argmin_merge(delta, j1, __shfl_xor_sync(0xffffffffu, delta, o), __shfl_xor_sync(0xffffffffu, j1, o));
      par ^= 1;
      // potentials: used columns (u[p[j]] += δ, v[j] −= δ), virtual column 0 (u[i] += δ), free minv −= δ
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const int j = 1 + tid + k * THREADS;
        if (j <= n) {
          if ((used >> k) & 1ull) {
            u[prow[k]] = __dadd_rn(u[prow[k]], delta);
            v[k] = __dsub_rn(v[k], delta);
          } else {
            minv[k] = __dsub_rn(minv[k], delta);
          }
        }
      }
      if (tid == 0) u[i] = __dadd_rn(u[i], delta);
      j0 = j1;
      i0 = p[j1];                                     // p is not modified during a search
      if (i0 == 0) break;
    }
    __syncthreads();                                  // all reads of p / writes of way and u done
    if (tid == 0) {                                   // augment along way[]
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
  if (n <= 512) return launch_t<512, 1>(N, n, ld, perm, work, st);
  if (n <= 1024) return launch_t<1024, 1>(N, n, ld, perm, work, st);
  if (n <= 2048) return launch_t<1024, 2>(N, n, ld, perm, work, st);
  if (n <= 4096) return launch_t<1024, 4>(N, n, ld, perm, work, st);
  if (n <= 8192) return launch_t<1024, 8>(N, n, ld, perm, work, st);
  if (n <= 16384) return launch_t<1024, 16>(N, n, ld, perm, work, st);
  if (n <= 65536) return launch_t<1024, 64>(N, n, ld, perm, work, st);
  return cudaErrorInvalidValue;
}

}  // namespace fram
