// lap.cu — K7: discretisation M = argmax_P ⟨P, N⟩ (Eq.(2); Alg.1 step 10 P:337; Hungarian
// P:316), the deterministic shortest-augmenting-path Kuhn–Munkres of reading R17, bit-exact with
// the oracle's LAP given the same N:
//   * rows inserted in order 1..n; potentials u, v; C = −N; every float op is an FP64 add/sub in
//     the oracle's association order ((C − u[i0]) − v[j]), so no FMA contraction can occur;
//   * each Dijkstra step's argmin over free columns is a block reduction on (minv[j], j) with ties
//     to the lowest j — the sequential strict-< scan's choice.
// One CTA of up to 1024 threads.  Column j is owned by thread (j−1) mod THREADS for the whole solve:
// its minv[j], v[j], used[j] and (once used) p[j] live in that thread's REGISTERS, so a Dijkstra
// step is one coalesced read of row i0 of N (issued before the previous step's potential updates),
// a register scan, a warp argmin by three redux.sync on an order-preserving key, ONE __syncthreads
// (per-warp candidates double-buffered by step parity; every warp then reduces the candidates
// itself) and register/shared potential updates.  Row potentials u[], the assignment
// p[] and way[] live in shared memory (global workspace when n is too large).  u[i0] can be read
// without a second barrier because the row about to enter the tree is never updated in the step
// that selects it.
#include <math_constants.h>
#include <type_traits>
#include <stdio.h>
#include <stdlib.h>
#include "common.cuh"
#include "internal.h"

// The records arrive by st.async in this CTA's own shared memory and complete on this CTA's mbarrier,
// so observing the phase with the default (CTA-scope acquire) semantics orders the reads after the
// data; ".acquire.cluster" made ptxas add an L1 invalidation (CCTL.IVALL) to every wait: 87.6 → 84.6 ms
// for the C4 LAP without it (profiles/r02/ab_mbar.log).
#ifndef MBAR_SEM
#define MBAR_SEM ""
#endif

namespace fram {
namespace {

// Order-preserving map FP64 → uint64 (negative: flip all bits; non-negative: flip the sign bit),
// so that unsigned comparison of keys equals numeric comparison of the doubles (no NaN here).
__device__ __forceinline__ uint64_t okey(double x) {
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  return b ^ ((b >> 63) ? 0xffffffffffffffffull : 0x8000000000000000ull);
}
__device__ __forceinline__ double unkey(uint64_t k) {
  const uint64_t b = k ^ ((k >> 63) ? 0x8000000000000000ull : 0xffffffffffffffffull);
  return __longlong_as_double((long long)b);
}
// Warp argmin over (key, j): lexicographic — the smallest value, ties to the lowest column j
// (the sequential strict-< scan's choice, R17).  Three redux.sync instead of a shuffle tree.
__device__ __forceinline__ void warp_argmin(uint64_t& key, int& j) {
  const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
  const unsigned mhi = __reduce_min_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_min_sync(0xffffffffu, hi == mhi ? lo : 0xffffffffu);
  const bool win = (hi == mhi) && (lo == mlo);
  j = (int)__reduce_min_sync(0xffffffffu, win ? (unsigned)j : 0x7fffffffu);
  key = ((uint64_t)mhi << 32) | mlo;
}

template <int THREADS, int CPT, bool SMEM>
__global__ void __launch_bounds__(THREADS, 1) lap_kernel(const double* __restrict__ N, int n, long ld,
                                                         int32_t* perm, void* gwork, int* err) {
  constexpr int WARPS = THREADS / 32;
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ uint64_t s_k[2][WARPS];                  // per-warp argmin candidates, double-buffered
  __shared__ int s_j[2][WARPS];                       // by step parity (one barrier per step)
  unsigned char* base = SMEM ? dsm : reinterpret_cast<unsigned char*>(gwork);
  const int m = n + 1;
  double* u = reinterpret_cast<double*>(base);        // row potentials u[0..n]
  int* p = reinterpret_cast<int*>(u + m);             // p[j]: row owning column j (0 = free)
  int* way = p + m;                                   // predecessor column on the search tree
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // column j = 1 + tid + k·THREADS lives in this thread's registers
  double minv[CPT], v[CPT], cv[CPT];
  double vs[CPT];                                     // scan copy of v: −inf for used / absent columns
  int prow[CPT];                                      // row owning a USED column (fixed during a search)
  using Mask = typename std::conditional<(CPT > 32), uint64_t, uint32_t>::type;
  constexpr Mask one = 1;
  Mask inr = 0;                                       // bit k: column j ≤ n exists
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    v[k] = 0.0;
    prow[k] = 0;
    if (1 + tid + k * THREADS <= n) inr |= one << k;
  }
  for (int j = tid; j < m; j += THREADS) { u[j] = 0.0; p[j] = 0; way[j] = 0; }
  __syncthreads();

  auto load_row = [&](int row) {                      // row `row` (1-based) of N into cv[]
    const double* crow = N + (long)(row - 1) * ld + tid;
#pragma unroll
    for (int k = 0; k < CPT; ++k) cv[k] = ((inr >> k) & one) ? __ldcg(crow + k * THREADS) : 0.0;
  };

  int par = 0;
  for (int i = 1; i <= n; ++i) {
    Mask fr = inr;                                    // bit k: column free (not yet in the tree)
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      minv[k] = CUDART_INF;
      vs[k] = ((inr >> k) & one) ? v[k] : -CUDART_INF;
    }
    if (tid == 0) p[0] = i;                           // read only by thread 0's augmentation
    int j0 = 0, i0 = i;
    load_row(i0);
    while (true) {
      // used[j0] = true (the owner remembers p[j0] = i0 for the potential updates).  A used column's
      // minv is never read again in this search (oracle: only free columns are scanned and updated),
      // so it is parked at +inf, and its scan copy of v at −inf (its cur is then +inf, never < minv):
      // the scan and the `minv −= δ` update need no free-column mask.  A free column's v does not
      // change during a search, so vs = v there and cur is the oracle's value.
      if (j0 > 0 && ((j0 - 1) % THREADS) == tid) {
        const int kk = (j0 - 1) / THREADS;
        fr &= ~(one << kk);
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
          prow[k] = (k == kk) ? i0 : prow[k];
          minv[k] = (k == kk) ? CUDART_INF : minv[k];
          vs[k] = (k == kk) ? -CUDART_INF : vs[k];
        }
      }
      const double ui0 = u[i0];                       // not written during this step (i0 ∉ tree)
      double bv[CPT];
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const double cur = __dsub_rn(__dsub_rn(-cv[k], ui0), vs[k]);    // (C[i0][j] − u[i0]) − v[j]
        const bool upd = cur < minv[k];
        minv[k] = upd ? cur : minv[k];
        if (upd) way[1 + tid + k * THREADS] = j0;
        bv[k] = minv[k];                              // +inf for used / absent columns
      }
      // thread-local argmin as a tree over k (j ascending with k: strict < keeps the lower j)
      int bk[CPT];
#pragma unroll
      for (int k = 0; k < CPT; ++k) bk[k] = k;
#pragma unroll
      for (int w = 1; w < CPT; w *= 2)
#pragma unroll
        for (int k = 0; k + w < CPT; k += 2 * w)
          if (bv[k + w] < bv[k]) { bv[k] = bv[k + w]; bk[k] = bk[k + w]; }
      const double best = bv[0];
      int bj = best < CUDART_INF ? 1 + tid + bk[0] * THREADS : 0x7fffffff;
      uint64_t key = okey(best);
      warp_argmin(key, bj);
      if (lane == 0) { s_k[par][warp] = key; s_j[par][warp] = bj; }
      __syncthreads();
      // every warp reduces the WARPS candidates itself (no second barrier)
      uint64_t dkey = (lane < WARPS) ? s_k[par][lane] : ~0ull;
      int j1 = (lane < WARPS) ? s_j[par][lane] : 0x7fffffff;
      warp_argmin(dkey, j1);
      const double delta = unkey(dkey);
      par ^= 1;
      if (j1 > n) {                                   // no finite candidate (non-finite N): give up cleanly
        if (tid == 0) *err = 1;
        return;                                       // j1 is the same in every thread
      }
      const int i0n = p[j1];                          // p is not modified during a search
      if (i0n != 0) load_row(i0n);                    // next row's loads overlap the updates below
      // potentials: used columns (u[p[j]] += δ, v[j] −= δ), virtual column 0 (u[i] += δ), free minv −= δ
      // The used columns' rows prow[k] are distinct (one owner per column), so all u loads are issued
      // before any store: the read-modify-writes overlap instead of forming one latency chain.
      const Mask usd = inr & ~fr;
      double ut[CPT];
#pragma unroll
      for (int k = 0; k < CPT; ++k)
        if ((usd >> k) & one) ut[k] = u[prow[k]];
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        if ((usd >> k) & one) {
          ut[k] = __dadd_rn(ut[k], delta);
          v[k] = __dsub_rn(v[k], delta);
        }
        minv[k] = __dsub_rn(minv[k], delta);         // free: as the oracle; used/absent: +inf stays +inf
      }
#pragma unroll
      for (int k = 0; k < CPT; ++k)
        if ((usd >> k) & one) u[prow[k]] = ut[k];
      if (tid == 0) u[i] = __dadd_rn(u[i], delta);
      j0 = j1;
      i0 = i0n;
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

// ---- K7c: the same R17 Hungarian on a thread-block cluster of CS CTAs (one per SM) -------------
// The single-CTA step is issue-bound on its SM (ncu: IPC 2.25–2.4), so the columns are split over CS
// SMs: CTA c owns columns [c·CH+1, (c+1)·CH] (CH = 512·CPT), each thread CPT of them in registers as
// in lap_kernel.  Per Dijkstra step every warp sends its argmin candidate {key, j, way[j]} to every
// CTA of the cluster with st.async (16 B, completing bytes on the receiver's mbarrier for that step's
// parity), and every warp of every CTA reduces the CS·16 records itself.  Kept identical in every
// CTA without further exchange: p[] (changed only by the augmentation, which every CTA walks the
// same way), u[] (a step updates the root and the rows that entered the tree earlier in this search,
// trow[], known to all from the records, by the same FP64 adds in the same order) and pw[j] = way[j]
// of the tree columns (final once a column is used, sent in its record).  way[] of the free columns
// stays local (wl[]).  All float operations equal lap_kernel's, so the result is bit-exact with R17.
//
// Deferred row potentials.  Within one search u is read only for the row entering the tree (u[i0]),
// which the search has not touched yet; the root and the tree rows are never read again before the
// search ends.  So instead of adding δ_s to every tree row at every step (O(tree) shared-memory
// read-modify-writes per step, up to ~13 per thread in the longest C4 searches), step s only records
// δ_s, and at the search end every tree row replays ITS suffix of the δ sequence, u += δ_e, δ_{e+1}, …,
// δ_{S−1} (e = the step after it entered; the root: all steps) — the same FP64 adds in the same order,
// so u is bit-identical to the step-by-step update.  A thread replays 4 rows at once (independent
// add chains).  The δ history lives in global memory (one store by one thread per step).
template <int CS, int CPT, int THREADS, bool UG>
__global__ void __launch_bounds__(THREADS, 1) lap_cluster_kernel(const double* __restrict__ N, int n, long ld,
                                                                 int32_t* perm, double* ug, double* dhist,
                                                                 int* err) {
  constexpr int WARPS = THREADS / 32, CH = THREADS * CPT, NREC = CS * WARPS;
  constexpr uint32_t REC_BYTES = NREC * 16;
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ __align__(16) uint4 s_rec[2][NREC];     // {key lo, key hi, j, way[j]} per warp per CTA
  __shared__ __align__(8) uint64_t s_mb[2];          // records of step parity q complete
  const int m = n + 1;
  // [m] replicated row potentials: in shared memory, or (UG, n > 8192, where 20 B per row no longer
  // fit) in this CTA's private copy in global memory — u is read once per step (u[i0], issued with
  // the row loads) and updated for the tree rows by the same thread every step
  double* u = UG ? ug + (size_t)blockIdx.x * m : reinterpret_cast<double*>(dsm);
  double* dh = dhist + (size_t)blockIdx.x * m;          // δ of each step of the current search
  int* p = UG ? reinterpret_cast<int*>(dsm) : reinterpret_cast<int*>(u + m);   // [m] replicated matching
  int* pw = p + m;                                    // [m] way of tree columns (replicated)
  int* trow = pw + m;                                 // [m] rows that entered the tree (this search)
  int* wl = trow + m;                                 // [CH] way of this CTA's columns
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned crank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const int c = (int)crank;
  const int jbase = c * CH + 1;                       // global column of (tid 0, k 0)

  double minv[CPT], v[CPT], vs[CPT], cv[CPT];
  int prow[CPT];
  uint32_t inr = 0;
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    v[k] = 0.0;
    prow[k] = 0;
    if (jbase + tid + k * THREADS <= n) inr |= 1u << k;
  }
  for (int j = tid; j < m; j += THREADS) { u[j] = 0.0; p[j] = 0; pw[j] = 0; }
  const uint32_t mb0 = (uint32_t)__cvta_generic_to_shared(&s_mb[0]);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0 + 8));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // remote addresses of every CTA's record slots and mbarriers
  const uint32_t rec0 = (uint32_t)__cvta_generic_to_shared(&s_rec[0][0]);
  uint32_t rrec[CS], rmb[CS];
#pragma unroll
  for (int r = 0; r < CS; ++r) {
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rrec[r]) : "r"(rec0), "r"(r));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rmb[r]) : "r"(mb0), "r"(r));
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");

  auto load_row = [&](int row) {
    const double* crow = N + (long)(row - 1) * ld + (jbase - 1) + tid;
#pragma unroll
    for (int k = 0; k < CPT; ++k) cv[k] = ((inr >> k) & 1u) ? __ldcg(crow + k * THREADS) : 0.0;
  };

  int step = 0;                                       // global step counter (buffer / phase parity)
  for (int i = 1; i <= n; ++i) {
    uint32_t fr = inr;
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      minv[k] = CUDART_INF;
      vs[k] = ((inr >> k) & 1u) ? v[k] : -CUDART_INF;
    }
    if (tid == 0) p[0] = i;
    int j0 = 0, i0 = i, ntree = 0;
    load_row(i0);
    __syncthreads();                                  // p[0] and the previous augmentation visible
    while (true) {
      if (j0 > 0) {
        const int jl = j0 - jbase;                    // used[j0] = true; its row i0 joins the tree
        if (jl >= 0 && jl < CH && (jl % THREADS) == tid) {
          const int kk = jl / THREADS;
          fr &= ~(1u << kk);
#pragma unroll
          for (int k = 0; k < CPT; ++k) {
            minv[k] = (k == kk) ? CUDART_INF : minv[k];
            vs[k] = (k == kk) ? -CUDART_INF : vs[k];
            prow[k] = (k == kk) ? i0 : prow[k];
          }
        }
        trow[ntree] = i0;                             // every thread writes the same value
        ++ntree;
      }
      const int q = step & 1;
      const uint32_t ph = (uint32_t)(step >> 1) & 1u;
      if (tid == 0)                                   // this step's records: NREC·16 bytes expected
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb0 + 8 * q), "r"(REC_BYTES) : "memory");
      const double ui0 = u[i0];
      double bv[CPT];
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const double cur = __dsub_rn(__dsub_rn(-cv[k], ui0), vs[k]);    // (C[i0][j] − u[i0]) − v[j]
        const bool upd = cur < minv[k];
        minv[k] = upd ? cur : minv[k];
        if (upd) wl[tid + k * THREADS] = j0;
        bv[k] = minv[k];
      }
      int bk[CPT];
#pragma unroll
      for (int k = 0; k < CPT; ++k) bk[k] = k;
#pragma unroll
      for (int w = 1; w < CPT; w *= 2)
#pragma unroll
        for (int k = 0; k + w < CPT; k += 2 * w)
          if (bv[k + w] < bv[k]) { bv[k] = bv[k + w]; bk[k] = bk[k + w]; }
      const double best = bv[0];
      int bj = best < CUDART_INF ? jbase + tid + bk[0] * THREADS : 0x7fffffff;
      uint64_t key = okey(best);
      warp_argmin(key, bj);
      __syncwarp();                                   // this step's wl[] writes → the sending lanes
      if (lane < CS) {                                // lane r sends the warp's record to CTA r
        const int wy = bj != 0x7fffffff ? wl[bj - jbase] : 0;
        const uint32_t off = (uint32_t)((q * NREC + c * WARPS + warp) * 16);
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
                     ::"r"(rrec[lane] + off), "r"((unsigned)key), "r"((unsigned)(key >> 32)), "r"(bj), "r"(wy),
                     "r"(rmb[lane] + 8 * q) : "memory");
      }
      {                                               // wait for all CS·16 records of this step
        uint32_t done = 0;
        while (!done)
          asm volatile("{ .reg .pred pp; mbarrier.try_wait.parity" MBAR_SEM ".shared::cta.b64 pp, [%1], %2; selp.u32 %0, 1, 0, pp; }"
                       : "=r"(done) : "r"(mb0 + 8 * q), "r"(ph) : "memory");
      }
      uint64_t dkey = ~0ull;
      int j1 = 0x7fffffff, wy1 = 0;
#pragma unroll
      for (int r = lane; r < NREC; r += 32) {
        const uint4 rr = s_rec[q][r];
        const uint64_t kr = ((uint64_t)rr.y << 32) | rr.x;
        if (kr < dkey || (kr == dkey && (int)rr.z < j1)) { dkey = kr; j1 = (int)rr.z; wy1 = (int)rr.w; }
      }
      const int mine = j1;
      // the row owning this lane's candidate column, loaded while the argmin reduces (p is fixed
      // during a search), so the winner's row index needs no dependent load after the reduction
      const int pl = (mine >= 1 && mine <= n) ? p[mine] : 0;
      warp_argmin(dkey, j1);
      const unsigned who = __ballot_sync(0xffffffffu, mine == j1);
      wy1 = __shfl_sync(0xffffffffu, wy1, __ffs(who) - 1);
      const int pwin = __shfl_sync(0xffffffffu, pl, __ffs(who) - 1);
      const double delta = unkey(dkey);
      ++step;
      if (j1 > n) {                                   // no finite candidate (non-finite N): give up cleanly
        if (c == 0 && tid == 0) *err = 1;
        return;                                       // every CTA reduced the same records: all return
      }
      if (tid == 0) { pw[j1] = wy1; dh[ntree] = delta; }   // way of the entering column (final); δ_s, s = ntree
      const int i0n = pwin;                           // = p[j1]
      if (i0n != 0) load_row(i0n);
      const uint32_t usd = inr & ~fr;
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        if ((usd >> k) & 1u) v[k] = __dsub_rn(v[k], delta);
        minv[k] = __dsub_rn(minv[k], delta);
      }
      j0 = j1;
      i0 = i0n;
      if (i0 == 0) break;
    }
    __syncthreads();                                  // pw[], p[], trow[] and the δ history final
    {   // replay: row q = 0 is the root (δ_0 … δ_{S−1}), row q ≥ 1 is trow[q−1] (δ_q … δ_{S−1}), S = ntree + 1
      const int S = ntree + 1;
      for (int q0 = tid; q0 <= ntree; q0 += 4 * THREADS) {
        double uu[4];
        int rr[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int q = q0 + k * THREADS;
          rr[k] = q <= ntree ? (q == 0 ? i : trow[q - 1]) : 0;
          uu[k] = q <= ntree ? u[rr[k]] : 0.0;
        }
#pragma unroll 4
        for (int s = q0; s < S; ++s) {
          const double d = dh[s];
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (s >= q0 + k * THREADS) uu[k] = __dadd_rn(uu[k], d);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (q0 + k * THREADS <= ntree) u[rr[k]] = uu[k];
      }
    }
    __syncthreads();                                  // u final for this search
    if (tid == 0) {                                   // augment along way[] (every CTA, same walk)
      int jj = j0;
      do {
        const int jw = pw[jj];
        p[jj] = p[jw];
        jj = jw;
      } while (jj != 0);
    }
  }
  __syncthreads();
  if (c == 0)
    for (int j = tid + 1; j < m; j += THREADS) perm[p[j] - 1] = (int32_t)(j - 1);
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int CS, int CPT, int THREADS = 512, bool UG = false>
cudaError_t launch_cluster_t(const double* N, long n, long ld, int32_t* perm, void* work, cudaStream_t st) {
  // work: [UG: CS × (n+1) u copies] [CS × (n+1) δ histories] [error word]
  double* ug = reinterpret_cast<double*>(work);
  double* dhist = ug + (UG ? (size_t)CS * (n + 1) : 0);
  int* err = reinterpret_cast<int*>(static_cast<char*>(work) + lap_err_offset(n));
  auto fn = lap_cluster_kernel<CS, CPT, THREADS, UG>;
  const size_t m = (size_t)n + 1;
  const size_t bytes = m * ((UG ? 0 : sizeof(double)) + 3 * sizeof(int)) + (size_t)THREADS * CPT * sizeof(int) + 64;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess && CS > 8) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, N, (int)n, ld, perm, ug, dhist, err);
}

template <int THREADS, int CPT>
cudaError_t launch_t(const double* N, long n, long ld, int32_t* perm, void* work, cudaStream_t st) {
  const size_t bytes = (size_t)(n + 1) * (sizeof(double) + 2 * sizeof(int)) + 64;   // u, p, way
  int* err = reinterpret_cast<int*>(static_cast<char*>(work) + lap_err_offset(n));
  if (bytes <= 200 * 1024) {
    auto fn = lap_kernel<THREADS, CPT, true>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    fn<<<1, THREADS, bytes, st>>>(N, (int)n, ld, perm, work, err);
  } else {
    lap_kernel<THREADS, CPT, false><<<1, THREADS, 0, st>>>(N, (int)n, ld, perm, work, err);
  }
  return cudaGetLastError();
}

}  // namespace

// single-CTA kernel: u, p, way in global memory; cluster kernel: per CTA of the cluster (≤ 16) a δ
// history and, for n > 8192, a u copy, then an error word
size_t lap_work_bytes(long n) {
  const size_t single = (size_t)(n + 1) * (sizeof(double) + 2 * sizeof(int)) + 64;
  const size_t cl = (size_t)(n + 1) * sizeof(double) * 16 * (n > 8192 ? 2 : 1) + 64;
  return single > cl ? single : cl;
}

size_t lap_err_offset(long n) {            // byte offset of the error word (past every kernel's arrays)
  return lap_work_bytes(n) - 8;
}

cudaError_t launch_lap(const double* N, long n, long ld, int32_t* perm, void* work, cudaStream_t st) {
  cudaError_t e0 = cudaMemsetAsync(static_cast<char*>(work) + lap_err_offset(n), 0, sizeof(int), st);
  if (e0 != cudaSuccess) return e0;
  if (n <= 256) return launch_t<256, 1>(N, n, ld, perm, work, st);
  if (n <= 512) return launch_t<512, 1>(N, n, ld, perm, work, st);
  if (n <= 1024) return launch_t<512, 2>(N, n, ld, perm, work, st);
  // 1024 < n ≤ 2048: a cluster of 4 CTAs × 128 threads × 4 columns (round 2: 40.2 vs 47.6 ms on one CTA
  // for a flat n = 2000 N, 2.1 vs 1.9 ms on a near-permutation one; profiles/r02/ab_lapsizes.log)
  if (n <= 2048) return launch_cluster_t<4, 4, 128>(N, n, ld, perm, work, st);
  // 2048 < n ≤ 8192: a cluster of 4 CTAs × 256 threads (C4, n = 4096: 86.7 ms against 120.0 ms on
  // one CTA; measured 2/4/8/16 CTAs × 128–1024 threads: 86.7–125 ms); the replicated u/p/way/tree arrays
  // (20 B per row) must fit in shared memory
  // n ≤ 4096: 8 CTAs × 128 threads × 4 columns (round 2, after the deferred potentials and the CTA-scope
  // record wait: 82.2 ms at C4 against 84.6 ms for 4 × 256 × 4; 2/4/8/16 CTAs × 64-512 threads measured
  // 82.2-107.7 ms, profiles/r02/ab_lapcfg*.log)
  if (n <= 4096) return launch_cluster_t<8, 4, 128>(N, n, ld, perm, work, st);
  if (n <= 8192) return launch_cluster_t<8, 8, 128>(N, n, ld, perm, work, st);   // 3% faster than 4 × 256 (r02)
  // n ≤ 16384: 8 CTAs × 256 threads × 8 columns, u in global memory (4×16 and 16×4 measured slower)
  if (n <= 16384) return launch_cluster_t<8, 8, 256, true>(N, n, ld, perm, work, st);
  if (n <= 65536) return launch_t<1024, 64>(N, n, ld, perm, work, st);
  return cudaErrorInvalidValue;
}

}  // namespace fram
