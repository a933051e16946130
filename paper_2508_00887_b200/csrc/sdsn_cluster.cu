// sdsn_cluster.cu — K4c: SDSN (Alg. 2) for small n on ONE thread-block cluster
// of C ≤ 16 CTAs (one per SM).  The whole iterate stays in the CTAs' shared memory, and the per-pass
// all-reduce of the column sums and the mass goes through distributed shared memory (DSMEM) —
// st.async stores completing on the receivers' mbarriers, no cluster barrier per pass — instead of
// the L2 round trips that dominate K4/K4r when a pass has only 20–800 columns (C1, C2).
//
// Same arithmetic as K4/K4r (readings R5, R9-R13): γ_j = S_j/n − 1 (lagged test),
// a_i = (1/n + S/n²) − r_i/n and b_j = −c_j/n in FP64 rounded to T, y' = max(0, (y + a_i) + b_j); S/n,
// S/n², r_i/n and c_j/n as RN(x/d) from a precomputed reciprocal and one FMA correction.
//
// CTA c owns rows [c·n/C, (c+1)·n/C) (R ≤ 64); warp w of the CTA sweeps rows w, w+8, …, lane l the
// columns l, l+32, … (≤ 28 per lane).  Row sums: one warp per row (FP64 for T = double; FP32 per lane,
// then FP64 for T = float).  Column sums: per-lane register partials → the 8 warps summed in order in
// shared memory → CTA partial → DSMEM reduce-scatter: CTA k receives the partials of column slice k
// from every CTA and sums them in CTA order (FP64) → b_j all-gathered into every CTA (DSMEM).  The
// per-CTA masses are all-gathered the same way and summed in CTA order by every CTA, so γ and the
// stop decision are identical everywhere.
#include <math_constants.h>
#include <algorithm>
#include <type_traits>
#include "common.cuh"
#include "internal.h"

namespace fram {
namespace {

constexpr int kCThreads = 256, kCWarps = 8, kCMaxCols = 28, kCMaxRows = 64, kCMaxCluster = 16;
constexpr int kCColsPerThread = (32 * kCMaxCols + kCThreads - 1) / kCThreads;   // 4

__device__ __forceinline__ uint32_t dsmem(const void* p, unsigned rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void dst_f64(uint32_t a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// st.async: a remote shared-memory store that completes its bytes on the receiver's mbarrier
__device__ __forceinline__ void ast_b32(uint32_t a, uint32_t v, uint32_t mb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(a), "r"(v), "r"(mb) : "memory");
}
__device__ __forceinline__ void ast_b64(uint32_t a, unsigned long long v, uint32_t mb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(a), "l"(v), "r"(mb) : "memory");
}
template <typename T> __device__ __forceinline__ void ast_t(uint32_t a, T v, uint32_t mb);
template <> __device__ __forceinline__ void ast_t<float>(uint32_t a, float v, uint32_t mb) { ast_b32(a, __float_as_uint(v), mb); }
template <> __device__ __forceinline__ void ast_t<double>(uint32_t a, double v, uint32_t mb) {
  ast_b64(a, (unsigned long long)__double_as_longlong(v), mb);
}
__device__ __forceinline__ void mb_wait(uint32_t mb, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred pp; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 pp, [%1], %2; selp.u32 %0, 1, 0, pp; }"
                 : "=r"(done) : "r"(mb), "r"(parity) : "memory");
}

template <typename T, int MC>                              // MC ≥ ⌈n/32⌉ columns per lane
__global__ void __launch_bounds__(kCThreads, 1) sdsn_cluster_kernel(SdsnParams P, int ldn) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const int n = (int)P.n;
  unsigned crank, csize;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
  const int c = (int)crank, C = (int)csize;
  const int r0 = (int)((long)c * n / C), r1 = (int)((long)(c + 1) * n / C), R = r1 - r0;
  const int SL = (n + C - 1) / C;                        // ≥ every column slice
  const int k0 = (int)((long)c * n / C), k1 = (int)((long)(c + 1) * n / C);   // my column slice
  // the same layout in every CTA (DSMEM addresses are mapped from the local ones): sized by the
  // largest row count, ceil(n/C)
  const int Rmax = (n + C - 1) / C;
  T* Ys = reinterpret_cast<T*>(dsm);                     // [Rmax][ldn] my rows
  T* s_cp = Ys + (size_t)Rmax * ldn;                     // [8][ldn] per-warp column partials
  T* s_recv = s_cp + (size_t)kCWarps * ldn;              // [C][SL] partials of my column slice
  T* s_b = s_recv + (size_t)kCMaxCluster * SL;           // [ldn] b_j, all columns
  __shared__ double s_Sp[2][kCMaxCluster];               // per-CTA masses (all-gathered), by call parity:
                                                         // with the mbarrier hand-off a fast CTA's next
                                                         // masses may land before a slow thread read these
  __shared__ double s_M[kCMaxCluster];                   // per-CTA maxima (all-gathered)
  __shared__ double s_r[kCMaxRows], s_rn[kCMaxRows];     // row sums and r_i/n of my rows
  __shared__ T s_a[kCMaxRows];
  __shared__ __align__(8) uint64_t s_mb[2];              // [0]: my slice's partials + masses, [1]: all b
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t mb0 = (uint32_t)__cvta_generic_to_shared(&s_mb[0]);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0 + 8));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const double dn = (double)n, nn = dn * dn;
  const double rn = __drcp_rn(dn), rnn = __drcp_rn(nn);
  auto div_n = [&](double x, double d, double r) {
    const double q = x * r;
    return fma(r, fma(-q, d, x), q);
  };
  const T* X = reinterpret_cast<const T*>(P.Y);

  // ---- load my rows and their max (Alg.2 step 1), max all-gathered through DSMEM ----
  double lmax = 0.0;
  for (int i = warp; i < R; i += kCWarps)
    for (int j = lane; j < n; j += 32) {
      const T x = X[(long)(r0 + i) * P.ld + j];
      Ys[i * ldn + j] = x;
      lmax = fmax(lmax, (double)x);
    }
  lmax = warp_max_d(lmax);
  __shared__ double s_w[kCWarps];
  if (lane == 0) s_w[warp] = lmax;
  __syncthreads();
  if (tid < C) {
    double m = 0.0;
    for (int w = 0; w < kCWarps; ++w) m = fmax(m, s_w[w]);
    dst_f64(dsmem(&s_M[c], (unsigned)tid), m);           // my max into CTA tid's s_M[c]
  }
  cluster_sync();
  double m = 0.0;
  for (int k = 0; k < C; ++k) m = fmax(m, s_M[k]);
  if (P.scale && m == 0.0) {                                        // R10 (θ-scaling on): all-zero ⇒ 11ᵀ/n, 0 passes
    for (int i = warp; i < R; i += kCWarps)
      for (int j = lane; j < n; j += 32) reinterpret_cast<T*>(P.Y)[(long)(r0 + i) * P.ld + j] = (T)(1.0 / dn);
    if (c == 0 && tid == 0) {
      *P.passes_out = 0;
      P.sdsn_out[0] = 0.0; P.sdsn_out[1] = 0.0; P.sdsn_out[2] = 0.0;
    }
    cluster_sync();
    return;
  }
  const double sc = (P.theta / 2.0) / m;                 // R11
  if (c == 0 && tid == 0) P.sdsn_out[1] = m;

  // the DSMEM slot of each of my columns in its owner's s_recv (owner k: k·n/C ≤ j < (k+1)·n/C),
  // computed once (64-bit integer divisions are slow)
  uint32_t dst_addr[kCColsPerThread];
#pragma unroll
  for (int u = 0; u < kCColsPerThread; ++u) {
    const int j = tid + u * kCThreads;
    dst_addr[u] = 0;
    if (j < n) {
      int kk = (int)min((long)(C - 1), (long)j * C / n);
      while (kk > 0 && (long)kk * n / C > j) --kk;
      while (kk + 1 < C && (long)(kk + 1) * n / C <= j) ++kk;
      dst_addr[u] = dsmem(&s_recv[c * SL + (j - (int)((long)kk * n / C))], (unsigned)kk);
    }
  }
  uint32_t sp_addr = 0, sp_mb = 0;                       // my mass slot in CTA `lane`'s s_Sp (+ its mbarrier)
  if (warp == 0 && lane < C) {
    sp_addr = dsmem(&s_Sp[0][c], (unsigned)lane);
    sp_mb = dsmem(&s_mb[0], (unsigned)lane);
  }
  // owner of each of my columns' mbarrier (partials), computed with the slots above
  uint32_t dst_mb[kCColsPerThread];
#pragma unroll
  for (int u = 0; u < kCColsPerThread; ++u) {
    const int j = tid + u * kCThreads;
    dst_mb[u] = 0;
    if (j < n) {
      int kk = (int)min((long)(C - 1), (long)j * C / n);
      while (kk > 0 && (long)kk * n / C > j) --kk;
      while (kk + 1 < C && (long)(kk + 1) * n / C <= j) ++kk;
      dst_mb[u] = dsmem(&s_mb[0], (unsigned)kk);
    }
  }
  int call = 0;                                          // sweep_and_reduce calls: mbarrier phase parity
  double S = 0.0;                                       // mass of the current iterate (all CTAs)
  // ---- one sweep over my rows, then the cluster all-reduce of column sums and mass ----
  // mode 0: y ← fl(s·y) (or y when !scale); mode 1: y ← max(0, (y + a_i) + b_j)
  auto sweep_and_reduce = [&](int mode) {
    const uint32_t par = (uint32_t)(call & 1);
    ++call;
    if (tid == 0) {                                      // bytes this pass brings: my slice from every
      const uint32_t bp = (uint32_t)(C * ((k1 - k0) * (int)sizeof(T) + 8));   // CTA + C masses; all of b
      const uint32_t bb = (uint32_t)(n * (int)sizeof(T));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb0), "r"(bp) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb0 + 8), "r"(bb) : "memory");
    }
    T colacc[MC], bl[MC];
#pragma unroll
    for (int m2 = 0; m2 < MC; ++m2) {
      const int j = lane + 32 * m2;
      colacc[m2] = (T)0;
      bl[m2] = (mode && j < n) ? s_b[j] : (T)0;           // b of my columns, for every row
    }
    // one row of this warp: y ← op(y) on the lane's ≤ MC columns, column partials, returns the lane's
    // row partial.  Loads, arithmetic and stores in separate unrolled loops (no branch between columns,
    // so the columns' dependency chains overlap); columns ≥ n read and contribute 0
    auto row = [&](int i) -> T {
      const T a = mode ? s_a[i] : (T)0;
      T rs = (T)0;
      T xv[MC];
#pragma unroll
      for (int m2 = 0; m2 < MC; ++m2) {
        const int j = lane + 32 * m2;
        xv[m2] = j < n ? Ys[i * ldn + j] : (T)0;
      }
#pragma unroll
      for (int m2 = 0; m2 < MC; ++m2) {
        const int j = lane + 32 * m2;
        T y;
        if (mode) {
          y = (xv[m2] + a) + bl[m2];                     // P1 then P2 (R9 grouping)
          y = y > (T)0 ? y : (T)0;
        } else {
          y = P.scale ? (T)(sc * (double)xv[m2]) : xv[m2];
        }
        y = j < n ? y : (T)0;
        xv[m2] = y;
        rs += y;
        colacc[m2] += y;
      }
#pragma unroll
      for (int m2 = 0; m2 < MC; ++m2) {
        const int j = lane + 32 * m2;
        if (j < n) Ys[i * ldn + j] = xv[m2];
      }
      return rs;
    };
    // n > 32 (R = 32 rows, 4 per warp): the warp's row partials are reduced together by one transpose-
    // reduce after its rows (5-9% faster per pass at n = 64-500, profiles/r02/ab_k4c4.log); n ≤ 32 (one
    // CTA, ≤ 3 rows per warp): row by row, as before
    constexpr int RB = kCMaxRows / kCWarps;             // 8
    constexpr bool batch_rows = MC > 1;
    T rsv[RB];
    if constexpr (batch_rows) {
#pragma unroll
      for (int q = 0; q < RB; ++q) rsv[q] = (T)0;
#pragma unroll
      for (int q = 0; q < RB; ++q) {
        const int i = warp + q * kCWarps;
        if (i >= R) break;
        rsv[q] = row(i);
      }
    } else {
      for (int i = warp; i < R; i += kCWarps) {
        const T rs = row(i);
        double r;
        if constexpr (sizeof(T) == 8) r = warp_sum_d((double)rs);
        else r = (double)warp_sum_f((float)rs);
        if (lane == 0) {
          s_r[i] = r;
          s_rn[i] = div_n(r, dn, rn);
        }
      }
    }
    if constexpr (batch_rows) {   // transpose-reduce of the RB = 8 rows: xor 16, 8, 4 halve the rows a
      // lane carries, xor 2, 1 finish; lane 4q ends with row q's sum (fixed tree, deterministic; FP64 adds
      // for T = double, FP32 partials then FP64 for T = float as before)
      using A = typename std::conditional<sizeof(T) == 8, double, float>::type;
      A v[RB];
#pragma unroll
      for (int q = 0; q < RB; ++q) v[q] = (A)rsv[q];
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        const int off = 16 >> l, m = RB >> (l + 1);
        const bool hi = lane & off;
#pragma unroll
        for (int q = 0; q < m; ++q) v[q] = (hi ? v[q + m] : v[q]) + __shfl_xor_sync(0xffffffffu, hi ? v[q] : v[q + m], off);
      }
      A z = v[0];
      z += __shfl_xor_sync(0xffffffffu, z, 2);
      z += __shfl_xor_sync(0xffffffffu, z, 1);
      const int i = warp + (lane >> 2) * kCWarps;
      if ((lane & 3) == 0 && i < R) {
        const double r = (double)z;
        s_r[i] = r;
        s_rn[i] = div_n(r, dn, rn);
      }
    }
#pragma unroll
    for (int m2 = 0; m2 < MC; ++m2) {
      const int j = lane + 32 * m2;
      if (j < n) s_cp[warp * ldn + j] = colacc[m2];
    }
    __syncthreads();
    // CTA partial of column j (8 warps in order) → the owner CTA of j (DSMEM); my mass → every CTA
#pragma unroll
    for (int u = 0; u < kCColsPerThread; ++u) {
      const int j = tid + u * kCThreads;
      if (j < n) {
        T p = s_cp[j];
        for (int w = 1; w < kCWarps; ++w) p += s_cp[w * ldn + j];
        ast_t<T>(dst_addr[u], p, dst_mb[u]);
      }
    }
    if (warp == 0) {
      double s = 0.0;
      for (int i = lane; i < R; i += 32) s += s_r[i];
      s = warp_sum_d(s);
      if (lane < C) {
        ast_t<double>(sp_addr + par * (uint32_t)(kCMaxCluster * sizeof(double)), s, sp_mb);
      }
    }
    mb_wait(mb0, par);                                   // my slice's partials and every mass arrived
    S = 0.0;                                             // every CTA: the masses in CTA order
    if constexpr (MC > 1) {
      double mv[kCMaxCluster];
#pragma unroll
      for (int k = 0; k < kCMaxCluster; ++k) mv[k] = k < C ? s_Sp[par][k] : 0.0;
#pragma unroll
      for (int k = 0; k < kCMaxCluster; ++k)
        if (k < C) S += mv[k];
    } else {
      for (int k = 0; k < C; ++k) S += s_Sp[par][k];
    }
    // my column slice: c_j = Σ over CTAs in order (FP64); b_j = −c_j/n → every CTA (DSMEM)
    for (int j = k0 + tid; j < k1; j += kCThreads) {
      double cs = 0.0;
      if constexpr (MC > 1) {
        T pv[kCMaxCluster];                             // all loads in flight, then the sum in CTA order
#pragma unroll
        for (int k = 0; k < kCMaxCluster; ++k) pv[k] = k < C ? s_recv[k * SL + (j - k0)] : (T)0;
#pragma unroll
        for (int k = 0; k < kCMaxCluster; ++k)
          if (k < C) cs += (double)pv[k];
      } else {                                          // n ≤ 32: one CTA
        for (int k = 0; k < C; ++k) cs += (double)s_recv[k * SL + (j - k0)];
      }
      const T bj = (T)(-div_n(cs, dn, rn));
      for (int k = 0; k < C; ++k) {
        ast_t<T>(dsmem(&s_b[j], (unsigned)k), bj, dsmem(&s_mb[1], (unsigned)k));
      }
    }
    mb_wait(mb0 + 8, par);                               // every b_j arrived
  };

  sweep_and_reduce(0);
  int jp = 0;
  double gam = 0.0;
  for (;; ++jp) {
    gam = div_n(S, dn, rn) - 1.0;                        // γ_j
    if (c == 0 && tid == 0 && P.gamma_hist) P.gamma_hist[jp] = gam;
    const bool last = P.sdsn_fixed > 0 ? (jp + 1 >= P.sdsn_fixed)
                                       : ((jp >= 1 && gam <= P.gamma_th) || jp + 1 >= P.sdsn_max);
    const double abase = rn + div_n(S, nn, rnn);         // 1/n + S/n²
    for (int i = tid; i < R; i += kCThreads) s_a[i] = (T)(abase - s_rn[i]);
    __syncthreads();
    const double S_in = S;
    sweep_and_reduce(1);                                 // the last pass's exchange is harmless
    if (last) {
      S = S_in;                                          // sdsn_out[2]: S of the last pass input
      break;
    }
  }
  // D → global
  for (int i = warp; i < R; i += kCWarps)
    for (int j = lane; j < n; j += 32) reinterpret_cast<T*>(P.Y)[(long)(r0 + i) * P.ld + j] = Ys[i * ldn + j];
  if (c == 0 && tid == 0) {
    *P.passes_out = jp + 1;
    P.sdsn_out[0] = gam;
    P.sdsn_out[2] = S;
  }
  cluster_sync();                                        // no CTA exits while remote stores may target it
}

int cluster_size_for(long n) { return (int)std::min<long>(kCMaxCluster, std::max<long>(1, (n + 31) / 32)); }

size_t cluster_smem(long n, int C, size_t ts) {
  const long ldn = (n + 3) & ~3L;
  const long R = (n + C - 1) / C, SL = (n + C - 1) / C;
  return ((size_t)R * ldn + (size_t)kCWarps * ldn + (size_t)kCMaxCluster * SL + (size_t)ldn) * ts;
}

}  // namespace

bool sdsn_cluster_supported(long n, bool f64) {
  if (n < 1 || (n + 31) / 32 > kCMaxCols) return false;
  const int C = cluster_size_for(n);
  if ((n + C - 1) / C > kCMaxRows) return false;
  return cluster_smem(n, C, f64 ? 8 : 4) <= (size_t)(227 * 1024 - 4096);
}

cudaError_t launch_sdsn_cluster(const SdsnParams& p, bool f64, cudaStream_t st) {
  if (!sdsn_cluster_supported(p.n, f64)) return cudaErrorInvalidValue;
  const int C = cluster_size_for(p.n);
  const int ldn = (int)((p.n + 3) & ~3L);
  const size_t dsm = cluster_smem(p.n, C, f64 ? 8 : 4);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kCThreads);
  cfg.dynamicSmemBytes = dsm;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int mc = (int)((p.n + 31) / 32);
  auto go = [&](auto tag, auto mc_c) -> cudaError_t {
    using T = decltype(tag);
    auto fn = sdsn_cluster_kernel<T, decltype(mc_c)::value>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
    if (e != cudaSuccess) return e;
    if (C > 8 && (e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess) return e;
    return cudaLaunchKernelEx(&cfg, fn, p, ldn);
  };
  auto pick = [&](auto tag) -> cudaError_t {
    if (mc <= 1) return go(tag, std::integral_constant<int, 1>{});
    if (mc <= 2) return go(tag, std::integral_constant<int, 2>{});
    if (mc <= 4) return go(tag, std::integral_constant<int, 4>{});
    if (mc <= 8) return go(tag, std::integral_constant<int, 8>{});
    if (mc <= 16) return go(tag, std::integral_constant<int, 16>{});
    return go(tag, std::integral_constant<int, kCMaxCols>{});
  };
  return f64 ? pick(double{}) : pick(float{});
}

}  // namespace fram
