// sdsn.cu — K4: SDSN (Scaling Doubly Stochastic Normalization), Alg. 2 of arXiv 2508.00887
// (PAPER.md P:344-361), as ONE persistent cooperative kernel per SDSN call.
//
// Per pass j on Y_j (mass S_j, row sums r, column sums c of Y_j, all known before the pass):
//   γ_j = S_j/n − 1                                 (Alg.2 step 7, lagged, P:355 / P:642)
//   a_i = (1/n + S_j/n²) − r_i/n ;  b_j = −c_j/n     (steps 3-5 elementwise, R9)
//   Y_{j+1} = max(0, (Y_j + a_i) + b_j)              (step 6: P2 ∘ P1)
//   and, fused into the same sweep, the row sums, column partials and mass of Y_{j+1}.
// Stop after pass j iff (j ≥ 1 ∧ γ_j ≤ γ_th) ∨ j+1 = sdsn_max (R5, R16) — known BEFORE the pass.
//
// Data layout: Y row-major n×ld in HBM (T = float in mixed modes, double in FP64 mode); CTA b
// owns rows [b·n/G, (b+1)·n/G); thread t owns 16-byte column vectors q = t + k·THREADS.
//   row sums  : per-thread partials → warp shuffle → fixed-order cross-warp sum (FP64) — local;
//   col sums  : per-thread register partials over the CTA's rows → colpart[b][:] →
//               grid barrier → CTA b reduces column slice b over all CTAs in a fixed order
//               (deterministic, no float atomics: S:375) → grid barrier.
//   S         : Σ per-CTA row-sum partials, summed identically by every CTA (FP64).
// Bytes per pass: 8n² (FP32) / 16n² (FP64) of Y + O(G·n) partials.
#include "common.cuh"
#include "internal.h"

namespace fram {

template <typename T> struct VecT;
template <> struct VecT<float>  { using t = float4;  static constexpr int W = 4; };
template <> struct VecT<double> { using t = double2; static constexpr int W = 2; };

constexpr int kSdsnThreads = 512;
constexpr int kSdsnWarps = kSdsnThreads / 32;
constexpr int kSdsnMaxRows = 1024;

template <typename T> __device__ __forceinline__ void vget(const typename VecT<T>::t& v, T* o);
template <> __device__ __forceinline__ void vget<float>(const float4& v, float* o) { o[0]=v.x; o[1]=v.y; o[2]=v.z; o[3]=v.w; }
template <> __device__ __forceinline__ void vget<double>(const double2& v, double* o) { o[0]=v.x; o[1]=v.y; }
template <typename T> __device__ __forceinline__ typename VecT<T>::t vmake(const T* o);
template <> __device__ __forceinline__ float4 vmake<float>(const float* o) { return make_float4(o[0],o[1],o[2],o[3]); }
template <> __device__ __forceinline__ double2 vmake<double>(const double* o) { return make_double2(o[0],o[1]); }

__device__ __forceinline__ float tmax0(float x) { return fmaxf(0.0f, x); }
__device__ __forceinline__ double tmax0(double x) { return fmax(0.0, x); }
__device__ __forceinline__ float warp_sum_t(float v) { return warp_sum_f(v); }
__device__ __forceinline__ double warp_sum_t(double v) { return warp_sum_d(v); }

// Fixed-order block reduction of RB per-thread row partials → s_r[row0 .. row0+cnt) (FP64).
template <typename T, int RB>
__device__ __forceinline__ void block_rows_reduce(T (&acc)[RB], double (*s_part)[kSdsnWarps][RB],
                                                  int buf, double* s_r, int row0, int cnt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int rr = 0; rr < RB; ++rr) {
    T v = warp_sum_t(acc[rr]);
    if (lane == 0) s_part[buf][warp][rr] = (double)v;
  }
  __syncthreads();
  if (threadIdx.x < cnt) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kSdsnWarps; ++w) s += s_part[buf][w][threadIdx.x];
    s_r[row0 + threadIdx.x] = s;
  }
}

template <typename T, int NV>
__global__ void __launch_bounds__(kSdsnThreads, 1) sdsn_kernel(SdsnParams P) {
  using VT = typename VecT<T>::t;
  constexpr int W = VecT<T>::W;
  constexpr int RB = (8 / NV) > 0 ? (8 / NV) : 1;           // rows per chunk: 8 vectors in flight
  __shared__ double s_r[kSdsnMaxRows];
  __shared__ T s_a[kSdsnMaxRows];
  __shared__ double s_part[2][kSdsnWarps][RB];
  __shared__ double s_red[kSdsnWarps][32];
  __shared__ double s_scal[2];

  const unsigned G = gridDim.x;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long n = P.n, ld = P.ld;
  const long r0 = (long)b * n / G, r1 = (long)(b + 1) * n / G;
  const int R = (int)(r1 - r0);
  const long nvec = (n + W - 1) / W;
  T* Y = reinterpret_cast<T*>(P.Y);
  T* colpart = reinterpret_cast<T*>(P.colpart);
  const double dn = (double)n, nn = dn * dn, inv_n = 1.0 / dn;

  // ---------------- column-slice reduction + S (after barrier 1) ----------------
  auto reduce_columns_and_S = [&]() {
    const long cb = (long)b * n / G, ce = (long)(b + 1) * n / G;
    for (long c0 = cb; c0 < ce; c0 += 32) {
      const long col = c0 + lane;
      double acc = 0.0;
      if (col < ce)
        for (unsigned k = warp; k < G; k += kSdsnWarps) acc += (double)ldcg(colpart + (long)k * ld + col);
      s_red[warp][lane] = acc;
      __syncthreads();
      if (tid < 32 && c0 + tid < ce) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < kSdsnWarps; ++w) s += s_red[w][tid];
        P.cvec[c0 + tid] = s;
      }
      __syncthreads();
    }
    if (warp == 0) {
      double s = 0.0;
      for (unsigned k = lane; k < G; k += 32) s += ldcg(P.Spart + k);
      s = warp_sum_d(s);
      if (lane == 0) s_scal[0] = s;
    }
  };
  // per-CTA Σ of own row sums (fixed order) → Spart[b]
  auto publish_rows = [&]() {
    __syncthreads();
    if (warp == 0) {
      double s = 0.0;
      for (int i = lane; i < R; i += 32) s += s_r[i];
      s = warp_sum_d(s);
      if (lane == 0) P.Spart[b] = s;
    }
  };

  // ---------------- phase M: m = max X (Alg.2 step 1) ----------------
  double sc = 1.0;
  if (P.scale) {
    double m = 0.0;
    for (int i = 0; i < R; ++i) {
      const VT* row = reinterpret_cast<const VT*>(Y + (r0 + i) * ld);
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const long q = tid + (long)k * kSdsnThreads;
        if (q < nvec) {
          T e[W];
          vget<T>(ldcg(row + q), e);
#pragma unroll
          for (int w = 0; w < W; ++w)
            if (q * W + w < n) m = fmax(m, (double)e[w]);
        }
      }
    }
    m = warp_max_d(m);
    if (lane == 0) s_red[warp][0] = m;
    __syncthreads();
    if (tid == 0) {
      double mm = 0.0;
      for (int w = 0; w < kSdsnWarps; ++w) mm = fmax(mm, s_red[w][0]);
      P.Mpart[b] = mm;
    }
    grid_barrier(P.bar, G);
    if (warp == 0) {
      double mm = 0.0;
      for (unsigned k = lane; k < G; k += 32) mm = fmax(mm, ldcg(P.Mpart + k));
      mm = warp_max_d(mm);
      if (lane == 0) s_scal[1] = mm;
    }
    __syncthreads();
    m = s_scal[1];
    if (m == 0.0) {                                   // R10: all-zero ⇒ 11ᵀ/n, 0 passes
      for (int i = 0; i < R; ++i) {
        VT* row = reinterpret_cast<VT*>(Y + (r0 + i) * ld);
        for (long q = tid; q < ld / W; q += kSdsnThreads) {
          T e[W];
#pragma unroll
          for (int w = 0; w < W; ++w) e[w] = (q * W + w < n) ? (T)inv_n : (T)0;
          row[q] = vmake<T>(e);
        }
      }
      if (b == 0 && tid == 0) {
        *P.passes_out = 0;
        P.sdsn_out[0] = 0.0; P.sdsn_out[1] = 0.0; P.sdsn_out[2] = 0.0;
      }
      return;
    }
    sc = (P.theta / 2.0) / m;                         // R11: s = (θ/2)/max X, FP64
    if (b == 0 && tid == 0) P.sdsn_out[1] = m;
  }

  // ---------------- phase S: Y0 = s·X (in place) and its sums ----------------
  T colacc[NV][W];
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int w = 0; w < W; ++w) colacc[k][w] = (T)0;
  {
    int buf = 0;
    for (int i0 = 0; i0 < R; i0 += RB, buf ^= 1) {
      T racc[RB];
#pragma unroll
      for (int rr = 0; rr < RB; ++rr) {
        racc[rr] = (T)0;
        const int i = i0 + rr;
        if (i < R) {
          VT* row = reinterpret_cast<VT*>(Y + (r0 + i) * ld);
#pragma unroll
          for (int k = 0; k < NV; ++k) {
            const long q = tid + (long)k * kSdsnThreads;
            if (q < nvec) {
              T e[W];
              vget<T>(row[q], e);
#pragma unroll
              for (int w = 0; w < W; ++w) {
                T y = P.scale ? (T)(sc * (double)e[w]) : e[w];
                y = (q * W + w < n) ? y : (T)0;
                e[w] = y;
                racc[rr] += y;
                colacc[k][w] += y;
              }
              if (P.scale) row[q] = vmake<T>(e);
            }
          }
        }
      }
      block_rows_reduce<T, RB>(racc, s_part, buf, s_r, i0, min(RB, R - i0));
    }
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const long q = tid + (long)k * kSdsnThreads;
    if (q < nvec) reinterpret_cast<VT*>(colpart + (long)b * ld)[q] = vmake<T>(colacc[k]);
  }
  publish_rows();
  grid_barrier(P.bar, G);
  reduce_columns_and_S();
  grid_barrier(P.bar, G);

  // ---------------- pass loop ----------------
  int j = 0;
  double gam = 0.0;
  for (;; ++j) {
    const double S = s_scal[0];
    gam = S / dn - 1.0;                                                // γ_j
    if (b == 0 && tid == 0 && P.gamma_hist) P.gamma_hist[j] = gam;
    const bool last = P.sdsn_fixed > 0 ? (j + 1 >= P.sdsn_fixed)
                                       : ((j >= 1 && gam <= P.gamma_th) || j + 1 >= P.sdsn_max);
    const double abase = 1.0 / dn + S / nn;
    for (int i = tid; i < R; i += kSdsnThreads) s_a[i] = (T)(abase - s_r[i] / dn);
    __syncthreads();
    T bv[NV][W];                                                       // b for owned columns
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const long q = tid + (long)k * kSdsnThreads;
#pragma unroll
      for (int w = 0; w < W; ++w)
        bv[k][w] = (q * W + w < n) ? (T)(-ldcg(P.cvec + q * W + w) / dn) : (T)0;
#pragma unroll
      for (int w = 0; w < W; ++w) colacc[k][w] = (T)0;
    }
    int buf = 0;
    for (int i0 = 0; i0 < R; i0 += RB, buf ^= 1) {
      VT v[RB][NV];
#pragma unroll
      for (int rr = 0; rr < RB; ++rr) {
        const int i = i0 + rr;
        if (i < R) {
          const VT* row = reinterpret_cast<const VT*>(Y + (r0 + i) * ld);
#pragma unroll
          for (int k = 0; k < NV; ++k) {
            const long q = tid + (long)k * kSdsnThreads;
            if (q < nvec) v[rr][k] = __ldcg(row + q);
          }
        }
      }
      T racc[RB];
#pragma unroll
      for (int rr = 0; rr < RB; ++rr) {
        racc[rr] = (T)0;
        const int i = i0 + rr;
        if (i < R) {
          const T a = s_a[i];
          VT* row = reinterpret_cast<VT*>(Y + (r0 + i) * ld);
#pragma unroll
          for (int k = 0; k < NV; ++k) {
            const long q = tid + (long)k * kSdsnThreads;
            if (q < nvec) {
              T e[W];
              vget<T>(v[rr][k], e);
#pragma unroll
              for (int w = 0; w < W; ++w) {
                T y = tmax0((e[w] + a) + bv[k][w]);                    // P2(P1(Y)) elementwise
                y = (q * W + w < n) ? y : (T)0;
                e[w] = y;
                racc[rr] += y;
                colacc[k][w] += y;
              }
              __stcg(row + q, vmake<T>(e));
            }
          }
        }
      }
      block_rows_reduce<T, RB>(racc, s_part, buf, s_r, i0, min(RB, R - i0));
    }
    if (last) break;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const long q = tid + (long)k * kSdsnThreads;
      if (q < nvec) reinterpret_cast<VT*>(colpart + (long)b * ld)[q] = vmake<T>(colacc[k]);
    }
    publish_rows();
    grid_barrier(P.bar, G);
    reduce_columns_and_S();
    grid_barrier(P.bar, G);
  }
  if (b == 0 && tid == 0) {
    *P.passes_out = j + 1;
    P.sdsn_out[0] = gam;
    P.sdsn_out[2] = s_scal[0];
  }
}

static int nv_for(long n, bool f64) {
  const int W = f64 ? 2 : 4;
  const long nvec = (n + W - 1) / W;
  const long per = (nvec + kSdsnThreads - 1) / kSdsnThreads;
  if (per <= 1) return 1;
  if (per <= 2) return 2;
  if (per <= 4) return 4;
  if (per <= 8) return 8;
  return 0;
}

bool sdsn_supported(long n, bool f64) { return n >= 1 && nv_for(n, f64) > 0; }

int sdsn_grid_for(long n, int num_sms) {
  long g = n / 16;
  if (g < 1) g = 1;
  if (g > num_sms) g = num_sms;
  while ((n + g - 1) / g > kSdsnMaxRows) ++g;   // (only for n > 1024·num_sms)
  return (int)g;
}

template <typename T, int NV>
static cudaError_t launch_t(const SdsnParams& p, cudaStream_t st, int grid) {
  auto fn = sdsn_kernel<T, NV>;
  SdsnParams pp = p;
  void* args[] = {&pp};
  return cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(kSdsnThreads), args, 0, st);
}

cudaError_t launch_sdsn(const SdsnParams& p, bool f64, cudaStream_t st, int num_sms, int* grid_out) {
  const int nv = nv_for(p.n, f64);
  if (nv == 0) return cudaErrorInvalidValue;
  const int grid = sdsn_grid_for(p.n, num_sms);
  if (grid_out) *grid_out = grid;
  cudaError_t e = cudaMemsetAsync(p.bar, 0, 2 * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  if (f64) {
    switch (nv) {
      case 1: return launch_t<double, 1>(p, st, grid);
      case 2: return launch_t<double, 2>(p, st, grid);
      case 4: return launch_t<double, 4>(p, st, grid);
      default: return launch_t<double, 8>(p, st, grid);
    }
  }
  switch (nv) {
    case 1: return launch_t<float, 1>(p, st, grid);
    case 2: return launch_t<float, 2>(p, st, grid);
    case 4: return launch_t<float, 4>(p, st, grid);
    default: return launch_t<float, 8>(p, st, grid);
  }
}

}  // namespace fram
