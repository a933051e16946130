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
// Data layout and work split: Y row-major n×ld (T = float in mixed modes, double in FP64 mode).
// CTA b owns rows [b·n/G, (b+1)·n/G).  Its 16 warps form CG column groups × RG row groups
// (CG·RG = 16); a warp streams every row of its row group over its column slice, with a register
// ring keeping PD rows of 16-byte loads in flight (no CTA barrier inside the sweep):
//   row sums : warp shuffle per row → s_rowpart[row][cg] → fixed-order sum over cg (FP64);
//   col sums : per-lane register partials over the warp's rows → (RG>1: fixed-order smem combine)
//              → colpart[b][:] → grid barrier → CTA b reduces column slice b over all CTAs in a
//              fixed order (deterministic, no float atomics: S:375) → grid barrier;
//   S        : Σ per-CTA row-sum partials, summed identically by every CTA (FP64).
// Algorithmic bytes per pass: 8n² (FP32) / 16n² (FP64) of Y, + O(G·n) of partials.
#include <stdlib.h>
#include <type_traits>
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

enum { SWEEP_SCALE = 0, SWEEP_PASS = 1 };

template <typename T, int VPL>
__global__ void __launch_bounds__(kSdsnThreads, 1) sdsn_kernel(SdsnParams P, int CG) {
  using VT = typename VecT<T>::t;
  constexpr int W = VecT<T>::W;
  constexpr int PD = VPL >= 8 ? 1 : 16 / VPL;                // rows in flight per warp
  extern __shared__ __align__(16) unsigned char dsm[];
  const long rows_max = (P.n + gridDim.x - 1) / gridDim.x + 1;
  double* s_rowpart = reinterpret_cast<double*>(dsm);       // [rows_max][CG]
  T* s_colstage = reinterpret_cast<T*>(dsm + ((sizeof(double) * rows_max * CG + 15) & ~15ul));   // [RG][ld]
  __shared__ double s_r[kSdsnMaxRows];
  __shared__ T s_a[kSdsnMaxRows];
  __shared__ double s_red[kSdsnWarps][32];
  __shared__ double s_scal[2];

  const unsigned G = gridDim.x;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int RG = kSdsnWarps / CG;
  const int cg = warp % CG, rg = warp / CG;
  const long n = P.n, ld = P.ld;
  const long r0 = (long)b * n / G, r1 = (long)(b + 1) * n / G;
  const int R = (int)(r1 - r0);
  const long nvec = (n + W - 1) / W;
  const int nrw = (R > rg) ? (R - rg + RG - 1) / RG : 0;     // rows handled by this warp
  T* Y = reinterpret_cast<T*>(P.Y);
  T* colpart = reinterpret_cast<T*>(P.colpart);
  const double dn = (double)n, nn = dn * dn;
  // vector index of slot k for this lane: q = (cg·VPL + k)·32 + lane
  auto qidx = [&](int k) -> long { return ((long)cg * VPL + k) * 32 + lane; };

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

  // ---------------- one sweep over the CTA's rows ----------------
  // MODE SCALE: y ← fl(s·y) (written only if P.scale); MODE PASS: y ← max(0, (y + a_i) + b_j).
  // Both accumulate the row sums (s_r) and column partials (colpart[b]) of the new values.
  auto sweep = [&](auto mode_c, double sc, const T (&bv)[VPL][W]) {
    constexpr int mode = decltype(mode_c)::value;
    T colacc[VPL][W];
#pragma unroll
    for (int k = 0; k < VPL; ++k)
#pragma unroll
      for (int w = 0; w < W; ++w) colacc[k][w] = (T)0;
    // per-slot constants (32-bit indexing: n·ld < 2^31 for every supported n)
    const int ldv = (int)(ld / W);
    VT* Yc = reinterpret_cast<VT*>(Y) + (long)r0 * ldv;        // this CTA's first row
    int qv[VPL], kind[VPL];                                   // kind: 0 skip, 1 full vector, 2 tail
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      qv[k] = (int)qidx(k);
      kind[k] = qv[k] >= (int)nvec ? 0 : ((qv[k] + 1) * W <= (int)n ? 1 : 2);
    }
    VT buf[PD][VPL];
    auto load_row = [&](int s, int rr) {
      const VT* row = Yc + (rg + rr * RG) * ldv;
#pragma unroll
      for (int k = 0; k < VPL; ++k)
        if (kind[k]) buf[s][k] = __ldcg(row + qv[k]);
    };
    bool full = true;                                          // every slot a full vector?
#pragma unroll
    for (int k = 0; k < VPL; ++k) full = full && (kind[k] == 1);
    full = __all_sync(0xffffffffu, full);
#pragma unroll
    for (int s = 0; s < PD; ++s)
      if (s < nrw) load_row(s, s);
    auto run = [&](auto full_c) {
      constexpr bool FULL = decltype(full_c)::value;
      for (int base = 0; base < nrw; base += PD) {
        T rs[PD];
#pragma unroll
        for (int s = 0; s < PD; ++s) {
          rs[s] = (T)0;
          const int rr = base + s;
          if (rr < nrw) {
            const int il = rg + rr * RG;                     // local row index
            VT* row = Yc + il * ldv;
            const T a = (mode == SWEEP_PASS) ? s_a[il] : (T)0;
#pragma unroll
            for (int k = 0; k < VPL; ++k) {
              if (FULL || kind[k]) {
                T e[W];
                vget<T>(buf[s][k], e);
#pragma unroll
                for (int w = 0; w < W; ++w) {
                  T y;
                  if constexpr (mode == SWEEP_PASS) y = tmax0((e[w] + a) + bv[k][w]);   // P2(P1(Y))
                  else y = P.scale ? (T)(sc * (double)e[w]) : e[w];
                  if (!FULL && kind[k] == 2 && qv[k] * W + w >= (int)n) y = (T)0;     // ragged tail
                  e[w] = y;
                  rs[s] += y;
                  colacc[k][w] += y;
                }
                if (mode == SWEEP_PASS || P.scale) __stcg(row + qv[k], vmake<T>(e));
              }
            }
            if (rr + PD < nrw) load_row(s, rr + PD);
          }
        }
#pragma unroll
        for (int s = 0; s < PD; ++s) rs[s] = warp_sum_t(rs[s]);      // converged: PD chains interleave
        if (lane == 0) {
#pragma unroll
          for (int s = 0; s < PD; ++s)
            if (base + s < nrw) s_rowpart[(rg + (base + s) * RG) * CG + cg] = (double)rs[s];
        }
      }
    };
    if (full) run(std::true_type{});
    else run(std::false_type{});
    // column partials of this CTA → colpart[b]
    if (RG == 1) {
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        const long q = qidx(k);
        if (q < nvec) reinterpret_cast<VT*>(colpart + (long)b * ld)[q] = vmake<T>(colacc[k]);
      }
      __syncthreads();
    } else {
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        const long q = qidx(k);
        if (q < nvec) reinterpret_cast<VT*>(s_colstage + (long)rg * ld)[q] = vmake<T>(colacc[k]);
      }
      __syncthreads();
      for (long q = tid; q < nvec; q += kSdsnThreads) {
        T acc[W];
        vget<T>(reinterpret_cast<const VT*>(s_colstage)[q], acc);
        for (int g = 1; g < RG; ++g) {
          T e[W];
          vget<T>(reinterpret_cast<const VT*>(s_colstage + (long)g * ld)[q], e);
#pragma unroll
          for (int w = 0; w < W; ++w) acc[w] += e[w];
        }
        reinterpret_cast<VT*>(colpart + (long)b * ld)[q] = vmake<T>(acc);
      }
    }
    // row sums (fixed order over column groups) and the CTA's mass partial
    for (int i = tid; i < R; i += kSdsnThreads) {
      double s = 0.0;
      for (int g = 0; g < CG; ++g) s += s_rowpart[i * CG + g];
      s_r[i] = s;
    }
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
    for (int rr = 0; rr < nrw; ++rr) {
      const VT* row = reinterpret_cast<const VT*>(Y + (r0 + rg + (long)rr * RG) * ld);
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        const long q = qidx(k);
        if (q < nvec) {
          T e[W];
          vget<T>(__ldcg(row + q), e);
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
          for (int w = 0; w < W; ++w) e[w] = (q * W + w < n) ? (T)(1.0 / dn) : (T)0;
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
  {
    T bz[VPL][W];
#pragma unroll
    for (int k = 0; k < VPL; ++k)
#pragma unroll
      for (int w = 0; w < W; ++w) bz[k][w] = (T)0;
    sweep(std::integral_constant<int, SWEEP_SCALE>{}, sc, bz);
  }
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
    T bv[VPL][W];                                                      // b for this lane's columns
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const long q = qidx(k);
#pragma unroll
      for (int w = 0; w < W; ++w)
        bv[k][w] = (q * W + w < n) ? (T)(-ldcg(P.cvec + q * W + w) / dn) : (T)0;
    }
    __syncthreads();
    sweep(std::integral_constant<int, SWEEP_PASS>{}, 1.0, bv);
    if (last) break;
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

// VPL (16-byte vectors per lane per row slice) and CG (column groups, CG·RG = 16 warps).
static bool plan(long n, bool f64, int* vpl, int* cg) {
  const int W = f64 ? 2 : 4;
  const long nvec = (n + W - 1) / W;
  int v = 1;
  while (v <= 8 && (nvec + 32L * v * kSdsnWarps - 1) / (32L * v * kSdsnWarps) > 1) v *= 2;
  if (v > 8) return false;
  const long groups = (nvec + 32L * v - 1) / (32L * v);      // warps needed to cover a row
  int c = 1;
  while (c < groups) c *= 2;
  if (c > kSdsnWarps) return false;
  *vpl = v;
  *cg = c;
  return true;
}

bool sdsn_supported(long n, bool f64) {
  int v, c;
  return n >= 1 && plan(n, f64, &v, &c);
}

int sdsn_grid_for(long n, int num_sms) {
  long g = n / 16;
  if (g < 1) g = 1;
  if (g > num_sms) g = num_sms;
  while ((n + g - 1) / g > kSdsnMaxRows) ++g;   // (only for n > 1024·num_sms)
  return (int)g;
}

template <typename T, int VPL>
static cudaError_t launch_t(const SdsnParams& p, cudaStream_t st, int grid, int cg) {
  auto fn = sdsn_kernel<T, VPL>;
  const int RG = kSdsnWarps / cg;
  const long rows_max = (p.n + grid - 1) / grid + 1;
  const size_t dsm = ((sizeof(double) * rows_max * cg + 15) & ~15ul) + (RG > 1 ? (size_t)RG * p.ld * sizeof(T) : 0);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
  if (e != cudaSuccess) return e;
  SdsnParams pp = p;
  int cgv = cg;
  void* args[] = {&pp, &cgv};
  return cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(kSdsnThreads), args, dsm, st);
}

cudaError_t launch_sdsn(const SdsnParams& p, bool f64, cudaStream_t st, int num_sms, int* grid_out) {
  int vpl, cg;
  if (!plan(p.n, f64, &vpl, &cg)) return cudaErrorInvalidValue;
  const int grid = sdsn_grid_for(p.n, num_sms);
  if (grid_out) *grid_out = grid;
  cudaError_t e = cudaMemsetAsync(p.bar, 0, 2 * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  if (f64) {
    switch (vpl) {
      case 1: return launch_t<double, 1>(p, st, grid, cg);
      case 2: return launch_t<double, 2>(p, st, grid, cg);
      case 4: return launch_t<double, 4>(p, st, grid, cg);
      default: return launch_t<double, 8>(p, st, grid, cg);
    }
  }
  switch (vpl) {
    case 1: return launch_t<float, 1>(p, st, grid, cg);
    case 2: return launch_t<float, 2>(p, st, grid, cg);
    case 4: return launch_t<float, 4>(p, st, grid, cg);
    default: return launch_t<float, 8>(p, st, grid, cg);
  }
}

}  // namespace fram
