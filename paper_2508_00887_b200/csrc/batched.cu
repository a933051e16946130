// batched.cu — K8: `batch` independent FRAM solves (Alg. 1) of size n ≤ 64 in
// ONE launch, one CTA per instance with the whole state in shared memory (the paper
// has no batched mode).  Per instance, inside the CTA:
//   K1 precondition (c = max(A,Ã,K); A/√c, Ã/√c, K/c), the outer loop of
//   GEMM1 U = N·Ã' (transposed, operand-rounded), GEMM2 G = A'·U + λK' (mma.sync m16n8k16 for
//   BF16/FP16 operands with FP32 accumulation; FP32-accumulated FMA on TF32-rounded operands; FP64
//   FMA in FP64 mode), SDSN passes (Alg. 2) with warp-shuffle row sums and fixed-order column
//   sums, the FP64 update and δ, and finally the R17 Hungarian on one warp.
// No grid-wide synchronisation and no inter-CTA traffic: instances are independent, so the
// result of an instance does not depend on the batch it is launched in (bit-identical splits).
#include <math_constants.h>
#include <vector>
#include "batched.h"
#include "common.cuh"
#include "internal.h"

namespace fram {
namespace {

constexpr int NP = 64;            // padded instance size
constexpr int BT = 256;           // threads per CTA
constexpr int BW = BT / 32;

template <int OP> struct BC;
template <> struct BC<0> { using OT = double; using T = double; static constexpr int LDO = 65; };
template <> struct BC<1> { using OT = float; using T = float; static constexpr int LDO = 65; };
template <> struct BC<2> { using OT = __nv_bfloat16; using T = float; static constexpr int LDO = 72; };
template <> struct BC<3> { using OT = __half; using T = float; static constexpr int LDO = 72; };
constexpr int LDY = 68;

template <int OP> __device__ __forceinline__ typename BC<OP>::OT rnd(double x);
template <> __device__ __forceinline__ double rnd<0>(double x) { return x; }
template <> __device__ __forceinline__ float rnd<1>(double x) { return tf32_rne(__double2float_rn(x)); }
template <> __device__ __forceinline__ __nv_bfloat16 rnd<2>(double x) { return __double2bfloat16(x); }
template <> __device__ __forceinline__ __half rnd<3>(double x) { return __double2half(x); }
template <int OP> __device__ __forceinline__ typename BC<OP>::OT rndf(typename BC<OP>::T x);
template <> __device__ __forceinline__ double rndf<0>(double x) { return x; }
template <> __device__ __forceinline__ float rndf<1>(float x) { return tf32_rne(x); }
template <> __device__ __forceinline__ __nv_bfloat16 rndf<2>(float x) { return __float2bfloat16_rn(x); }
template <> __device__ __forceinline__ __half rndf<3>(float x) { return __float2half_rn(x); }

__device__ __forceinline__ double ld_in(const void* p, int dt, long idx) {
  if (dt == 0) return reinterpret_cast<const double*>(p)[idx];
  if (dt == 1) return (double)reinterpret_cast<const float*>(p)[idx];
  return (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[idx]);
}

template <int OP>
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  if constexpr (OP == 2) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  } else {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
}

// D = Aop · Bopᵀ over the padded 64×64 tile; epi(row, col, value) for row, col < n.
template <int OP, typename Epi>
__device__ __forceinline__ void bgemm(const typename BC<OP>::OT* A, const typename BC<OP>::OT* B, int n, Epi epi) {
  constexpr int LDO = BC<OP>::LDO;
  const int tid = threadIdx.x;
  if constexpr (OP >= 2) {
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int mt = warp & 3, ntb = (warp >> 2) * 4;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    const int kmax = (n + 15) / 16;
    for (int kk = 0; kk < kmax; ++kk) {
      const int k0 = kk * 16;
      const typename BC<OP>::OT* ar = A + (16 * mt + g) * LDO + k0 + 2 * t;
      const uint32_t a0 = *reinterpret_cast<const uint32_t*>(ar);
      const uint32_t a1 = *reinterpret_cast<const uint32_t*>(ar + 8 * LDO);
      const uint32_t a2 = *reinterpret_cast<const uint32_t*>(ar + 8);
      const uint32_t a3 = *reinterpret_cast<const uint32_t*>(ar + 8 * LDO + 8);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const typename BC<OP>::OT* br = B + (8 * (ntb + nt) + g) * LDO + k0 + 2 * t;
        const uint32_t b0 = *reinterpret_cast<const uint32_t*>(br);
        const uint32_t b1 = *reinterpret_cast<const uint32_t*>(br + 8);
        mma16816<OP>(acc[nt], a0, a1, a2, a3, b0, b1);
      }
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int r = 16 * mt + g, c = 8 * (ntb + nt) + 2 * t;
      if (r < n && c < n) epi(r, c, acc[nt][0]);
      if (r < n && c + 1 < n) epi(r, c + 1, acc[nt][1]);
      if (r + 8 < n && c < n) epi(r + 8, c, acc[nt][2]);
      if (r + 8 < n && c + 1 < n) epi(r + 8, c + 1, acc[nt][3]);
    }
  } else {
    using T = typename BC<OP>::T;
    const int ty = tid >> 4, tx = tid & 15;
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = (T)0;
    for (int k = 0; k < n; ++k) {
      T av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = (T)A[(4 * ty + i) * LDO + k];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = (T)B[(4 * tx + j) * LDO + k];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = 4 * ty + i, c = 4 * tx + j;
        if (r < n && c < n) epi(r, c, acc[i][j]);
      }
  }
}

struct BatchParams {
  const void *A, *B, *K;
  const double* X0;
  int dt;
  int n;
  long batch;
  double lambda, theta, alpha, gamma_th, delta_th;
  int max_outer, sdsn_max, sdsn_fixed, flags;
  const int32_t* replay;       // device, nullable
  int replay_len;
  double* X_out;
  int32_t* perm_out;
  int32_t* inst;               // [batch][4]: outer, passes, converged, status
};

template <int OP>
__global__ void __launch_bounds__(BT) fram_batched_kernel(BatchParams P) {
  using OT = typename BC<OP>::OT;
  using T = typename BC<OP>::T;
  constexpr int LDO = BC<OP>::LDO;
  extern __shared__ __align__(16) unsigned char sm[];
  // ---- carve shared memory ----
  size_t off = 0;
  auto carve = [&](size_t bytes) { unsigned char* p = sm + off; off += (bytes + 15) & ~size_t(15); return p; };
  OT* sA = reinterpret_cast<OT*>(carve(sizeof(OT) * NP * LDO));
  OT* sBT = reinterpret_cast<OT*>(carve(sizeof(OT) * NP * LDO));
  OT* sUT = reinterpret_cast<OT*>(carve(sizeof(OT) * NP * LDO));
  OT* sNq = (OP == 0) ? nullptr : reinterpret_cast<OT*>(carve(sizeof(OT) * NP * LDO));
  // TF32 (OP 1): the FP64 iterate N lives in registers — thread tid owns elements e = tid + k·BT, the
  // update's own partition — which frees 33 KB and lets 2 CTAs share an SM instead of 1 (BF16 / FP16
  // already fit 2, and 3 would not fit their registers; FP64 uses sN as the GEMM operand).  The LAP
  // and X_out then read N from the sA|sBT region, written once after the outer loop.
  constexpr bool NREG = (OP == 1);
  constexpr int NK = NP * NP / BT;
  double* sN = NREG ? nullptr : reinterpret_cast<double*>(carve(sizeof(double) * NP * LDO));
  double nreg[NK];
  T* sK = reinterpret_cast<T*>(carve(sizeof(T) * NP * LDY));
  T* sY = reinterpret_cast<T*>(carve(sizeof(T) * NP * LDY));
  double* sr = reinterpret_cast<double*>(carve(sizeof(double) * NP));
  T* sa = reinterpret_cast<T*>(carve(sizeof(T) * NP));
  T* sb = reinterpret_cast<T*>(carve(sizeof(T) * NP));
  T* cpart = reinterpret_cast<T*>(carve(sizeof(T) * BW * NP));
  double* red = reinterpret_cast<double*>(carve(sizeof(double) * BW * 4));
  double* lu = reinterpret_cast<double*>(carve(sizeof(double) * (NP + 1) * 3));
  int* lp = reinterpret_cast<int*>(carve(sizeof(int) * (NP + 1) * 2));
  unsigned char* lused = carve(NP + 1);
  __shared__ double s_scal[4];
  __shared__ unsigned long long s_bad[3];

  const long inst = blockIdx.x;
  const int n = P.n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long nn = (long)n * n;
  const double dn = (double)n;
  // x/n and x/n² as RN(x/d) from a precomputed correctly rounded reciprocal plus one FMA correction
  // (Markstein; exactly the IEEE quotient, see tools/div_probe.cu) — no FP64 division per pass
  const double rdn = __drcp_rn(dn), rdnn = __drcp_rn(dn * dn);
  auto div_n = [&](double x, double d, double r) {
    const double q = x * r;
    return fma(r, fma(-q, d, x), q);
  };
  for (size_t i = tid * 16; i < off; i += BT * 16) *reinterpret_cast<uint4*>(sm + i) = make_uint4(0, 0, 0, 0);
  if (tid < 3) s_bad[tid] = 0;
  __syncthreads();

  // ---- K1: validation + c = max(A, Ã, K) ----
  const void* Ai = reinterpret_cast<const unsigned char*>(P.A) + inst * nn * (P.dt == 0 ? 8 : P.dt == 1 ? 4 : 2);
  const void* Bi = reinterpret_cast<const unsigned char*>(P.B) + inst * nn * (P.dt == 0 ? 8 : P.dt == 1 ? 4 : 2);
  const void* Ki = P.K ? reinterpret_cast<const unsigned char*>(P.K) + inst * nn * (P.dt == 0 ? 8 : P.dt == 1 ? 4 : 2)
                       : nullptr;
  double mx = 0.0;
  unsigned long long bad = 0, asym = 0;
  for (long e = tid; e < nn; e += BT) {
    const long i = e / n, j = e % n;
    const double a = ld_in(Ai, P.dt, e), b = ld_in(Bi, P.dt, e), k = Ki ? ld_in(Ki, P.dt, e) : 0.0;
    if (!isfinite(a) || !isfinite(b) || !isfinite(k) || a < 0 || b < 0 || k < 0) ++bad;
    else mx = fmax(mx, fmax(a, fmax(b, k)));
    if (P.flags & FRAM_FLAG_CHECK_SYMMETRY) {
      if (ld_in(Ai, P.dt, j * n + i) != a || ld_in(Bi, P.dt, j * n + i) != b) ++asym;
    }
  }
  mx = warp_max_d(mx);
  if (lane == 0) red[warp] = mx;
  if (bad) atomicAdd(&s_bad[0], bad);
  if (asym) atomicAdd(&s_bad[1], asym);
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int w = 0; w < BW; ++w) m = fmax(m, red[w]);
    s_scal[0] = m;
  }
  __syncthreads();
  const double c = s_scal[0];
  if (s_bad[0] || s_bad[1] || !(c > 0)) {
    if (tid == 0) {
      int32_t* st = P.inst + inst * 4;
      st[0] = 0; st[1] = 0; st[2] = 0; st[3] = FRAM_ERR_DATA;
    }
    return;
  }
  const double sqc = sqrt(c);
  for (long e = tid; e < nn; e += BT) {
    const int i = (int)(e / n), j = (int)(e % n);
    sA[i * LDO + j] = rnd<OP>(ld_in(Ai, P.dt, e) / sqc);
    sBT[j * LDO + i] = rnd<OP>(ld_in(Bi, P.dt, e) / sqc);           // Ã'ᵀ
    if (Ki) sK[i * LDY + j] = (T)(ld_in(Ki, P.dt, e) / c);
    if constexpr (!NREG) {
      const double x0 = P.X0 ? P.X0[inst * nn + e] : 1.0 / dn;
      sN[i * LDO + j] = x0;
      if constexpr (OP != 0) sNq[i * LDO + j] = rnd<OP>(x0);
    }
  }
  if constexpr (NREG) {
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      const long e = tid + (long)k * BT;
      nreg[k] = 0.0;
      if (e < nn) {
        const double x0 = P.X0 ? P.X0[inst * nn + e] : 1.0 / dn;
        nreg[k] = x0;
        sNq[(e / n) * LDO + (e % n)] = rnd<OP>(x0);
      }
    }
  }
  __syncthreads();

  const int T_outer = P.replay ? P.replay_len : P.max_outer;
  int t = 0, total = 0;
  bool converged = false;
  const bool scale = (P.flags & FRAM_FLAG_NO_THETA_SCALE) == 0;
  for (t = 1; t <= T_outer; ++t) {
    // ---- Alg.1 step 5: G = A'·(N·Ã') + λK' ----
    const OT* Nop = (OP == 0) ? reinterpret_cast<const OT*>(sN) : sNq;
    bgemm<OP>(Nop, sBT, n, [&](int r, int cc, T v) { sUT[cc * LDO + r] = rndf<OP>(v); });
    __syncthreads();
    bgemm<OP>(sA, sUT, n, [&](int r, int cc, T v) {
      sY[r * LDY + cc] = v + (Ki ? (T)P.lambda * sK[r * LDY + cc] : (T)0);
    });
    __syncthreads();

    // ---- Alg.2 SDSN on sY ----
    double m = 0.0;
    for (long e = tid; e < nn; e += BT) m = fmax(m, (double)sY[(e / n) * LDY + (e % n)]);
    m = warp_max_d(m);
    if (lane == 0) red[warp] = m;
    __syncthreads();
    if (tid == 0) {
      double mm = 0.0;
      for (int w = 0; w < BW; ++w) mm = fmax(mm, red[w]);
      s_scal[1] = mm;
    }
    __syncthreads();
    m = s_scal[1];
    int passes = 0;
    const int fixed = P.replay ? P.replay[t - 1] : P.sdsn_fixed;
    if (scale && m == 0.0) {
      for (long e = tid; e < nn; e += BT) sY[(e / n) * LDY + (e % n)] = (T)(1.0 / dn);
      __syncthreads();
    } else {
      const double s = scale ? (P.theta / 2.0) / m : 1.0;
      // Y0 = s·G and its sums; warp w owns rows w, w+8, ...; lane owns columns lane, lane+32
      auto sums = [&]() {
        T cp0 = (T)0, cp1 = (T)0;
        for (int i = warp; i < n; i += BW) {
          const T y0 = lane < n ? sY[i * LDY + lane] : (T)0;
          const T y1 = lane + 32 < n ? sY[i * LDY + lane + 32] : (T)0;
          cp0 += y0;
          cp1 += y1;
          T rs = y0 + y1;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
          if (lane == 0) sr[i] = (double)rs;
        }
        cpart[warp * NP + lane] = cp0;
        cpart[warp * NP + lane + 32] = cp1;
      };
      // after a sync: c_j (fixed order over warps) → b_j, and (warp 2) S (fixed order) → a_i for the
      // next pass, so a pass needs one barrier after its sweep and one after this step
      auto finish = [&]() {
        if (tid < NP) {
          double cs = 0.0;
#pragma unroll
          for (int w = 0; w < BW; ++w) cs += (double)cpart[w * NP + tid];
          sb[tid] = (T)(-div_n(cs, dn, rdn));
        } else if (warp == 2) {
          double S = (lane < n ? sr[lane] : 0.0) + (lane + 32 < n ? sr[lane + 32] : 0.0);
          S = warp_sum_d(S);
          if (lane == 0) s_scal[2] = S;
          const double ab = rdn + div_n(S, dn * dn, rdnn);
          sa[lane] = (T)(ab - div_n(sr[lane], dn, rdn));
          sa[lane + 32] = (T)(ab - div_n(sr[lane + 32], dn, rdn));
        }
      };
      if (scale)
        for (long e = tid; e < nn; e += BT) {
          T& y = sY[(e / n) * LDY + (e % n)];
          y = (T)(s * (double)y);
        }
      __syncthreads();
      sums();
      __syncthreads();
      finish();
      __syncthreads();
      for (int j = 0;; ++j) {
        const double S = s_scal[2];
        const double gam = div_n(S, dn, rdn) - 1.0;
        const bool last = fixed > 0 ? (j + 1 >= fixed) : ((j >= 1 && gam <= P.gamma_th) || j + 1 >= P.sdsn_max);
        T cp0 = (T)0, cp1 = (T)0;
        const T b0 = sb[lane], b1 = sb[lane + 32];
        // the warp's (≤ NP/BW = 8) rows: per-lane row partials kept in registers and reduced together
        // by one transpose-reduce (xor 16, 8, 4 halve the rows a lane carries, xor 2, 1 finish)
        T rv[NP / BW];
#pragma unroll
        for (int k = 0; k < NP / BW; ++k) {
          const int i = warp + k * BW;
          T y0 = (T)0, y1 = (T)0;
          if (i < n) {
            const T a = sa[i];
            if (lane < n) { y0 = (sY[i * LDY + lane] + a) + b0; y0 = y0 > (T)0 ? y0 : (T)0; sY[i * LDY + lane] = y0; }
            if (lane + 32 < n) {
              y1 = (sY[i * LDY + lane + 32] + a) + b1;
              y1 = y1 > (T)0 ? y1 : (T)0;
              sY[i * LDY + lane + 32] = y1;
            }
          }
          cp0 += y0;
          cp1 += y1;
          rv[k] = y0 + y1;
        }
        {
          static_assert(NP / BW == 8, "transpose-reduce of 8 rows");
          const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
          T w4[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) w4[q] = (b4 ? rv[q + 4] : rv[q]) + __shfl_xor_sync(0xffffffffu, b4 ? rv[q] : rv[q + 4], 16);
          T w2[2];
#pragma unroll
          for (int q = 0; q < 2; ++q) w2[q] = (b3 ? w4[q + 2] : w4[q]) + __shfl_xor_sync(0xffffffffu, b3 ? w4[q] : w4[q + 2], 8);
          T z = (b2 ? w2[1] : w2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? w2[0] : w2[1], 4);
          z += __shfl_xor_sync(0xffffffffu, z, 2);
          z += __shfl_xor_sync(0xffffffffu, z, 1);
          const int i = warp + (lane >> 2) * BW;           // lane 4k holds row k of this warp
          if ((lane & 3) == 0 && i < n) sr[i] = (double)z;
        }
        cpart[warp * NP + lane] = cp0;
        cpart[warp * NP + lane + 32] = cp1;
        passes = j + 1;
        __syncthreads();
        if (last) break;
        finish();
        __syncthreads();
      }
    }
    total += passes;
    // ---- Alg.1 steps 7-8: update and δ ----
    double dd = 0.0, nv2 = 0.0;
    if constexpr (NREG) {
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        const long e = tid + (long)k * BT;
        if (e < nn) {
          const int i = (int)(e / n), j = (int)(e % n);
          const double old = nreg[k];
          const double nv = __dadd_rn(__dmul_rn(1.0 - P.alpha, old), __dmul_rn(P.alpha, (double)sY[i * LDY + j]));
          const double df = __dsub_rn(nv, old);
          dd = __fma_rn(df, df, dd);
          nv2 = __fma_rn(nv, nv, nv2);
          nreg[k] = nv;
          sNq[i * LDO + j] = rnd<OP>(nv);
        }
      }
    } else {
      for (long e = tid; e < nn; e += BT) {
        const int i = (int)(e / n), j = (int)(e % n);
        const double old = sN[i * LDO + j];
        const double nv = __dadd_rn(__dmul_rn(1.0 - P.alpha, old), __dmul_rn(P.alpha, (double)sY[i * LDY + j]));
        const double df = __dsub_rn(nv, old);
        dd = __fma_rn(df, df, dd);
        nv2 = __fma_rn(nv, nv, nv2);
        sN[i * LDO + j] = nv;
        if constexpr (OP != 0) sNq[i * LDO + j] = rnd<OP>(nv);
      }
    }
    dd = warp_sum_d(dd);
    nv2 = warp_sum_d(nv2);
    if (lane == 0) { red[warp] = dd; red[BW + warp] = nv2; }
    __syncthreads();
    if (tid == 0) {
      double a = 0.0, b = 0.0;
      for (int w = 0; w < BW; ++w) { a += red[w]; b += red[BW + w]; }
      s_scal[3] = sqrt(a) / sqrt(b);
    }
    __syncthreads();
    const double delta = s_scal[3];
    if (delta <= P.delta_th) {
      converged = true;
      if (!P.replay) break;
    } else if (P.replay) {
      converged = false;
    }
  }
  if (t > T_outer) t = T_outer;
  if constexpr (NREG) {                            // N → the sA|sBT region (free now) for the LAP / X_out
    static_assert(!NREG || 2 * ((sizeof(OT) * NP * LDO + 15) / 16 * 16) >= sizeof(double) * NP * LDO, "sN alias");
    __syncthreads();
    sN = reinterpret_cast<double*>(sA);
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      const long e = tid + (long)k * BT;
      if (e < nn) sN[(e / n) * LDO + (e % n)] = nreg[k];
    }
    __syncthreads();
  }

  // ---- Alg.1 step 10: R17 Hungarian on warp 0 ----
  if (warp == 0) {
    double* u = lu;
    double* v = lu + (NP + 1);
    double* minv = lu + 2 * (NP + 1);
    int* p = lp;
    int* way = lp + (NP + 1);
    for (int j = lane; j <= n; j += 32) { u[j] = 0.0; v[j] = 0.0; p[j] = 0; way[j] = 0; }
    __syncwarp();
    for (int i = 1; i <= n; ++i) {
      for (int j = lane; j <= n; j += 32) { minv[j] = CUDART_INF; lused[j] = 0; }
      if (lane == 0) p[0] = i;
      __syncwarp();
      int j0 = 0;
      while (true) {
        if (lane == 0) lused[j0] = 1;
        __syncwarp();
        const int i0 = p[j0];
        const double ui0 = u[i0];
        double best = CUDART_INF;
        int bj = 0x7fffffff;
        for (int j = lane + 1; j <= n; j += 32) {
          if (!lused[j]) {
            const double cur = __dsub_rn(__dsub_rn(-sN[(i0 - 1) * LDO + (j - 1)], ui0), v[j]);
            double mv = minv[j];
            if (cur < mv) { mv = cur; minv[j] = cur; way[j] = j0; }
            if (mv < best) { best = mv; bj = j; }
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, best, o);
          const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
          if (ov < best || (ov == best && oj < bj)) { best = ov; bj = oj; }
        }
        __syncwarp();
        for (int j = lane; j <= n; j += 32) {
          if (lused[j]) { u[p[j]] = __dadd_rn(u[p[j]], best); v[j] = __dsub_rn(v[j], best); }
          else minv[j] = __dsub_rn(minv[j], best);
        }
        __syncwarp();
        j0 = bj;
        if (p[j0] == 0) break;
      }
      if (lane == 0) {
        do { const int j1 = way[j0]; p[j0] = p[j1]; j0 = j1; } while (j0 != 0);
      }
      __syncwarp();
    }
    if (P.perm_out)
      for (int j = lane + 1; j <= n; j += 32) P.perm_out[inst * n + p[j] - 1] = j - 1;
  }
  if (P.X_out)
    for (long e = tid; e < nn; e += BT) P.X_out[inst * nn + e] = sN[(e / n) * LDO + (e % n)];
  if (tid == 0) {
    int32_t* st = P.inst + inst * 4;
    st[0] = t; st[1] = total; st[2] = converged ? 1 : 0; st[3] = converged ? FRAM_OK : FRAM_NOT_CONVERGED;
  }
}

template <int OP>
size_t smem_bytes() {
  using OT = typename BC<OP>::OT;
  using T = typename BC<OP>::T;
  constexpr int LDO = BC<OP>::LDO;
  auto r = [](size_t b) { return (b + 15) & ~size_t(15); };
  size_t s = 3 * r(sizeof(OT) * NP * LDO);
  if (OP != 0) s += r(sizeof(OT) * NP * LDO);
  if (OP != 1) s += r(sizeof(double) * NP * LDO);   // OP 1 keeps N in registers (fram_batched_kernel)
  s += 2 * r(sizeof(T) * NP * LDY) + r(sizeof(double) * NP) +
       2 * r(sizeof(T) * NP) + r(sizeof(T) * BW * NP) + r(sizeof(double) * BW * 4) + r(sizeof(double) * (NP + 1) * 3) +
       r(sizeof(int) * (NP + 1) * 2) + r(NP + 1);
  return s;
}

template <int OP>
cudaError_t launch_b(const BatchParams& p, cudaStream_t st) {
  const size_t sm = smem_bytes<OP>();
  auto fn = fram_batched_kernel<OP>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  // the whole unified L1 as shared memory, so the 2 CTAs per SM the kernel is sized for always fit (left
  // to the driver, the carveout — and C3 TF32 throughput — varied between runs: 107K vs 137K inst/s)
  e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  fn<<<(unsigned)p.batch, BT, sm, st>>>(p);
  return cudaGetLastError();
}

bool is_dev(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

cudaError_t grow(void** p, size_t* have, size_t need) {
  if (need <= *have && *p) return cudaSuccess;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *have = 0;
  cudaError_t e = cudaMalloc(p, need);
  if (e == cudaSuccess) *have = need;
  return e;
}

}  // namespace

void batched_release(BatchedWs& ws) {
  if (ws.inst_stats) cudaFree(ws.inst_stats);
  if (ws.staging) cudaFree(ws.staging);
  if (ws.out_staging) cudaFree(ws.out_staging);
  ws = BatchedWs{};
}

fram_status batched_solve(BatchedWs& ws, long n, double lambda, const fram_schedule& sched, long batch, int dt,
                          const void* A, const void* B, const void* K, const double* X0, int prec, cudaStream_t st,
                          double* X_out, int32_t* perm_out, int32_t* status_out, fram_stats* stats, int num_sms,
                          std::string* err) {
  (void)num_sms;
  if (n > NP) { *err = "fram_solve_batched supports n <= 64"; return FRAM_ERR_USAGE; }
  if (batch == 0) return FRAM_OK;
  auto cf = [&](cudaError_t e, const char* what) {
    cudaGetLastError();
    *err = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? FRAM_ERR_OOM : FRAM_ERR_CUDA;
  };
  const size_t es = dt == 0 ? 8 : (dt == 1 ? 4 : 2);
  const size_t mat = (size_t)batch * n * n;
  // stage host inputs into one device buffer
  size_t need = 0;
  const bool hA = !is_dev(A), hB = !is_dev(B), hK = K && !is_dev(K), hX = X0 && !is_dev(X0);
  need += (hA ? mat * es : 0) + (hB ? mat * es : 0) + (hK ? mat * es : 0) + (hX ? mat * 8 : 0);
  cudaError_t e;
  if (need) {
    if ((e = grow(&ws.staging, &ws.staging_bytes, need)) != cudaSuccess) return cf(e, "staging alloc");
  }
  unsigned char* sp = reinterpret_cast<unsigned char*>(ws.staging);
  auto stage = [&](const void* src, bool host, size_t bytes) -> const void* {
    if (!host) return src;
    cudaMemcpyAsync(sp, src, bytes, cudaMemcpyHostToDevice, st);
    const void* r = sp;
    sp += bytes;
    return r;
  };
  const void* dA = stage(A, hA, mat * es);
  const void* dB = stage(B, hB, mat * es);
  const void* dK = K ? stage(K, hK, mat * es) : nullptr;
  const double* dX0 = X0 ? reinterpret_cast<const double*>(stage(X0, hX, mat * 8)) : nullptr;
  const bool hXo = X_out && !is_dev(X_out), hP = perm_out && !is_dev(perm_out);
  size_t oneed = (hXo ? mat * 8 : 0) + (hP ? (size_t)batch * n * 4 : 0) + (size_t)batch * 16 + 1024;
  if ((e = grow(&ws.out_staging, &ws.out_bytes, oneed)) != cudaSuccess) return cf(e, "out alloc");
  unsigned char* op = reinterpret_cast<unsigned char*>(ws.out_staging);
  int32_t* dinst = reinterpret_cast<int32_t*>(op);
  op += ((size_t)batch * 16 + 255) & ~size_t(255);
  double* dXo = hXo ? reinterpret_cast<double*>(op) : X_out;
  if (hXo) op += mat * 8;
  int32_t* dP = hP ? reinterpret_cast<int32_t*>(op) : perm_out;
  // replay schedule to device (small)
  int32_t* drep = nullptr;
  std::vector<int32_t> rep(sched.replay_passes, sched.replay_passes + sched.replay_len);
  if (!rep.empty()) {
    if ((e = grow(&ws.inst_stats, &ws.inst_bytes, rep.size() * 4)) != cudaSuccess) return cf(e, "replay alloc");
    drep = reinterpret_cast<int32_t*>(ws.inst_stats);
    cudaMemcpyAsync(drep, rep.data(), rep.size() * 4, cudaMemcpyHostToDevice, st);
  }
  BatchParams p{};
  p.A = dA; p.B = dB; p.K = dK; p.X0 = dX0; p.dt = dt; p.n = (int)n; p.batch = batch;
  p.lambda = lambda; p.theta = sched.theta; p.alpha = sched.alpha; p.gamma_th = sched.gamma_th;
  p.delta_th = sched.delta_th; p.max_outer = sched.max_outer; p.sdsn_max = sched.sdsn_max;
  p.sdsn_fixed = sched.sdsn_fixed; p.flags = sched.flags; p.replay = drep; p.replay_len = (int)rep.size();
  p.X_out = dXo; p.perm_out = dP; p.inst = dinst;
  switch (prec) {
    case 0: e = launch_b<0>(p, st); break;
    case 1: e = launch_b<1>(p, st); break;
    case 2: e = launch_b<2>(p, st); break;
    default: e = launch_b<3>(p, st); break;
  }
  if (e != cudaSuccess) return cf(e, "batched launch");
  if (hXo) cudaMemcpyAsync(X_out, dXo, mat * 8, cudaMemcpyDeviceToHost, st);
  if (hP) cudaMemcpyAsync(perm_out, dP, (size_t)batch * n * 4, cudaMemcpyDeviceToHost, st);
  std::vector<int32_t> hinst((size_t)batch * 4);
  cudaMemcpyAsync(hinst.data(), dinst, (size_t)batch * 16, cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cf(e, "batched sync");
  fram_status worst = FRAM_OK;
  int maxo = 0, allc = 1;
  int64_t tot = 0;
  std::vector<int32_t> sts((size_t)batch);
  for (long b = 0; b < batch; ++b) {
    const int32_t s = hinst[b * 4 + 3];
    sts[b] = s;
    if (s == FRAM_ERR_DATA) worst = FRAM_ERR_DATA;
    else if (s == FRAM_NOT_CONVERGED && worst == FRAM_OK) worst = FRAM_NOT_CONVERGED;
    maxo = std::max(maxo, hinst[b * 4]);
    tot += hinst[b * 4 + 1];
    allc &= hinst[b * 4 + 2];
  }
  if (status_out) {
    if (is_dev(status_out)) cudaMemcpy(status_out, sts.data(), (size_t)batch * 4, cudaMemcpyHostToDevice);
    else memcpy(status_out, sts.data(), (size_t)batch * 4);
  }
  if (stats) {
    stats->outer_iters = maxo;
    stats->converged = allc;
    stats->total_passes = tot;
    stats->kernel_launches = 1;
  }
  if (worst == FRAM_ERR_DATA) *err = "one or more instances have invalid data (status_out)";
  else if (worst == FRAM_NOT_CONVERGED) *err = "one or more instances did not converge (status_out)";
  return worst;
}

}  // namespace fram
