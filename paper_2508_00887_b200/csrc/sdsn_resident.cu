// sdsn_resident.cu — K4r: SDSN (Scaling Doubly Stochastic Normalization), Alg. 2 of arXiv
// 2508.00887, FP32, with the iterate Y held ON-CHIP for the whole call.
//
// Same arithmetic and stopping rule as the streaming kernel (sdsn.cu, readings R5, R9-R13):
//   γ_j = S_j/n − 1;  a_i = (1/n + S_j/n²) − r_i/n;  b_j = −c_j/n  (FP64, rounded to FP32)
//   Y_{j+1} = max(0, (Y_j + a_i) + b_j)   with r, c, S of Y_{j+1} fused into the same sweep.
//
// Why on-chip: at n = 4096 the FP32 iterate is 64 MiB; read + written once per pass it is bound
// by L2/HBM bandwidth (8n² B per pass, ~24 us).  The 148 SMs together hold 148 × (256 KB TMEM +
// 227 KB shared memory) ≈ 71 MB, so each CTA keeps its row block resident: the first RT = 512/CPT
// rows in TMEM (tcgen05.ld/st, 32x32b shape: TMEM lane = column-owner thread), the rest in
// shared memory.  Per pass only the column-sum partials (4·n B per CTA) and the b vector cross
// L2, and the pass becomes ALU-bound (5 FP32 ops per element) plus two grid barriers.
//
// Work split.  CTA b owns rows [b·n/G, (b+1)·n/G).  Thread t = 32·(warp%4) + lane owns columns
// [t·CPT, (t+1)·CPT) of every row (128 owners cover 128·CPT ≥ n columns; columns ≥ n are padding
// held at 0 by b_pad = −∞).  Warps w and w+4 (row groups g = w/4) share a TMEM lane quarter and
// split the rows (r ≡ g mod 2).  Row sums: FP32 per thread → warp shuffle → 4 quarter partials
// combined in FP64 in a fixed order.  Column sums: per-thread FP32 register partials over its
// rows → the two row groups combined in shared memory → colpart[b] → grid barrier → CTA b reduces
// slot slice b over all CTAs in CTA order (FP64, deterministic, no float atomics: S:375) and
// writes b = −c/n → grid barrier → every CTA reads b.  S = Σ of per-CTA FP64 row-sum partials,
// summed identically by every CTA, so every CTA takes the same stop decision (R5).
//
// Vectors that cross CTAs (colpart, bvec) use the "slot" layout: slot (c·128 + t)·4 + e holds
// column t·CPT + 4c + e, so every access by the owner threads is a coalesced float4.
// Grid barriers: one monotonic arrival counter (red.release.gpu), one acquire poller per CTA.
#include <math_constants.h>
#include <stdlib.h>
#include <type_traits>
#include "common.cuh"
#include "internal.h"
#include "tmem_ldst.cuh"

namespace fram {
namespace {

constexpr int kResThreads = 256;             // 8 warps = 4 TMEM lane quarters × 2 row groups
constexpr int kResSmemMax = 232448 - 2304;   // 227 KB opt-in minus static shared memory (2128 B)
constexpr int kResMinSmem = 120 * 1024;      // forces one CTA per SM (TMEM: 512 columns per CTA)

template <int CPT> struct RC {
  static constexpr int V = CPT / 4;          // float4 chunks per owner thread per row
  static constexpr int NS = 128 * CPT;       // slots = padded columns
  static constexpr int RT = 512 / CPT;       // rows held in TMEM
};

constexpr int kResMaxRows = 32;             // rows per CTA (the grid is sized so R ≤ 32)
constexpr int kResKMax = 5;                  // G ≤ 32·kResKMax CTAs (148 SMs)

// dynamic shared memory: SMEM-resident rows, column staging, per-thread row partials, s_r, s_a
size_t res_smem_bytes(int cpt, int rs, int R) {
  const size_t ns = 128 * (size_t)cpt;
  return (size_t)rs * ns * 4 + ns * 4 + (size_t)R * 128 * 4 + (size_t)R * 8 + (size_t)R * 4 + 64;
}

// two FP32 adds in one instruction (FADD2, sm_100): d = (a.x + b.x, a.y + b.y), each RN
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n add.rn.f32x2 rd, ra, rb;\n"
      " mov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

template <int CPT>
__global__ void __launch_bounds__(kResThreads, 1) sdsn_res_kernel(ResParams P) {
  using C = RC<CPT>;
  constexpr int V = C::V, NS = C::NS, RT = C::RT;
  extern __shared__ __align__(16) unsigned char dsm[];
  const int RS = P.rs;
  const int Rmax = P.rmax;
  float4* s_rows = reinterpret_cast<float4*>(dsm);                    // [RS][V·128] slot layout
  float4* s_col = s_rows + (size_t)RS * V * 128;                      // [V·128] column staging
  float* s_rowthr = reinterpret_cast<float*>(s_col + V * 128);        // [Rmax][128] per-thread row partials
  double* s_r = reinterpret_cast<double*>(s_rowthr + Rmax * 128);    // [Rmax] row sums (FP64)
  float* s_a = reinterpret_cast<float*>(s_r + Rmax);                 // [Rmax] a_i (FP32)
  __shared__ uint32_t s_tmem;
  __shared__ double s_red[kResThreads / 32];
  __shared__ double s_S;
  __shared__ double s_red2[kResThreads / 32][32];

  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = warp & 3, g = warp >> 2;
  const int t = q * 32 + lane;
  const long n = P.n, ld = P.ld;
  const long r0 = (long)b * n / G, r1 = (long)(b + 1) * n / G;
  const int R = (int)(r1 - r0);
  const double dn = (double)n, nn = dn * dn;
  unsigned epoch = 0;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem + ((uint32_t)(q * 32) << 16);          // this warp's lane quarter

  auto load_row = [&](int r, float (&x)[CPT]) {
    if (r < RT) {
      uint32_t v[CPT];
      tmem_ld<CPT>(tmem + (uint32_t)(r * CPT), v);
      tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < CPT; ++k) x[k] = __uint_as_float(v[k]);
    } else {
      const float4* row = s_rows + (size_t)(r - RT) * (V * 128);
#pragma unroll
      for (int c = 0; c < V; ++c) {
        const float4 v = row[c * 128 + t];
        x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
      }
    }
  };
  auto store_row = [&](int r, const float (&x)[CPT]) {
    if (r < RT) {
      uint32_t v[CPT];
#pragma unroll
      for (int k = 0; k < CPT; ++k) v[k] = __float_as_uint(x[k]);
      tmem_st<CPT>(tmem + (uint32_t)(r * CPT), v);
    } else {
      float4* row = s_rows + (size_t)(r - RT) * (V * 128);
#pragma unroll
      for (int c = 0; c < V; ++c) row[c * 128 + t] = make_float4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
    }
  };
  // grid-wide barrier: one monotonic arrival counter (red.release), one acquire poller per CTA
  auto gbar = [&]() {
    ++epoch;
    __syncthreads();
    if (tid == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(P.flags) : "memory");
      const unsigned target = epoch * (unsigned)G;
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(P.flags) : "memory");
      } while (v < target);
    }
    __syncthreads();
  };
  auto dealloc = [&]() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(512));
  };

  // ---------------- phase L: X rows → on-chip, m = max X (Alg.2 step 1) ----------------
  {
    float lmax = 0.f;
    for (int r = g; r < R; r += 2) {
      const float* grow = P.Y + (r0 + r) * ld;
      float x[CPT];
#pragma unroll
      for (int c = 0; c < V; ++c) {
        const long col = (long)t * CPT + 4 * c;
        float4 v;
        if (col + 3 < n) {
          v = __ldcg(reinterpret_cast<const float4*>(grow + col));
        } else {
          v.x = col < n ? grow[col] : 0.f;
          v.y = col + 1 < n ? grow[col + 1] : 0.f;
          v.z = col + 2 < n ? grow[col + 2] : 0.f;
          v.w = col + 3 < n ? grow[col + 3] : 0.f;
        }
        x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
        lmax = fmaxf(lmax, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
      }
      store_row(r, x);
    }
    tmem_wait_st();
    double m = (double)lmax;
    m = warp_max_d(m);
    if (lane == 0) s_red[warp] = m;
    __syncthreads();
    if (tid == 0) {
      double mm = 0.0;
      for (int w = 0; w < kResThreads / 32; ++w) mm = fmax(mm, s_red[w]);
      P.Mpart[b] = mm;
    }
  }
  double sc = 1.0;
  if (P.scale) {
    gbar();
    if (warp == 0) {
      double mv[kResKMax], mm = 0.0;
#pragma unroll
      for (int i = 0; i < kResKMax; ++i) mv[i] = (lane + 32 * i < G) ? __ldcg(P.Mpart + lane + 32 * i) : 0.0;
#pragma unroll
      for (int i = 0; i < kResKMax; ++i) mm = fmax(mm, mv[i]);
      mm = warp_max_d(mm);
      if (lane == 0) s_S = mm;
    }
    __syncthreads();
    const double m = s_S;
    if (m == 0.0) {                                      // R10: all-zero ⇒ 11ᵀ/n, 0 passes
      for (int r = g; r < R; r += 2) {
        float* grow = P.Y + (r0 + r) * ld;
        for (long col = (long)t; col < n; col += 128) grow[col] = (float)(1.0 / dn);
      }
      if (b == 0 && tid == 0) {
        *P.passes_out = 0;
        P.sdsn_out[0] = 0.0; P.sdsn_out[1] = 0.0; P.sdsn_out[2] = 0.0;
      }
      dealloc();
      return;
    }
    sc = (P.theta / 2.0) / m;                            // R11: s = (θ/2)/max X in FP64
    if (b == 0 && tid == 0) P.sdsn_out[1] = m;
    __syncthreads();                                     // s_S is reused below
  }

  // ---------------- one sweep over the CTA's rows ----------------
  // PASS: y ← max(0, (y + a_i) + b_j);  SCALE: y ← fl(s·y).  Accumulates the new row sums
  // (s_r, Spart[b]) and column partials (colpart[b], slot layout).
  // after a sweep: column partials (two row groups combined in shared memory) → colpart[b];
  // row sums (per-thread partials → fixed-order tree) → s_r; Σ r → Spart[b]
  auto sweep_epilogue = [&](const float (&col)[CPT]) {
    tmem_wait_st();
    if (g == 1) {
#pragma unroll
      for (int c = 0; c < V; ++c) s_col[c * 128 + t] = make_float4(col[4 * c], col[4 * c + 1], col[4 * c + 2], col[4 * c + 3]);
    }
    __syncthreads();
    if (g == 0) {
      float4* dst = reinterpret_cast<float4*>(P.colpart + (long)b * NS);
#pragma unroll
      for (int c = 0; c < V; ++c) {
        float4 o = s_col[c * 128 + t];
        o.x += col[4 * c]; o.y += col[4 * c + 1]; o.z += col[4 * c + 2]; o.w += col[4 * c + 3];
        __stcg(dst + c * 128 + t, o);
      }
    }
    // row sums: warp w reduces rows w, w+8, …, up to 4 at a time (independent shuffle chains)
    for (int r = warp; r < R; r += 4 * (kResThreads / 32)) {
      float pr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int rr = r + u * (kResThreads / 32);
        const float* pp = s_rowthr + rr * 128;
        pr[u] = rr < R ? ((pp[lane] + pp[lane + 32]) + (pp[lane + 64] + pp[lane + 96])) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) pr[u] = warp_sum_f(pr[u]);
      if (lane == 0) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (r + u * (kResThreads / 32) < R) s_r[r + u * (kResThreads / 32)] = (double)pr[u];
      }
    }
    __syncthreads();
    if (warp == 0) {
      double s = 0.0;
      for (int i = lane; i < R; i += 32) s += s_r[i];
      s = warp_sum_d(s);
      if (lane == 0) __stcg(P.Spart + b, s);
    }
  };

  // Y0 = fl(s·X) (Alg.2 step 1; skipped when !P.scale) with its sums
  auto sweep_scale = [&]() {
    float col[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) col[k] = 0.f;
    for (int r = g; r < R; r += 2) {
      float x[CPT];
      load_row(r, x);
      float r0s = 0.f, r1s = 0.f;
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const float y = P.scale ? (float)(sc * (double)x[k]) : x[k];
        x[k] = y;
        col[k] += y;
        if (k & 1) r1s += y; else r0s += y;
      }
      if (P.scale) store_row(r, x);
      s_rowthr[r * 128 + t] = r0s + r1s;
    }
    sweep_epilogue(col);
  };

  // one SDSN pass: y ← max(0, (y + a_i) + b_j) (P2∘P1, R9 grouping), two rows at a time with
  // paired FP32 adds (add.rn.f32x2: x+a, +b, column and row accumulation)
  auto pass_rows = [&](float (&x)[CPT], float a, const float (&bv)[CPT], float2 (&col2)[CPT / 2]) -> float {
    float2 rs = make_float2(0.f, 0.f);
    const float2 a2 = make_float2(a, a);
#pragma unroll
    for (int k = 0; k < CPT; k += 2) {
      float2 y = add2(add2(make_float2(x[k], x[k + 1]), a2), make_float2(bv[k], bv[k + 1]));
      y.x = fmaxf(0.0f, y.x);
      y.y = fmaxf(0.0f, y.y);
      x[k] = y.x;
      x[k + 1] = y.y;
      col2[k / 2] = add2(col2[k / 2], y);
      rs = add2(rs, y);
    }
    return rs.x + rs.y;
  };
  auto sweep_pass = [&](const float (&bv)[CPT]) {
    float2 col2[CPT / 2];
#pragma unroll
    for (int k = 0; k < CPT / 2; ++k) col2[k] = make_float2(0.f, 0.f);
    int ra = g;
    for (; ra + 2 < R; ra += 4) {
      const int rb = ra + 2;
      float xa[CPT], xb[CPT];
      if (rb < RT) {                                     // both rows in TMEM: one wait for two loads
        uint32_t va[CPT], vb[CPT];
        tmem_ld<CPT>(tmem + (uint32_t)(ra * CPT), va);
        tmem_ld<CPT>(tmem + (uint32_t)(rb * CPT), vb);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < CPT; ++k) { xa[k] = __uint_as_float(va[k]); xb[k] = __uint_as_float(vb[k]); }
      } else {
        load_row(ra, xa);
        load_row(rb, xb);
      }
      const float sa = pass_rows(xa, s_a[ra], bv, col2);
      const float sb = pass_rows(xb, s_a[rb], bv, col2);
      store_row(ra, xa);
      store_row(rb, xb);
      s_rowthr[ra * 128 + t] = sa;
      s_rowthr[rb * 128 + t] = sb;
    }
    if (ra < R) {
      float xa[CPT];
      load_row(ra, xa);
      s_rowthr[ra * 128 + t] = pass_rows(xa, s_a[ra], bv, col2);
      store_row(ra, xa);
    }
    float col[CPT];
#pragma unroll
    for (int k = 0; k < CPT / 2; ++k) { col[2 * k] = col2[k].x; col[2 * k + 1] = col2[k].y; }
    sweep_epilogue(col);
  };

  // slot slice b: lane ↔ slot (coalesced rows of colpart), warp ↔ source CTA k ≡ warp (mod 8);
  // FP64 accumulation in the fixed order k = warp, warp+8, …, then the 8 warps combined in order.
  auto slice = [&]() {
    const int s0 = (int)((long)b * NS / G), s1 = (int)((long)(b + 1) * NS / G);
    constexpr int WS = kResThreads / 32;
    double sv[kResKMax];                                 // Spart loads issued first (overlap)
    if (warp == 0) {
#pragma unroll
      for (int i = 0; i < kResKMax; ++i) sv[i] = (lane + 32 * i < G) ? __ldcg(P.Spart + lane + 32 * i) : 0.0;
    }
    for (int sb = s0; sb < s1; sb += 32) {
      const int s = sb + lane;
      double acc = 0.0;
      if (s < s1) {
        float v[(32 * kResKMax + WS - 1) / WS];
#pragma unroll
        for (int i = 0; i < (32 * kResKMax + WS - 1) / WS; ++i) {
          const int k = warp + i * WS;
          v[i] = k < G ? __ldcg(P.colpart + (long)k * NS + s) : 0.f;
        }
#pragma unroll
        for (int i = 0; i < (32 * kResKMax + WS - 1) / WS; ++i) acc += (double)v[i];
      }
      s_red2[warp][lane] = acc;
      __syncthreads();
      if (warp == 0 && s < s1) {
        double cs = 0.0;
#pragma unroll
        for (int w = 0; w < WS; ++w) cs += s_red2[w][lane];
        const int f = s >> 2, e = s & 3, c = f >> 7, tt = f & 127;
        const long colj = (long)tt * CPT + 4 * c + e;
        __stcg(P.bvec + s, colj < n ? (float)(-cs / dn) : -CUDART_INF_F);
      }
      __syncthreads();
    }
    if (warp == 0) {
      double sacc = 0.0;
#pragma unroll
      for (int i = 0; i < kResKMax; ++i) sacc += sv[i];
      sacc = warp_sum_d(sacc);
      if (lane == 0) s_S = sacc;
    }
  };

  // ---------------- phase S: Y0 = s·X (on chip) and its sums ----------------
  sweep_scale();
  gbar();
  slice();
  gbar();

  // ---------------- pass loop (device-side stop decision, identical in every CTA) ----------------
  int j = 0;
  double gam = 0.0;
  long long tacc[6] = {0, 0, 0, 0, 0, 0};   // dev timing (P.dbg): bload, sweep, barA, slice, barB
  auto now = [&]() -> long long {
    long long v = 0;
    if (P.dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
  };
  for (;; ++j) {
    long long t0 = now();
    const double S = s_S;
    gam = S / dn - 1.0;                                                 // γ_j
    if (b == 0 && tid == 0 && P.gamma_hist) P.gamma_hist[j] = gam;
    const bool last = P.sdsn_fixed > 0 ? (j + 1 >= P.sdsn_fixed)
                                       : ((j >= 1 && gam <= P.gamma_th) || j + 1 >= P.sdsn_max);
    const double abase = 1.0 / dn + S / nn;
    for (int i = tid; i < R; i += kResThreads) s_a[i] = (float)(abase - s_r[i] / dn);
    float bv[CPT];
#pragma unroll
    for (int c = 0; c < V; ++c) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(P.bvec) + c * 128 + t);
      bv[4 * c] = v.x; bv[4 * c + 1] = v.y; bv[4 * c + 2] = v.z; bv[4 * c + 3] = v.w;
    }
    __syncthreads();
    long long t1 = now();
    sweep_pass(bv);
    __syncthreads();
    long long t2 = now();
    if (last) break;
    gbar();
    long long t3 = now();
    slice();
    __syncthreads();
    long long t4 = now();
    gbar();
    long long t5 = now();
    tacc[0] += t1 - t0; tacc[1] += t2 - t1; tacc[2] += t3 - t2; tacc[3] += t4 - t3; tacc[4] += t5 - t4;
    tacc[5] += 1;
  }
  if (P.dbg && tid == 0) {
    for (int k = 0; k < 6; ++k) P.dbg[b * 8 + k] = tacc[k];
  }

  // ---------------- D = Y_final → global (row-major, ld) ----------------
  for (int r = g; r < R; r += 2) {
    float x[CPT];
    load_row(r, x);
    float* grow = P.Y + (r0 + r) * ld;
#pragma unroll
    for (int c = 0; c < V; ++c) {
      const long col = (long)t * CPT + 4 * c;
      if (col + 3 < n) {
        *reinterpret_cast<float4*>(grow + col) = make_float4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
      } else {
        if (col < n) grow[col] = x[4 * c];
        if (col + 1 < n) grow[col + 1] = x[4 * c + 1];
        if (col + 2 < n) grow[col + 2] = x[4 * c + 2];
      }
    }
  }
  if (b == 0 && tid == 0) {
    *P.passes_out = j + 1;
    P.sdsn_out[0] = gam;
    P.sdsn_out[2] = s_S;
  }
  dealloc();
}

int cpt_for(long n) {
  if (n <= 512) return 4;
  if (n <= 1024) return 8;
  if (n <= 2048) return 16;
  if (n <= 4096) return 32;
  return 0;
}

int rows_target() {
  static int rt = -1;
  if (rt < 0) {
    const char* e = getenv("FRAM_RES_ROWS");
    rt = e ? atoi(e) : 16;
    if (rt < 1) rt = 16;
  }
  return rt;
}

template <int CPT>
cudaError_t launch_res_t(ResParams p, cudaStream_t st, int G) {
  auto fn = sdsn_res_kernel<CPT>;
  const long R = (p.n + G - 1) / G;
  if (R > kResMaxRows || G > 32 * kResKMax) return cudaErrorInvalidValue;
  p.rs = (int)(R > RC<CPT>::RT ? R - RC<CPT>::RT : 0);
  p.rmax = (int)R;
  size_t dsm = res_smem_bytes(CPT, p.rs, (int)R);
  if (dsm > (size_t)kResSmemMax) return cudaErrorInvalidValue;
  if (dsm < (size_t)kResMinSmem) dsm = kResMinSmem;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(p.flags, 0, sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  void* args[] = {&p};
  return cudaLaunchCooperativeKernel((const void*)fn, dim3(G), dim3(kResThreads), args, dsm, st);
}

}  // namespace

int sdsn_res_grid(long n, int num_sms) {
  const int cpt = cpt_for(n);
  if (cpt == 0) return 0;
  long G = (n + rows_target() - 1) / rows_target();
  if (G > num_sms) G = num_sms;
  if (G < 1) G = 1;
  auto R_of = [&](long G_) { return (int)((n + G_ - 1) / G_); };
  auto rs_of = [&](long G_) { const long e = R_of(G_) - 512 / cpt; return (int)(e > 0 ? e : 0); };
  auto fits = [&](long G_) {
    return R_of(G_) <= kResMaxRows && G_ <= 32 * kResKMax &&
           res_smem_bytes(cpt, rs_of(G_), R_of(G_)) <= (size_t)kResSmemMax;
  };
  while (G < num_sms && !fits(G)) ++G;
  if (!fits(G)) return 0;
  return (int)G;
}

long sdsn_res_slots(long n) { return 128L * cpt_for(n); }

cudaError_t launch_sdsn_resident(const ResParams& p, cudaStream_t st, int num_sms) {
  const int G = sdsn_res_grid(p.n, num_sms);
  if (G == 0) return cudaErrorInvalidValue;
  switch (cpt_for(p.n)) {
    case 4: return launch_res_t<4>(p, st, G);
    case 8: return launch_res_t<8>(p, st, G);
    case 16: return launch_res_t<16>(p, st, G);
    case 32: return launch_res_t<32>(p, st, G);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace fram
