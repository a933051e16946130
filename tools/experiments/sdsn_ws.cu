// EXPERIMENT (not built into libfram; measured slower, see DESIGN §10 and profiles/r02/ab_k4w_ws.log):
// 9.9 µs/pass at n = 4096 against 6.36 for K4r.  To try it, copy it into csrc/, declare sdsn_ws_grid /
// launch_sdsn_ws in internal.h and dispatch to it from launch_sdsn_resident.
//
// sdsn_ws.cu — K4w: the on-chip FP32 SDSN (Alg. 2 of arXiv 2508.00887) with
// warp-specialised exchange, for 2048 < n ≤ 4096 (C4).  Same arithmetic, stopping rule and on-chip
// residency as K4r (sdsn_resident.cu; readings R5, R9-R13):
//   γ_j = S_j/n − 1;  a_i = (1/n + S_j/n²) − r_i/n;  b_j = −c_j/n  (FP64, rounded to FP32)
//   Y_{j+1} = max(0, (Y_j + a_i) + b_j)   with r, c, S of Y_{j+1} fused into the same sweep.
//
// Why another kernel: in K4r every pass is sweep → column all-reduce (two L2 hops: partials → slot
// owner, b → every CTA) → sweep, and the same warps do both, so the ~2.6 µs exchange is exposed on
// every ~6.5 µs pass.  Here the columns of every row are split into two halves A and B, and
//   * 16 row warps sweep half A, publish its column partials, sweep half B, publish, reduce the row
//     sums (the only thing the next pass needs from both halves: a_i and S);
//   * 2 exchange warps per half ("chains") run the two-hop all-reduce of their half concurrently with
//     the row warps' sweep of the OTHER half: chain A reduces A's partials of Y_{j+1} while the row
//     warps sweep B of pass j, chain B reduces B's partials while they sweep A of pass j+1.
// What remains exposed per pass is the S hop (one tagged word per CTA, one L2 round trip), done by
// row warp 0 while the other row warps wait at the half-A barrier.
//
// Work split (CPT = 32 columns per owner thread, 8 float4 quads; half H = quads 4H..4H+3).
//   row warp w < 16: TMEM lane quarter q = w % 4, quad k = w / 4 of each half; thread t = 32q + lane
//     owns columns t·32 + 4(4H + k) + [0, 4) of every row of the CTA's row block, in both halves.
//   chain warps 16-17 (half A), 18-19 (half B).
// Rows: the first 16 in TMEM (lane t, column 32r + c), the rest (≤ 12) in shared memory ([row][quad][t]
// float4).  Row sums: FP32 float2 accumulators per lane and row across both halves → one 32-row
// transpose-reduce per warp per pass → [row][warp] in shared memory → row warp 0 combines the 16 warp
// partials of row `lane` in FP64 (fixed pairwise tree), publishes Σ r_i, waits for S.  Column sums:
// complete per thread over the CTA's rows (each column has exactly one owner thread), published
// straight from registers as tagged words.  Chains reduce slot slice b of their half over all CTAs
// (FP64, fixed order: source k ≡ g mod 4 per group g, groups combined pairwise), publish b, poll the
// whole half of b and hand it to the row warps through shared memory and a named barrier.
// Every cross-CTA word carries its epoch parity in the FP32/FP64 sign bit (xchg.cuh); the data
// dependencies make one bit sufficient, as in K4r.  Deterministic: no float atomics.
#include <math_constants.h>
#include "common.cuh"
#include "internal.h"
#include "tmem_ldst.cuh"
#include "xchg.cuh"

namespace fram {
namespace {

constexpr int kWsThreads = 640;          // 16 row warps + 4 chain warps
constexpr int kWsRowThreads = 512;
constexpr int kWsRT = 16;                // rows in TMEM (512 columns / 32)
constexpr int kWsRS = 12;                // rows in shared memory at most
constexpr int kWsRows = kWsRT + kWsRS;   // 28 rows per CTA at most
constexpr int kWsNSH = 2048;             // slots per half
constexpr int kWsGMax = 160;             // CTAs at most (40 sources per chain thread)
constexpr int kWsNI = kWsGMax / 4;
constexpr int kWsSmemMax = 232448 - 4096;   // 227 KB opt-in minus the static shared memory

#ifndef FRAM_DEV_WS_TIMING
#define FRAM_DEV_WS_TIMING 0
#endif
constexpr int kWsStampPass = 500;

// named barriers (0 is __syncthreads)
constexpr int kBarA = 1, kBarB = 2, kBarRows = 3, kBarChain = 4, kBarPub = 6;   // kBarChain + H, kBarPub + H

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

size_t ws_smem_bytes(int rs) { return (size_t)rs * 8 * 128 * 16 + 2 * 512 * 16; }

__global__ void __launch_bounds__(kWsThreads, 1) sdsn_ws_kernel(ResParams P) {
  extern __shared__ __align__(16) unsigned char dsm[];
  float4* s_rows = reinterpret_cast<float4*>(dsm);                     // [rs][8][128]
  float4* s_b = s_rows + (size_t)P.rs * 8 * 128;                       // [2][512] (−|b|, slot order)
  __shared__ uint32_t s_tmem;
  __shared__ float s_rowpart[16][32];       // [warp][row]
  __shared__ double s_rn[kWsRows];
  __shared__ float s_a[kWsRows];
  __shared__ double s_xc[2][2][16];
  __shared__ double s_red[20];
  __shared__ double s_S;
  __shared__ int s_last;
  __shared__ volatile int s_dec[2];                      // [j & 1] = (j + 1) | last << 30: pass j's stop decision

  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool rowwarp = warp < 16;
  const int q = warp & 3, k = (warp >> 2) & 3;
  const int t = q * 32 + lane;
  const long n = P.n, ld = P.ld;
  const long r0 = (long)b * n / G, r1 = (long)(b + 1) * n / G;
  const int R = (int)(r1 - r0);
  const int RT = R < kWsRT ? R : kWsRT;
  const double dn = (double)n, nn = dn * dn;
  const double rn = __drcp_rn(dn), rnn = __drcp_rn(nn);
  auto div_n = [&](double S_, double d, double r) {      // RN(S/d) (Markstein, as K4r)
    const double qq = S_ * r;
    return fma(r, fma(-qq, d, S_), qq);
  };

  if (tid < 2) s_dec[tid] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(4 * k);   // + 32r + 16H
  auto squad = [&](int r, int H) -> float4* { return s_rows + (size_t)(r - kWsRT) * 1024 + (4 * H + k) * 128 + t; };
  auto tm_ld = [&](int r, int H, uint32_t (&v)[4]) { tmem_ld<4>(tmem + (uint32_t)(32 * r + 16 * H), v); };
  auto tm_st = [&](int r, int H, const uint32_t (&v)[4]) { tmem_st<4>(tmem + (uint32_t)(32 * r + 16 * H), v); };
  // dev timeline (FRAM_DEV_WS_TIMING builds only; P.dbg is null in the product): absolute
  // %globaltimer stamps of pass kWsStampPass, [G*16 + b*16 + slot]
  auto stamp = [&](int slot, int jj) {
#if FRAM_DEV_WS_TIMING
    if (P.dbg && lane == 0 && jj == kWsStampPass) {
      long long v;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
      P.dbg[(size_t)G * 16 + b * 16 + slot] = v;
    }
#endif
  };
  auto dealloc = [&]() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(512));
  };

  // ---------------- phase L: X rows → on chip, m = max X (Alg.2 step 1) ----------------
  if (rowwarp) {
    float lmax = 0.f;
    for (int r = 0; r < R; ++r) {
      const float* grow = P.Y + (r0 + r) * ld;
#pragma unroll
      for (int H = 0; H < 2; ++H) {
        const long col = (long)t * 32 + 4 * (4 * H + k);
        float4 v;
        if (col + 3 < n) {
          v = __ldca(reinterpret_cast<const float4*>(grow + col));
        } else {
          v.x = col < n ? grow[col] : 0.f;
          v.y = col + 1 < n ? grow[col + 1] : 0.f;
          v.z = col + 2 < n ? grow[col + 2] : 0.f;
          v.w = col + 3 < n ? grow[col + 3] : 0.f;
        }
        lmax = fmaxf(lmax, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
        if (r < kWsRT) {
          const uint32_t u[4] = {__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z), __float_as_uint(v.w)};
          tm_st(r, H, u);
        } else {
          *squad(r, H) = v;
        }
      }
    }
    tmem_wait_st();
    double m = warp_max_d((double)lmax);
    if (lane == 0) s_red[warp] = m;
  }
  __syncthreads();
  if (tid == 0) {
    double mm = 0.0;
    for (int w = 0; w < 16; ++w) mm = fmax(mm, s_red[w]);
    st_d1(P.Mpart + b, mm, 1u);
  }
  double sc = 1.0;
  if (P.scale) {
    if (warp == 0) {
      double mm = 0.0;
      double v[5];
      wait_d1_lanes<5>(P.Mpart, G, lane, 1u, v);
#pragma unroll
      for (int i = 0; i < 5; ++i) mm = fmax(mm, v[i]);
      mm = warp_max_d(mm);
      if (lane == 0) s_S = mm;
    }
    __syncthreads();
    const double m = s_S;
    if (m == 0.0) {                                      // R10: all-zero ⇒ 11ᵀ/n, 0 passes
      if (rowwarp) {
        for (int r = 0; r < R; ++r) {
          float* grow = P.Y + (r0 + r) * ld;
          for (long col = (long)(k * 128 + t); col < n; col += 512) grow[col] = (float)(1.0 / dn);
        }
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

  // the stop rule of pass j from S_j (identical arithmetic in every warp that evaluates it)
  auto decide = [&](int j, double S, double* gam_out) -> bool {
    const double gam = div_n(S, dn, rn) - 1.0;                          // γ_j = S/n − 1
    if (gam_out) *gam_out = gam;
    return P.sdsn_fixed > 0 ? (j + 1 >= P.sdsn_fixed) : ((j >= 1 && gam <= P.gamma_th) || j + 1 >= P.sdsn_max);
  };
  auto poll_S = [&](unsigned e) -> double {              // S of epoch e (all lanes of the calling warp)
    double v[5];
    wait_d1_lanes<5>(P.Spart + (size_t)(e & 1) * G, G, lane, (e >> 1) & 1u, v);
    double sacc = 0.0;
#pragma unroll
    for (int i = 0; i < 5; ++i) sacc += v[i];
    return warp_sum_d(sacc);
  };

  if (!rowwarp) {
    // ======================= chains: the two-hop all-reduce of half H =======================
    const int H = (warp - 16) >> 1, cl = (warp - 16) & 1, ct = cl * 32 + lane;
    const int s0 = (int)((long)b * kWsNSH / G), s1 = (int)((long)(b + 1) * kWsNSH / G);
    const int so = lane & 15, grp = cl * 2 + (lane >> 4);
    const int s = s0 + so;
    const unsigned* cp = P.colpart + (size_t)H * G * kWsNSH;
    unsigned* bv = P.bvec + (size_t)H * kWsNSH;
    auto produce = [&](unsigned e) {
      const int jj = (int)e - 2, sb = 8 + 4 * H;       // b of Y_{jj+1}, produced during pass jj
      if (cl == 0) stamp(sb, jj);
      double acc = 0.0;
      if (s < s1) {                                      // ≤ 16 slots per CTA (G ≥ 128)
        unsigned w[kWsNI];
        const unsigned* base = cp + (size_t)grp * kWsNSH + s;   // source grp + 4i at base + 4i·NSH
        const int ni = (G - grp + 3) >> 2;                       // sources of this group
#pragma unroll
        for (int i = 0; i < kWsNI; ++i) w[i] = i < ni ? ld_w(base + (size_t)i * 4 * kWsNSH) : ptag(0.f, e);
        bool ok;
        do {
          ok = true;
#pragma unroll
          for (int i = 0; i < kWsNI; ++i)
            if (!pok(w[i], e)) { ok = false; w[i] = ld_w(base + (size_t)i * 4 * kWsNSH); }
        } while (!ok);
#pragma unroll
        for (int i = 0; i < kWsNI; ++i) acc += (double)pval(w[i]);
      }
      if (cl == 0) stamp(sb + 1, jj);
      acc += __shfl_xor_sync(0xffffffffu, acc, 16);    // groups 2cl and 2cl+1 (commutative: same in both)
      if (cl == 1 && lane < 16) s_xc[e & 1][H][lane] = acc;
      bar_sync(kBarChain + H, 64);
      if (cl == 0 && lane < 16 && s < s1) {
        const double cs = acc + s_xc[e & 1][H][lane];
        const int f = s >> 2, e4 = s & 3, kk = f >> 7, tt = f & 127;
        const long colj = (long)tt * 32 + 4 * (4 * H + kk) + e4;
        st_w(bv + s, ptag(colj < n ? (float)(cs / dn) : CUDART_INF_F, e));   // |b_j| = c_j/n
      }
      if (cl == 0) stamp(sb + 2, jj);
      // the whole half of b of epoch e → shared memory (negated: b = −|b|; −∞ on padding)
      uint4 wv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) wv[i] = ld_w4(bv + (size_t)(i * 64 + ct) * 4);
      bool ok;
      do {
        ok = true;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (!pok(wv[i].x, e) || !pok(wv[i].y, e) || !pok(wv[i].z, e) || !pok(wv[i].w, e)) {
            ok = false;
            wv[i] = ld_w4(bv + (size_t)(i * 64 + ct) * 4);
          }
      } while (!ok);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        s_b[H * 512 + i * 64 + ct] = make_float4(-pval(wv[i].x), -pval(wv[i].y), -pval(wv[i].z), -pval(wv[i].w));
      if (cl == 0) stamp(sb + 3, jj);
      bar_arrive(kBarA + H, kWsRowThreads + 64);
    };
    bar_sync(kBarPub + H, kWsRowThreads + 64);           // this CTA's row warps published half H of Y_0
    produce(1u);                                         // b of Y_0
    for (int j = 0;; ++j) {
      int dj;
      while (((dj = s_dec[j & 1]) & 0x3fffffff) != j + 1) __nanosleep(32);   // row warp 0's decision for pass j
      if (dj >> 30) break;                               // pass j is the last: nothing more to reduce
      bar_sync(kBarPub + H, kWsRowThreads + 64);         // this CTA published half H of Y_{j+1}
      produce((unsigned)j + 2);                          // b of Y_{j+1}
    }
    dealloc();
    return;
  }

  // ============================ row warps ============================
#ifndef WS_RACC_F32
#define WS_RACC_F32 1
#endif
#ifndef WS_TB
#define WS_TB 2
#endif
#if WS_RACC_F32
  float racc[kWsRows];
#else
  float2 racc[kWsRows];                                  // per-lane row partials (both halves)
#endif
  // one half of every row: y ← op(y), column partials → tagged words (e ≠ 0), row partials → racc
  auto sweep_half = [&](auto scale_tag, int H, unsigned e, float2 bq01, float2 bq23) {
    constexpr bool SCALE = decltype(scale_tag)::value;
    float2 c01 = make_float2(0.f, 0.f), c23 = make_float2(0.f, 0.f);
    auto body = [&](int r, float (&x)[4]) {
      float2 y01, y23;
      if (SCALE) {
        y01 = make_float2(x[0], x[1]);
        y23 = make_float2(x[2], x[3]);
        if (P.scale) {
          y01 = make_float2((float)(sc * (double)x[0]), (float)(sc * (double)x[1]));
          y23 = make_float2((float)(sc * (double)x[2]), (float)(sc * (double)x[3]));
        }
      } else {
        const float a = s_a[r];
        const float2 a2 = make_float2(a, a);
        y01 = add2(add2(make_float2(x[0], x[1]), a2), bq01);
        y23 = add2(add2(make_float2(x[2], x[3]), a2), bq23);
        y01.x = fmaxf(0.0f, y01.x); y01.y = fmaxf(0.0f, y01.y);
        y23.x = fmaxf(0.0f, y23.x); y23.y = fmaxf(0.0f, y23.y);
      }
      x[0] = y01.x; x[1] = y01.y; x[2] = y23.x; x[3] = y23.y;
      c01 = add2(c01, y01);
      c23 = add2(c23, y23);
      const float2 sr = add2(y01, y23);
#if WS_RACC_F32
      racc[r] = H == 0 ? sr.x + sr.y : racc[r] + (sr.x + sr.y);
#else
      racc[r] = H == 0 ? sr : add2(racc[r], sr);
#endif
    };
    // rows in rounds of 4 TMEM rows + 3 shared-memory rows, all loads of a round in flight before the
    // first wait, so the TMEM and shared-memory datapaths work concurrently (every warp holds rows of both)
    auto trow = [&](int r, uint32_t (&v)[4]) {
      float x[4] = {__uint_as_float(v[0]), __uint_as_float(v[1]), __uint_as_float(v[2]), __uint_as_float(v[3])};
      body(r, x);
      if (!SCALE || P.scale) {
        const uint32_t u[4] = {__float_as_uint(x[0]), __float_as_uint(x[1]), __float_as_uint(x[2]), __float_as_uint(x[3])};
        tm_st(r, H, u);
      }
    };
    auto srow = [&](int r, float4 v) {
      float x[4] = {v.x, v.y, v.z, v.w};
      body(r, x);
      if (!SCALE || P.scale) *squad(r, H) = make_float4(x[0], x[1], x[2], x[3]);
    };
    if (SCALE) {                                         // once per call: one row at a time
#pragma unroll
      for (int r = 0; r < kWsRT; ++r) {
        if (r < RT) {
          uint32_t v[4];
          tm_ld(r, H, v);
          tmem_wait_ld();
          trow(r, v);
        }
      }
#pragma unroll
      for (int r = kWsRT; r < kWsRows; ++r)
        if (r < R) srow(r, *squad(r, H));
    } else if (RT == kWsRT) {                            // full TMEM block: no predicates on tcgen05 ops
      constexpr int TB = WS_TB, NR = kWsRT / TB, SB = (kWsRS + NR - 1) / NR;
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) {
        uint32_t v[TB][4];
        float4 w[SB];
#pragma unroll
        for (int i = 0; i < TB; ++i) tm_ld(TB * rr + i, H, v[i]);
#pragma unroll
        for (int i = 0; i < SB; ++i)
          if (SB * rr + i < kWsRS && kWsRT + SB * rr + i < R) w[i] = *squad(kWsRT + SB * rr + i, H);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < TB; ++i) trow(TB * rr + i, v[i]);
#pragma unroll
        for (int i = 0; i < SB; ++i)
          if (SB * rr + i < kWsRS && kWsRT + SB * rr + i < R) srow(kWsRT + SB * rr + i, w[i]);
      }
    } else {                                             // R < 16: TMEM rows only, ragged
#pragma unroll
      for (int rb = 0; rb < kWsRT; rb += 4) {
        if (rb < RT) {
          uint32_t v[4][4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (rb + i < RT) tm_ld(rb + i, H, v[i]);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (rb + i < RT) trow(rb + i, v[i]);
        }
      }
    }
    tmem_wait_st();
    if (e != 0) {
      unsigned* dst = P.colpart + ((size_t)H * G + b) * kWsNSH + (size_t)(k * 128 + t) * 4;
      st_w4(dst, make_uint4(ptag(c01.x, e), ptag(c01.y, e), ptag(c23.x, e), ptag(c23.y, e)));
      bar_arrive(kBarPub + H, kWsRowThreads + 64);       // lets chain H start polling
    }
  };
  // row sums of the pass: one transpose-reduce of the 28 (padded to 32) per-lane partials per warp
  // (each level halves the rows a lane carries; lane l ends with row l), then [row][warp]
  auto reduce_rows = [&]() {
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
#if WS_RACC_F32
      v[i] = (i < kWsRows && i < R) ? racc[i < kWsRows ? i : 0] : 0.f;
#else
      v[i] = (i < kWsRows && i < R) ? racc[i < kWsRows ? i : 0].x + racc[i < kWsRows ? i : 0].y : 0.f;
#endif
    }
#pragma unroll
    for (int l = 0; l < 5; ++l) {
      const int off = 16 >> l, m = 16 >> l;
      const bool hi = lane & off;
#pragma unroll
      for (int i = 0; i < m; ++i) v[i] = (hi ? v[i + m] : v[i]) + __shfl_xor_sync(0xffffffffu, hi ? v[i] : v[i + m], off);
    }
    if (lane < R) s_rowpart[warp][lane] = v[0];
  };
  // S duty (row warp 0): r_i (FP64, fixed tree over the 16 warp partials), Σ r_i → Spart tagged e,
  // S_j of epoch e → γ_j, the stop decision, a_i for pass j
  auto s_duty = [&](int j, unsigned e) {
    double acc = 0.0;
    if (lane < R) {
      double v[16];
#pragma unroll
      for (int w = 0; w < 16; ++w) v[w] = (double)s_rowpart[w][lane];
#pragma unroll
      for (int st = 1; st < 16; st *= 2)
#pragma unroll
        for (int w = 0; w < 16; w += 2 * st) v[w] += v[w + st];
      acc = v[0];
    }
    const double rnl = acc / dn;
    const double sp = warp_sum_d(acc);
    if (lane == 0) st_d1(P.Spart + (size_t)(e & 1) * G + b, sp, (e >> 1) & 1u);
    stamp(5, j - 1);
    const double S = poll_S(e);
    double gam;
    const bool last = decide(j, S, &gam);
    const double abase = rn + div_n(S, nn, rnn);                        // 1/n + S/n²
    if (lane < R) s_a[lane] = (float)(abase - rnl);                     // a_i (FP64, rounded once)
    if (lane == 0) {
      s_last = last ? 1 : 0;
      s_dec[j & 1] = (j + 1) | (last ? 1 << 30 : 0);
      s_S = S;
      if (b == 0 && P.gamma_hist) P.gamma_hist[j] = gam;
      s_red[0] = gam;
    }
  };

  // ---------------- phase S: Y0 = s·X (on chip) and its sums, epoch 1 ----------------
  sweep_half(std::integral_constant<bool, true>{}, 0, 1u, make_float2(0.f, 0.f), make_float2(0.f, 0.f));
  sweep_half(std::integral_constant<bool, true>{}, 1, 1u, make_float2(0.f, 0.f), make_float2(0.f, 0.f));
  reduce_rows();
  bar_sync(kBarRows, kWsRowThreads);
  if (warp == 0) s_duty(0, 1u);

  // ---------------- pass loop ----------------
  int j = 0;
  unsigned ep = 1;                                       // epoch of Y_j's sums = j + 1
  for (;; ++j) {
    bar_sync(kBarA, kWsRowThreads + 64);                 // b of half A (epoch ep), a_i, the stop flag
    if (warp == 0) { stamp(0, j); stamp(7, j - 1); }
    const bool last = s_last != 0;
    float4 bq = s_b[k * 128 + t];
    sweep_half(std::integral_constant<bool, false>{}, 0, last ? 0u : ep + 1, make_float2(bq.x, bq.y), make_float2(bq.z, bq.w));
    if (warp == 0) stamp(1, j);
    bar_sync(kBarB, kWsRowThreads + 64);                 // b of half B (epoch ep)
    if (warp == 0) stamp(2, j);
    bq = s_b[512 + k * 128 + t];
    sweep_half(std::integral_constant<bool, false>{}, 1, last ? 0u : ep + 1, make_float2(bq.x, bq.y), make_float2(bq.z, bq.w));
    if (warp == 0) stamp(3, j);
    if (last) break;
    ++ep;
    reduce_rows();
    bar_sync(kBarRows, kWsRowThreads);
    if (warp == 0) { stamp(4, j); s_duty(j + 1, ep); stamp(6, j); }
  }

  // ---------------- D = Y_final → global (row-major, ld) ----------------
  for (int r = 0; r < R; ++r) {
    float* grow = P.Y + (r0 + r) * ld;
#pragma unroll
    for (int H = 0; H < 2; ++H) {
      float x[4];
      if (r < kWsRT) {
        uint32_t v[4];
        tm_ld(r, H, v);
        tmem_wait_ld();
        x[0] = __uint_as_float(v[0]); x[1] = __uint_as_float(v[1]); x[2] = __uint_as_float(v[2]); x[3] = __uint_as_float(v[3]);
      } else {
        const float4 v = *squad(r, H);
        x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
      }
      const long col = (long)t * 32 + 4 * (4 * H + k);
      if (col + 3 < n) {
        *reinterpret_cast<float4*>(grow + col) = make_float4(x[0], x[1], x[2], x[3]);
      } else {
        if (col < n) grow[col] = x[0];
        if (col + 1 < n) grow[col + 1] = x[1];
        if (col + 2 < n) grow[col + 2] = x[2];
      }
    }
  }
  if (b == 0 && tid == 0) {
    *P.passes_out = j + 1;
    P.sdsn_out[0] = s_red[0];
    P.sdsn_out[2] = s_S;
  }
  dealloc();
}

}  // namespace

// grid for K4w at n, or 0 when it does not apply (then K4r runs): 2048 < n ≤ 4096, one CTA per SM,
// ≤ 28 rows per CTA (16 in TMEM, ≤ 12 in shared memory), 128 ≤ G ≤ 160
int sdsn_ws_grid(long n, int num_sms) {
  if (n <= 2048 || n > 4096) return 0;
  const int G = sdsn_res_grid(n, num_sms);
  if (G < 128 || G > kWsGMax) return 0;
  const long R = (n + G - 1) / G;
  if (R > kWsRows) return 0;
  const int rs = R > kWsRT ? (int)(R - kWsRT) : 0;
  if (ws_smem_bytes(rs) > (size_t)kWsSmemMax) return 0;
  return G;
}

cudaError_t launch_sdsn_ws(ResParams p, cudaStream_t st, int num_sms) {
  const int G = sdsn_ws_grid(p.n, num_sms);
  if (G == 0) return cudaErrorInvalidValue;
  const long R = (p.n + G - 1) / G;
  p.rs = R > kWsRT ? (int)(R - kWsRT) : 0;
  p.rmax = (int)R;
  size_t dsm = ws_smem_bytes(p.rs);
  if (dsm < 120 * 1024) dsm = 120 * 1024;                // one CTA per SM (TMEM: 512 columns per CTA)
  cudaError_t e = cudaFuncSetAttribute(sdsn_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
  if (e != cudaSuccess) return e;
  const size_t ns = 2 * (size_t)kWsNSH;
  p.Spart = p.xchg;                                      // [2][G] u64, tag bit 1 initially in slot 1
  p.Mpart = p.Spart + 2 * (size_t)G;                     // [G] u64
  p.colpart = reinterpret_cast<unsigned*>(p.xchg + ((3 * (size_t)G + 1) & ~(size_t)1));   // [2][G][2048] u32
  p.bvec = p.colpart + (size_t)G * ns;                   // [2][2048] u32
  e = cudaMemsetAsync(p.Spart, 0, (size_t)G * sizeof(uint64_t), st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(p.Spart + G, 0x80, (size_t)G * sizeof(uint64_t), st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(p.Mpart, 0, (size_t)G * sizeof(uint64_t) + 8 + ((size_t)G * ns + ns) * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  void* args[] = {&p};
  return cudaLaunchCooperativeKernel((const void*)sdsn_ws_kernel, dim3(G), dim3(kWsThreads), args, dsm, st);
}

}  // namespace fram
