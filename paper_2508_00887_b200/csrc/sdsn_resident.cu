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
#include "xchg.cuh"

namespace fram {
namespace {

constexpr int kResSmemMax = 232448 - 4608;   // 227 KB opt-in minus static shared memory (≤ 4.3 KB)
constexpr int kResMinSmem = 120 * 1024;      // forces one CTA per SM (TMEM: 512 columns per CTA)

template <int CPT> struct RC {
  static constexpr int V = CPT / 4;          // float4 chunks per owner thread per row
  static constexpr int NS = 128 * CPT;       // slots = padded columns
  static constexpr int RT = 512 / CPT;       // rows held in TMEM
};

constexpr int kResMaxRows = 32;             // rows per CTA (the grid is sized so R ≤ 32)
constexpr int kResKMax = 5;                  // G ≤ 32·kResKMax CTAs (148 SMs)

// dynamic shared memory: SMEM-resident rows, column staging, per-warp row partials, s_r, s_rn
size_t res_smem_bytes(int cpt, int rs, int R) {
  const size_t ns = 128 * (size_t)cpt;
  return (size_t)rs * ns * 4 + ns * 4 + (size_t)R * 8 * 4 + (size_t)R * 8 + (size_t)R * 8 + 64;
}

template <int CPT> struct RK {
  static constexpr bool SPLIT = CPT >= 8;                // two warps share each TMEM lane's row slice
  static constexpr int NH = SPLIT ? 2 : 1;
  static constexpr int THREADS = SPLIT ? 512 : 256;
  static constexpr int NW = THREADS / 32;
  static constexpr int CH = CPT / NH;                    // columns per thread
  static constexpr int VH = CH / 4;                      // float4 chunks per thread per row
};

template <int CPT>
__global__ void __launch_bounds__(RK<CPT>::THREADS, 1) sdsn_res_kernel(ResParams P) {
  using C = RC<CPT>;
  using K = RK<CPT>;
  constexpr int V = C::V, NS = C::NS, RT = C::RT;
  constexpr int NW = K::NW, CH = K::CH, VH = K::VH;
  extern __shared__ __align__(16) unsigned char dsm[];
  const int RS = P.rs;
  const int Rmax = P.rmax;
  float4* s_rows = reinterpret_cast<float4*>(dsm);                    // [RS][V·128] slot layout
  float4* s_col = s_rows + (size_t)RS * V * 128;                      // [V·128] column staging
  float* s_rowpart = reinterpret_cast<float*>(s_col + V * 128);       // [Rmax][8] per-warp row partials
  double* s_r = reinterpret_cast<double*>(s_rowpart + Rmax * 8);     // [Rmax] row sums (FP64)
  double* s_rn = s_r + Rmax;                                          // [Rmax] r_i / n (FP64)
  __shared__ uint32_t s_tmem;
  __shared__ double s_red[NW];
  __shared__ double s_S;
  __shared__ double s_red2[NW][32];
  __shared__ float s_af[kResMaxRows];                    // a_i of the current pass (FP32)

  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = warp & 3;
  const int h = K::SPLIT ? (warp >> 2) & 1 : 0;
  const int g = K::SPLIT ? warp >> 3 : warp >> 2;
  const int t = q * 32 + lane;
  const int c0 = h * VH;                                 // first float4 chunk of this thread
  const long n = P.n, ld = P.ld;
  const long r0 = (long)b * n / G, r1 = (long)(b + 1) * n / G;
  const int R = (int)(r1 - r0);
  const double dn = (double)n, nn = dn * dn;
  // S/n and S/n² on the pass-start critical path without a full FP64 division: with the correctly
  // rounded reciprocal r = RN(1/d), q = RN(S·r) and one FMA correction q + r·(S − q·d) is RN(S/d)
  // (Markstein's theorem; tools/div_probe.cu: 0 mismatches against IEEE division in 3.6e10 cases)
  const double rn = __drcp_rn(dn), rnn = __drcp_rn(nn);
  auto div_n = [&](double S_, double d, double r) {
    const double q = S_ * r;
    return fma(r, fma(-q, d, S_), q);
  };

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * CH);   // lane quarter, half

  auto load_row = [&](int r, float (&x)[CH]) {
    if (r < RT) {
      uint32_t v[CH];
      tmem_ld<CH>(tmem + (uint32_t)(r * CPT), v);
      tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < CH; ++k) x[k] = __uint_as_float(v[k]);
    } else {
      const float4* row = s_rows + (size_t)(r - RT) * (V * 128);
#pragma unroll
      for (int c = 0; c < VH; ++c) {
        const float4 v = row[(c0 + c) * 128 + t];
        x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
      }
    }
  };
  auto store_row = [&](int r, const float (&x)[CH]) {
    if (r < RT) {
      uint32_t v[CH];
#pragma unroll
      for (int k = 0; k < CH; ++k) v[k] = __float_as_uint(x[k]);
      tmem_st<CH>(tmem + (uint32_t)(r * CPT), v);
    } else {
      float4* row = s_rows + (size_t)(r - RT) * (V * 128);
#pragma unroll
      for (int c = 0; c < VH; ++c)
        row[(c0 + c) * 128 + t] = make_float4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
    }
  };
  // Cross-CTA exchange without grid barriers: every published value travels in one 8-byte word
  // together with the epoch it belongs to (single-copy atomic), and a consumer re-reads a word
  // until its tag matches — it waits for exactly the data it needs.  Tags are zeroed by the
  // launcher; epochs start at 1.
  auto dealloc = [&]() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(512));
  };

  long long tk0 = 0;
  if (P.dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tk0));
  // ---------------- phase L: X rows → on-chip, m = max X (Alg.2 step 1) ----------------
  {
    float lmax = 0.f;
    // 4 rows of loads in flight per row group before their stores (tcgen05.st is an asm with a memory
    // clobber, so the compiler cannot hoist the next row's loads above it by itself).  The per-call time
    // did not move, but the pass loop of this build measured 0.5-1% faster at n = 4096
    // (profiles/r02/ab_k4r_loadrows.log; 2 rows: no change)
    constexpr int LB = 4;
    auto load_g = [&](int r, float (&x)[CH]) {
      const float* grow = P.Y + (r0 + r) * ld;
#pragma unroll
      for (int c = 0; c < VH; ++c) {
        const long col = (long)t * CPT + 4 * (c0 + c);
        float4 v;
        if (col + 3 < n) {
          // L1-allocating: a lane's 16-byte loads of one row are two per 32-byte sector (the column-
          // owner layout); the second one hits L1 (per call 320 → 300 us, `profiles/r02/ab_k4r_ldca.log`)
          v = __ldca(reinterpret_cast<const float4*>(grow + col));
        } else {
          v.x = col < n ? grow[col] : 0.f;
          v.y = col + 1 < n ? grow[col + 1] : 0.f;
          v.z = col + 2 < n ? grow[col + 2] : 0.f;
          v.w = col + 3 < n ? grow[col + 3] : 0.f;
        }
        x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
      }
    };
    for (int r = g; r < R; r += 2 * LB) {
      float x[LB][CH];
#pragma unroll
      for (int i = 0; i < LB; ++i)
        if (r + 2 * i < R) load_g(r + 2 * i, x[i]);
#pragma unroll
      for (int i = 0; i < LB; ++i) {
        if (r + 2 * i < R) {
#pragma unroll
          for (int k = 0; k < CH; ++k) lmax = fmaxf(lmax, x[i][k]);
          store_row(r + 2 * i, x[i]);
        }
      }
    }
    tmem_wait_st();
    double m = (double)lmax;
    m = warp_max_d(m);
    if (lane == 0) s_red[warp] = m;
    __syncthreads();
    if (tid == 0) {
      double mm = 0.0;
      for (int w = 0; w < NW; ++w) mm = fmax(mm, s_red[w]);
      st_d1(P.Mpart + b, mm, 1u);
    }
  }
  double sc = 1.0;
  if (P.scale) {
    if (warp == 0) {
      double mm = 0.0;
      double v[kResKMax];
      wait_d1_lanes<kResKMax>(P.Mpart, G, lane, 1u, v);
#pragma unroll
      for (int i = 0; i < kResKMax; ++i) mm = fmax(mm, v[i]);
      mm = warp_max_d(mm);
      if (lane == 0) s_S = mm;
    }
    __syncthreads();
    const double m = s_S;
    if (m == 0.0) {                                      // R10: all-zero ⇒ 11ᵀ/n, 0 passes
      for (int r = g; r < R; r += 2) {
        float* grow = P.Y + (r0 + r) * ld;
        for (long col = (long)(h * 128 + t); col < n; col += 128 * K::NH) grow[col] = (float)(1.0 / dn);
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

  // after a sweep: column partials (two row groups combined in shared memory) → colpart[b];
  // row sums (per-lane partials → fixed-order tree) → s_r; Σ r → Spart[b]; all tagged e
  // dev timing (P.dbg; set only by a -DFRAM_DEV_RES_TIMING=1 build of fram_api.cu, always null in the
  // product, where these branches are never taken): per-CTA slots accumulated in shared memory by one thread
  // (k < 9) or by the first warp of each row group (rows: 9 + g ns, 11 + g cycles), copied out at the end
  __shared__ long long s_dbg[16];
  if (tid < 16) s_dbg[tid] = 0;
  __syncthreads();
  auto dadd = [&](int k, long long v) { if (P.dbg && tid == 0) s_dbg[k] += v; };
  int jst = -1;                                          // pass whose timeline is stamped (dev timing)
  auto stamp = [&](int k) {
    if (P.dbg && tid == 0 && jst == 500) {
      long long v;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
      P.dbg[(size_t)G * 16 + b * 8 + k] = v;
    }
  };
  auto gt = [&]() -> long long {
    long long v = 0;
    if (P.dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
  };
  auto sweep_epilogue = [&](const float (&col)[CH], unsigned e) {
    const long long e0 = gt();
    tmem_wait_st();
    // the two row groups' column partials are combined through shared memory and published by
    // group 0 (splitting the stores between the groups measured slower)
    if (g == 1) {
#pragma unroll
      for (int c = 0; c < VH; ++c)
        s_col[(c0 + c) * 128 + t] = make_float4(col[4 * c], col[4 * c + 1], col[4 * c + 2], col[4 * c + 3]);
    }
    __syncthreads();
    const long long e1 = gt();
    if (g == 0 && e != 0) {
      unsigned* dst = P.colpart + (long)b * NS;
#pragma unroll
      for (int c = 0; c < VH; ++c) {
        float4 o = s_col[(c0 + c) * 128 + t];
        o.x += col[4 * c]; o.y += col[4 * c + 1]; o.z += col[4 * c + 2]; o.w += col[4 * c + 3];
        st_w4(dst + (size_t)((c0 + c) * 128 + t) * 4, make_uint4(ptag(o.x, e), ptag(o.y, e), ptag(o.z, e), ptag(o.w, e)));
      }
    }
    // row sums, off the critical path (group 0 goes on to the slice reduction): the first warp of
    // group 1 combines the 4·NH per-warp partials of row `lane` in FP64 in a fixed order, keeps
    // r_i and r_i/n, and publishes this CTA's Σ r_i (R ≤ 32 rows: one row per lane)
    if (warp == NW / 2) {
      double acc = 0.0;
      if (lane < R) {
        const float* pp = s_rowpart + lane * 8;
#pragma unroll
        for (int k = 0; k < 4 * K::NH; ++k) acc += (double)pp[k];
        s_r[lane] = acc;
        s_rn[lane] = acc / dn;
      }
      const double sp = warp_sum_d(acc);
      if (lane == 0 && e != 0) st_d1(P.Spart + (size_t)(e & 1) * G + b, sp, (e >> 1) & 1u);
    }
    const long long e1a = gt();
    dadd(4, e1a - e1);
  };
  // this warp's partials of rows ra and rb (rb < 0: none): two interleaved shuffle trees, lane 0
  // stores them at slot 4·h + q of the row (fixed order, deterministic)
  auto put_rowparts = [&](int ra, float va, int rb, float vb) {
    // transpose-reduce: one xor-16 exchange leaves lanes 0-15 with row a and lanes 16-31 with row b,
    // four more levels finish both (5 shuffles for two rows instead of 10); fixed tree, deterministic
    const bool lo = lane < 16;
    float keep = lo ? va : vb;
    keep += __shfl_xor_sync(0xffffffffu, lo ? vb : va, 16);
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) keep += __shfl_xor_sync(0xffffffffu, keep, o);
    if (lane == 0) s_rowpart[ra * 8 + 4 * h + q] = keep;
    if (lane == 16 && rb >= 0) s_rowpart[rb * 8 + 4 * h + q] = keep;
  };
  // this warp's partials of the NB rows i0 + k·rstep (k < NB, rows ≥ rend absent): one transpose-
  // reduce — each xor level (16, 8, …) halves the set of rows a lane carries, the remaining levels
  // finish the sum (NB = 8: 9 shuffles for 8 rows); lane k·32/NB ends with row k.  Fixed tree.
  auto put_rowparts_n = [&](auto nb, int i0, int rstep, int rend, float* v) {
    constexpr int NB = decltype(nb)::value;
    constexpr int LG = NB == 8 ? 3 : NB == 4 ? 2 : 1;
#pragma unroll
    for (int l = 0; l < LG; ++l) {
      const int off = 16 >> l, m = NB >> (l + 1);
      const bool hi = lane & off;
#pragma unroll
      for (int i = 0; i < m; ++i) v[i] = (hi ? v[i + m] : v[i]) + __shfl_xor_sync(0xffffffffu, hi ? v[i] : v[i + m], off);
    }
    float z = v[0];
#pragma unroll
    for (int off = 16 >> LG; off > 0; off >>= 1) z += __shfl_xor_sync(0xffffffffu, z, off);
    const int r = i0 + (lane >> (5 - LG)) * rstep;
    if ((lane & ((32 >> LG) - 1)) == 0 && r < rend) s_rowpart[r * 8 + 4 * h + q] = z;
  };

  // Y0 = fl(s·X) (Alg.2 step 1; skipped when !P.scale) with its sums
  auto sweep_scale = [&]() {
    float col[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) col[k] = 0.f;
    for (int r = g; r < R; r += 2) {
      float x[CH];
      load_row(r, x);
      float r0s = 0.f, r1s = 0.f;
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const float y = P.scale ? (float)(sc * (double)x[k]) : x[k];
        x[k] = y;
        col[k] += y;
        if (k & 1) r1s += y; else r0s += y;
      }
      if (P.scale) store_row(r, x);
      put_rowparts(r, r0s + r1s, -1, 0.f);
    }
    sweep_epilogue(col, 1u);
  };

  // one SDSN pass on one row slice: y ← max(0, (y + a_i) + b_j) (P2∘P1, R9 grouping) with paired
  // FP32 adds (add.rn.f32x2: x+a, +b, column and row accumulation).  For CPT = 32 the row partial goes
  // into two accumulators (alternate column pairs), halving its FADD2 dependency chain: 6.41 vs 6.58 µs
  // per pass at n = 4096 (A/B on one B200, profiles/r02/ab_k4r_r02n.log; at CPT = 16 it measured 2%
  // slower and four accumulators 7% slower at CPT = 32, so only CPT = 32 takes it)
  constexpr bool kRs2 = (CPT == 32);
  auto pass_rows = [&](float (&x)[CH], float a, const float2 (&bv)[CH / 2], float2 (&col2)[CH / 2]) -> float {
    float2 rs = make_float2(0.f, 0.f), rs2 = make_float2(0.f, 0.f);
    const float2 a2 = make_float2(a, a);
#pragma unroll
    for (int k = 0; k < CH; k += 2) {
      float2 y = add2(add2(make_float2(x[k], x[k + 1]), a2), bv[k / 2]);
      y.x = fmaxf(0.0f, y.x);
      y.y = fmaxf(0.0f, y.y);
      x[k] = y.x;
      x[k + 1] = y.y;
      col2[k / 2] = add2(col2[k / 2], y);
      if (kRs2 && ((k / 2) & 1)) rs2 = add2(rs2, y);
      else rs = add2(rs, y);
    }
    if (kRs2) rs = add2(rs, rs2);
    return rs.x + rs.y;
  };
  auto arow = [&](int r) -> float { return s_af[r]; };   // a_i, precomputed by the S warp (wait_S)
  auto sweep_pass = [&](const float2 (&bv)[CH / 2], unsigned e) {
    const long long l0 = gt();
    const long long c0k = P.dbg ? clock64() : 0;
    float2 col2[CH / 2];
#pragma unroll
    for (int k = 0; k < CH / 2; ++k) col2[k] = make_float2(0.f, 0.f);
    // rows of this row group: with rows in both TMEM and shared memory, group 0 takes the TMEM rows
    // and group 1 the shared-memory rows so the two datapaths work concurrently; otherwise rows
    // alternate between the groups.  Each datapath has its own loop (no per-row kind test).
    // A warp's rows rbeg, rbeg + rstep, … < rend go in batches of 8 (4 pairs); the per-lane row
    // partials of a batch stay in registers and are reduced together by put_rowparts8 after the
    // batch, so no shuffle chain sits between one pair's stores and the next pair's loads.
    auto rows_tmem = [&](int rbeg, int rend, int rstep) {
      for (int i0 = rbeg; i0 < rend; i0 += 8 * rstep) {
        float rsv[8];
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          const int ra = i0 + i * rstep, rb = ra + rstep;
          rsv[i] = 0.f;
          rsv[i + 1] = 0.f;
          if (rb < rend) {                               // two rows, one wait for both loads
            uint32_t va[CH], vb[CH];
            tmem_ld<CH>(tmem + (uint32_t)(ra * CPT), va);
            tmem_ld<CH>(tmem + (uint32_t)(rb * CPT), vb);
            tmem_wait_ld();
            float xa[CH], xb[CH];
#pragma unroll
            for (int k = 0; k < CH; ++k) { xa[k] = __uint_as_float(va[k]); xb[k] = __uint_as_float(vb[k]); }
            rsv[i] = pass_rows(xa, arow(ra), bv, col2);
            rsv[i + 1] = pass_rows(xb, arow(rb), bv, col2);
#pragma unroll
            for (int k = 0; k < CH; ++k) { va[k] = __float_as_uint(xa[k]); vb[k] = __float_as_uint(xb[k]); }
            tmem_st<CH>(tmem + (uint32_t)(ra * CPT), va);
            tmem_st<CH>(tmem + (uint32_t)(rb * CPT), vb);
          } else if (ra < rend) {
            float xa[CH];
            load_row(ra, xa);
            rsv[i] = pass_rows(xa, arow(ra), bv, col2);
            store_row(ra, xa);
          }
        }
        put_rowparts_n(std::integral_constant<int, 8>{}, i0, rstep, rend, rsv);
      }
    };
    auto rows_smem = [&](int rbeg, int rend) {
      for (int i0 = rbeg; i0 < rend; i0 += 4) {
        float rsv[4];
#pragma unroll
        for (int i = 0; i < 4; i += 2) {
          const int ra = i0 + i;
          rsv[i] = 0.f;
          rsv[i + 1] = 0.f;
          if (ra + 1 < rend) {
            float4* pa = s_rows + (size_t)(ra - RT) * (V * 128) + c0 * 128 + t;
            float4* pb = pa + V * 128;
            float xa[CH], xb[CH];
#pragma unroll
            for (int c = 0; c < VH; ++c) {
              const float4 u = pa[c * 128], w = pb[c * 128];
              xa[4 * c] = u.x; xa[4 * c + 1] = u.y; xa[4 * c + 2] = u.z; xa[4 * c + 3] = u.w;
              xb[4 * c] = w.x; xb[4 * c + 1] = w.y; xb[4 * c + 2] = w.z; xb[4 * c + 3] = w.w;
            }
            rsv[i] = pass_rows(xa, arow(ra), bv, col2);
            rsv[i + 1] = pass_rows(xb, arow(ra + 1), bv, col2);
#pragma unroll
            for (int c = 0; c < VH; ++c) {
              pa[c * 128] = make_float4(xa[4 * c], xa[4 * c + 1], xa[4 * c + 2], xa[4 * c + 3]);
              pb[c * 128] = make_float4(xb[4 * c], xb[4 * c + 1], xb[4 * c + 2], xb[4 * c + 3]);
            }
          } else if (ra < rend) {
            float xa[CH];
            load_row(ra, xa);
            rsv[i] = pass_rows(xa, arow(ra), bv, col2);
            store_row(ra, xa);
          }
        }
        put_rowparts_n(std::integral_constant<int, 4>{}, i0, 1, rend, rsv);
      }
    };
    if (R > RT) {
      if (g == 0) rows_tmem(0, RT, 1);
      else rows_smem(RT, R);
    } else {
      rows_tmem(g, R, 2);
    }
    float col[CH];
#pragma unroll
    for (int k = 0; k < CH / 2; ++k) { col[2 * k] = col2[k].x; col[2 * k + 1] = col2[k].y; }
    if (P.dbg && lane == 0 && (warp & 7) == 0) {
      s_dbg[9 + g] += gt() - l0;
      s_dbg[11 + g] += clock64() - c0k;
    }
    sweep_epilogue(col, e);
  };

  // slot slice b of epoch e: lane ↔ slot, warp ↔ source CTA k ≡ warp (mod NW); each source word is
  // re-read until it carries tag e.  FP64 accumulation in the fixed order k = warp, warp+NW, …,
  // then the NW warps combined in order (deterministic).  Publishes b = −c/n tagged e and
  // leaves S (Σ of the per-CTA row-sum partials, tagged e) in s_S.
  auto slice = [&](unsigned e) {
    // slice boundaries on whole 32-byte sectors (8 slots), so every sector of b is written by ONE
    // slot owner: with boundaries anywhere (b·NS/G) two CTAs wrote parts of a sector and every pass
    // paid for it — n = 4096: 6.38 → 6.23 µs per pass, n = 3000: 6.18 → 5.38, n = 2000: 4.53 → 3.61
    // (A/B on one B200, profiles/r02/ab_k4r_slice_align.log; 128-byte lines measured the same)
    constexpr int SA = 8;
    const int s0 = SA * (int)((long)b * (NS / SA) / G), s1 = SA * (int)((long)(b + 1) * (NS / SA) / G);
    constexpr int NI = (32 * kResKMax + NW - 1) / NW;
    for (int sb = s0; sb < s1; sb += 32) {
      const int s = sb + lane;
      double acc = 0.0;
      if (s < s1) {
        unsigned w[NI];
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const int k = warp + i * NW;
          w[i] = k < G ? ld_w(P.colpart + (long)k * NS + s) : ptag(0.f, e);
        }
        bool ok;
        do {
          ok = true;
#pragma unroll
          for (int i = 0; i < NI; ++i)
            if (!pok(w[i], e)) { ok = false; w[i] = ld_w(P.colpart + (long)(warp + i * NW) * NS + s); }
        } while (!ok);
#pragma unroll
        for (int i = 0; i < NI; ++i) acc += (double)pval(w[i]);
      }
      s_red2[warp][lane] = acc;
      __syncthreads();
      if (sb == s0) stamp(4);
      if (warp == 0 && s < s1) {
        double v[NW];                                    // the NW warp sums, fixed pairwise tree
#pragma unroll
        for (int w = 0; w < NW; ++w) v[w] = s_red2[w][lane];
#pragma unroll
        for (int st = 1; st < NW; st *= 2)
#pragma unroll
          for (int w = 0; w < NW; w += 2 * st) v[w] += v[w + st];
        const double cs = v[0];
        const int f = s >> 2, e4 = s & 3, c = f >> 7, tt = f & 127;
        const long colj = (long)tt * CPT + 4 * c + e4;
        // |b_j| = c_j/n by the one-FMA correction of the correctly rounded reciprocal (= the IEEE quotient,
        // see div_n): the FP64 division left the critical path of every pass (n = 4096: 6.25 → 6.19 µs,
        // profiles/r02/ab_k4r_bdiv.log; an earlier version of the kernel had measured no gain)
        st_w(P.bvec + s, ptag(colj < n ? (float)div_n(cs, dn, rn) : CUDART_INF_F, e));
      }
      if (sb + 32 < s1) __syncthreads();               // s_red2 is reused by the next chunk
    }
  };
  // S of epoch e (row-sum partials, parity buffer), waited for by one warp while the others wait for b
  auto wait_S = [&](unsigned e) {
    double sacc = 0.0;
    double v[kResKMax];
    wait_d1_lanes<kResKMax>(P.Spart + (size_t)(e & 1) * G, G, lane, (e >> 1) & 1u, v);
#pragma unroll
    for (int i = 0; i < kResKMax; ++i) sacc += v[i];      // absent words are +0: same sum as before
    sacc = warp_sum_d(sacc);
    if (lane == 0) s_S = sacc;
    // a_i = (1/n + S/n²) − r_i/n of every row, in FP64 and rounded once to FP32, for the coming sweep
    // (this warp wrote s_rn in the previous epilogue): the sweep then reads one float per row instead
    // of an FP64 subtract and convert; n = 3000: 5.38 → 5.12 µs per pass, n = 4096 within noise
    // (profiles/r02/ab_k4r_af.log)
    const double ab = rn + div_n(sacc, nn, rnn);
    if (lane < R) s_af[lane] = (float)(ab - s_rn[lane]);
  };

  // ---------------- phase S: Y0 = s·X (on chip) and its sums ----------------
  long long tk1 = 0;
  if (P.dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tk1));
  sweep_scale();
  unsigned ep = 1;                                       // epoch of the current exchange
  slice(ep);
  __syncthreads();

  // ---------------- pass loop (device-side stop decision, identical in every CTA) ----------------
  int j = 0;
  double gam = 0.0;
  auto now = [&]() -> long long {
    long long v = 0;
    if (P.dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
  };
  for (;; ++j) {
    jst = j;
    stamp(0);
    long long t0 = now();
    // pass boundary: row group 0 waits for the b values of epoch ep (its columns are those of group
    // 1) and hands them to group 1 through shared memory (s_col), while the first warp of group 1
    // collects S — half the L2 polling traffic of every thread polling its own words
    float2 bv[CH / 2];                                   // b_j pairs (register pairs for FADD2)
    if (g == 0) {
      uint4 w[VH];
      const unsigned* myb = P.bvec;
#pragma unroll
      for (int c = 0; c < VH; ++c) w[c] = ld_w4(myb + (size_t)((c0 + c) * 128 + t) * 4);
      bool ok;
      do {                                               // wait for every b of epoch ep
        ok = true;
#pragma unroll
        for (int c = 0; c < VH; ++c) {
          if (!pok(w[c].x, ep) || !pok(w[c].y, ep) || !pok(w[c].z, ep) || !pok(w[c].w, ep)) {
            ok = false;
            w[c] = ld_w4(myb + (size_t)((c0 + c) * 128 + t) * 4);
          }
        }
      } while (!ok);
      stamp(1);
#pragma unroll
      for (int c = 0; c < VH; ++c) {                     // b = −|b|; −0 and −∞ (padding) as stored
        const float4 v = make_float4(-pval(w[c].x), -pval(w[c].y), -pval(w[c].z), -pval(w[c].w));
        s_col[(c0 + c) * 128 + t] = v;
        bv[2 * c] = make_float2(v.x, v.y);
        bv[2 * c + 1] = make_float2(v.z, v.w);
      }
    } else if (warp == NW / 2) {
      wait_S(ep);
    }
    __syncthreads();
    if (g == 1) {
#pragma unroll
      for (int c = 0; c < VH; ++c) {
        const float4 v = s_col[(c0 + c) * 128 + t];
        bv[2 * c] = make_float2(v.x, v.y);
        bv[2 * c + 1] = make_float2(v.z, v.w);
      }
    }
    stamp(2);
    const double S = s_S;                               // written by wait_S, synced
    gam = div_n(S, dn, rn) - 1.0;                                       // γ_j = S/n − 1
    if (b == 0 && tid == 0 && P.gamma_hist) P.gamma_hist[j] = gam;
    const bool last = P.sdsn_fixed > 0 ? (j + 1 >= P.sdsn_fixed)
                                       : ((j >= 1 && gam <= P.gamma_th) || j + 1 >= P.sdsn_max);
    long long t1 = now();
    sweep_pass(bv, last ? 0u : ep + 1);
    long long t2 = now();
    stamp(3);
    if (last) {
      __syncthreads();
      break;
    }
    ++ep;
    slice(ep);
    stamp(5);
    long long t4 = now();
    dadd(0, t1 - t0); dadd(1, t2 - t1); dadd(8, t4 - t2);
  }
  if (P.dbg && tid == 0) {
    for (int k = 0; k < 16; ++k) P.dbg[b * 16 + k] = s_dbg[k];
    long long tk2;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tk2));
    P.dbg[b * 16 + 5] = (j & 0xffff) | ((tk1 - tk0) << 16);         // passes | load-phase ns
    P.dbg[b * 16 + 3] = tk2 - tk0;                                   // total ns to loop end
  }

  // ---------------- D = Y_final → global (row-major, ld) ----------------
  for (int r = g; r < R; r += 2) {
    float x[CH];
    load_row(r, x);
    float* grow = P.Y + (r0 + r) * ld;
#pragma unroll
    for (int c = 0; c < VH; ++c) {
      const long col = (long)t * CPT + 4 * (c0 + c);
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
  const size_t ns = RC<CPT>::NS;
  p.Spart = p.xchg;                                      // [2][G] u64, tag bit 1 initially (0x80 bytes)
  p.Mpart = p.Spart + 2 * (size_t)G;                     // [G] u64
  p.colpart = reinterpret_cast<unsigned*>(p.xchg + ((3 * (size_t)G + 1) & ~(size_t)1));   // [G][NS] u32, 16-B aligned
  p.bvec = p.colpart + (size_t)G * ns;                   // [NS] u32
  e = cudaMemsetAsync(p.Spart, 0, (size_t)G * sizeof(uint64_t), st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(p.Spart + G, 0x80, (size_t)G * sizeof(uint64_t), st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(p.Mpart, 0, (size_t)G * sizeof(uint64_t) + 8 + ((size_t)G * ns + ns) * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  void* args[] = {&p};
  return cudaLaunchCooperativeKernel((const void*)fn, dim3(G), dim3(RK<CPT>::THREADS), args, dsm, st);
}

}  // namespace

int sdsn_res_grid(long n, int num_sms) {
  const int cpt = cpt_for(n);
  if (cpt == 0) return 0;
  long G = (n + 15) / 16;                               // ~16 rows per CTA, more CTAs if needed
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

size_t sdsn_res_xchg_words(long n, int num_sms) {         // in 8-byte words
  const size_t ns = (size_t)sdsn_res_slots(n);
  return 3 * (size_t)num_sms + 2 + ((size_t)num_sms * ns + ns + 1) / 2;
}

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
