// sdsn_pipe.cu — K4p: SDSN (Alg. 2 of arXiv 2508.00887), FP32, iterate held
// ON-CHIP (TMEM + shared memory) like K4r (sdsn_resident.cu), with the per-pass column all-reduce
// PIPELINED behind the sweep.
//
// Same arithmetic and stopping rule as K4r / K4 (readings R5, R9-R13):
//   γ_j = S_j/n − 1;  a_i = (1/n + S_j/n²) − r_i/n;  b_j = −c_j/n  (FP64, rounded to FP32)
//   Y_{j+1} = max(0, (Y_j + a_i) + b_j)   with r, c, S of Y_{j+1} fused into the same sweep.
//
// Why.  In K4r a pass is: sweep all columns (≈3.1 µs at n = 4096) → publish column partials → hop 1
// (owners poll the partials of all 148 CTAs) → owners reduce and publish b → hop 2 (every CTA polls
// b) → next sweep: the two L2 hops and their polling (≈3.4 µs) sit on the critical path of every pass.
// Here every pass sweeps the columns in two halves, A then B (for thread t: A = its first CPT/2
// columns, B = the last CPT/2), and publishes each half's column partials as soon as that half is
// swept.  So hop 1 of half A travels while half B is swept, the owners reduce half A without waiting,
// and b_A of the next pass is visible before it is needed; b_B's hops travel while the owners reduce
// half A and wait for the mass S (the one exchange that needs the whole pass on every CTA), and
// while half A of the next pass is swept.  Per pass: sweep A + sweep B + the S hop + two slice
// reductions, instead of a sweep + two hops + one reduction.
//
// Work split (n ≤ 4096, CPT = 32 or 16 columns per owner thread t = 32·(warp%4) + lane, as K4r).
// 16 warps: q = warp%4 (TMEM lane quarter), g = warp/4 (row group).  With R rows per CTA, RT = 512/CPT
// of them in TMEM and the rest in shared memory: g0 / g1 take the two halves of the TMEM rows, g2 / g3
// the two halves of the shared-memory rows (the two datapaths run concurrently; K4r measured 16 TMEM
// rows ≈ 12 shared-memory rows per 8 warps).  A thread sweeps its group's rows over the CPT/2 columns
// of the current half.  Column partials: groups 1 and 3 hand theirs to groups 0 and 2 through shared
// memory, and groups 0 and 2 publish (g0+g1) and (g2+g3): two sources per CTA, 2G in total.  Row sums:
// per warp and half in s_rowpart[row][half·4 + q], combined in FP64 in a fixed order after half B.
// Every published value is a tagged word (epoch parity in the sign bit, K4r's exchange, xchg.cuh);
// one parity bit suffices because nobody publishes epoch e+1 of a word before every reader of epoch e
// has read it (each such publication needs data that every reader produces only after reading).
#include <math_constants.h>
#include <type_traits>
#include "common.cuh"
#include "internal.h"
#include "tmem_ldst.cuh"
#include "xchg.cuh"

namespace fram {
namespace {

constexpr int kPipeSmemMax = 232448 - 2048;   // 227 KB opt-in minus static shared memory (≤ 2 KB)
constexpr int kPipeMinSmem = 120 * 1024;      // one CTA per SM (TMEM: 512 columns per CTA)
constexpr int kPipeMaxRows = 32;              // rows per CTA (lane ↔ row in the row-sum combine)
constexpr int kThreads = 512, kWarps = 16;

template <int CPT> struct PC {
  static constexpr int V = CPT / 4;           // float4 chunks per thread per row
  static constexpr int NS = 128 * CPT;        // slots = padded columns
  static constexpr int HS = NS / 2;           // slots per half
  static constexpr int RT = 512 / CPT;        // rows held in TMEM
  static constexpr int CH = CPT / 2;          // columns per thread per half
  static constexpr int VH = CH / 4;           // float4 chunks per thread per half
};

// dynamic shared memory: shared-memory rows, column hand-off (2 × half), b hand-off (half),
// per-warp row partials, s_r, s_rn
size_t pipe_smem_bytes(int cpt, int rs, int R) {
  const size_t ns = 128 * (size_t)cpt;
  return (size_t)rs * ns * 4 + ns * 4 + ns / 2 * 4 + (size_t)R * 8 * 4 + (size_t)R * 8 * 2 + 64;
}

template <int CPT>
__global__ void __launch_bounds__(kThreads, 1) sdsn_pipe_kernel(ResParams P) {
  using C = PC<CPT>;
  constexpr int V = C::V, NS = C::NS, HS = C::HS, RT = C::RT, CH = C::CH, VH = C::VH;
  constexpr int NI = (2 * 32 * 5 + kWarps - 1) / kWarps;      // sources per lane per warp (2G ≤ 320)
  extern __shared__ __align__(16) unsigned char dsm[];
  const int RS = P.rs;
  const int Rmax = P.rmax;
  float4* s_rows = reinterpret_cast<float4*>(dsm);                    // [RS][V·128] slot layout
  float4* s_col = s_rows + (size_t)RS * V * 128;                      // [2][VH·128] column hand-off
  float4* s_bh = s_col + 2 * VH * 128;                                // [VH·128] b hand-off (one half)
  float* s_rowpart = reinterpret_cast<float*>(s_bh + VH * 128);       // [Rmax][8] per-warp row partials
  double* s_r = reinterpret_cast<double*>(s_rowpart + Rmax * 8);     // [Rmax] row sums (FP64)
  double* s_rn = s_r + Rmax;                                          // [Rmax] r_i / n
  __shared__ uint32_t s_tmem;
  __shared__ double s_red[kWarps];
  __shared__ double s_S;

  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = warp & 3, g = warp >> 2;
  const int t = q * 32 + lane;
  const long n = P.n, ld = P.ld;
  const long r0 = (long)b * n / G, r1 = (long)(b + 1) * n / G;
  const int R = (int)(r1 - r0);
  const double dn = (double)n, nn = dn * dn;
  const double rn = __drcp_rn(dn), rnn = __drcp_rn(nn);
  auto div_n = [&](double S_, double d, double r) {     // RN(S/d) by one FMA correction (as K4r)
    const double qq = S_ * r;
    return fma(r, fma(-qq, d, S_), qq);
  };
  // this group's rows: TMEM rows [0, RTu) split by g0/g1, shared-memory rows [RT, R) by g2/g3; with no
  // shared-memory rows all four groups split the TMEM rows
  const int RTu = R < RT ? R : RT;
  int rb, re;
  if (R > RT) {
    const int hs = RT + (R - RT + 1) / 2;
    rb = g == 0 ? 0 : g == 1 ? RT / 2 : g == 2 ? RT : hs;
    re = g == 0 ? RT / 2 : g == 1 ? RT : g == 2 ? hs : R;
  } else {
    rb = g * RTu / 4;
    re = (g + 1) * RTu / 4;
  }
  const bool in_tmem = rb < RT;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem + ((uint32_t)(q * 32) << 16);           // lane quarter
  auto dealloc = [&]() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(512));
  };
  // half `hh` of row r: TMEM columns r·CPT + hh·CH, or float4 chunks hh·VH … of the shared-memory row
  auto load_half = [&](int r, int hh, float (&x)[CH]) {
    if (r < RT) {
      uint32_t v[CH];
      tmem_ld<CH>(tmem + (uint32_t)(r * CPT + hh * CH), v);
      tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < CH; ++k) x[k] = __uint_as_float(v[k]);
    } else {
      const float4* row = s_rows + (size_t)(r - RT) * (V * 128) + hh * VH * 128 + t;
#pragma unroll
      for (int c = 0; c < VH; ++c) {
        const float4 v = row[c * 128];
        x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
      }
    }
  };
  auto store_half = [&](int r, int hh, const float (&x)[CH]) {
    if (r < RT) {
      uint32_t v[CH];
#pragma unroll
      for (int k = 0; k < CH; ++k) v[k] = __float_as_uint(x[k]);
      tmem_st<CH>(tmem + (uint32_t)(r * CPT + hh * CH), v);
    } else {
      float4* row = s_rows + (size_t)(r - RT) * (V * 128) + hh * VH * 128 + t;
#pragma unroll
      for (int c = 0; c < VH; ++c) row[c * 128] = make_float4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
    }
  };

  // ---------------- phase L: X rows → on-chip, m = max X (Alg.2 step 1) ----------------
  {
    float lmax = 0.f;
    for (int r = rb; r < re; ++r) {
      const float* grow = P.Y + (r0 + r) * ld;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        float x[CH];
#pragma unroll
        for (int c = 0; c < VH; ++c) {
          const long col = (long)t * CPT + hh * CH + 4 * c;
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
        store_half(r, hh, x);
      }
    }
    tmem_wait_st();
    double m = warp_max_d((double)lmax);
    if (lane == 0) s_red[warp] = m;
    __syncthreads();
    if (tid == 0) {
      double mm = 0.0;
      for (int w = 0; w < kWarps; ++w) mm = fmax(mm, s_red[w]);
      st_d1(P.Mpart + b, mm, 1u);
    }
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
      for (int r = rb; r < re; ++r) {
        float* grow = P.Y + (r0 + r) * ld;
        for (long col = t; col < n; col += 128) grow[col] = (float)(1.0 / dn);
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

  // this warp's partials of the NB rows i0 + k (k < NB, rows ≥ rend absent), half hh: one transpose-
  // reduce (NB = 8: 9 shuffles for 8 rows) into s_rowpart[row][hh·4 + q] (fixed tree, deterministic)
  auto put_rowparts8 = [&](int i0, int rend, int hh, float* v) {
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      const int off = 16 >> l, m = 8 >> (l + 1);
      const bool hi = lane & off;
#pragma unroll
      for (int i = 0; i < m; ++i) v[i] = (hi ? v[i + m] : v[i]) + __shfl_xor_sync(0xffffffffu, hi ? v[i] : v[i + m], off);
    }
    float z = v[0];
#pragma unroll
    for (int off = 2; off > 0; off >>= 1) z += __shfl_xor_sync(0xffffffffu, z, off);
    const int r = i0 + (lane >> 2);
    if ((lane & 3) == 0 && r < rend) s_rowpart[r * 8 + hh * 4 + q] = z;
  };
  // y ← max(0, (y + a_i) + b_j) on CH columns, paired FP32 adds (add.rn.f32x2)
  auto pass_cols = [&](float (&x)[CH], float a, const float2 (&bv)[CH / 2], float2 (&col2)[CH / 2]) -> float {
    float2 rs = make_float2(0.f, 0.f);
    const float2 a2 = make_float2(a, a);
#pragma unroll
    for (int k = 0; k < CH; k += 2) {
      float2 y = add2(add2(make_float2(x[k], x[k + 1]), a2), bv[k / 2]);
      y.x = fmaxf(0.0f, y.x);
      y.y = fmaxf(0.0f, y.y);
      x[k] = y.x;
      x[k + 1] = y.y;
      col2[k / 2] = add2(col2[k / 2], y);
      rs = add2(rs, y);
    }
    return rs.x + rs.y;
  };
  auto scale_cols = [&](float (&x)[CH], float2 (&col2)[CH / 2]) -> float {
    float r0s = 0.f, r1s = 0.f;
#pragma unroll
    for (int k = 0; k < CH; k += 2) {
      const float y0 = P.scale ? (float)(sc * (double)x[k]) : x[k];
      const float y1 = P.scale ? (float)(sc * (double)x[k + 1]) : x[k + 1];
      x[k] = y0;
      x[k + 1] = y1;
      col2[k / 2] = add2(col2[k / 2], make_float2(y0, y1));
      r0s += y0;
      r1s += y1;
    }
    return r0s + r1s;
  };
  double abase = 0.0;                                    // 1/n + S/n² of the current pass
  // one half-sweep of this group's rows; col2 returns the thread's column partials over the rows
  auto sweep_half = [&](int hh, bool scale_mode, const float2 (&bv)[CH / 2], float2 (&col2)[CH / 2]) {
#pragma unroll
    for (int k = 0; k < CH / 2; ++k) col2[k] = make_float2(0.f, 0.f);
    for (int i0 = rb; i0 < re; i0 += 8) {
      float rsv[8];
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        const int ra = i0 + i, rb2 = ra + 1;
        rsv[i] = 0.f;
        rsv[i + 1] = 0.f;
        if (rb2 < re) {
          float xa[CH], xb[CH];
          if (in_tmem) {                                 // two rows, one wait for both loads
            uint32_t va[CH], vb[CH];
            tmem_ld<CH>(tmem + (uint32_t)(ra * CPT + hh * CH), va);
            tmem_ld<CH>(tmem + (uint32_t)(rb2 * CPT + hh * CH), vb);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < CH; ++k) { xa[k] = __uint_as_float(va[k]); xb[k] = __uint_as_float(vb[k]); }
          } else {
            load_half(ra, hh, xa);
            load_half(rb2, hh, xb);
          }
          if (scale_mode) {
            rsv[i] = scale_cols(xa, col2);
            rsv[i + 1] = scale_cols(xb, col2);
          } else {
            rsv[i] = pass_cols(xa, (float)(abase - s_rn[ra]), bv, col2);
            rsv[i + 1] = pass_cols(xb, (float)(abase - s_rn[rb2]), bv, col2);
          }
          store_half(ra, hh, xa);
          store_half(rb2, hh, xb);
        } else if (ra < re) {
          float xa[CH];
          load_half(ra, hh, xa);
          rsv[i] = scale_mode ? scale_cols(xa, col2) : pass_cols(xa, (float)(abase - s_rn[ra]), bv, col2);
          store_half(ra, hh, xa);
        }
      }
      put_rowparts8(i0, re, hh, rsv);
    }
    tmem_wait_st();
  };
  // groups 1 / 3 hand their column partials of half hh to groups 0 / 2 (call before a barrier)
  auto handoff_cols = [&](const float2 (&col2)[CH / 2]) {
    if (g & 1) {
      float4* dst = s_col + (g >> 1) * VH * 128 + t;
#pragma unroll
      for (int c = 0; c < VH; ++c)
        dst[c * 128] = make_float4(col2[2 * c].x, col2[2 * c].y, col2[2 * c + 1].x, col2[2 * c + 1].y);
    }
  };
  // groups 0 / 2 publish (own + partner) as source 2b + g/2, slots hh·HS + …, tag e (after the barrier)
  auto publish_cols = [&](int hh, const float2 (&col2)[CH / 2], unsigned e) {
    if (!(g & 1)) {
      const float4* src = s_col + (g >> 1) * VH * 128 + t;
      unsigned* dst = P.colpart + (size_t)(2 * b + (g >> 1)) * NS + (size_t)hh * HS;
#pragma unroll
      for (int c = 0; c < VH; ++c) {
        float4 o = src[c * 128];
        o.x += col2[2 * c].x; o.y += col2[2 * c].y; o.z += col2[2 * c + 1].x; o.w += col2[2 * c + 1].y;
        st_w4(dst + (size_t)(c * 128 + t) * 4, make_uint4(ptag(o.x, e), ptag(o.y, e), ptag(o.z, e), ptag(o.w, e)));
      }
    }
  };
  // slot slice b of half hh, epoch e: lane ↔ slot, warp ↔ sources k ≡ warp (mod 16) of the 2G; each
  // source word is re-read until it carries tag e.  FP64 accumulation in the fixed order k = warp,
  // warp+16, …, then the 16 warps combined by a fixed pairwise tree.  Publishes |b_j| = c_j/n tagged e.
  auto reduce_slice = [&](int hh, unsigned e) {
    const int K = 2 * G;
    const int s0 = (int)((long)b * HS / G), s1 = (int)((long)(b + 1) * HS / G);
    // [16 warps][32] FP64 partials.  Half A's live in s_bh (free from SYNC3's reads until the next pass's
    // poll_b, which the g0 warps reach only after reduce B's barrier, i.e. after warp 0 read them);
    // half B's in s_col (its publish_cols reads precede reduce A's barrier; the next writes follow SYNC1)
    double (*red)[32] = reinterpret_cast<double (*)[32]>(hh == 0 ? s_bh : s_col);
    for (int sb = s0; sb < s1; sb += 32) {
      const int s = sb + lane;
      double acc = 0.0;
      if (s < s1) {
        const unsigned* base = P.colpart + (size_t)hh * HS + s;
        unsigned w[NI];
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const int k = warp + i * kWarps;
          w[i] = k < K ? ld_w(base + (size_t)k * NS) : ptag(0.f, e);
        }
        bool ok;
        do {
          ok = true;
#pragma unroll
          for (int i = 0; i < NI; ++i)
            if (!pok(w[i], e)) { ok = false; w[i] = ld_w(base + (size_t)(warp + i * kWarps) * NS); }
        } while (!ok);
#pragma unroll
        for (int i = 0; i < NI; ++i) acc += (double)pval(w[i]);
      }
      red[warp][lane] = acc;
      __syncthreads();
      if (warp == 0 && s < s1) {
        double v[kWarps];
#pragma unroll
        for (int w2 = 0; w2 < kWarps; ++w2) v[w2] = red[w2][lane];
#pragma unroll
        for (int st = 1; st < kWarps; st *= 2)
#pragma unroll
          for (int w2 = 0; w2 < kWarps; w2 += 2 * st) v[w2] += v[w2 + st];
        const int gs = hh * HS + s;                      // global slot → column
        const int f = gs >> 2, e4 = gs & 3, c = f >> 7, tt = f & 127;
        const long colj = (long)tt * CPT + 4 * c + e4;
        st_w(P.bvec + gs, ptag(colj < n ? (float)(v[0] / dn) : CUDART_INF_F, e));
      }
      if (sb + 32 < s1) __syncthreads();               // red is reused by the next chunk
    }
  };
  // g0 threads: poll |b| of half hh (epoch e) for columns of owner t into registers and s_bh
  auto poll_b = [&](int hh, unsigned e, float2 (&bv)[CH / 2]) {
    uint4 w[VH];
    const unsigned* myb = P.bvec + (size_t)hh * HS;
#pragma unroll
    for (int c = 0; c < VH; ++c) w[c] = ld_w4(myb + (size_t)(c * 128 + t) * 4);
    bool ok;
    do {
      ok = true;
#pragma unroll
      for (int c = 0; c < VH; ++c) {
        if (!pok(w[c].x, e) || !pok(w[c].y, e) || !pok(w[c].z, e) || !pok(w[c].w, e)) {
          ok = false;
          w[c] = ld_w4(myb + (size_t)(c * 128 + t) * 4);
        }
      }
    } while (!ok);
#pragma unroll
    for (int c = 0; c < VH; ++c) {                     // b = −|b|; −0 and −∞ (padding) as stored
      const float4 v = make_float4(-pval(w[c].x), -pval(w[c].y), -pval(w[c].z), -pval(w[c].w));
      s_bh[c * 128 + t] = v;
      bv[2 * c] = make_float2(v.x, v.y);
      bv[2 * c + 1] = make_float2(v.z, v.w);
    }
  };
  auto read_b = [&](float2 (&bv)[CH / 2]) {
#pragma unroll
    for (int c = 0; c < VH; ++c) {
      const float4 v = s_bh[c * 128 + t];
      bv[2 * c] = make_float2(v.x, v.y);
      bv[2 * c + 1] = make_float2(v.z, v.w);
    }
  };
  // after half B: row sums r_i (FP64, fixed order over the 8 per-warp partials), r_i/n, and this CTA's
  // Σ r_i published tagged (S partial of epoch e, parity buffer as K4r)
  auto rows_and_S = [&](unsigned e) {
    double acc = 0.0;
    if (lane < R) {
      const float* pp = s_rowpart + lane * 8;
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += (double)pp[k];
      s_r[lane] = acc;
      s_rn[lane] = acc / dn;
    }
    const double sp = warp_sum_d(acc);
    if (lane == 0) st_d1(P.Spart + (size_t)(e & 1) * G + b, sp, (e >> 1) & 1u);
  };
  auto wait_S = [&](unsigned e) {
    double sacc = 0.0;
    double v[5];
    wait_d1_lanes<5>(P.Spart + (size_t)(e & 1) * G, G, lane, (e >> 1) & 1u, v);
#pragma unroll
    for (int i = 0; i < 5; ++i) sacc += v[i];
    sacc = warp_sum_d(sacc);
    if (lane == 0) s_S = sacc;
  };

  // ---------------- phase S (epoch 1): Y0 = s·X on chip, its sums, b and S of Y0 ----------------
  float2 bv[CH / 2], col2[CH / 2];
#pragma unroll
  for (int k = 0; k < CH / 2; ++k) bv[k] = make_float2(0.f, 0.f);
  sweep_half(0, true, bv, col2);
  handoff_cols(col2);
  __syncthreads();
  publish_cols(0, col2, 1u);
  sweep_half(1, true, bv, col2);
  handoff_cols(col2);
  __syncthreads();
  publish_cols(1, col2, 1u);
  if (warp == 4) rows_and_S(1u);
  reduce_slice(0, 1u);
  reduce_slice(1, 1u);

  // ---------------- pass loop (device-side stop decision, identical in every CTA) ----------------
  int j = 0;
  double gam = 0.0;
  unsigned ein = 1;                                      // epoch of the pass input's b, S
  for (;; ++j, ++ein) {
    // pass start: g0 polls b_A(ein) → s_bh; warp 4 collects S(ein)
    if (g == 0) poll_b(0, ein, bv);
    else if (warp == 4) wait_S(ein);
    __syncthreads();                                     // SYNC1
    if (g != 0) read_b(bv);
    const double S = s_S;
    gam = div_n(S, dn, rn) - 1.0;                        // γ_j = S/n − 1
    if (b == 0 && tid == 0 && P.gamma_hist) P.gamma_hist[j] = gam;
    const bool last = P.sdsn_fixed > 0 ? (j + 1 >= P.sdsn_fixed)
                                       : ((j >= 1 && gam <= P.gamma_th) || j + 1 >= P.sdsn_max);
    abase = rn + div_n(S, nn, rnn);                      // 1/n + S/n²
    const unsigned eout = ein + 1;
    // half A
    sweep_half(0, false, bv, col2);
    handoff_cols(col2);
    __syncthreads();                                     // SYNC2: partner partials in s_col, s_bh free
    if (!last) publish_cols(0, col2, eout);
    if (g == 0) poll_b(1, ein, bv);                      // b_B(ein): published during our half A
    __syncthreads();                                     // SYNC3
    if (g != 0) read_b(bv);
    // half B
    sweep_half(1, false, bv, col2);
    handoff_cols(col2);
    __syncthreads();                                     // SYNC4
    if (last) break;
    publish_cols(1, col2, eout);
    if (warp == 4) rows_and_S(eout);
    reduce_slice(0, eout);                               // half A partials travelled during half B
    reduce_slice(1, eout);
  }

  // ---------------- D = Y_final → global (row-major, ld) ----------------
  for (int r = rb; r < re; ++r) {
    float* grow = P.Y + (r0 + r) * ld;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      float x[CH];
      load_half(r, hh, x);
#pragma unroll
      for (int c = 0; c < VH; ++c) {
        const long col = (long)t * CPT + hh * CH + 4 * c;
        if (col + 3 < n) {
          *reinterpret_cast<float4*>(grow + col) = make_float4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
        } else {
          if (col < n) grow[col] = x[4 * c];
          if (col + 1 < n) grow[col + 1] = x[4 * c + 1];
          if (col + 2 < n) grow[col + 2] = x[4 * c + 2];
        }
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

int cpt_pipe(long n) {
  if (n > 1024 && n <= 2048) return 16;
  if (n > 2048 && n <= 4096) return 32;
  return 0;
}

template <int CPT>
cudaError_t launch_pipe_t(ResParams p, cudaStream_t st, int G) {
  auto fn = sdsn_pipe_kernel<CPT>;
  const long R = (p.n + G - 1) / G;
  if (R > kPipeMaxRows || 2 * G > 2 * 32 * 5) return cudaErrorInvalidValue;
  p.rs = (int)(R > PC<CPT>::RT ? R - PC<CPT>::RT : 0);
  p.rmax = (int)R;
  size_t dsm = pipe_smem_bytes(CPT, p.rs, (int)R);
  if (dsm > (size_t)kPipeSmemMax) return cudaErrorInvalidValue;
  if (dsm < (size_t)kPipeMinSmem) dsm = kPipeMinSmem;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
  if (e != cudaSuccess) return e;
  const size_t ns = PC<CPT>::NS;
  p.Spart = p.xchg;                                      // [2][G] u64, tag bit 1 initially (0x80 bytes)
  p.Mpart = p.Spart + 2 * (size_t)G;                     // [G] u64
  p.colpart = reinterpret_cast<unsigned*>(p.xchg + ((3 * (size_t)G + 1) & ~(size_t)1));   // [2G][NS] u32
  p.bvec = p.colpart + 2 * (size_t)G * ns;               // [NS] u32
  e = cudaMemsetAsync(p.Spart, 0, (size_t)G * sizeof(uint64_t), st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(p.Spart + G, 0x80, (size_t)G * sizeof(uint64_t), st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(p.Mpart, 0, (size_t)G * sizeof(uint64_t) + 8 + (2 * (size_t)G * ns + ns) * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  void* args[] = {&p};
  return cudaLaunchCooperativeKernel((const void*)fn, dim3(G), dim3(kThreads), args, dsm, st);
}

}  // namespace

int sdsn_pipe_grid(long n, int num_sms) {
  const int cpt = cpt_pipe(n);
  if (cpt == 0) return 0;
  long G = (n + 15) / 16;
  if (G > num_sms) G = num_sms;
  if (G < 1) G = 1;
  auto R_of = [&](long G_) { return (int)((n + G_ - 1) / G_); };
  auto rs_of = [&](long G_) { const long e = R_of(G_) - 512 / cpt; return (int)(e > 0 ? e : 0); };
  auto fits = [&](long G_) {
    return R_of(G_) <= kPipeMaxRows && G_ <= 32 * 5 &&
           pipe_smem_bytes(cpt, rs_of(G_), R_of(G_)) <= (size_t)kPipeSmemMax;
  };
  while (G < num_sms && !fits(G)) ++G;
  if (!fits(G)) return 0;
  return (int)G;
}

size_t sdsn_pipe_xchg_words(long n, int num_sms) {        // in 8-byte words
  const size_t ns = 128 * (size_t)(cpt_pipe(n) ? cpt_pipe(n) : 32);
  return 3 * (size_t)num_sms + 2 + (2 * (size_t)num_sms * ns + ns + 1) / 2;
}

cudaError_t launch_sdsn_pipe(const ResParams& p, cudaStream_t st, int num_sms) {
  const int G = sdsn_pipe_grid(p.n, num_sms);
  if (G == 0) return cudaErrorInvalidValue;
  switch (cpt_pipe(p.n)) {
    case 16: return launch_pipe_t<16>(p, st, G);
    case 32: return launch_pipe_t<32>(p, st, G);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace fram
