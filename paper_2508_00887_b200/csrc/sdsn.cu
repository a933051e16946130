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
//              → colpart[b][:] → CTA b reduces column slice b over all CTAs in a fixed order
//              (deterministic, no float atomics: S:375) → c (FP64) → read by every CTA;
//   S        : Σ per-CTA row-sum partials, summed identically by every CTA (FP64).
// No grid barriers: every exchanged word carries its epoch's parity in the sign bit (the values
// are non-negative) and is re-read until the tag matches (the K4r exchange, xchg.cuh).
// Algorithmic bytes per pass: 8n² (FP32) / 16n² (FP64) of Y, + O(G·n) of partials.
#include <stdlib.h>
#include <algorithm>
#include <type_traits>
#include "common.cuh"
#include "internal.h"
#include "xchg.cuh"
#include "tmem_ldst.cuh"

namespace fram {

// Tagged words of the cross-CTA exchange (as in K4r, xchg.cuh): non-negative values with the epoch
// parity in the sign bit; a consumer re-reads a word until its tag matches, so no grid barrier is
// needed.  T = float: 4-byte words; T = double: 8-byte words.
template <typename T> struct Tag;
template <> struct Tag<float> {
  using W = unsigned;
  static __device__ __forceinline__ W make(float v, unsigned e) { return __float_as_uint(v) | ((e & 1u) << 31); }
  static __device__ __forceinline__ bool ok(W w, unsigned e) { return (w >> 31) == (e & 1u); }
  static __device__ __forceinline__ float val(W w) { return __uint_as_float(w & 0x7fffffffu); }
  static __device__ __forceinline__ W ld(const float* p) { return ld_w(reinterpret_cast<const unsigned*>(p)); }
  static __device__ __forceinline__ void st(float* p, float v, unsigned e) { st_w(reinterpret_cast<unsigned*>(p), make(v, e)); }
  static __device__ __forceinline__ void st4(float* p, const float* v, unsigned e) {
    st_w4(reinterpret_cast<unsigned*>(p), make_uint4(make(v[0], e), make(v[1], e), make(v[2], e), make(v[3], e)));
  }
};
template <> struct Tag<double> {
  using W = uint64_t;
  static __device__ __forceinline__ W make(double v, unsigned e) {
    return (uint64_t)__double_as_longlong(v) | ((uint64_t)(e & 1u) << 63);
  }
  static __device__ __forceinline__ bool ok(W w, unsigned e) { return (unsigned)(w >> 63) == (e & 1u); }
  static __device__ __forceinline__ double val(W w) { return __longlong_as_double((long long)(w & 0x7fffffffffffffffull)); }
  static __device__ __forceinline__ W ld(const double* p) { return ld_tag(reinterpret_cast<const uint64_t*>(p)); }
  static __device__ __forceinline__ void st(double* p, double v, unsigned e) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(make(v, e)) : "memory");
  }
  static __device__ __forceinline__ void st4(double* p, const double* v, unsigned e) {   // 2 words (double2)
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(make(v[0], e)), "l"(make(v[1], e))
                 : "memory");
  }
};

template <typename T> struct VecT;
template <> struct VecT<float>  { using t = float4;  static constexpr int W = 4; };
template <> struct VecT<double> { using t = double2; static constexpr int W = 2; };

#ifndef SDSN_PAIR
#define SDSN_PAIR 1
#endif
#ifndef SDSN_ONCHIP
#define SDSN_ONCHIP 1
#endif
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
// max(0, x) for FP64 by the sign bit (3 integer ops; fmax is a DSETP on the FP64 pipe plus 4-5
// selects for its NaN / signed-zero rules, which finite iterates never need: −0 → +0 either way)
__device__ __forceinline__ double tmax0(double x) {
  const long long v = __double_as_longlong(x);
  return __longlong_as_double(v & ~(v >> 63));
}
__device__ __forceinline__ float warp_sum_t(float v) { return warp_sum_f(v); }
__device__ __forceinline__ double warp_sum_t(double v) { return warp_sum_d(v); }

enum { SWEEP_SCALE = 0, SWEEP_PASS = 1 };

// OO ("on-chip only"): every row of every CTA is held in TMEM / shared memory (FP64, n ≲ 2070 on 148
// SMs); that instantiation has no streamed-row loop and takes the on-chip rows in pairs, which the
// streamed-row loop's registers do not allow (FP64 n = 4096 with pairs: 22.1 → 41.4 us/pass)
template <typename T, int VPL, bool OO>
__global__ void __launch_bounds__(kSdsnThreads, 1) sdsn_kernel(SdsnParams P, int CG, int NT, int NSM) {
  using VT = typename VecT<T>::t;
  constexpr int W = VecT<T>::W;
  // rows in flight per warp: 2 for VPL = 2 and 4 (16/VPL measured slower — the deeper ring pushed
  // the sweep into spills: FP64 n = 4096 32.4 → 27.4 us/pass, FP64 n = 2048 11.8 → 10.2, FP32
  // n = 6000 44.4 → 35.6; PD = 3 / 4 for VPL = 4 / 2 in between)
  constexpr int PD = VPL >= 8 ? 1 : VPL >= 2 ? 2 : 16;
  constexpr int WPR = VPL * (int)sizeof(VT) / 4;             // 32-bit words per thread per row
  extern __shared__ __align__(16) unsigned char dsm[];
  const long rows_max = (P.n + gridDim.x - 1) / gridDim.x + 1;
  // b of the thread's column slots in shared memory for VPL = 8 ([VPL][threads], conflict-free):
  // in registers they pushed the sweep into spills (32 FP32 / 64 FP64 registers); with the 2-row
  // ring VPL = 4 keeps them in registers without spills (and one more on-chip row fits)
  constexpr bool BSM = VPL >= 8;
  double* s_rowpart = reinterpret_cast<double*>(dsm);       // [rows_max][CG]
  VT* s_bv = reinterpret_cast<VT*>(dsm + ((sizeof(double) * rows_max * CG + 15) & ~15ul));   // [VPL][threads] (BSM)
  // column accumulators in shared memory as well for FP64 with VPL = 8 (CSM; one 16-byte read-modify-
  // write per vector instead of 16 FP64 registers): FP64 n = 8192 221.7 → 174.6 us/pass; FP32 VPL = 8
  // (365 vs 355) and VPL = 4 (+3-5%) are faster with register accumulators
  constexpr bool CSM = VPL >= 8 && sizeof(T) == 8;
  VT* s_cacc = s_bv + (BSM ? VPL * kSdsnThreads : 0);                                            // [VPL][threads] (CSM)
  T* s_colstage = reinterpret_cast<T*>(s_cacc + (CSM ? VPL * kSdsnThreads : 0));                 // [RG][ld]
  // On-chip rows (RG = 1 only, NT + NSM > 0): a warp's first NT rows live in TMEM (lane quarter
  // warp%4, column block (row·4 + warp/4)·WPR), the next NSM rows in shared memory, the rest stream
  // through L2/HBM.  A pass then moves only the streamed rows through the memory system (FP64 at
  // n = 4096: about half of the 128 MB iterate, which then fits in L2).
  VT* s_on = reinterpret_cast<VT*>(s_colstage);              // [NSM][nvec] (RG = 1: no column staging)
  __shared__ uint32_t s_tmem;
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
  if (NT > 0) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&s_tmem)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  const uint32_t tmem = NT > 0 ? s_tmem + ((uint32_t)((warp & 3) * 32) << 16) : 0u;
  auto tmem_free = [&]() {
    if (NT > 0) {
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(512));
    }
  };
  const int nrw = (R > rg) ? (R - rg + RG - 1) / RG : 0;     // rows handled by this warp
  T* Y = reinterpret_cast<T*>(P.Y);
  T* colpart = reinterpret_cast<T*>(P.colpart);
  const double dn = (double)n, nn = dn * dn;
  // vector index of slot k for this lane: q = (cg·VPL + k)·32 + lane
  auto qidx = [&](int k) -> long { return ((long)cg * VPL + k) * 32 + lane; };

  // S/n, S/n² and c/n without full FP64 divisions: r = RN(1/d), then q + r·(x − q·d) = RN(x/d)
  // (Markstein; see K4r and tools/div_probe.cu)
  const double rn = __drcp_rn(dn), rnn = __drcp_rn(nn);
  auto div_n = [&](double x, double d, double r) {
    const double q = x * r;
    return fma(r, fma(-q, d, x), q);
  };
  using TG = Tag<T>;
  // ---------------- column-slice reduction + S of epoch e ----------------
  // CTA b sums column slice b over all CTAs' tagged partials (warp ↔ source CTA k ≡ warp mod 16,
  // all loads in flight, then re-read until tagged e; FP64 in CTA order, warps combined in order)
  // and publishes c (tagged e); warp 0 collects S from the per-CTA masses (tagged, parity buffer).
  constexpr int NI = (32 * 5 + kSdsnWarps - 1) / kSdsnWarps;   // G ≤ 160 sources
  auto reduce_columns_and_S = [&](unsigned e) {
    const long cb = (long)b * n / G, ce = (long)(b + 1) * n / G;
    for (long c0 = cb; c0 < ce; c0 += 32) {
      const long col = c0 + lane;
      double acc = 0.0;
      if (col < ce) {
        typename TG::W w[NI];
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const unsigned k = warp + i * kSdsnWarps;
          w[i] = k < G ? TG::ld(colpart + (long)k * ld + col) : TG::make((T)0, e);
        }
        bool ok;
        do {
          ok = true;
#pragma unroll
          for (int i = 0; i < NI; ++i)
            if (!TG::ok(w[i], e)) { ok = false; w[i] = TG::ld(colpart + (long)(warp + i * kSdsnWarps) * ld + col); }
        } while (!ok);
#pragma unroll
        for (int i = 0; i < NI; ++i) acc += (double)TG::val(w[i]);
      }
      s_red[warp][lane] = acc;
      __syncthreads();
      if (tid < 32 && c0 + tid < ce) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < kSdsnWarps; ++w) sum += s_red[w][tid];
        Tag<double>::st(P.cvec + c0 + tid, sum, e);
      }
      __syncthreads();
    }
    if (warp == 0) {
      double v[5];
      wait_d1_lanes<5>(reinterpret_cast<const uint64_t*>(P.Spart) + (size_t)(e & 1) * G, (int)G, lane, (e >> 1) & 1u, v);
      double sum = 0.0;
#pragma unroll
      for (int i = 0; i < 5; ++i) sum += v[i];
      sum = warp_sum_d(sum);
      if (lane == 0) s_scal[0] = sum;
    }
  };

  // ---------------- one sweep over the CTA's rows ----------------
  // MODE SCALE: y ← fl(s·y) (written only if P.scale); MODE PASS: y ← max(0, (y + a_i) + b_j).
  // Both accumulate the row sums (s_r) and column partials (colpart[b]) of the new values.
  auto sweep = [&](auto mode_c, double sc, const T (&bv)[VPL][W], unsigned e, bool rev, bool wb) {
    constexpr int mode = decltype(mode_c)::value;
    T colacc[CSM ? 1 : VPL][W];
#pragma unroll
    for (int k = 0; k < (CSM ? 1 : VPL); ++k)
#pragma unroll
      for (int w = 0; w < W; ++w) colacc[k][w] = (T)0;
    if constexpr (CSM) {
      T z[W];
#pragma unroll
      for (int w = 0; w < W; ++w) z[w] = (T)0;
#pragma unroll
      for (int k = 0; k < VPL; ++k) s_cacc[k * kSdsnThreads + tid] = vmake<T>(z);
    }
    // column accumulation of one vector of new values (same per-column add order either way)
    auto cadd = [&](int k, const T (&y)[W]) {
      if constexpr (CSM) {
        T c[W];
        vget<T>(s_cacc[k * kSdsnThreads + tid], c);
#pragma unroll
        for (int w = 0; w < W; ++w) c[w] += y[w];
        s_cacc[k * kSdsnThreads + tid] = vmake<T>(c);
      } else {
#pragma unroll
        for (int w = 0; w < W; ++w) colacc[CSM ? 0 : k][w] += y[w];
      }
    };
    auto cget = [&](int k, T (&c)[W]) {
      if constexpr (CSM) vget<T>(s_cacc[k * kSdsnThreads + tid], c);
      else {
#pragma unroll
        for (int w = 0; w < W; ++w) c[w] = colacc[CSM ? 0 : k][w];
      }
    };
    // per-slot constants (32-bit indexing: n·ld < 2^31 for every supported n)
    const int ldv = (int)(ld / W);
    VT* Yc = reinterpret_cast<VT*>(Y) + (long)r0 * ldv;        // this CTA's first row
    // slot k's vector index and kind (0 skip, 1 full vector, 2 ragged tail), derived on use rather
    // than kept in 2·VPL registers
    const int q0 = (int)qidx(0);
    auto qvf = [&](int k) -> int { return q0 + 32 * k; };
    auto kindf = [&](int k) -> int {
      const int q = q0 + 32 * k;
      return q >= (int)nvec ? 0 : ((q + 1) * W <= (int)n ? 1 : 2);
    };
    auto getb = [&](int k, T (&bb)[W]) {
      if constexpr (BSM) {
        if constexpr (decltype(mode_c)::value == SWEEP_PASS) vget<T>(s_bv[k * kSdsnThreads + tid], bb);
      } else {
#pragma unroll
        for (int w = 0; w < W; ++w) bb[w] = bv[k][w];
      }
    };
    VT buf[PD][VPL];
    // on-chip rows first (local rows [0, non)), then the streamed rows with the register ring.
    // rev: the streamed rows in reverse order (odd passes), so a pass starts on the rows the
    // previous pass wrote last — still in L2 when they are about the L2 size
    const int non = RG == 1 ? min(NT + NSM, nrw) : 0;
    const int nrs = OO ? 0 : nrw - non;
    auto rmap = [&](int rr) { return non + (rev ? nrs - 1 - rr : rr); };
    auto load_row = [&](int s, int rr) {
      const VT* row = Yc + (rg + rmap(rr) * RG) * ldv;
#pragma unroll
      for (int k = 0; k < VPL; ++k)
        if (kindf(k)) buf[s][k] = __ldcg(row + qvf(k));
    };
    bool full = true;                                          // every slot a full vector?
#pragma unroll
    for (int k = 0; k < VPL; ++k) full = full && (kindf(k) == 1);
    full = __all_sync(0xffffffffu, full);
    // the first streamed rows' loads are in flight while the on-chip rows are processed
#pragma unroll
    for (int s = 0; s < PD; ++s)
      if (s < nrs) load_row(s, s);
    // on-chip rows: one at a time (TMEM or shared memory; the scale sweep reads X from global).  The
    // TMEM and shared-memory rows are separate code paths and full rows skip the ragged-tail tests:
    // one shared register array with per-element tail checks cost ~330 instructions per row and
    // warp (ncu source page, FP64 n = 4096: the on-chip rows took as long as the streamed ones).
  auto rowbody = [&](auto full_c, VT (&v)[VPL], T a) -> T {
    constexpr bool FULL = decltype(full_c)::value;
      T r = (T)0;
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        if (FULL || kindf(k)) {
          T x[W], bb[W];
          vget<T>(v[k], x);
          getb(k, bb);
#pragma unroll
          for (int w = 0; w < W; ++w) {
            T y;
            if constexpr (decltype(mode_c)::value == SWEEP_PASS) y = tmax0((x[w] + a) + bb[w]);
            else y = P.scale ? (T)(sc * (double)x[w]) : x[w];
            if (!FULL && kindf(k) == 2 && qvf(k) * W + w >= (int)n) y = (T)0;
            x[w] = y;
            r += y;
          }
          cadd(k, x);
          v[k] = vmake<T>(x);
        }
      }
      return r;
    };
    auto onchip = [&](auto full_c, int il) {
      constexpr bool FULL = decltype(full_c)::value;
      const T a = (mode_c.value == SWEEP_PASS) ? s_a[il] : (T)0;
      VT* row = Yc + il * ldv;
      T r;
      if (mode_c.value == SWEEP_SCALE || il >= NT) {
        VT v[VPL];
        VT* src = il >= NT ? s_on + (long)(il - NT) * nvec : nullptr;
#pragma unroll
        for (int k = 0; k < VPL; ++k)
          if (FULL || kindf(k)) v[k] = mode_c.value == SWEEP_SCALE ? __ldcg(row + qvf(k)) : src[qvf(k)];
        r = rowbody(full_c, v, a);
        if (wb) {
#pragma unroll
          for (int k = 0; k < VPL; ++k)
            if (FULL || kindf(k)) __stcg(row + qvf(k), v[k]);
        }
        if (il < NT) {
          uint32_t wv[WPR];
#pragma unroll
          for (int k = 0; k < VPL; ++k) *reinterpret_cast<VT*>(&wv[k * (WPR / VPL)]) = v[k];
          tmem_st<WPR>(tmem + (uint32_t)((il * 4 + (warp >> 2)) * WPR), wv);
        } else {
#pragma unroll
          for (int k = 0; k < VPL; ++k)
            if (FULL || kindf(k)) s_on[(long)(il - NT) * nvec + qvf(k)] = v[k];
        }
      } else {
        uint32_t wv[WPR];
        tmem_ld<WPR>(tmem + (uint32_t)((il * 4 + (warp >> 2)) * WPR), wv);
        tmem_wait_ld();
        VT v[VPL];
#pragma unroll
        for (int k = 0; k < VPL; ++k) v[k] = *reinterpret_cast<const VT*>(&wv[k * (WPR / VPL)]);
        r = rowbody(full_c, v, a);
        if (wb) {
#pragma unroll
          for (int k = 0; k < VPL; ++k)
            if (FULL || kindf(k)) __stcg(row + qvf(k), v[k]);
        }
#pragma unroll
        for (int k = 0; k < VPL; ++k) *reinterpret_cast<VT*>(&wv[k * (WPR / VPL)]) = v[k];
        tmem_st<WPR>(tmem + (uint32_t)((il * 4 + (warp >> 2)) * WPR), wv);
      }
      r = warp_sum_t(r);
      if (lane == 0) s_rowpart[il * CG + cg] = (double)r;
    };
    // two on-chip rows of the same kind at once (PASS sweeps): independent chains for the TMEM / shared-
    // memory latency and the FP64 adds, and one paired warp reduction (xor 16 splits the two rows
    // between the half-warps: 5 shuffle rounds for both rows instead of 10)
    auto onchip2 = [&](auto full_c, int il) {
      constexpr bool FULL = decltype(full_c)::value;
      const T a0 = s_a[il], a1 = s_a[il + 1];
      VT v0[VPL], v1[VPL];
      if (il < NT) {
        uint32_t w0[WPR], w1[WPR];
        tmem_ld<WPR>(tmem + (uint32_t)((il * 4 + (warp >> 2)) * WPR), w0);
        tmem_ld<WPR>(tmem + (uint32_t)(((il + 1) * 4 + (warp >> 2)) * WPR), w1);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
          v0[k] = *reinterpret_cast<const VT*>(&w0[k * (WPR / VPL)]);
          v1[k] = *reinterpret_cast<const VT*>(&w1[k * (WPR / VPL)]);
        }
      } else {
        const VT* s0 = s_on + (long)(il - NT) * nvec;
#pragma unroll
        for (int k = 0; k < VPL; ++k)
          if (FULL || kindf(k)) { v0[k] = s0[qvf(k)]; v1[k] = s0[nvec + qvf(k)]; }
      }
      T r0 = rowbody(full_c, v0, a0);
      T r1 = rowbody(full_c, v1, a1);
      if (wb) {
        VT* row0 = Yc + il * ldv;
#pragma unroll
        for (int k = 0; k < VPL; ++k)
          if (FULL || kindf(k)) { __stcg(row0 + qvf(k), v0[k]); __stcg(row0 + ldv + qvf(k), v1[k]); }
      }
      if (il < NT) {
        uint32_t w0[WPR], w1[WPR];
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
          *reinterpret_cast<VT*>(&w0[k * (WPR / VPL)]) = v0[k];
          *reinterpret_cast<VT*>(&w1[k * (WPR / VPL)]) = v1[k];
        }
        tmem_st<WPR>(tmem + (uint32_t)((il * 4 + (warp >> 2)) * WPR), w0);
        tmem_st<WPR>(tmem + (uint32_t)(((il + 1) * 4 + (warp >> 2)) * WPR), w1);
      } else {
        VT* s0 = s_on + (long)(il - NT) * nvec;
#pragma unroll
        for (int k = 0; k < VPL; ++k)
          if (FULL || kindf(k)) { s0[qvf(k)] = v0[k]; s0[nvec + qvf(k)] = v1[k]; }
      }
      const bool hi = (lane & 16) != 0;
      T keep = hi ? r1 : r0;
      keep += __shfl_xor_sync(0xffffffffu, hi ? r0 : r1, 16);
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) keep += __shfl_xor_sync(0xffffffffu, keep, o);
      if ((lane & 15) == 0) s_rowpart[(il + (hi ? 1 : 0)) * CG + cg] = (double)keep;
    };
    // the on-chip rows of a PASS sweep: pairs within the TMEM rows, then within the shared-memory rows
    auto onchip_all = [&](auto full_c) {
      int il = 0;
      if constexpr (OO && SDSN_PAIR && decltype(mode_c)::value == SWEEP_PASS) {
        const int nt = min(NT, non);
        for (; il + 1 < nt; il += 2) onchip2(full_c, il);
        if (il < nt) onchip(full_c, il++);
        for (; il + 1 < non; il += 2) onchip2(full_c, il);
      }
      for (; il < non; ++il) onchip(full_c, il);
    };
    // FP32 on-chip rows: the round-1 row body (one register array for TMEM / shared memory /
    // global words; the split body below measured slower for FP32: n = 16384 354 → 436 us/pass)
    auto onchip32 = [&](int il) {
      // one register array holds the row slice: TMEM words, shared-memory or global vectors
      uint32_t wv[WPR];
      VT* row = Yc + il * ldv;
      auto vec = [&](int k) -> VT& { return *reinterpret_cast<VT*>(&wv[k * (WPR / VPL)]); };
      if (mode_c.value == SWEEP_SCALE) {
#pragma unroll
        for (int k = 0; k < VPL; ++k)
          if (kindf(k)) vec(k) = __ldcg(row + qvf(k));
      } else if (il < NT) {
        tmem_ld<WPR>(tmem + (uint32_t)((il * 4 + (warp >> 2)) * WPR), wv);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int k = 0; k < VPL; ++k)
          if (kindf(k)) vec(k) = s_on[(long)(il - NT) * nvec + qvf(k)];
      }
      const T a = (mode_c.value == SWEEP_PASS) ? s_a[il] : (T)0;
      T r = (T)0;
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        if (kindf(k)) {
          T x[W], bb[W];
          vget<T>(vec(k), x);
          getb(k, bb);
#pragma unroll
          for (int w = 0; w < W; ++w) {
            T y;
            if constexpr (decltype(mode_c)::value == SWEEP_PASS) y = tmax0((x[w] + a) + bb[w]);
            else y = P.scale ? (T)(sc * (double)x[w]) : x[w];
            if (kindf(k) == 2 && qvf(k) * W + w >= (int)n) y = (T)0;
            x[w] = y;
            r += y;
          }
          cadd(k, x);
          vec(k) = vmake<T>(x);
          if (il >= NT) s_on[(long)(il - NT) * nvec + qvf(k)] = vec(k);
          if (wb) __stcg(row + qvf(k), vec(k));
        }
      }
      if (il < NT) tmem_st<WPR>(tmem + (uint32_t)((il * 4 + (warp >> 2)) * WPR), wv);
      r = warp_sum_t(r);
      if (lane == 0) s_rowpart[il * CG + cg] = (double)r;
    };
    // FP64: the split row body inside the full / ragged dispatch (with the sign-bit max: FP64
    // n = 4096 26.7 → 22.1 us/pass, n = 2048 10.2 → 7.5; `profiles/r02/ab_k4lean2.log`)
    constexpr bool kF64Body = sizeof(T) == 8;
    if constexpr (!kF64Body)
      for (int il = 0; il < non; ++il) onchip32(il);
    auto run = [&](auto full_c) {
      constexpr bool FULL = decltype(full_c)::value;
      if constexpr (kF64Body) onchip_all(full_c);
      for (int base = 0; base < nrs; base += PD) {
        T rs[PD];
#pragma unroll
        for (int s = 0; s < PD; ++s) {
          rs[s] = (T)0;
          const int rr = base + s;
          if (rr < nrs) {
            const int il = rg + rmap(rr) * RG;               // local row index
            VT* row = Yc + il * ldv;
            [[maybe_unused]] const T a = (mode == SWEEP_PASS) ? s_a[il] : (T)0;
#pragma unroll
            for (int k = 0; k < VPL; ++k) {
              if (FULL || kindf(k)) {
                T e[W], bb[W];
                vget<T>(buf[s][k], e);
                getb(k, bb);
#pragma unroll
                for (int w = 0; w < W; ++w) {
                  T y;
                  if constexpr (mode == SWEEP_PASS) y = tmax0((e[w] + a) + bb[w]);   // P2(P1(Y))
                  else y = P.scale ? (T)(sc * (double)e[w]) : e[w];
                  if (!FULL && kindf(k) == 2 && qvf(k) * W + w >= (int)n) y = (T)0;     // ragged tail
                  e[w] = y;
                  rs[s] += y;
                }
                cadd(k, e);
                if (mode == SWEEP_PASS || P.scale) __stcg(row + qvf(k), vmake<T>(e));
              }
            }
            if (rr + PD < nrs) load_row(s, rr + PD);
          }
        }
#pragma unroll
        for (int s = 0; s < PD; ++s) rs[s] = warp_sum_t(rs[s]);      // converged: PD chains interleave
        if (lane == 0) {
#pragma unroll
          for (int s = 0; s < PD; ++s)
            if (base + s < nrs) s_rowpart[(rg + rmap(base + s) * RG) * CG + cg] = (double)rs[s];
        }
      }
    };
    if (full) run(std::true_type{});
    else run(std::false_type{});
    if (NT > 0) tmem_wait_st();
    // column partials of this CTA → colpart[b] (tagged e; e = 0: last pass, nothing published)
    if (RG == 1) {
      if (e != 0) {
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
          const long q = qidx(k);
          if (q < nvec) {
            T c[W];
            cget(k, c);
            TG::st4(colpart + (long)b * ld + q * W, c, e);
          }
        }
      }
      __syncthreads();
    } else {
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        const long q = qidx(k);
        if (q < nvec) {
          T c[W];
          cget(k, c);
          reinterpret_cast<VT*>(s_colstage + (long)rg * ld)[q] = vmake<T>(c);
        }
      }
      __syncthreads();
      if (e != 0) {
        for (long q = tid; q < nvec; q += kSdsnThreads) {
          T acc[W];
          vget<T>(reinterpret_cast<const VT*>(s_colstage)[q], acc);
          for (int g = 1; g < RG; ++g) {
            T x[W];
            vget<T>(reinterpret_cast<const VT*>(s_colstage + (long)g * ld)[q], x);
#pragma unroll
            for (int w = 0; w < W; ++w) acc[w] += x[w];
          }
          TG::st4(colpart + (long)b * ld + q * W, acc, e);
        }
      }
    }
    // row sums (fixed order over column groups) and the CTA's mass partial (tagged, parity buffer)
    for (int i = tid; i < R; i += kSdsnThreads) {
      double s = 0.0;
      for (int g = 0; g < CG; ++g) s += s_rowpart[i * CG + g];
      s_r[i] = s;
    }
    __syncthreads();
    if (warp == 0 && e != 0) {
      double s = 0.0;
      for (int i = lane; i < R; i += 32) s += s_r[i];
      s = warp_sum_d(s);
      if (lane == 0) st_d1(reinterpret_cast<uint64_t*>(P.Spart) + (size_t)(e & 1) * G + b, s, (e >> 1) & 1u);
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
      st_d1(reinterpret_cast<uint64_t*>(P.Mpart) + b, mm, 1u);
    }
    if (warp == 0) {
      double v[5];
      wait_d1_lanes<5>(reinterpret_cast<const uint64_t*>(P.Mpart), (int)G, lane, 1u, v);
      double mm = 0.0;
#pragma unroll
      for (int i = 0; i < 5; ++i) mm = fmax(mm, v[i]);
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
      tmem_free();
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
    sweep(std::integral_constant<int, SWEEP_SCALE>{}, sc, bz, 1u, false, false);
  }
  unsigned ep = 1;                                   // epoch of the current exchange
  reduce_columns_and_S(ep);

  // ---------------- pass loop ----------------
  int j = 0;
  double gam = 0.0;
  for (;; ++j) {
    T bv[VPL][W];                                     // b for this lane's columns: −c/n of epoch ep
    {
      typename Tag<double>::W cw[VPL][W];
#pragma unroll
      for (int k = 0; k < VPL; ++k)
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const long col = qidx(k) * W + w;
          cw[k][w] = col < n ? Tag<double>::ld(P.cvec + col) : Tag<double>::make(0.0, ep);
        }
      bool ok;
      do {
        ok = true;
#pragma unroll
        for (int k = 0; k < VPL; ++k)
#pragma unroll
          for (int w = 0; w < W; ++w)
            if (!Tag<double>::ok(cw[k][w], ep)) { ok = false; cw[k][w] = Tag<double>::ld(P.cvec + qidx(k) * W + w); }
      } while (!ok);
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        T x[W];
#pragma unroll
        for (int w = 0; w < W; ++w) x[w] = (qidx(k) * W + w < n) ? (T)(-div_n(Tag<double>::val(cw[k][w]), dn, rn)) : (T)0;
        if constexpr (BSM) s_bv[k * kSdsnThreads + tid] = vmake<T>(x);
        else {
#pragma unroll
          for (int w = 0; w < W; ++w) bv[k][w] = x[w];
        }
      }
    }
    __syncthreads();                                  // s_scal[0] (S of epoch ep) from the reduction
    const double S = s_scal[0];
    gam = div_n(S, dn, rn) - 1.0;                                      // γ_j = S/n − 1
    if (b == 0 && tid == 0 && P.gamma_hist) P.gamma_hist[j] = gam;
    const bool last = P.sdsn_fixed > 0 ? (j + 1 >= P.sdsn_fixed)
                                       : ((j >= 1 && gam <= P.gamma_th) || j + 1 >= P.sdsn_max);
    const double abase = rn + div_n(S, nn, rnn);                       // 1/n + S/n²
    for (int i = tid; i < R; i += kSdsnThreads) s_a[i] = (T)(abase - div_n(s_r[i], dn, rn));
    __syncthreads();
    sweep(std::integral_constant<int, SWEEP_PASS>{}, 1.0, bv, last ? 0u : ep + 1, (j & 1) == 0, last);
    if (last) break;
    ++ep;
    reduce_columns_and_S(ep);
  }
  if (b == 0 && tid == 0) {
    *P.passes_out = j + 1;
    P.sdsn_out[0] = gam;
    P.sdsn_out[2] = s_scal[0];
  }
  tmem_free();
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
  const int RG = kSdsnWarps / cg;
  const long rows_max = (p.n + grid - 1) / grid + 1;
  size_t dsm = ((sizeof(double) * rows_max * cg + 15) & ~15ul) + (RG > 1 ? (size_t)RG * p.ld * sizeof(T) : 0) +
               (VPL >= 8 ? (size_t)VPL * kSdsnThreads * sizeof(typename VecT<T>::t) : 0) +  // s_bv
               (VPL >= 8 && sizeof(T) == 8 ? (size_t)VPL * kSdsnThreads * sizeof(typename VecT<T>::t) : 0);   // s_cacc
  // on-chip rows (one row group only): up to 128/WPR rows in TMEM and as many rows as fit in the
  // shared memory that is left (227 KB opt-in minus the static arrays)
  int nt = 0, nsm = 0;
  if (RG == 1 && SDSN_ONCHIP) {
    constexpr int WPR = VPL * (int)sizeof(typename VecT<T>::t) / 4;
    const long R = (p.n + grid - 1) / grid;
    nt = (int)std::min<long>(128 / WPR, R);
    const long row_bytes = ((p.n + VecT<T>::W - 1) / VecT<T>::W) * (long)sizeof(typename VecT<T>::t);
    const long stat = (long)(kSdsnMaxRows * (sizeof(double) + sizeof(T)) + kSdsnWarps * 32 * 8 + 256);
    const long avail = 232448 - stat - (long)dsm;
    nsm = (int)std::max<long>(0, std::min<long>(R - nt, avail / row_bytes));
    dsm += (size_t)nsm * row_bytes;
  }
  auto fn = sdsn_kernel<T, VPL, false>;
  if constexpr (sizeof(T) == 8 && VPL <= 4)
    if (RG == 1 && SDSN_ONCHIP && nt + nsm >= (p.n + grid - 1) / grid) fn = sdsn_kernel<T, VPL, true>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
  if (e != cudaSuccess) return e;
  SdsnParams pp = p;
  int cgv = cg;
  void* args[] = {&pp, &cgv, &nt, &nsm};
  return cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(kSdsnThreads), args, dsm, st);
}

cudaError_t launch_sdsn(const SdsnParams& p, bool f64, cudaStream_t st, int num_sms, int* grid_out) {
  int vpl, cg;
  if (!plan(p.n, f64, &vpl, &cg)) return cudaErrorInvalidValue;
  const int grid = sdsn_grid_for(p.n, num_sms);
  if (grid > 160) return cudaErrorInvalidValue;          // the tagged reductions cover ≤ 160 CTAs
  if (grid_out) *grid_out = grid;
  // tagged exchange words start "not ready" for every epoch's first read: colpart, cvec and Mpart
  // zero (tag 0 ≠ epoch 1), Spart buffer 1 (epoch 1, tag 0) set to tag 1, buffer 0 (epoch 2, tag 1)
  // zero.  Spart and Mpart hold 2·grid and grid words.
  const size_t ts = f64 ? 8 : 4;
  cudaError_t e = cudaMemsetAsync(p.colpart, 0, (size_t)grid * p.ld * ts, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(p.cvec, 0, (size_t)p.ld * 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(p.Mpart, 0, (size_t)grid * 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(p.Spart, 0, (size_t)grid * 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(p.Spart + grid, 0x80, (size_t)grid * 8, st);
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
