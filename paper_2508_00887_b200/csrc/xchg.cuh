// xchg.cuh — device helpers for the on-chip SDSN kernels (K4r, K4p): cross-CTA words that carry their
// own epoch tag (single-copy-atomic 4/8-byte accesses at gpu scope) and the paired FP32 add.
#pragma once
#include <stdint.h>

namespace fram {
namespace {

__device__ __forceinline__ unsigned tag_of(uint64_t w) { return (unsigned)(w >> 32); }
__device__ __forceinline__ uint64_t ld_tag(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// an FP64 value published as two tagged words (hi, lo halves)
// 32-bit words: a non-negative FP32 magnitude with the epoch parity in the (otherwise zero) sign bit.
// A slot read for epoch e can only hold epoch e−1 or e (see the ordering argument in the kernel),
// so one bit distinguishes them.
__device__ __forceinline__ unsigned ptag(float mag, unsigned e) { return __float_as_uint(mag) | ((e & 1u) << 31); }
__device__ __forceinline__ bool pok(unsigned w, unsigned e) { return (w >> 31) == (e & 1u); }
__device__ __forceinline__ float pval(unsigned w) { return __uint_as_float(w & 0x7fffffffu); }
__device__ __forceinline__ unsigned ld_w(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint4 ld_w4(const unsigned* p) {
  uint4 v;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_w(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_w4(unsigned* p, uint4 v) {
  asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
// a non-negative FP64 value with a 1-bit tag in the sign bit (one single-copy-atomic 8-byte word)
__device__ __forceinline__ void st_d1(uint64_t* p, double v, unsigned bit) {
  const uint64_t w = (uint64_t)__double_as_longlong(v) | ((uint64_t)bit << 63);
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ double wait_d1(const uint64_t* p, unsigned bit) {
  uint64_t w;
  do { w = ld_tag(p); } while ((unsigned)(w >> 63) != bit);
  return __longlong_as_double((long long)(w & 0x7fffffffffffffffull));
}

// NW tagged FP64 words p[lane + 32·i] (i < NW, index < cnt; absent words read as 0): all loads are
// issued before any is waited on, so the wait costs one L2 round trip, not NW of them
template <int NW>
__device__ __forceinline__ void wait_d1_lanes(const uint64_t* p, int cnt, int lane, unsigned bit, double (&out)[NW]) {
  uint64_t w[NW];
#pragma unroll
  for (int i = 0; i < NW; ++i) w[i] = lane + 32 * i < cnt ? ld_tag(p + lane + 32 * i) : ((uint64_t)bit << 63);
  bool ok;
  do {
    ok = true;
#pragma unroll
    for (int i = 0; i < NW; ++i)
      if ((unsigned)(w[i] >> 63) != bit) { ok = false; w[i] = ld_tag(p + lane + 32 * i); }
  } while (!ok);
#pragma unroll
  for (int i = 0; i < NW; ++i) out[i] = __longlong_as_double((long long)(w[i] & 0x7fffffffffffffffull));
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

// Threads: warp w → TMEM lane quarter q = w%4, column half h (SPLIT only), row group g.
// Thread (q, lane, h) owns columns [t·CPT + h·CH, +CH) of every row, t = 32q + lane, CH = CPT/NH.

}  // namespace
}  // namespace fram
