// Dev probe: on-chip SDSN sweep throughput without the exchange (one CTA per SM, 512 threads,
// n = 4096 → CPT = 32, two column halves of 16 per thread).  Row kinds: TMEM rows, shared-memory
// rows and register-resident rows; each row group g ∈ {0,1} (8 warps) gets its own mix.  Reports
// cycles per pass per group and for the whole pass (one __syncthreads per pass, as in K4r).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2508_00887_b200/csrc
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tmem_ldst.cuh"
#include "xchg.cuh"
using namespace fram;

constexpr int CPT = 32, CH = 16, VH = 4, NS = 128 * CPT;

template <int T0, int S0, int G0, int T1, int S1, int G1, int MODE>
__global__ void __launch_bounds__(512, 1) sweep(int passes, float* out, long long* cyc) {
  extern __shared__ __align__(16) unsigned char dsm[];
  float4* s_rows = reinterpret_cast<float4*>(dsm);
  __shared__ float s_rowpart[64 * 8];
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, q = warp & 3, h = (warp >> 2) & 1, g = warp >> 3;
  const int t = q * 32 + lane, c0 = h * VH;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * CH);
  constexpr int TT = T0 + T1;          // TMEM rows: group 0 takes [0,T0), group 1 [T0, T0+T1)
  static_assert(TT * CPT <= 512, "TMEM");
  const int tbeg = g == 0 ? 0 : T0, tcnt = g == 0 ? T0 : T1;
  const int sbeg = g == 0 ? 0 : S0, scnt = g == 0 ? S0 : S1;   // shared rows
  constexpr int GM = G0 > G1 ? G0 : G1;
  float reg[GM > 0 ? GM : 1][CH];
#pragma unroll
  for (int r = 0; r < (GM > 0 ? GM : 1); ++r)
#pragma unroll
    for (int k = 0; k < CH; ++k) reg[r][k] = 0.001f * (k + r + t);
  // init TMEM/shared rows
  for (int r = tbeg; r < tbeg + tcnt; ++r) {
    uint32_t v[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) v[k] = __float_as_uint(0.001f * (k + r + t));
    tmem_st<CH>(tmem + (uint32_t)(r * CPT), v);
  }
  tmem_wait_st();
  for (int r = sbeg; r < sbeg + scnt; ++r)
#pragma unroll
    for (int c = 0; c < VH; ++c) s_rows[(size_t)r * (NS / 4) + (c0 + c) * 128 + t] = make_float4(0.001f, 0.002f, 0.f, 0.003f);
  float2 bv[CH / 2];
#pragma unroll
  for (int k = 0; k < CH / 2; ++k) bv[k] = make_float2(-0.0001f * k, -0.0002f);
  __syncthreads();

  auto relu = [&](float v) -> float {
    if (MODE == 3) return __int_as_float(max(__float_as_int(v), 0));
    if (MODE == 4) return v;
    return fmaxf(0.0f, v);
  };
  auto pass_row = [&](float (&x)[CH], float a, float2 (&col2)[CH / 2]) -> float {
    float2 rs = make_float2(0.f, 0.f);
    const float2 a2 = make_float2(a, a);
    if (MODE == 5) {                    // scalar FADDs
      float r0 = 0.f, r1 = 0.f;
#pragma unroll
      for (int k = 0; k < CH; k += 2) {
        float y0 = fmaxf(0.f, (x[k] + a) + bv[k / 2].x), y1 = fmaxf(0.f, (x[k + 1] + a) + bv[k / 2].y);
        x[k] = y0; x[k + 1] = y1;
        col2[k / 2].x += y0; col2[k / 2].y += y1;
        r0 += y0; r1 += y1;
      }
      return r0 + r1;
    }
    if (MODE == 6) {                    // FADD2 with two independent row-sum chains
      float2 r0 = make_float2(0.f, 0.f), r1 = make_float2(0.f, 0.f);
#pragma unroll
      for (int k = 0; k < CH; k += 2) {
        float2 y = add2(add2(make_float2(x[k], x[k + 1]), a2), bv[k / 2]);
        y.x = fmaxf(0.0f, y.x); y.y = fmaxf(0.0f, y.y);
        x[k] = y.x; x[k + 1] = y.y;
        col2[k / 2] = add2(col2[k / 2], y);
        if (k & 2) r1 = add2(r1, y); else r0 = add2(r0, y);
      }
      r0 = add2(r0, r1);
      return r0.x + r0.y;
    }
#pragma unroll
    for (int k = 0; k < CH; k += 2) {
      float2 y = add2(add2(make_float2(x[k], x[k + 1]), a2), bv[k / 2]);
      y.x = relu(y.x);
      y.y = relu(y.y);
      x[k] = y.x;
      x[k + 1] = y.y;
      col2[k / 2] = add2(col2[k / 2], y);
      rs = add2(rs, y);
    }
    return rs.x + rs.y;
  };
  // deferred: 8 per-lane row partials → one transpose-reduce (9 shuffles for 8 rows)
  auto put8 = [&](int rbase, float (&v)[8], int cnt) {
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
    float w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float snd = b4 ? v[i] : v[i + 4];
      const float kp = b4 ? v[i + 4] : v[i];
      w[i] = kp + __shfl_xor_sync(0xffffffffu, snd, 16);
    }
    float u[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float snd = b3 ? w[i] : w[i + 2];
      const float kp = b3 ? w[i + 2] : w[i];
      u[i] = kp + __shfl_xor_sync(0xffffffffu, snd, 8);
    }
    float z = (b2 ? u[1] : u[0]) + __shfl_xor_sync(0xffffffffu, b2 ? u[0] : u[1], 4);
    z += __shfl_xor_sync(0xffffffffu, z, 2);
    z += __shfl_xor_sync(0xffffffffu, z, 1);
    const int rr = lane >> 2;
    if ((lane & 3) == 0 && rr < cnt) s_rowpart[((rbase + rr) & 63) * 8 + 4 * h + q] = z;
  };
  auto put2 = [&](int ra, float va, int rb, float vb) {
    const bool lo = lane < 16;
    float keep = lo ? va : vb;
    keep += __shfl_xor_sync(0xffffffffu, lo ? vb : va, 16);
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) keep += __shfl_xor_sync(0xffffffffu, keep, o);
    if (lane == 0) s_rowpart[(ra & 63) * 8 + 4 * h + q] = keep;
    if (lane == 16 && rb >= 0) s_rowpart[(rb & 63) * 8 + 4 * h + q] = keep;
  };
  long long tg = 0, tall = 0;
  float2 colkeep = make_float2(0.f, 0.f);
  for (int p = 0; p < passes; ++p) {
    const long long p0 = clock64();
    float2 col2[CH / 2];
#pragma unroll
    for (int k = 0; k < CH / 2; ++k) col2[k] = make_float2(0.f, 0.f);
    const float a = -1e-6f * (p & 7);
    // register rows
    if (g == 0) {
#pragma unroll
      for (int r = 0; r < G0; r += 2) {
        const float sa = pass_row(reg[r], a, col2);
        const float sb = r + 1 < G0 ? pass_row(reg[r + 1], a, col2) : 0.f;
        put2(40 + r, sa, r + 1 < G0 ? 41 + r : -1, sb);
      }
    } else {
#pragma unroll
      for (int r = 0; r < G1; r += 2) {
        const float sa = pass_row(reg[r], a, col2);
        const float sb = r + 1 < G1 ? pass_row(reg[r + 1], a, col2) : 0.f;
        put2(50 + r, sa, r + 1 < G1 ? 51 + r : -1, sb);
      }
    }
    if (MODE == 7) {                      // compute only, four rows interleaved
      const int nrows = tcnt + scnt;
      for (int rb8 = 0; rb8 < nrows; rb8 += 8) {
        float rsv[8];
#pragma unroll
        for (int i = 0; i < 8; i += 4) {
          float2 r[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) r[u] = make_float2(0.f, 0.f);
          const float2 a2 = make_float2(a, a);
#pragma unroll
          for (int k = 0; k < CH; k += 2) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              float2 y = add2(add2(make_float2(reg[u][k], reg[u][k + 1]), a2), bv[k / 2]);
              y.x = fmaxf(0.f, y.x); y.y = fmaxf(0.f, y.y);
              reg[u][k] = y.x; reg[u][k + 1] = y.y;
              col2[k / 2] = add2(col2[k / 2], y);
              r[u] = add2(r[u], y);
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) rsv[i + u] = r[u].x + r[u].y;
        }
        put8(rb8, rsv, nrows - rb8);
      }
    } else if (MODE >= 2) {                      // compute only: the same two register rows, no loads/stores
      const int nrows = tcnt + scnt;
      for (int rb8 = 0; rb8 < nrows; rb8 += 8) {
        float rsv[8];
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          rsv[i] = 0.f; rsv[i + 1] = 0.f;
          if (rb8 + i + 1 < nrows) { rsv[i] = pass_row(reg[0], a, col2); rsv[i + 1] = pass_row(reg[1], a, col2); }
        }
        put8(rb8, rsv, nrows - rb8);
      }
    } else if (MODE == 1) {
      for (int rb8 = tbeg; rb8 < tbeg + tcnt; rb8 += 8) {
        float rsv[8];
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          rsv[i] = 0.f; rsv[i + 1] = 0.f;
          const int r = rb8 + i;
          if (r + 1 < tbeg + tcnt) {
            uint32_t va[CH], vb[CH];
            tmem_ld<CH>(tmem + (uint32_t)(r * CPT), va);
            tmem_ld<CH>(tmem + (uint32_t)((r + 1) * CPT), vb);
            tmem_wait_ld();
            float xa[CH], xb[CH];
#pragma unroll
            for (int k = 0; k < CH; ++k) { xa[k] = __uint_as_float(va[k]); xb[k] = __uint_as_float(vb[k]); }
            rsv[i] = pass_row(xa, a, col2); rsv[i + 1] = pass_row(xb, a, col2);
#pragma unroll
            for (int k = 0; k < CH; ++k) { va[k] = __float_as_uint(xa[k]); vb[k] = __float_as_uint(xb[k]); }
            tmem_st<CH>(tmem + (uint32_t)(r * CPT), va);
            tmem_st<CH>(tmem + (uint32_t)((r + 1) * CPT), vb);
          }
        }
        put8(rb8, rsv, tbeg + tcnt - rb8);
      }
      for (int rb8 = sbeg; rb8 < sbeg + scnt; rb8 += 8) {
        float rsv[8];
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          rsv[i] = 0.f; rsv[i + 1] = 0.f;
          const int r = rb8 + i;
          if (r + 1 < sbeg + scnt) {
            float xa[CH], xb[CH];
            const float4* ra = s_rows + (size_t)r * (NS / 4);
            const float4* rb = ra + NS / 4;
#pragma unroll
            for (int c = 0; c < VH; ++c) {
              const float4 u = ra[(c0 + c) * 128 + t], w = rb[(c0 + c) * 128 + t];
              xa[4 * c] = u.x; xa[4 * c + 1] = u.y; xa[4 * c + 2] = u.z; xa[4 * c + 3] = u.w;
              xb[4 * c] = w.x; xb[4 * c + 1] = w.y; xb[4 * c + 2] = w.z; xb[4 * c + 3] = w.w;
            }
            rsv[i] = pass_row(xa, a, col2); rsv[i + 1] = pass_row(xb, a, col2);
            float4* wa = s_rows + (size_t)r * (NS / 4);
            float4* wb = wa + NS / 4;
#pragma unroll
            for (int c = 0; c < VH; ++c) {
              wa[(c0 + c) * 128 + t] = make_float4(xa[4 * c], xa[4 * c + 1], xa[4 * c + 2], xa[4 * c + 3]);
              wb[(c0 + c) * 128 + t] = make_float4(xb[4 * c], xb[4 * c + 1], xb[4 * c + 2], xb[4 * c + 3]);
            }
          }
        }
        put8(20 + rb8, rsv, sbeg + scnt - rb8);
      }
    } else {
    // TMEM rows in pairs
    for (int r = tbeg; r + 1 < tbeg + tcnt; r += 2) {
      uint32_t va[CH], vb[CH];
      tmem_ld<CH>(tmem + (uint32_t)(r * CPT), va);
      tmem_ld<CH>(tmem + (uint32_t)((r + 1) * CPT), vb);
      tmem_wait_ld();
      float xa[CH], xb[CH];
#pragma unroll
      for (int k = 0; k < CH; ++k) { xa[k] = __uint_as_float(va[k]); xb[k] = __uint_as_float(vb[k]); }
      const float sa = pass_row(xa, a, col2), sb = pass_row(xb, a, col2);
#pragma unroll
      for (int k = 0; k < CH; ++k) { va[k] = __float_as_uint(xa[k]); vb[k] = __float_as_uint(xb[k]); }
      tmem_st<CH>(tmem + (uint32_t)(r * CPT), va);
      tmem_st<CH>(tmem + (uint32_t)((r + 1) * CPT), vb);
      put2(r, sa, r + 1, sb);
    }
    // shared rows in pairs
    for (int r = sbeg; r + 1 < sbeg + scnt; r += 2) {
      float xa[CH], xb[CH];
      const float4* ra = s_rows + (size_t)r * (NS / 4);
      const float4* rb = ra + NS / 4;
#pragma unroll
      for (int c = 0; c < VH; ++c) {
        const float4 u = ra[(c0 + c) * 128 + t], w = rb[(c0 + c) * 128 + t];
        xa[4 * c] = u.x; xa[4 * c + 1] = u.y; xa[4 * c + 2] = u.z; xa[4 * c + 3] = u.w;
        xb[4 * c] = w.x; xb[4 * c + 1] = w.y; xb[4 * c + 2] = w.z; xb[4 * c + 3] = w.w;
      }
      const float sa = pass_row(xa, a, col2), sb = pass_row(xb, a, col2);
      float4* wa = s_rows + (size_t)r * (NS / 4);
      float4* wb = wa + NS / 4;
#pragma unroll
      for (int c = 0; c < VH; ++c) {
        wa[(c0 + c) * 128 + t] = make_float4(xa[4 * c], xa[4 * c + 1], xa[4 * c + 2], xa[4 * c + 3]);
        wb[(c0 + c) * 128 + t] = make_float4(xb[4 * c], xb[4 * c + 1], xb[4 * c + 2], xb[4 * c + 3]);
      }
      put2(20 + r, sa, 21 + r, sb);
    }
    }
    tmem_wait_st();
    const long long p1 = clock64();
    __syncthreads();
    const long long p2 = clock64();
    tg += p1 - p0;
    tall += p2 - p0;
#pragma unroll
    for (int k = 0; k < CH / 2; ++k) colkeep = add2(colkeep, col2[k]);
  }
  float acc = colkeep.x + colkeep.y;
  __syncthreads();
  for (int i = 0; i < 8; ++i) acc += s_rowpart[(tid * 8 + i) & 511];
#pragma unroll
  for (int r = 0; r < (GM > 0 ? GM : 1); ++r)
#pragma unroll
    for (int k = 0; k < CH; ++k) acc += reg[r][k];
  if (acc == 1.2345f) out[0] = acc;
  if (lane == 0) {
    atomicMax((unsigned long long*)&cyc[blockIdx.x * 3 + g], (unsigned long long)tg);
    atomicMax((unsigned long long*)&cyc[blockIdx.x * 3 + 2], (unsigned long long)tall);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(512));
}

template <int T0, int S0, int G0, int T1, int S1, int G1, int MODE = 0>
void run(const char* name) {
  auto fn = sweep<T0, S0, G0, T1, S1, G1, MODE>;
  const int smem = (S0 + S1) * NS * 4 + 16;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem < 120 * 1024 ? 120 * 1024 : smem);
  float* out; long long* cyc;
  cudaMalloc(&out, 4); cudaMalloc(&cyc, 148 * 3 * 8);
  const int passes = 2000;
  for (int it = 0; it < 2; ++it) {
    cudaMemset(cyc, 0, 148 * 3 * 8);
    fn<<<148, 512, smem < 120 * 1024 ? 120 * 1024 : smem>>>(passes, out, cyc);
  }
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148 * 3];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  double m[3] = {0, 0, 0};
  for (int b = 0; b < 148; ++b) for (int k = 0; k < 3; ++k) m[k] += h[b * 3 + k] / 148.0;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, fn);
  printf("%-34s rows T%d/S%d/R%d | T%d/S%d/R%d  regs %3d spill %4zu  grp0 %6.0f grp1 %6.0f pass %6.0f cyc  (%.2f us @1.965GHz) %s\n",
         name, T0, S0, G0, T1, S1, G1, fa.numRegs, fa.localSizeBytes, m[0] / passes, m[1] / passes, m[2] / passes,
         m[2] / passes / 1965.0, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(out); cudaFree(cyc);
}

int main() {
  run<16, 0, 4, 0, 12, 4, 2>("compute only, FADD2 pairs");
  run<16, 0, 4, 0, 12, 4, 7>("compute only, FADD2 quads");
  return 0;
}
