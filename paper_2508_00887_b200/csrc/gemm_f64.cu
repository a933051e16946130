// gemm_f64.cu — K2d/K3d: the gradient GEMMs in FP64 mode (all steps FP64: the paper's "GPU-FP64"
// comparison).  tcgen05 has no f64 kind, so this uses the FP64 tensor path through
// mma.sync.m8n8k4.f64 (DMMA), with a cp.async multi-stage SMEM ring.
// Same NT contract and epilogues as gemm_tc.cu: D = Aop·Bopᵀ; epi 0 stores Dᵀ, epi 1 stores
// G = D + λK' (FP64).
#include "common.cuh"
#include "internal.h"

namespace fram {
namespace {

// CTA tile TM×TN, k-slab TK, NS-stage cp.async ring; one warp per 32×32 sub-tile (4×4 DMMA 8×8×4).
// Shared-memory row pitch TK + 4 doubles (≡ 8 words mod 32: conflict-free fragment loads).  Measured
// alternatives (profiles/r02/ab_dmma.log): NS = 3 / 4, 128×64 and 128×128 tiles, TK = 32 — equal or
// slower (the DMMA pipe is ~90% busy).
constexpr int TM = 64, TN = 64, TK = 16, NS = 2, PADK = TK + 4;
constexpr int THREADS = (TM / 32) * (TN / 32) * 32;
constexpr size_t SMEM = (size_t)NS * (TM + TN) * PADK * sizeof(double);

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool pred) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  const int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool pred) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  const int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N_> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N_) : "memory"); }

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(THREADS) gemm_f64_kernel(const double* __restrict__ A, const double* __restrict__ B,
                                                           long M, long N, long K, long ld, int epi, double* out,
                                                           long ldo, const double* Kq, double lam, long kchunk) {
  extern __shared__ __align__(16) double gsm[];
  auto As = [&](int buf, int r, int k) -> double& { return gsm[((size_t)buf * (TM + TN) + r) * PADK + k]; };
  auto Bs = [&](int buf, int r, int k) -> double& { return gsm[((size_t)buf * (TM + TN) + TM + r) * PADK + k]; };
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long m0 = (long)blockIdx.y * TM, n0 = (long)blockIdx.x * TN;
  const int wm = (warp / (TN / 32)) * 32, wn = (warp % (TN / 32)) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto load_stage = [&](int buf, long k0) {
    // TM×TK (and TN×TK) doubles in 16-byte chunks, TK/2 chunks per row
#pragma unroll
    for (int c = tid; c < TM * TK / 2; c += THREADS) {
      const int r = c / (TK / 2), kc = (c % (TK / 2)) * 2;
      const long gr = m0 + r, gk = k0 + kc;
      const bool ok = gr < M && gk < K;
      cp_async16(&As(buf, r, kc), ok ? (const void*)(A + gr * ld + gk) : (const void*)A, ok);
    }
#pragma unroll
    for (int c = tid; c < TN * TK / 2; c += THREADS) {
      const int r = c / (TK / 2), kc = (c % (TK / 2)) * 2;
      const long gk = k0 + kc, gn = n0 + r;
      const bool okb = gn < N && gk < K;
      if (kchunk & 1) {                               // odd blocks: 8-byte copies (no 16-B alignment)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const long k = gk + e;
          const bool oke = gn < N && k < K;
          const double* bp = B + (k / kchunk) * N * kchunk + gn * kchunk + k % kchunk;
          cp_async8(&Bs(buf, r, kc + e), oke ? (const void*)bp : (const void*)B, oke);
        }
      } else {
        const double* bp = kchunk ? B + (gk / kchunk) * N * kchunk + gn * kchunk + gk % kchunk : B + gn * ld + gk;
        cp_async16(&Bs(buf, r, kc), okb ? (const void*)bp : (const void*)B, okb);
      }
    }
  };

  const int nk = (int)((K + TK - 1) / TK);
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) {
    if (s < nk) load_stage(s, (long)s * TK);
    cp_commit();
  }
  for (int kb = 0; kb < nk; ++kb) {
    const int buf = kb % NS;
    cp_wait<NS - 2>();                                // slab kb has landed (this thread's copies)
    __syncthreads();                                  // ... everyone's; slab kb−1's buffer is free
    if (kb + NS - 1 < nk) load_stage((kb + NS - 1) % NS, (long)(kb + NS - 1) * TK);
    cp_commit();
#pragma unroll
    for (int kk = 0; kk < TK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As(buf, wm + i * 8 + (lane >> 2), kk + (lane & 3));
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs(buf, wn + j * 8 + (lane >> 2), kk + (lane & 3));
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  // epilogue: acc[i][j][e] = D[m0+wm+i*8+lane/4][n0+wn+j*8+2*(lane%4)+e]
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long r = m0 + wm + i * 8 + (lane >> 2);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const long c = n0 + wn + j * 8 + 2 * (lane & 3) + e;
        if (r < M && c < N) {
          if (epi == 0) out[c * ldo + r] = acc[i][j][e];
          else out[r * ldo + c] = Kq ? acc[i][j][e] + lam * Kq[r * ldo + c] : acc[i][j][e];
        }
      }
    }
  }
}

}  // namespace

cudaError_t launch_gemm_f64(const GemmArgs& g, cudaStream_t st) {
  cudaError_t attr = cudaFuncSetAttribute(gemm_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
  // 4 CTAs per SM (register-limited) need 4 × 41 KB of shared memory: ask for the full carveout
  if (attr == cudaSuccess)
    attr = cudaFuncSetAttribute(gemm_f64_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                (int)cudaSharedmemCarveoutMaxShared);
  if (attr != cudaSuccess) return attr;
  dim3 grid((unsigned)((g.N + TN - 1) / TN), (unsigned)((g.M + TM - 1) / TM));
  gemm_f64_kernel<<<grid, THREADS, SMEM, st>>>((const double*)g.Aop, (const double*)g.Bop, g.M, g.N, g.K, g.ld, g.epi,
                                            (double*)g.out, g.ldo, (const double*)g.Kq, g.lam, g.kchunk);
  return cudaGetLastError();
}

}  // namespace fram
