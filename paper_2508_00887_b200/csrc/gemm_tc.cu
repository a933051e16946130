// gemm_tc.cu — K2/K3: the gradient contraction X = A'·N·Ã' + λK' (Alg.1 step 5)
// on 5th-generation tensor cores: TMA → SMEM (128B swizzle) → tcgen05.mma (kind::f16 for
// BF16/FP16, kind::tf32 for TF32; FP32 accumulation in TMEM) → tcgen05.ld epilogue.
//
// One NT GEMM shape serves both products: D[M×N] = Aop[M×K] · Bop[N×K]ᵀ, both operands row-major
// with K contiguous ("K-major").
//   GEMM1 (epi 0): Aop = N_q, Bop = Ã'ᵀ  → D = N·Ã' = U, stored TRANSPOSED as Uᵀ in the operand
//                  format (R12: the intermediate is rounded to the operand format).
//   GEMM2 (epi 1): Aop = A',  Bop = Uᵀ   → D = A'·U, stored as G = D + λK' in FP32.
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer (one elected lane), w2 TMEM allocator,
// w4-w7 epilogue (TMEM lane quarter = warp % 4).  Tile 128×256×(128 B of K), 4-stage mbarrier ring.
// Persistent: one CTA per SM walks the tiles t = blockIdx.x, +gridDim.x, …; the accumulator is
// double-buffered in TMEM (2 × 256 columns), so the epilogue of tile i overlaps the MMAs of tile i+1.
#include <cuda.h>
#include "common.cuh"
#include "internal.h"

namespace fram {
namespace {

constexpr int BM = 128, BN = 256, STAGES = 4, GEMM_THREADS = 256;
constexpr int TILE_A = BM * 128;            // bytes: 128 rows × 128 B
constexpr int TILE_B = BN * 128;            // bytes: 256 rows × 128 B
constexpr int STAGE_BYTES = TILE_A + TILE_B;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
constexpr uint32_t TMEM_COLS = 512;                 // two 128×256 FP32 accumulators

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
// UMMA shared-memory descriptor, K-major, SWIZZLE_128B (sm_100 format: version 1 at bit 46,
// layout type 2 at bits 61-63, SBO = 1024 B between 8-row swizzle atoms, LBO unused = 16 B).
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
template <int OP>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (OP == 1) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  } else {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  }
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
        "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
        "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct EpiArgs {
  long M, N, K;
  long kchunk;   // > 0: B operand K-blocked (3-D tensor map: {kchunk, N, K/kchunk})
  int epi;
  void* out;
  long ldo;
  const float* Kq;
  float lam;
};

template <int OP> struct OpStore;
template <> struct OpStore<1> { __device__ static void st(void* o, long idx, float v) { reinterpret_cast<float*>(o)[idx] = tf32_rne(v); } };
template <> struct OpStore<2> { __device__ static void st(void* o, long idx, float v) { reinterpret_cast<__nv_bfloat16*>(o)[idx] = __float2bfloat16_rn(v); } };
template <> struct OpStore<3> { __device__ static void st(void* o, long idx, float v) { reinterpret_cast<__half*>(o)[idx] = __float2half_rn(v); } };

template <int OP>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, EpiArgs ea) {
  constexpr int ESZ = (OP == 1) ? 4 : 2;       // operand element size (TF32 stored as FP32)
  constexpr int BK = 128 / ESZ;                // K elements per 128-byte stage row
  constexpr int UK = 32 / ESZ;                 // K per tcgen05.mma (32 bytes)
  constexpr uint32_t FMT = (OP == 1) ? 2u : (OP == 2 ? 1u : 0u);   // TF32 / BF16 / F16
  constexpr uint32_t IDESC = (1u << 4) | (FMT << 7) | (FMT << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(BM >> 4) << 24);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * TILE_A;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;                    // [2] accumulator b ready (MMA → epilogue)
  uint64_t* tempty = tfull + 2;                        // [2] accumulator b drained (epilogue → MMA)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (int)((ea.K + BK - 1) / BK);
  const int ntn = (int)((ea.N + BN - 1) / BN), ntm = (int)((ea.M + BM - 1) / BM);
  const int ntiles = ntm * ntn;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(tfull + b, 1); mbar_init(tempty + b, 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {                                   // ---- TMA producer (ring continues across tiles)
      int it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int m0 = (tile / ntn) * BM, n0 = (tile % ntn) * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
          mbar_wait(empty + s, ph ^ 1u);
          mbar_expect_tx(full + s, STAGE_BYTES);
          tma_load_2d(&tmA, full + s, sA + s * TILE_A, kb * BK, m0);
          if (ea.kchunk > 0) {
            const long k0 = (long)kb * BK;
            tma_load_3d(&tmB, full + s, sB + s * TILE_B, (int)(k0 % ea.kchunk), n0, (int)(k0 / ea.kchunk));
          } else {
            tma_load_2d(&tmB, full + s, sB + s * TILE_B, kb * BK, n0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {                                   // ---- MMA issuer
      int it = 0, ti = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ti) {
        const int b = ti & 1;
        const uint32_t use = (uint32_t)(ti >> 1) & 1u;
        mbar_wait(tempty + b, use ^ 1u);               // accumulator b drained by the epilogue
        tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)(b * BN);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
          mbar_wait(full + s, ph);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * TILE_A), b0 = smem_u32(sB + s * TILE_B);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)
            umma<OP>(acc, sdesc_sw128(a0 + k * 32), sdesc_sw128(b0 + k * 32), IDESC, (kb | k) != 0 ? 1u : 0u);
          umma_commit(empty + s);                      // frees the SMEM slot when these MMAs finish
        }
        umma_commit(tfull + b);                        // accumulator b complete
      }
    }
  } else if (warp >= 4) {                              // ---- epilogue: TMEM → registers → HBM
    const int q = warp & 3;
    int ti = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ti) {
      const int b = ti & 1;
      const int m0 = (tile / ntn) * BM, n0 = (tile % ntn) * BN;
      mbar_wait(tfull + b, (uint32_t)(ti >> 1) & 1u);
      tc_fence_after();
      const long row = (long)m0 + q * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN + c * 32), v);
        const long col0 = (long)n0 + c * 32;
        if (row < ea.M && col0 < ea.N) {
          if (ea.epi == 0) {
            // transposed store: out[col][row]; lanes of a warp write consecutive rows (coalesced)
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
              const long col = col0 + jj;
              if (col < ea.N) OpStore<OP>::st(ea.out, col * ea.ldo + row, __uint_as_float(v[jj]));
            }
          } else {
            float* g = reinterpret_cast<float*>(ea.out) + row * ea.ldo;
            const float* kr = ea.Kq ? ea.Kq + row * ea.ldo : nullptr;
            if (col0 + 32 <= ea.N) {
#pragma unroll
              for (int jj = 0; jj < 32; jj += 4) {
                float4 o = make_float4(__uint_as_float(v[jj]), __uint_as_float(v[jj + 1]),
                                       __uint_as_float(v[jj + 2]), __uint_as_float(v[jj + 3]));
                if (kr) {
                  const float4 kk = *reinterpret_cast<const float4*>(kr + col0 + jj);
                  o.x += ea.lam * kk.x; o.y += ea.lam * kk.y; o.z += ea.lam * kk.z; o.w += ea.lam * kk.w;
                }
                *reinterpret_cast<float4*>(g + col0 + jj) = o;
              }
            } else {
              for (int jj = 0; jj < 32; ++jj) {
                const long col = col0 + jj;
                if (col < ea.N) {
                  float o = __uint_as_float(v[jj]);
                  if (kr) o += ea.lam * kr[col];
                  g[col] = o;
                }
              }
            }
          }
        }
      }
      tc_fence_before();                               // this warp's TMEM reads of buffer b are done
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(tempty + b)) : "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static const EncodeTiledFn fn = [] {              // thread-safe one-time lookup (virtual-shard threads)
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiledFn>(p);
    return (EncodeTiledFn) nullptr;
  }();
  return fn;
}

bool make_map(CUtensorMap* m, const void* base, int op, long rows, long kdim, long ld, int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  const int esz = (op == 1) ? 4 : 2;
  CUtensorMapDataType dt = (op == 1) ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                     : (op == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
  cuuint64_t gdim[2] = {(cuuint64_t)kdim, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)(ld * esz)};
  cuuint32_t box[2] = {(cuuint32_t)(128 / esz), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void*>(base), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// K-blocked operand: {kchunk, rows, K/kchunk}, 128B-swizzled boxes of {128 B of K, box_rows, 1}
bool make_map_blocked(CUtensorMap* m, const void* base, int op, long rows, long kdim, long kchunk, int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc || kchunk <= 0 || kdim % kchunk) return false;
  const int esz = (op == 1) ? 4 : 2;
  CUtensorMapDataType dt = (op == 1) ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                     : (op == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
  cuuint64_t gdim[3] = {(cuuint64_t)kchunk, (cuuint64_t)rows, (cuuint64_t)(kdim / kchunk)};
  cuuint64_t gstride[2] = {(cuuint64_t)(kchunk * esz), (cuuint64_t)(rows * kchunk * esz)};
  cuuint32_t box[3] = {(cuuint32_t)(128 / esz), (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, dt, 3, const_cast<void*>(base), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int OP>
cudaError_t launch_op(const GemmArgs& g, cudaStream_t st) {
  CUtensorMap ta, tb;
  if (!make_map(&ta, g.Aop, OP, g.M, g.K, g.ld, BM)) return cudaErrorInvalidValue;
  if (g.kchunk > 0) {
    if (g.kchunk % (128 / ((OP == 1) ? 4 : 2)) || !make_map_blocked(&tb, g.Bop, OP, g.N, g.K, g.kchunk, BN))
      return cudaErrorInvalidValue;
  } else if (!make_map(&tb, g.Bop, OP, g.N, g.K, g.ld, BN)) {
    return cudaErrorInvalidValue;
  }
  EpiArgs ea{g.M, g.N, g.K, g.kchunk, g.epi, g.out, g.ldo, reinterpret_cast<const float*>(g.Kq), (float)g.lam};
  auto fn = gemm_tc_kernel<OP>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  static const int nsm = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  const long tiles = ((g.N + BN - 1) / BN) * ((g.M + BM - 1) / BM);
  fn<<<(unsigned)(tiles < nsm ? tiles : nsm), GEMM_THREADS, SMEM_BYTES, st>>>(ta, tb, ea);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gemm_tc(const GemmArgs& g, int op, cudaStream_t st) {
  switch (op) {
    case 1: return launch_op<1>(g, st);
    case 2: return launch_op<2>(g, st);
    case 3: return launch_op<3>(g, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace fram
