// common.cuh — device helpers shared by the libfram kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#if !defined(__CUDA_ARCH__) || (__CUDA_ARCH__ >= 1000)
#else
#error "libfram targets sm_100a only"
#endif

namespace fram {

constexpr int kWarp = 32;

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Grid-wide barrier for a cooperative launch (all CTAs co-resident).  `bar[0]` = arrival count,
// `bar[1]` = generation.  Both zero-initialised by the host before the launch.
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nblocks) {
  __syncthreads();
  if (nblocks > 1 && threadIdx.x == 0) {
    volatile unsigned int* gen = bar + 1;
    unsigned int g = *gen;
    __threadfence();
    unsigned int arrived = atomicAdd(bar, 1u);
    if (arrived == nblocks - 1) {
      bar[0] = 0u;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) { }
    }
    __threadfence();
  }
  __syncthreads();
}

// L1-bypassing loads for data written by other CTAs during the same launch.
template <typename T> __device__ __forceinline__ T ldcg(const T* p) { return __ldcg(p); }

// ---- operand-format rounding (round-to-nearest-even) -------------------------------------
__device__ __forceinline__ float tf32_rne(float x) {
  uint32_t b = __float_as_uint(x);
  if ((b & 0x7f800000u) == 0x7f800000u) return x;      // inf / nan untouched
  b += 0xfffu + ((b >> 13) & 1u);
  b &= ~0x1fffu;
  return __uint_as_float(b);
}

}  // namespace fram
