// Dev probe (not part of libfram): on-chip bandwidth of TMEM (tcgen05.ld/st), shared memory and
// register-resident elementwise work, to size the on-chip-resident SDSN design.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_probe tools/tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Each warp: ITERS times { ld 32 cols x32 of its lane quarter at column c, add 1, st back }.
template <int X>
__global__ void __launch_bounds__(512, 1) tmem_rw(int iters, int ncols, float* out, long long* cyc) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  const int q = warp & 3, g = warp >> 2, ng = blockDim.x / 128;
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int c = g * X; c < ncols; c += ng * X) {
      const uint32_t addr = tm + ((uint32_t)(q * 32) << 16) + (uint32_t)c;
      uint32_t v[X];
      if constexpr (X == 32) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(addr));
      } else {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(addr));
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int k = 0; k < X; ++k) {
        float f = __uint_as_float(v[k]) + 1.0f;
        acc += f;
        v[k] = __float_as_uint(f);
      }
      if constexpr (X == 32) {
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
            ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
      } else {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                     ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
      }
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  long long t1 = clock64();
  if (acc == 12345.f) out[0] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

// Shared memory: each thread float4 read-modify-write over `bytes` of smem, conflict-free.
__global__ void __launch_bounds__(512, 1) smem_rw(int iters, int bytes, float* out, long long* cyc) {
  extern __shared__ float4 sm[];
  const int nv = bytes / 16;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) sm[i] = make_float4(0, 0, 0, 0);
  __syncthreads();
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll 4
    for (int i = threadIdx.x; i < nv; i += blockDim.x) {
      float4 v = sm[i];
      v.x += 1.f; v.y += 1.f; v.z += 1.f; v.w += 1.f;
      acc += v.x + v.y + v.z + v.w;
      sm[i] = v;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (acc == 12345.f) out[0] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// Register-resident SDSN-like elementwise work: E elements per thread, ops per element:
// y = max(0, (y + a) + b); col += y; row += y.
template <int E>
__global__ void __launch_bounds__(512, 1) reg_alu(int iters, float* out, long long* cyc) {
  float y[E], col[E], bb[E];
#pragma unroll
  for (int k = 0; k < E; ++k) { y[k] = threadIdx.x * 1e-3f + k; col[k] = 0; bb[k] = -1e-3f * k; }
  float row = 0.f;
  const float a = 1e-4f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < E; ++k) {
      float t = fmaxf(0.f, (y[k] + a) + bb[k]);
      y[k] = t;
      col[k] += t;
      row += t;
    }
  }
  long long t1 = clock64();
  float s = row;
#pragma unroll
  for (int k = 0; k < E; ++k) s += col[k] + y[k];
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}


__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;
}
__device__ __forceinline__ unsigned long long pk(float x, float y) {
  return ((unsigned long long)__float_as_uint(y) << 32) | __float_as_uint(x);
}
// Same as reg_alu with the four adds done two elements at a time (FADD2).
template <int E>
__global__ void __launch_bounds__(512, 1) reg_alu2(int iters, float* out, long long* cyc) {
  unsigned long long y[E / 2], col[E / 2], bb[E / 2];
#pragma unroll
  for (int k = 0; k < E / 2; ++k) { y[k] = pk(threadIdx.x * 1e-3f + k, k); col[k] = 0; bb[k] = pk(-1e-3f * k, -2e-3f * k); }
  unsigned long long row = 0;
  const unsigned long long a = pk(1e-4f, 1e-4f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < E / 2; ++k) {
      unsigned long long t = add2(add2(y[k], a), bb[k]);
      float lo = fmaxf(0.f, __uint_as_float((unsigned)t)), hi = fmaxf(0.f, __uint_as_float((unsigned)(t >> 32)));
      t = pk(lo, hi);
      y[k] = t;
      col[k] = add2(col[k], t);
      row = add2(row, t);
    }
  }
  long long t1 = clock64();
  float s = __uint_as_float((unsigned)row);
#pragma unroll
  for (int k = 0; k < E / 2; ++k) s += __uint_as_float((unsigned)col[k]) + __uint_as_float((unsigned)y[k]);
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// Grid barrier latency: monotonic counter, one red.release + acquire poll per CTA.
__global__ void __launch_bounds__(512, 1) gbar(int iters, unsigned* ctr, long long* cyc) {
  long long t0 = clock64();
  for (int it = 1; it <= iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
      const unsigned target = (unsigned)it * gridDim.x;
      unsigned v;
      do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; long long h[148];
  cudaMalloc(&out, 4); cudaMalloc(&cyc, 148 * 8);
  auto report = [&](const char* name, double bytes_per_sm) {
    cudaDeviceSynchronize();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("%s: error %s\n", name, cudaGetErrorString(e)); return; }
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("%-40s %10lld cyc  %.1f B/cyc/SM\n", name, mx, bytes_per_sm / mx);
  };
  const int iters = 200;
  tmem_rw<32><<<148, 512>>>(iters, 512, out, cyc);
  report("tmem ld+st x32, 16 warps, 512 cols", 2.0 * iters * 512 * 128 * 4);
  tmem_rw<32><<<148, 128>>>(iters, 512, out, cyc);
  report("tmem ld+st x32, 4 warps", 2.0 * iters * 512 * 128 * 4);
  tmem_rw<32><<<148, 256>>>(iters, 512, out, cyc);
  report("tmem ld+st x32, 8 warps", 2.0 * iters * 512 * 128 * 4);
  tmem_rw<8><<<148, 512>>>(iters, 512, out, cyc);
  report("tmem ld+st x8, 16 warps", 2.0 * iters * 512 * 128 * 4);
  cudaFuncSetAttribute(smem_rw, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  smem_rw<<<148, 512, 196608>>>(iters, 196608, out, cyc);
  report("smem float4 rmw 192KB, 16 warps", 2.0 * iters * 196608);
  smem_rw<<<148, 256, 196608>>>(iters, 196608, out, cyc);
  report("smem float4 rmw 192KB, 8 warps", 2.0 * iters * 196608);
  reg_alu<32><<<148, 512>>>(iters * 16, out, cyc);
  report("reg alu E=32, 512 thr (B = elem*8)", 8.0 * iters * 16 * 32 * 512);
  reg_alu<64><<<148, 256>>>(iters * 16, out, cyc);
  report("reg alu E=64, 256 thr (B = elem*8)", 8.0 * iters * 16 * 64 * 256);
  reg_alu2<32><<<148, 512>>>(iters * 16, out, cyc);
  report("reg alu FADD2 E=32, 512 thr (B = elem*8)", 8.0 * iters * 16 * 32 * 512);
  unsigned* ctr; cudaMalloc(&ctr, 4); cudaMemset(ctr, 0, 4);
  int nb = 1000; void* args[] = {&nb, &ctr, &cyc};
  cudaLaunchCooperativeKernel((void*)gbar, 148, 512, args, 0, 0);
  report("grid barrier x1000 (B/cyc meaningless)", 1.0);
  printf("=> per barrier: %.0f cycles\n", (double)h[0] / nb);
  return 0;
}
