// Dev probe: per-SMSP throughput of FADD2 / FADD / FMNMX / mixes (16 warps per SM, 8 independent chains).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  float2 d;
  asm volatile("{.reg .b64 ra, rb, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n add.rn.f32x2 rd, ra, rb;\n mov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(int iters, float* out, long long* cyc) {
  float2 x[8]; float y[16];
  for (int i = 0; i < 8; ++i) { x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f); }
  for (int i = 0; i < 16; ++i) y[i] = threadIdx.x * 1e-3f + i;
  const float2 c = make_float2(1e-7f, -1e-7f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (MODE == 0) {               // 8 FADD2
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = add2(x[i], c);
      } else if (MODE == 1) {        // 16 FADD
#pragma unroll
        for (int i = 0; i < 16; ++i) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(y[i]) : "f"(1e-7f));
      } else if (MODE == 2) {        // 16 FMNMX
#pragma unroll
        for (int i = 0; i < 16; ++i) asm volatile("max.f32 %0, %0, %1;" : "+f"(y[i]) : "f"(0.5f));
      } else if (MODE == 3) {        // 8 FADD2 + 8 FMNMX interleaved
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          x[i] = add2(x[i], c);
          asm volatile("max.f32 %0, %0, %1;" : "+f"(y[i]) : "f"(0.5f));
        }
      } else if (MODE == 4) {        // 16 FFMA
#pragma unroll
        for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(y[i]) : "f"(1.0f), "f"(1e-7f));
      } else if (MODE == 5) {        // 8 IMNMX
#pragma unroll
        for (int i = 0; i < 16; ++i) asm volatile("max.s32 %0, %0, %1;" : "+r"(*(int*)&y[i]) : "r"(5));
      }
    }
  }
  long long t1 = clock64();
  float acc = 0.f;
  for (int i = 0; i < 8; ++i) acc += x[i].x + x[i].y;
  for (int i = 0; i < 16; ++i) acc += y[i];
  if (acc == 1.234f) out[0] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE> void run(const char* nm, int per_iter) {
  float* o; long long* c; cudaMalloc(&o, 4); cudaMalloc(&c, 148 * 8);
  const int iters = 4096;
  k<MODE><<<148, 512>>>(iters, o, c); cudaDeviceSynchronize();
  k<MODE><<<148, 512>>>(iters, o, c); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  // per SMSP: 4 warps × iters × per_iter instructions
  printf("%-28s %.2f cycles per warp-instruction per SMSP\n", nm, (double)h / (4.0 * iters * per_iter));
}
int main() {
  run<0>("FADD2", 32); run<1>("FADD", 64); run<2>("FMNMX", 64); run<3>("FADD2+FMNMX (8+8)", 64); run<4>("FFMA", 64); run<5>("IMNMX", 64);
}
