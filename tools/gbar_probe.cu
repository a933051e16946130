// Dev probe (not part of libfram): grid-barrier variants for a 148-CTA persistent kernel.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gbar_probe.bin tools/gbar_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) { unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) { unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) { asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ unsigned atom_rel(unsigned* p, unsigned v) { unsigned o; asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory"); return o; }
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) { asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }

// V0: one counter, red.release + acquire poll
// V1: two-level: groups of 16 CTAs; last arriver of a group (atom return) bumps the top counter; all poll top
// V2: one counter, relaxed poll + fence after
// V3: one counter on its own 128B line, poll with nanosleep(32)
// V4: V0 but the counter arrive by every warp's lane 0 is replaced by... (same as V0 with 256-thread CTAs)
template <int V>
__global__ void __launch_bounds__(256, 1) gbar(int iters, unsigned* ctr, long long* cyc) {
  const unsigned G = gridDim.x;
  long long t0 = clock64();
  for (unsigned it = 1; it <= (unsigned)iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      if (V == 0 || V == 3) {
        red_rel(ctr, 1);
        while (ld_acq(ctr) < it * G) { if (V == 3) __nanosleep(32); }
      } else if (V == 2) {
        red_rel(ctr, 1);
        while (ld_rlx(ctr) < it * G) {}
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else if (V == 1) {
        const unsigned grp = blockIdx.x / 16, ng = (G + 15) / 16;
        const unsigned gsz = min(16u, G - grp * 16);
        unsigned* gc = ctr + 32 * (1 + grp);
        const unsigned o = atom_rel(gc, 1);
        if (o + 1 == it * gsz) red_rel(ctr, 1);
        while (ld_acq(ctr) < it * ng) {}
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  unsigned* ctr; long long* cyc; long long h[148];
  cudaMalloc(&ctr, 64 * 1024); cudaMalloc(&cyc, 148 * 8);
  int nb = 2000;
  auto run = [&](const char* name, void* fn) {
    cudaMemset(ctr, 0, 64 * 1024);
    void* args[] = {&nb, &ctr, &cyc};
    cudaLaunchCooperativeKernel(fn, 148, 256, args, 0, 0);
    cudaDeviceSynchronize();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-40s %.0f cycles/barrier\n", name, (double)h[0] / nb);
  };
  for (int rep = 0; rep < 2; ++rep) {
    run("V0 counter red.release + acquire poll", (void*)gbar<0>);
    run("V1 two-level (16) atom + top counter", (void*)gbar<1>);
    run("V2 counter + relaxed poll + fence", (void*)gbar<2>);
    run("V3 V0 + nanosleep(32)", (void*)gbar<3>);
  }
  return 0;
}
