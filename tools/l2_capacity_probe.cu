// Dev probe: effective L2 capacity seen by a small cluster of SMs reading random rows, the LAP's
// access pattern (K7c: 8 CTAs, each reads its 4 KB slice of a random 32 KB row of an FP64 matrix).
// For working sets W = 16 … 160 MB: warm up, then time dependent random row reads (each step waits
// for its row, like a Dijkstra step) and report ns per step; ncu's lts__t_sector_hit_rate on the
// same command gives the hit rate.  A knee near half of the 126 MB would mean the cluster's die
// caches far-homed lines in its own L2 half.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2cap tools/l2_capacity_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int CS = 8, THREADS = 128, CPT = 4, ROWLEN = CS * THREADS * CPT;   // 4096 doubles per row

__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(THREADS, 1)
rowwalk(const double* __restrict__ N, int rows, int steps, unsigned seed, double* out, long long* ns) {
  unsigned crank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const int tid = threadIdx.x;
  double acc = 0.0;
  unsigned x = seed;
  long long t0 = 0;
  for (int s = 0; s < steps; ++s) {
    if (s == steps / 2) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    x = x * 1664525u + 1013904223u;                       // same sequence in every thread
    // the row depends on the previous step's data (like p[j1] → row), so steps are serial
    const int row = (int)((x ^ (unsigned)(acc < 0.0)) % (unsigned)rows);
    const double* r = N + (size_t)row * ROWLEN + crank * THREADS * CPT + tid;
#pragma unroll
    for (int k = 0; k < CPT; ++k) acc += __ldcg(r + k * THREADS);
    acc = __shfl_sync(0xffffffffu, acc, 0);              // warp-uniform dependency
  }
  long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (tid == 0 && crank == 0) ns[0] = t1 - t0;
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  const size_t maxb = 160ull << 20;
  double* N; double* out; long long* ns;
  cudaMalloc(&N, maxb); cudaMalloc(&out, 8); cudaMalloc(&ns, 8);
  cudaMemset(N, 0, maxb);
  const int Ws[] = {16, 32, 48, 56, 64, 72, 80, 96, 112, 128, 144, 160};
  for (int W : Ws) {
    const int rows = (int)(((size_t)W << 20) / (ROWLEN * 8));
    const int steps = 200000;
    rowwalk<<<CS, THREADS>>>(N, rows, steps, 12345u, out, ns);
    rowwalk<<<CS, THREADS>>>(N, rows, steps, 777u, out, ns);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    long long t;
    cudaMemcpy(&t, ns, 8, cudaMemcpyDeviceToHost);
    printf("W = %3d MB (%6d rows): %.1f ns per dependent row step\n", W, rows, (double)t / (steps - steps / 2));
  }
  return 0;
}
