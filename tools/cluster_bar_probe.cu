// Dev probe: cost of one cluster-wide barrier (barrier.cluster.arrive.release + wait.acquire) and of a
// DSMEM store + cluster barrier round, per iteration, for clusters of 2 and 4 CTAs (512 threads each).
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(int iters, long long* out) {
  __shared__ unsigned long long slot[2][8];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank(), nb = cl.num_blocks();
  cl.sync();
  long long t0 = clock64();
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 1 && threadIdx.x < nb) {       // every CTA writes its candidate into every CTA's slot
      unsigned long long* dst = cl.map_shared_rank(&slot[it & 1][rank], threadIdx.x);
      *dst = (unsigned long long)it * 8 + rank;
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (MODE == 1) acc += slot[it & 1][(it + 1) % nb];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = acc; }
}
template <int MODE> void run(int cs) {
  long long* o; cudaMalloc(&o, 16);
  cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(cs); cfg.blockDim = dim3(512);
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  const int iters = 100000;
  cudaLaunchKernelEx(&cfg, k<MODE>, iters, o); cudaDeviceSynchronize();
  cudaLaunchKernelEx(&cfg, k<MODE>, iters, o); cudaError_t e = cudaDeviceSynchronize();
  long long h[2]; cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  printf("cluster %d mode %d: %.0f cycles per iteration %s\n", cs, MODE, (double)h[0] / iters, cudaGetErrorString(e));
}
int main() { run<0>(2); run<1>(2); run<0>(4); run<1>(4); 
  // reference: __syncthreads loop in one CTA
  return 0; }
