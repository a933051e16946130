// Dev probe: max active clusters for 1-CTA/SM kernels and cooperative + cluster launches on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* o) { extern __shared__ float s[]; s[threadIdx.x] = 1; __syncthreads(); if (o) o[blockIdx.x] = s[0]; }
int main() {
  int smem = 200 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148 / cs * cs); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: max active clusters %d (%d CTAs) %s\n", cs, n, n * cs, cudaGetErrorString(e));
  }
  // cooperative + cluster launch
  for (int cs : {2, 4}) {
    cudaLaunchConfig_t cfg = {};
    int G = 148 / cs * cs;
    cfg.gridDim = dim3(G); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[2]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative; at[1].val.cooperative = 1;
    cfg.attrs = at; cfg.numAttrs = 2;
    float* o; cudaMalloc(&o, 4 * 148);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, o);
    cudaError_t e2 = cudaDeviceSynchronize();
    printf("coop+cluster %d grid %d: launch %s sync %s\n", cs, G, cudaGetErrorString(e), cudaGetErrorString(e2));
  }
  return 0;
}
