// Dev probe: can one TMA load put a row of an FP32 n×ld matrix into K4r's slot layout?
// 4-D view {e = 4 floats, t = 128 owner threads, c = V chunks, row} with byte strides {128·V/… :
// t → CPT·4 B, c → 16 B, row → ld·4 B}; box {4, 128, V, 1} lands in shared memory as [c][t][e], i.e.
// float4 (c·128 + t) = columns t·CPT + 4c … +3, exactly s_rows' layout.  Also times 28 rows per CTA ×
// 148 CTAs (the C4 load phase) against the current per-thread 16-byte loads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_slot tools/tma_slot_probe.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

constexpr int CPT = 32, V = CPT / 4, NS = 128 * CPT;   // n = 4096

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(512, 1) tma_rows(const __grid_constant__ CUtensorMap tm, const float* Y, long n, long ld,
                                                   int rows_per_cta, int mode, float* out, long long* ns) {
  extern __shared__ __align__(128) float4 srow[];        // [rows][V][128]
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const long r0 = (long)blockIdx.x * rows_per_cta;
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (mode == 0) {
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(rows_per_cta * NS * 4) : "memory");
      for (int r = 0; r < rows_per_cta; ++r)
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     ::"r"(sa(srow + (size_t)r * V * 128)), "l"(&tm), "r"(0), "r"(0), "r"(0), "r"((int)(r0 + r)), "r"(sa(&bar))
                     : "memory");
    }
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(sa(&bar)), "r"(0) : "memory");
  } else {                                               // K4r's current pattern: thread t, 16-byte loads
    const int t = tid & 127, h = tid >> 7;               // 4 groups of 128 threads split the rows
    for (int r = h; r < rows_per_cta; r += 4) {
      const float* g = Y + (r0 + r) * ld;
#pragma unroll
      for (int c = 0; c < V; ++c) srow[(size_t)r * V * 128 + c * 128 + t] = __ldca(reinterpret_cast<const float4*>(g + t * CPT + 4 * c));
    }
    __syncthreads();
  }
  long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (tid == 0) ns[blockIdx.x] = t1 - t0;
  // checksum of the slot layout: float4 (c·128 + t) of row r must hold Y[r][t·CPT + 4c .. +3]
  __syncthreads();
  float bad = 0.f;
  for (int r = 0; r < rows_per_cta; ++r)
    for (int f = tid; f < V * 128; f += 512) {
      const int c = f / 128, t = f % 128;
      const float4 v = srow[(size_t)r * V * 128 + f];
      const float* g = Y + (r0 + r) * ld + t * CPT + 4 * c;
      bad += (v.x != g[0]) + (v.y != g[1]) + (v.z != g[2]) + (v.w != g[3]);
    }
  if (bad > 0.f) atomicAdd(out, bad);
}

int main() {
  const long n = NS, ld = NS;
  const int G = 148, R = 12;
  const long rows = (long)G * R;
  float* Y; float* out; long long* ns;
  cudaMalloc(&Y, rows * ld * 4); cudaMalloc(&out, 4); cudaMalloc(&ns, G * 8);
  std::vector<float> h(rows * ld);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)(i % 9973) * 0.5f;
  cudaMemcpy(Y, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* fp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<decltype(&cuTensorMapEncodeTiled)>(fp);
  CUtensorMap tm;
  cuuint64_t gdim[4] = {4, 128, (cuuint64_t)V, (cuuint64_t)rows};
  cuuint64_t gstr[3] = {(cuuint64_t)CPT * 4, 16, (cuuint64_t)ld * 4};
  cuuint32_t box[4] = {4, 128, (cuuint32_t)V, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, Y, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)cr);
  if (cr != CUDA_SUCCESS) return 1;
  const int smem = R * NS * 4;
  cudaFuncSetAttribute(tma_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 2; ++mode)
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(out, 0, 4);
      tma_rows<<<G, 512, smem>>>(tm, Y, n, ld, R, mode, out, ns);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      float bad; cudaMemcpy(&bad, out, 4, cudaMemcpyDeviceToHost);
      std::vector<long long> t(G); cudaMemcpy(t.data(), ns, G * 8, cudaMemcpyDeviceToHost);
      long long mx = 0, sum = 0; for (auto v : t) { mx = std::max(mx, v); sum += v; }
      printf("%s: %d rows x 16 KB per CTA: mean %.1f us, max %.1f us, mismatches %.0f\n", mode == 0 ? "TMA 4-D slot load " : "per-thread ld.ca   ",
             R, sum / 1e3 / G, mx / 1e3, bad);
    }
  return 0;
}
