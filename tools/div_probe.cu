// Dev probe: S/d via a precomputed correctly rounded reciprocal and one FMA correction (Markstein)
// against IEEE division, for random S and d = n, n^2.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned long long seed, int iters, unsigned long long* bad) {
  unsigned long long x = seed ^ (0x9e3779b97f4a7c15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1));
  unsigned long long nb = 0;
  for (int it = 0; it < iters; ++it) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    const int n = 1 + (int)((x >> 40) % 70000);
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    const double S = __longlong_as_double((long long)((x & 0x000fffffffffffffull) | (((x >> 52) % 120 + 960ull) << 52)));  // ~[2^-63, 2^56]
    const double dn = (double)n, nn = dn * dn;
    const double rn = __drcp_rn(dn), rnn = __drcp_rn(nn);
    double q = S * rn; double e = fma(-q, dn, S); const double a1 = fma(rn, e, q);
    q = S * rnn; e = fma(-q, nn, S); const double a2 = fma(rnn, e, q);
    if (a1 != S / dn) ++nb;
    if (a2 != S / nn) ++nb;
    if (rn != 1.0 / dn) ++nb;
  }
  atomicAdd(bad, nb);
}
int main() {
  unsigned long long* b; cudaMalloc(&b, 8); cudaMemset(b, 0, 8);
  for (int r = 0; r < 4; ++r) k<<<148 * 4, 256>>>(1234567ull + r, 20000, b);
  cudaDeviceSynchronize();
  unsigned long long h; cudaMemcpy(&h, b, 8, cudaMemcpyDeviceToHost);
  printf("mismatches: %llu of %.3g\n", h, 4.0 * 148 * 4 * 256 * 20000 * 3);
}
