// update.cu — K5/K6: FRAM update and outer stopping test (Alg.1 steps 7-8).
//   N⁽ᵗ⁾ = (1−α)N⁽ᵗ⁻¹⁾ + αD⁽ᵗ⁾  (FP64, evaluated unfused as in R15: __dmul_rn/__dadd_rn)
//   δ⁽ᵗ⁾ = ‖N⁽ᵗ⁾ − N⁽ᵗ⁻¹⁾‖_F / ‖N⁽ᵗ⁾‖_F  (R14)
// plus N_q = N rounded to the GEMM operand format for the next gradient.  The two sums of squares
// are reduced deterministically: per-CTA partials, then the last CTA to finish sums them in CTA
// order and writes out3 = {ΣΔ², ΣN², δ}.
#include "common.cuh"
#include "internal.h"

namespace fram {
namespace {

constexpr int UPD_THREADS = 512;

template <int OP> __device__ __forceinline__ void store_op(void* p, long idx, double v);
template <> __device__ __forceinline__ void store_op<0>(void*, long, double) {}
template <> __device__ __forceinline__ void store_op<1>(void* p, long idx, double v) {
  reinterpret_cast<float*>(p)[idx] = tf32_rne(__double2float_rn(v));
}
template <> __device__ __forceinline__ void store_op<2>(void* p, long idx, double v) {
  reinterpret_cast<__nv_bfloat16*>(p)[idx] = __double2bfloat16(v);
}
template <> __device__ __forceinline__ void store_op<3>(void* p, long idx, double v) {
  reinterpret_cast<__half*>(p)[idx] = __double2half(v);
}

// two adjacent N_q entries with one store (idx even, ld even)
template <int OP> __device__ __forceinline__ void store_op2(void* p, long idx, double v0, double v1);
template <> __device__ __forceinline__ void store_op2<0>(void*, long, double, double) {}
template <> __device__ __forceinline__ void store_op2<1>(void* p, long idx, double v0, double v1) {
  *reinterpret_cast<float2*>(reinterpret_cast<float*>(p) + idx) =
      make_float2(tf32_rne(__double2float_rn(v0)), tf32_rne(__double2float_rn(v1)));
}
template <> __device__ __forceinline__ void store_op2<2>(void* p, long idx, double v0, double v1) {
  __nv_bfloat162 t;
  t.x = __double2bfloat16(v0);
  t.y = __double2bfloat16(v1);
  *reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(p) + idx) = t;
}
template <> __device__ __forceinline__ void store_op2<3>(void* p, long idx, double v0, double v1) {
  __half2 t;
  t.x = __double2half(v0);
  t.y = __double2half(v1);
  *reinterpret_cast<__half2*>(reinterpret_cast<__half*>(p) + idx) = t;
}
template <typename TD> struct Pair;
template <> struct Pair<float> { using t = float2; };
template <> struct Pair<double> { using t = double2; };

template <int OP, typename TD>
__global__ void __launch_bounds__(UPD_THREADS) update_kernel(double* __restrict__ N, const TD* __restrict__ D,
                                                             void* Nq, long rows, long n, long ld, double alpha,
                                                             double* partials, unsigned* counter, double* out3) {
  __shared__ double s1[UPD_THREADS / 32], s2[UPD_THREADS / 32];
  __shared__ bool is_last;
  const double oma = 1.0 - alpha;
  double dd = 0.0, nn = 0.0;
  auto upd1 = [&](double old, double d, double& nv) {
    nv = __dadd_rn(__dmul_rn(oma, old), __dmul_rn(alpha, d));
    const double df = __dsub_rn(nv, old);
    dd = __fma_rn(df, df, dd);
    nn = __fma_rn(nv, nv, nn);
  };
  const bool vec = (ld % 2 == 0);
  const long npair = vec ? n / 2 : 0;                   // column pairs handled two-wide
  for (long i = blockIdx.x; i < rows; i += gridDim.x) {
    double* nr = N + i * ld;
    const TD* dr = D + i * ld;
    // pairs of columns: 16-byte N and 8/16-byte D accesses, four pairs per thread in flight
    constexpr int UNR = 4;
    for (long p0 = threadIdx.x; p0 < npair; p0 += (long)UNR * UPD_THREADS) {
      double2 o[UNR];
      double d0[UNR], d1[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const long pp = p0 + (long)u * UPD_THREADS;
        if (pp < npair) {
          o[u] = reinterpret_cast<const double2*>(nr)[pp];
          const typename Pair<TD>::t dv = reinterpret_cast<const typename Pair<TD>::t*>(dr)[pp];
          d0[u] = (double)dv.x;
          d1[u] = (double)dv.y;
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const long pp = p0 + (long)u * UPD_THREADS;
        if (pp < npair) {
          double2 nv;
          upd1(o[u].x, d0[u], nv.x);
          upd1(o[u].y, d1[u], nv.y);
          reinterpret_cast<double2*>(nr)[pp] = nv;
          store_op2<OP>(Nq, i * ld + 2 * pp, nv.x, nv.y);
        }
      }
    }
    for (long j = 2 * npair + threadIdx.x; j < n; j += UPD_THREADS) {   // odd tail / odd ld
      double nv;
      upd1(nr[j], (double)dr[j], nv);
      nr[j] = nv;
      store_op<OP>(Nq, i * ld + j, nv);
    }
  }
  dd = warp_sum_d(dd);
  nn = warp_sum_d(nn);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { s1[warp] = dd; s2[warp] = nn; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < UPD_THREADS / 32; ++w) { a += s1[w]; b += s2[w]; }
    partials[2 * blockIdx.x] = a;
    partials[2 * blockIdx.x + 1] = b;
    __threadfence();
    const unsigned done = atomicAdd(counter, 1u);
    is_last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last && threadIdx.x == 0) {
    __threadfence();
    double a = 0.0, b = 0.0;
    for (unsigned k = 0; k < gridDim.x; ++k) { a += __ldcg(partials + 2 * k); b += __ldcg(partials + 2 * k + 1); }
    out3[0] = a;
    out3[1] = b;
    out3[2] = sqrt(a) / sqrt(b);
    *counter = 0u;
  }
}

template <int OP>
__global__ void init_n_kernel(double* N, void* Nq, const double* X0, long rows, long n, long ld) {
  const double u = 1.0 / (double)n;
  for (long i = blockIdx.x; i < rows; i += gridDim.x)
    for (long j = threadIdx.x; j < n; j += blockDim.x) {
      const double v = X0 ? X0[i * n + j] : u;
      N[i * ld + j] = v;
      store_op<OP>(Nq, i * ld + j, v);
    }
}

// dst (drows × dcols, leading dim ldd, FP64) ← src (rows × cols of dtype dt, leading dim lds), zero
// outside the source block (padding of attributed graphs, R30)
__global__ void pad_convert_kernel(double* dst, long ldd, long drows, long dcols, const void* src, int dt, long lds,
                                   long rows, long cols) {
  for (long i = blockIdx.x; i < drows; i += gridDim.x)
    for (long j = threadIdx.x; j < dcols; j += blockDim.x) {
      double v = 0.0;
      if (i < rows && j < cols) {
        const long idx = i * lds + j;
        if (dt == 0) v = reinterpret_cast<const double*>(src)[idx];
        else if (dt == 1) v = (double)reinterpret_cast<const float*>(src)[idx];
        else v = (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(src)[idx]);
      }
      dst[i * ldd + j] = v;
    }
}

__global__ void copy2d_kernel(double* dst, long ldd, const double* src, long lds, long rows, long cols) {
  for (long i = blockIdx.x; i < rows; i += gridDim.x)
    for (long j = threadIdx.x; j < cols; j += blockDim.x) dst[i * ldd + j] = src[i * lds + j];
}

}  // namespace

template <int OP, typename TD>
static void launch_upd(double* N, const void* D, void* Nq, long rows, long n, long ld, double alpha,
                       double* partials, unsigned* counter, double* out3, cudaStream_t st, int num_sms) {
  // exactly the resident CTAs: one wave (the partials buffer holds at most 4 CTAs per SM); computed
  // once per instantiation (thread-safe static initialisation; every device here is an sm_100a B200)
  static const int per_sm = []() {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, update_kernel<OP, TD>, UPD_THREADS, 0) !=
                        cudaSuccess || occ <= 0)
      return 4;
    return occ < 4 ? occ : 4;
  }();
  const int grid = (int)((rows < (long)num_sms * per_sm) ? rows : (long)num_sms * per_sm);
  update_kernel<OP, TD><<<grid, UPD_THREADS, 0, st>>>(N, (const TD*)D, Nq, rows, n, ld, alpha, partials, counter,
                                                      out3);
}

cudaError_t launch_update(double* N, const void* D, bool d_f64, void* Nq, int op, long rows, long n, long ld,
                          double alpha, double* partials, unsigned* counter, double* out3, cudaStream_t st,
                          int num_sms) {
#define UPD_CASE(OPV)                                                                                        \
  if (d_f64) launch_upd<OPV, double>(N, D, Nq, rows, n, ld, alpha, partials, counter, out3, st, num_sms);      \
  else launch_upd<OPV, float>(N, D, Nq, rows, n, ld, alpha, partials, counter, out3, st, num_sms);
  switch (op) {
    case 0: UPD_CASE(0) break;
    case 1: UPD_CASE(1) break;
    case 2: UPD_CASE(2) break;
    case 3: UPD_CASE(3) break;
    default: return cudaErrorInvalidValue;
  }
#undef UPD_CASE
  return cudaGetLastError();
}

cudaError_t launch_init_n(double* N, void* Nq, int op, const double* X0, long rows, long n, long ld,
                          cudaStream_t st) {
  const int grid = (int)(rows < 1024 ? rows : 1024);
  switch (op) {
    case 0: init_n_kernel<0><<<grid, 256, 0, st>>>(N, Nq, X0, rows, n, ld); break;
    case 1: init_n_kernel<1><<<grid, 256, 0, st>>>(N, Nq, X0, rows, n, ld); break;
    case 2: init_n_kernel<2><<<grid, 256, 0, st>>>(N, Nq, X0, rows, n, ld); break;
    case 3: init_n_kernel<3><<<grid, 256, 0, st>>>(N, Nq, X0, rows, n, ld); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_pad_convert(double* dst, long ldd, long drows, long dcols, const void* src, int dt, long lds,
                               long rows, long cols, cudaStream_t st) {
  const int grid = (int)(drows < 2048 ? drows : 2048);
  pad_convert_kernel<<<grid < 1 ? 1 : grid, 256, 0, st>>>(dst, ldd, drows, dcols, src, dt, lds, rows, cols);
  return cudaGetLastError();
}

cudaError_t launch_copy2d_f64(double* dst, long ldd, const double* src, long lds, long rows, long cols,
                              cudaStream_t st) {
  const int grid = (int)(rows < 1024 ? rows : 1024);
  copy2d_kernel<<<grid < 1 ? 1 : grid, 256, 0, st>>>(dst, ldd, src, lds, rows, cols);
  return cudaGetLastError();
}

}  // namespace fram
