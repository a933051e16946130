// precond.cu — K1: preconditioning, Alg.1 steps 2-3 (rationale P:1025).
//   c = max(A, Ã, K) (FP64);  A' = A/√c, Ã' = Ã/√c, K' = K/c (FP64), then quantised to the GEMM
//   operand format (mixed modes) or kept FP64 (FP64 mode).  Ã' is written TRANSPOSED so that the
//   first gradient GEMM (U = N·Ã') sees its B operand K-major without assuming Ã symmetric.
// Validation (R28): non-finite, negative and (optionally) asymmetric entries are
// counted; the orchestrator turns any count into FRAM_ERR_DATA before touching outputs.
#include "common.cuh"
#include "internal.h"

namespace fram {

__device__ __forceinline__ double load_as_f64(const void* p, int dt, long idx) {
  if (dt == 0) return reinterpret_cast<const double*>(p)[idx];
  if (dt == 1) return (double)reinterpret_cast<const float*>(p)[idx];
  return (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[idx]);
}

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  // valid for v >= 0: the IEEE order of non-negative doubles equals the order of their bits
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

// 32×32 tiles; block (32, 8).  Tile (ti, tj) and its mirror (tj, ti) for the symmetry test.
__global__ void precond_scan_kernel(const void* A, const void* B, const void* K, int dt, long n,
                                    int check_sym, PrecondScan* out) {
  __shared__ double t1[32][33];
  __shared__ double t2[32][33];
  __shared__ double s_max[8];
  __shared__ unsigned long long s_cnt[3];
  const long ti = blockIdx.y, tj = blockIdx.x;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const void* mats[3] = {A, B, K};
  for (int mi = 0; mi < 3; ++mi) {
    const void* M = mats[mi];
    if (M == nullptr) continue;
    if (tid < 3) s_cnt[tid] = 0;
    __syncthreads();
    double mx = 0.0;
    unsigned long long nf = 0, ng = 0, as = 0;
    for (int r = ty; r < 32; r += 8) {
      const long i = ti * 32 + r, j = tj * 32 + tx;
      double v = 0.0;
      if (i < n && j < n) {
        v = load_as_f64(M, dt, i * n + j);
        if (!isfinite(v)) ++nf;
        else {
          if (v < 0.0) ++ng;
          mx = fmax(mx, v);
        }
      }
      t1[r][tx] = v;
      const long i2 = tj * 32 + r, j2 = ti * 32 + tx;
      t2[r][tx] = (check_sym && mi < 2 && i2 < n && j2 < n) ? load_as_f64(M, dt, i2 * n + j2) : 0.0;
    }
    __syncthreads();
    if (check_sym && mi < 2) {
      for (int r = ty; r < 32; r += 8) {
        const long i = ti * 32 + r, j = tj * 32 + tx;
        if (i < n && j < n) {
          const double a = t1[r][tx], b = t2[tx][r];     // M[i][j] vs M[j][i]
          if (!(a == b) && isfinite(a) && isfinite(b)) ++as;
        }
      }
    }
    mx = warp_max_d(mx);
    if (tx == 0) s_max[ty] = mx;
    if (nf) atomicAdd(&s_cnt[0], nf);
    if (ng) atomicAdd(&s_cnt[1], ng);
    if (as) atomicAdd(&s_cnt[2], as);
    __syncthreads();
    if (tid == 0) {
      double m = 0.0;
      for (int w = 0; w < 8; ++w) m = fmax(m, s_max[w]);
      atomic_max_nonneg(&out->maxv[mi], m);
      if (s_cnt[0]) atomicAdd(&out->bad_nonfinite, s_cnt[0]);
      if (s_cnt[1]) atomicAdd(&out->bad_negative, s_cnt[1]);
      if (s_cnt[2]) atomicAdd(&out->bad_asym, s_cnt[2]);
    }
    __syncthreads();
  }
}

cudaError_t launch_precond_scan(const void* A, const void* B, const void* K, int in_dt, long n,
                                bool check_sym, PrecondScan* out_dev, double*, unsigned*,
                                cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out_dev, 0, sizeof(PrecondScan), st);
  if (e != cudaSuccess) return e;
  const long nt = (n + 31) / 32;
  precond_scan_kernel<<<dim3((unsigned)nt, (unsigned)nt), dim3(32, 8), 0, st>>>(A, B, K, in_dt, n,
                                                                               check_sym ? 1 : 0, out_dev);
  return cudaGetLastError();
}

template <int OP> struct OpT;
template <> struct OpT<0> { using t = double; };
template <> struct OpT<1> { using t = float; };
template <> struct OpT<2> { using t = __nv_bfloat16; };
template <> struct OpT<3> { using t = __half; };

template <int OP> __device__ __forceinline__ typename OpT<OP>::t to_op(double x);
template <> __device__ __forceinline__ double to_op<0>(double x) { return x; }
template <> __device__ __forceinline__ float to_op<1>(double x) { return tf32_rne(__double2float_rn(x)); }
template <> __device__ __forceinline__ __nv_bfloat16 to_op<2>(double x) { return __double2bfloat16(x); }
template <> __device__ __forceinline__ __half to_op<3>(double x) { return __double2half(x); }

// A' (row-major) and Ã'ᵀ (row-major) into ld-padded buffers; K' = K/c (f32 or f64).
__global__ void precond_scan_rows_kernel(const void* A, const void* K, int dt, long rows, long n,
                                         PrecondScan* out) {
  const void* mats[2] = {A, K};
  for (int mi = 0; mi < 2; ++mi) {
    const void* M = mats[mi];
    if (!M) continue;
    double mx = 0.0;
    unsigned long long nf = 0, ng = 0;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < rows * n; idx += (long)gridDim.x * blockDim.x) {
      const double v = load_as_f64(M, dt, idx);
      if (!isfinite(v)) ++nf;
      else if (v < 0.0) ++ng;
      else mx = fmax(mx, v);
    }
    mx = warp_max_d(mx);
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(&out->maxv[mi == 0 ? 0 : 2], mx);
    if (nf) atomicAdd(&out->bad_nonfinite, nf);
    if (ng) atomicAdd(&out->bad_negative, ng);
  }
}

cudaError_t launch_precond_scan_rows(const void* A, const void* K, int in_dt, long rows, long n,
                                     PrecondScan* out_dev, cudaStream_t st) {
  precond_scan_rows_kernel<<<296, 256, 0, st>>>(A, K, in_dt, rows, n, out_dev);
  return cudaGetLastError();
}

template <int OP>
__global__ void precond_apply_kernel(const void* A, const void* B, const void* K, int dt, long n,
                                     long ld, const double* cmax, void* Aq, void* BqT, void* Kq,
                                     int k_f64, long rows_a) {
  using OT = typename OpT<OP>::t;
  __shared__ double tb[32][33];
  const double c = fmax(fmax(cmax[0], cmax[1]), cmax[2]);
  const double sA = sqrt(c);                                  // A/√c, IEEE-rounded sqrt
  const long ti = blockIdx.y, tj = blockIdx.x;
  const int tx = threadIdx.x, ty = threadIdx.y;
  OT* aq = reinterpret_cast<OT*>(Aq);
  OT* bq = reinterpret_cast<OT*>(BqT);
  for (int r = ty; r < 32; r += 8) {
    const long i = ti * 32 + r, j = tj * 32 + tx;
    if (i < n && j < n) {
      if (i < rows_a) {
        aq[i * ld + j] = to_op<OP>(load_as_f64(A, dt, i * n + j) / sA);
        if (K) {
          const double kv = load_as_f64(K, dt, i * n + j) / c;
          if (k_f64) reinterpret_cast<double*>(Kq)[i * ld + j] = kv;
          else reinterpret_cast<float*>(Kq)[i * ld + j] = __double2float_rn(kv);
        }
      }
      tb[r][tx] = load_as_f64(B, dt, i * n + j) / sA;
    }
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const long i = tj * 32 + r, j = ti * 32 + tx;          // BqT[i][j] = B'[j][i]
    if (i < n && j < n) bq[i * ld + j] = to_op<OP>(tb[tx][r]);
  }
}

cudaError_t launch_precond_apply(const void* A, const void* B, const void* K, int in_dt, long n,
                                 long ld, const double* c_dev, int op, void* Aq, void* BqT,
                                 void* Kq, bool k_f64, cudaStream_t st, long rows_a) {
  if (rows_a < 0) rows_a = n;
  const long nt = (n + 31) / 32;
  dim3 grid((unsigned)nt, (unsigned)nt), block(32, 8);
  const int kf = k_f64 ? 1 : 0;
  switch (op) {
    case 0: precond_apply_kernel<0><<<grid, block, 0, st>>>(A, B, K, in_dt, n, ld, c_dev, Aq, BqT, Kq, kf, rows_a); break;
    case 1: precond_apply_kernel<1><<<grid, block, 0, st>>>(A, B, K, in_dt, n, ld, c_dev, Aq, BqT, Kq, kf, rows_a); break;
    case 2: precond_apply_kernel<2><<<grid, block, 0, st>>>(A, B, K, in_dt, n, ld, c_dev, Aq, BqT, Kq, kf, rows_a); break;
    case 3: precond_apply_kernel<3><<<grid, block, 0, st>>>(A, B, K, in_dt, n, ld, c_dev, Aq, BqT, Kq, kf, rows_a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// Standalone input checks: SDSN counts negative or non-finite entries; the LAP (any real N,
// Eq.2) counts non-finite entries only.
template <typename T>
__global__ void scan_nonneg_kernel(const T* X, long n, unsigned long long* bad) {
  unsigned long long cnt = 0;
  const long total = n * n;
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
    const double v = (double)X[idx];
    if (!(v >= 0.0) || !isfinite(v)) ++cnt;
  }
  if (cnt) atomicAdd(bad, cnt);
}

__global__ void scan_finite_kernel(const double* X, long count, unsigned long long* bad) {
  unsigned long long cnt = 0;
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < count; idx += (long)gridDim.x * blockDim.x)
    if (!isfinite(X[idx])) ++cnt;
  if (cnt) atomicAdd(bad, cnt);
}

cudaError_t launch_scan_nonneg(const void* X, bool f64, long n, unsigned long long* bad, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  const int blocks = 592, threads = 256;
  if (f64) scan_nonneg_kernel<double><<<blocks, threads, 0, st>>>((const double*)X, n, bad);
  else scan_nonneg_kernel<float><<<blocks, threads, 0, st>>>((const float*)X, n, bad);
  return cudaGetLastError();
}

// `count` consecutive doubles (an ld-padded buffer whose padding is zero may be scanned whole)
cudaError_t launch_scan_finite(const double* X, long count, unsigned long long* bad, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  scan_finite_kernel<<<592, 256, 0, st>>>(X, count, bad);
  return cudaGetLastError();
}

}  // namespace fram
