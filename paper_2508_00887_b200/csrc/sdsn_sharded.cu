// sdsn_sharded.cu — K4s: SDSN (Alg. 2) on a ROW BLOCK of the iterate, for the
// row-sharded solve of config C5: rank r owns rows [r·n/W, (r+1)·n/W) of Y.
//
// Row sums are local to a rank; column sums and the mass S are global.  One pass is
//   pass kernel  : y ← max(0, (y + a_i) + b_j) on the local rows (a_i from the local row sums and
//                  the global S, b_j = −c_j/n from the all-reduced column sums), accumulating the new
//                  local row sums (FP64 per row) and per-CTA column partials (T);
//   reduce kernel: c_j(local) = Σ_CTA partials (FP64, CTA order), S(local) = Σ_i r_i (FP64, fixed
//                  tree) → send[0..n]
//   ncclAllReduce(send → recv, n+1 FP64, sum)   — issued by the host between the kernels
// so that every rank holds identical (c, S) and takes the same stop decision (R5).  The stop test
// (lagged γ, R5/R16) is evaluated on the device by every CTA of the next pass kernel; after the last
// pass a `done` flag turns the remaining queued passes into no-ops, and the host polls it once per
// chunk of passes.  Same arithmetic and groupings as the single-GPU kernels (R9, R11, R13).
#include <math_constants.h>
#include "common.cuh"
#include "internal.h"

namespace fram {
namespace {

constexpr int kShThreads = 512;                  // 256 / 1024 measured slower (418 / 386 vs 375 us at C5)

template <typename T> struct V4;
template <> struct V4<float> { using t = float4; static constexpr int W = 4; };
template <> struct V4<double> { using t = double2; static constexpr int W = 2; };

template <typename T>
__device__ __forceinline__ void vsplit(const typename V4<T>::t& v, T* o);
template <> __device__ __forceinline__ void vsplit<float>(const float4& v, float* o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
template <> __device__ __forceinline__ void vsplit<double>(const double2& v, double* o) { o[0] = v.x; o[1] = v.y; }
template <typename T>
__device__ __forceinline__ typename V4<T>::t vjoin(const T* o);
template <> __device__ __forceinline__ float4 vjoin<float>(const float* o) { return make_float4(o[0], o[1], o[2], o[3]); }
template <> __device__ __forceinline__ double2 vjoin<double>(const double* o) { return make_double2(o[0], o[1]); }

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

// local max of the row block (non-negative values: max as unsigned bit patterns)
template <typename T>
__global__ void sh_max_kernel(const T* __restrict__ Y, long rows, long n, long ld, double* out) {
  double m = 0.0;
  for (long i = blockIdx.x; i < rows; i += gridDim.x)
    for (long j = threadIdx.x; j < n; j += blockDim.x) m = fmax(m, (double)Y[i * ld + j]);
  m = warp_max_d(m);
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, m);
}

// One sweep over the CTA's rows.  mode 0: scale (y ← fl(s·y), s = (θ/2)/m from recv[0]; m = 0 ⇒
// 11ᵀ/n and done); mode 1: SDSN pass p.  Column partials in shared memory (one owner per column).
template <typename T>
__global__ void __launch_bounds__(kShThreads, 1) sh_pass_kernel(ShardSdsnParams P, int mode) {
  using VT = typename V4<T>::t;
  constexpr int W = V4<T>::W;
  extern __shared__ __align__(16) unsigned char dsm[];
  ShardSdsnState* st = P.state;
  if (st->done) return;
  const int p = st->pass;                                        // pass index (mode 1), device-side
  const long n = P.n, ld = P.ld, rows = P.rows;
  T* s_col = reinterpret_cast<T*>(dsm);                          // [ld] column partials
  T* s_b = s_col + ld;                                           // [ld] b_j = −c_j/n (FP32 mode only)
  constexpr bool BS = sizeof(T) == 4;
  const double dn = (double)n, nn = dn * dn;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long r0 = (long)blockIdx.x * rows / gridDim.x, r1 = (long)(blockIdx.x + 1) * rows / gridDim.x;
  const long nvec = ld / W;
  T* Y = reinterpret_cast<T*>(P.Y);

  double sc = 1.0, S = 0.0, abase = 0.0;
  bool last = false;
  if (mode == 0) {
    const double m = P.recv[0];
    if (P.scale && m == 0.0) {                                              // R10 (θ-scaling on): all-zero ⇒ 11ᵀ/n, 0 passes
      for (long i = r0; i < r1; ++i)
        for (long j = tid; j < n; j += kShThreads) Y[i * ld + j] = (T)(1.0 / dn);
      if (blockIdx.x == 0 && tid == 0) {
        st->done = 1; st->passes = 0; st->gamma_last = 0.0; st->maxx = 0.0;
      }
      return;
    }
    sc = P.scale ? (P.theta / 2.0) / m : 1.0;                    // R11
    if (blockIdx.x == 0 && tid == 0) st->maxx = m;
  } else {
    S = P.recv[n];
    const double gam = S / dn - 1.0;                             // γ_p of the pass input
    last = P.sdsn_fixed > 0 ? (p + 1 >= P.sdsn_fixed) : ((p >= 1 && gam <= P.gamma_th) || p + 1 >= P.sdsn_max);
    abase = 1.0 / dn + S / nn;
    if (blockIdx.x == 0 && tid == 0) {
      if (P.gamma_hist) P.gamma_hist[p] = gam;
      if (last) { st->passes = p + 1; st->gamma_last = gam; st->S_last = S; }
    }
  }
  for (long q = tid; q < nvec; q += kShThreads) {
    T z[W];
#pragma unroll
    for (int w = 0; w < W; ++w) z[w] = (T)0;
    reinterpret_cast<VT*>(s_col)[q] = vjoin<T>(z);
    if (BS && mode) {
#pragma unroll
      for (int w = 0; w < W; ++w) z[w] = (q * W + w < n) ? (T)(-P.recv[q * W + w] / dn) : (T)0;   // R9
      reinterpret_cast<VT*>(s_b)[q] = vjoin<T>(z);
    }
  }
  __syncthreads();
  // row partials per warp in shared memory (no barrier per row); combined once after the sweep
  double* s_rp = reinterpret_cast<double*>(BS ? s_b + ld : s_col + ld);   // [rows of this CTA][warps]
  // odd passes walk the rows in reverse ("snake" order): a pass starts on the rows the previous one
  // wrote last, which are still in L2 when the row block is about the L2 size (K4 does the same)
  const bool rev = mode == 1 && (p & 1);
  // Work unit = (row, chunk of NB·kShThreads vectors); thread tid owns vectors tid + u·kShThreads of
  // a chunk and issues all NB loads before using any.  One CTA per SM: the warps run through the
  // units independently (no barrier per row), so one warp's loads overlap another's arithmetic.
  // (Double-buffering the next unit in registers measured slower: 396 vs 375 us per pass at C5.)
  constexpr int NB = 4096 / kShThreads;                          // vectors per thread per unit
  const long nch = (nvec + (long)NB * kShThreads - 1) / ((long)NB * kShThreads);
  const long nunits = (r1 - r0) * nch;
  auto unit_row = [&](long k) { const long ii = r0 + k / nch; return rev ? r0 + r1 - 1 - ii : ii; };
  auto load_unit = [&](long k, VT (&buf)[NB]) {
    const VT* row = reinterpret_cast<const VT*>(Y + unit_row(k) * ld);
    const long q0 = (k % nch) * NB * kShThreads + tid;
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      const long q = q0 + (long)u * kShThreads;
      if (q < nvec) buf[u] = __ldcg(row + q);
    }
  };
  VT cur[NB];
  double rs = 0.0;
  for (long k = 0; k < nunits; ++k) {
    load_unit(k, cur);
    const long i = unit_row(k), c = k % nch;
    VT* row = reinterpret_cast<VT*>(Y + i * ld);
    const T a = mode ? (T)(abase - P.rsum[i] / dn) : (T)0;      // R9: a_i in FP64, rounded
    const long q0 = c * NB * kShThreads + tid;
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      const long q = q0 + (long)u * kShThreads;
      if (q >= nvec) break;
      T e[W], cc[W], bb[W];
      vsplit<T>(cur[u], e);
      vsplit<T>(reinterpret_cast<VT*>(s_col)[q], cc);
      if (BS && mode) vsplit<T>(reinterpret_cast<VT*>(s_b)[q], bb);
      T rp = (T)0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const long j = q * W + w;
        T y;
        if (j >= n) y = (T)0;
        else if (mode) {                                         // P2(P1(Y)), R9 grouping
          const T bj = BS ? bb[w] : (T)(-P.recv[j] / dn);
          y = (e[w] + a) + bj;
          y = y > (T)0 ? y : (T)0;
        }
        else y = P.scale ? (T)(sc * (double)e[w]) : e[w];
        e[w] = y;
        cc[w] += y;
        rp += y;
      }
      __stcg(row + q, vjoin<T>(e));
      reinterpret_cast<VT*>(s_col)[q] = vjoin<T>(cc);
      rs += (double)rp;
    }
    if (c == nch - 1) {                                          // row complete: per-warp partial
      rs = warp_sum_d(rs);
      if (lane == 0) s_rp[(i - r0) * (kShThreads / 32) + warp] = rs;
      rs = 0.0;
    }
  }
  __syncthreads();
  for (long i = r0 + tid; i < r1; i += kShThreads) {             // fixed order over warps
    double r = 0.0;
#pragma unroll
    for (int w = 0; w < kShThreads / 32; ++w) r += s_rp[(i - r0) * (kShThreads / 32) + w];
    P.rsum[i] = r;
  }
  T* dst = reinterpret_cast<T*>(P.colpart) + (long)blockIdx.x * ld;
  for (long q = tid; q < nvec; q += kShThreads) reinterpret_cast<VT*>(dst)[q] = reinterpret_cast<VT*>(s_col)[q];
  if (mode && last) {
    __syncthreads();
    if (blockIdx.x == 0 && tid == 0) st->done_pending = 1;      // becomes `done` after this pass
  }
}

// c_j = Σ_CTA partials (FP64, CTA order), S_local = Σ_i r_i → send[0..n]; then thread 0 of CTA 0
// advances the pass index (mode 1) and promotes done_pending → done for the next pass kernel (the
// all-reduce of the final pass still runs, harmlessly).  Another CTA of this kernel may then see done
// and skip its columns: only after the last pass, whose sums nothing reads.
template <typename T>
__global__ void sh_reduce_kernel(ShardSdsnParams P, int nctas, int mode) {
  ShardSdsnState* st = P.state;
  if (st->done) return;
  const long n = P.n, ld = P.ld;
  const T* cp = reinterpret_cast<const T*>(P.colpart);
  for (long j = blockIdx.x * (long)blockDim.x + threadIdx.x; j < n; j += (long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int b = 0; b < nctas; ++b) acc += (double)cp[(long)b * ld + j];
    P.send[j] = acc;
  }
  if (blockIdx.x == 0) {
    __shared__ double s_w[32];
    double s = 0.0;
    for (long i = threadIdx.x; i < P.rows; i += blockDim.x) s += P.rsum[i];
    s = warp_sum_d(s);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_w[w];
      P.send[n] = t;
      if (st->done_pending) st->done = 1;
      if (mode == 1) st->pass += 1;
    }
  }
}

}  // namespace

int sdsn_sh_grid(long rows, int num_sms, bool f64) {
  (void)f64;
  long g = (long)num_sms;                                        // one CTA per SM (pipelined sweep)
  if (g > rows) g = rows;
  return (int)(g < 1 ? 1 : g);
}

// column partials + b (FP32 mode) + per-warp row partials of up to rows_max rows
size_t sdsn_sh_smem(long ld, bool f64, long rows_max) {
  return (size_t)ld * (f64 ? 8 : 8) + (size_t)rows_max * (kShThreads / 32) * 8;
}

cudaError_t launch_sdsn_sh_max(const ShardSdsnParams& p, bool f64, cudaStream_t st, int num_sms) {
  cudaError_t e = cudaMemsetAsync(p.send, 0, sizeof(double), st);
  if (e != cudaSuccess) return e;
  const int g = (int)(p.rows < 2L * num_sms ? p.rows : 2L * num_sms);
  if (f64) sh_max_kernel<double><<<g, 256, 0, st>>>((const double*)p.Y, p.rows, p.n, p.ld, p.send);
  else sh_max_kernel<float><<<g, 256, 0, st>>>((const float*)p.Y, p.rows, p.n, p.ld, p.send);
  return cudaGetLastError();
}

cudaError_t prepare_sdsn_sh(const ShardSdsnParams& p, bool f64, int num_sms) {
  const int g = sdsn_sh_grid(p.rows, num_sms, f64);
  const size_t sm = sdsn_sh_smem(p.ld, f64, (p.rows + g - 1) / g + 1);
  return f64 ? cudaFuncSetAttribute(sh_pass_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)
             : cudaFuncSetAttribute(sh_pass_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
}

cudaError_t launch_sdsn_sh_sweep(const ShardSdsnParams& p, bool f64, int mode, cudaStream_t st, int num_sms) {
  const int g = sdsn_sh_grid(p.rows, num_sms, f64);
  const size_t sm = sdsn_sh_smem(p.ld, f64, (p.rows + g - 1) / g + 1);
  if (f64) {
    sh_pass_kernel<double><<<g, kShThreads, sm, st>>>(p, mode);
    sh_reduce_kernel<double><<<(unsigned)((p.n + 255) / 256), 256, 0, st>>>(p, g, mode);
  } else {
    sh_pass_kernel<float><<<g, kShThreads, sm, st>>>(p, mode);
    sh_reduce_kernel<float><<<(unsigned)((p.n + 255) / 256), 256, 0, st>>>(p, g, mode);
  }
  return cudaGetLastError();
}

}  // namespace fram
