/*
 * fram.h — C ABI of libfram.so, a B200-native (sm_100a) implementation of the inner loop of
 * FRAM, "Frobenius-Regularized Assignment Matching" (arXiv 2508.00887).
 *
 * Citation keys: P:n = PAPER.md line n (Alg. 1 "FRAM" P:322-342, Alg. 2 "SDSN" P:344-361);
 * S:n = SPEC.md line n (conventions only); R<k> = a reading listed in DESIGN.md §3.
 *
 * Conventions (all entry points):
 *  - Matrices are n×n, row-major, contiguous (leading dimension n), caller-owned.  A pointer may
 *    be CUDA device memory or host memory (pinned or pageable); the library detects which with
 *    cudaPointerGetAttributes and, for host memory, stages through its own device workspace
 *    (the copies are enqueued on `stream`).  The library never frees caller memory and never
 *    retains a caller pointer after the call returns.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Every entry
 *    point enqueues its work on `stream` and returns after cudaStreamSynchronize(stream), so
 *    status, outputs and stats are final on return.  (fram_solve copies X_out on a handle-owned
 *    non-blocking stream while the LAP runs; that copy is joined into `stream` before return.)
 *  - A handle is created for one n and one device; it owns all workspace (allocated lazily on
 *    first use, sized for n).  A handle is not thread-safe; distinct handles are independent.
 *  - On any status other than FRAM_OK / FRAM_NOT_CONVERGED, outputs are left untouched and
 *    fram_last_error() returns a thread-local message.
 *  - There is no CPU fallback: every arithmetic step of the path runs in this library's CUDA
 *    kernels; without a usable sm_100 device every compute call returns FRAM_ERR_CUDA.
 */
#ifndef FRAM_H
#define FRAM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FRAM_ABI_VERSION 1

#if defined(__GNUC__)
#define FRAM_API __attribute__((visibility("default")))
#else
#define FRAM_API
#endif

typedef enum {
  FRAM_OK = 0,
  FRAM_ERR_USAGE = 1,        /* bad argument: null required pointer, n mismatch, bad enum, θ≤0,
                                α∉(0,1], γ_th≤0, n%W≠0                            */
  FRAM_ERR_DATA = 2,         /* non-finite or negative entry; c = max(A,Ã,K) = 0;
                                asymmetric A or Ã when FRAM_FLAG_CHECK_SYMMETRY is set (R28)  */
  FRAM_NOT_CONVERGED = 3,    /* max_outer reached: outputs ARE written (R16)          */
  FRAM_ERR_CUDA = 4,         /* CUDA runtime / launch failure, or no sm_100 device           */
  FRAM_ERR_NCCL = 5,         /* NCCL failure (sharded handles)                                */
  FRAM_ERR_OOM = 6           /* device workspace allocation failed                            */
} fram_status;

/* GEMM operand format of Alg.1 step 5.  Mixed modes: operands in this format, FP32
 * accumulation in TMEM (tcgen05), G and SDSN in FP32 (step 6), update/δ/LAP in FP64 (steps 7,
 * 8, 10).  FRAM_PREC_FP64: every step FP64 (the paper's "GPU-FP64" comparison). */
typedef enum {
  FRAM_PREC_FP64 = 0,
  FRAM_PREC_TF32 = 1,        /* the paper's choice for step 5                 */
  FRAM_PREC_BF16 = 2,
  FRAM_PREC_FP16 = 3
} fram_precision;

/* Storage type of the caller's A, B (Ã) and K buffers. */
typedef enum {
  FRAM_DT_F64 = 0,
  FRAM_DT_F32 = 1,
  FRAM_DT_BF16 = 2
} fram_dtype;

/* fram_schedule.flags */
#define FRAM_FLAG_TRACE           0x1  /* record per-outer-iteration passes/δ/γ into fram_stats arrays */
#define FRAM_FLAG_CHECK_SYMMETRY  0x2  /* validate A = Aᵀ and Ã = Ãᵀ (R28) → FRAM_ERR_DATA        */
#define FRAM_FLAG_NO_THETA_SCALE  0x4  /* DSPFP projection: skip Alg.2 step 1 (NEXT-1)  */
#define FRAM_FLAG_TIME_PHASES     0x8  /* CUDA-event timing of GEMM / SDSN / update / LAP phases       */

typedef struct {
  double  theta;        /* θ of Alg.2 step 1: 10 sparse / 2 dense                        */
  double  alpha;        /* step size α of Alg.1 step 7: 0.95                              */
  double  gamma_th;     /* SDSN threshold γ_th (Alg.2 line 2): 1e-3 (R3; paper gives no value)    */
  double  delta_th;     /* FRAM threshold δ_th (Alg.1 line 4): 1e-4 (R3)                          */
  int32_t max_outer;    /* cap on outer iterations: 100 (R3, R16)                                 */
  int32_t sdsn_max;     /* cap on SDSN passes per call: 1000 (R3)                                 */
  int32_t sdsn_fixed;   /* 0 = γ test; >0 = exactly this many passes per call (DSPFP / parity)    */
  int32_t flags;        /* FRAM_FLAG_*                                                            */
  const int32_t* replay_passes;  /* host, nullable: pass count for outer iteration t (0-based);
                                    when set, exactly replay_len outer iterations run;
                                    replay_len > max_outer → FRAM_ERR_USAGE                       */
  int32_t replay_len;
} fram_schedule;

/* Host memory, caller-owned; arrays nullable, each sized max_outer (filled when FLAG_TRACE). */
typedef struct {
  int32_t outer_iters;       /* outer iterations run (t at exit)                                 */
  int32_t converged;         /* 1 if δ ≤ δ_th was reached                                         */
  int32_t sdsn_capped_calls; /* SDSN calls that stopped on sdsn_max                               */
  int32_t sdsn_kernel;       /* SDSN kernel used: 1 streaming (K4), 2 on-chip resident (K4r),
                                3 row-sharded per-pass kernels + NCCL (K4s), 4 one thread-block
                                cluster with a DSMEM all-reduce (K4c, small n)                      */
  int64_t total_passes;      /* Σ_t passes_t                                                     */
  int32_t* passes_per_iter;  /* [max_outer] SDSN passes of outer iteration t                     */
  double*  delta_trace;      /* [max_outer] δ_t                                          */
  double*  gamma_last;       /* [max_outer] γ of the last pass's input                           */
  double ms_precond, ms_gemm, ms_sdsn, ms_update, ms_lap, ms_total;   /* FLAG_TIME_PHASES        */
  int64_t kernel_launches;   /* number of this library's kernels launched by the call            */
} fram_stats;

typedef struct fram_ctx* fram_handle;

/* Create a handle for problems of size n on CUDA device `device`.  λ ≥ 0 weights the unary term
 * (Alg.1 step 5).  `s` is copied (nullable ⇒ defaults θ=10, α=0.95, γ_th=1e-3, δ_th=1e-4,
 * max_outer=100, sdsn_max=1000).  No device memory is allocated until first use. */
FRAM_API fram_status fram_create(int64_t n, double lambda, const fram_schedule* s, int device,
                        fram_handle* out);

/* Replace the handle's schedule (copied). */
FRAM_API fram_status fram_set_schedule(fram_handle h, const fram_schedule* s);

/* One FRAM solve: Alg. 1 end to end.
 *  A, B : n×n edge-attribute matrices of G and G̃ (B = Ã), nonnegative, symmetric, `dt`.
 *  K    : n×n unary term K = F F̃ᵀ or NULL (⇒ 0).
 *  X0   : n×n FP64 initial N⁽⁰⁾ or NULL (⇒ 11ᵀ/n, R1).
 *  X_out: n×n FP64 final N (device or host), nullable.   perm_out: int32[n], perm[i] = column of
 *         Ã matched to row i (the LAP of step 10, R17), nullable.
 *  Returns FRAM_OK, FRAM_NOT_CONVERGED (outputs written), or an error (outputs untouched). */
FRAM_API fram_status fram_solve(fram_handle h, fram_dtype dt, const void* A, const void* B, const void* K,
                       const double* X0, fram_precision p, void* stream,
                       double* X_out, int32_t* perm_out, fram_stats* stats);

/* `batch` independent solves of size n (not in the paper).  n ≤ 64: one launch, one CTA
 * per instance with the whole state on chip (K8).  n > 64: 4 worker threads with their own streams
 * run the single-instance solve on the instances in turn (several instances on the GPU at once).
 * Inputs are batch×n×n contiguous; X0 nullable;
 * status_out: int32[batch] per-instance fram_status (device or host), nullable; the call
 * returns the worst per-instance status.  stats (nullable) aggregates outer_iters (max),
 * total_passes (sum) and converged (1 iff all converged). */
FRAM_API fram_status fram_solve_batched(fram_handle h, int64_t batch, fram_dtype dt, const void* A,
                               const void* B, const void* K, const double* X0,
                               fram_precision p, void* stream, double* X_out, int32_t* perm_out,
                               int32_t* status_out, fram_stats* stats);

/* Attributed graphs of possibly unequal size (reading R30).
 *  G has n1 nodes (A: n1×n1, features F: n1×d), G̃ has n2 nodes (B = Ã: n2×n2, F̃: n2×d), all
 *  row-major contiguous in dtype `dt`, n1, n2 ≤ the handle's n =: m.  Both graphs are padded to m nodes
 *  with isolated zero-attribute nodes ("n = ñ for simplicity"); the unary term
 *  K = F·F̃ᵀ (Eq.(1), gradient term λK P:82) is computed on the device in FP64 (DMMA GEMM; zero
 *  on padding; F, F̃ nullable together ⇒ K = 0) and must be ≥ 0; then Alg. 1 runs as in fram_solve.
 *  perm_out: int32[n1] — the node of G̃ matched to each node of G, or −1 when it is matched to a padding
 *  node (n1 > n2).  X_out (nullable): m×m FP64 final N of the padded problem.  Not available on
 *  sharded handles. */
FRAM_API fram_status fram_solve_attributed(fram_handle h, fram_dtype dt, int64_t n1, int64_t n2, int64_t d,
                                  const void* A, const void* B, const void* F, const void* Ft,
                                  fram_precision p, void* stream, double* X_out, int32_t* perm_out,
                                  fram_stats* stats);

FRAM_API void fram_destroy(fram_handle h);

/* Thread-local message for the last non-OK status on this thread ("" if none). */
FRAM_API const char* fram_last_error(void);

/* ---- sharded (row-partitioned) solves, SURVEY §3.3 / §8(e) -------------------------------
 * The library owns an ncclComm; Python broadcasts the 128-byte id through torch.distributed.
 * In a sharded handle fram_solve's A, K, X0, X_out are the local row block
 * [rank·n/W, (rank+1)·n/W) (n % W == 0, row-major n/W × n); B (Ã) is full on every rank;
 * perm_out is full on every rank.  NCCL is loaded at run time (dlopen of libnccl.so.2).
 * Per outer iteration (Alg.1 steps 5-8): U_rᵀ = (N_r·Ã')ᵀ locally, all-gather of the U_rᵀ blocks
 * (n²·esz bytes in total), G_r = A'_r·U + λK'_r, SDSN on the row block with one all-reduce of the
 * n column sums and the mass per pass (FP64, n+1 values), the local update, and an all-reduce of
 * (ΣΔ², ΣN²) for δ.  After the loop every rank all-gathers N and runs the same LAP (step 10).
 * Mixed modes need (n/W) % 64 == 0.  The symmetry check (FRAM_FLAG_CHECK_SYMMETRY) covers Ã only
 * (a row block of A cannot see its transpose).  fram_sdsn / fram_gradient / fram_lap /
 * fram_solve_batched return FRAM_ERR_USAGE on a sharded handle. */
FRAM_API fram_status fram_get_unique_id(uint8_t id[128]);
FRAM_API fram_status fram_create_sharded(int64_t n, double lambda, const fram_schedule* s,
                                const uint8_t id[128], int rank, int world, int device,
                                fram_handle* out);

/* Virtual-shard group (test harness for the W > 1 sharded path on ONE GPU; SURVEY §4 L-d): a handle
 * whose fram_solve runs `world` ranks of the row-sharded solve (exactly the code of a real sharded
 * handle: row-block GEMMs with the K-blocked operand, K4s SDSN, row-block update, LAP on the gathered
 * N), one host thread and CUDA stream per rank, with the NCCL collectives replaced by fixed-order
 * (rank 0..W−1) device sums and copies between the ranks' buffers.  fram_solve on this handle takes
 * the FULL n×n A, B, K, X0 and X_out (rank r works on rows [r·n/W, (r+1)·n/W)); perm_out and stats
 * come from rank 0.  world ∈ [1, 16], n % world == 0 (mixed precision: (n/world) % 64 == 0).
 * fram_sdsn / fram_gradient / fram_lap / batched / attributed calls are FRAM_ERR_USAGE on it. */
FRAM_API fram_status fram_create_sharded_virtual(int64_t n, double lambda, const fram_schedule* s, int world,
                                                int device, fram_handle* out);

/* Evaluation of a discrete matching (not on the solve's path): M[i, perm[i]] = 1 for the handle's n.
 *  out[0] = ½‖A − MÃMᵀ‖_F + ‖F − MF̃‖_F   — the paper's matching error (with F = NULL only
 *           the edge term, as P:380 prescribes for graphs without node attributes)
 *  out[1] = ½‖A − MÃMᵀ‖_F                 out[2] = ‖F − MF̃‖_F
 *  out[3] = Φ(M) = ½⟨MᵀAM, Ã⟩ + λ⟨MᵀF, F̃⟩  (Eq.(1), λ of the handle; K = F F̃ᵀ)
 *  A, B: n×n, F, Ft: n×d (NULL ⇒ no feature term), all of storage `dt`, device or host; perm: int32[n]
 *  (device or host); out: host double[4].  Sums in FP64 in a fixed order (deterministic).  A perm
 *  entry outside [0, n) → FRAM_ERR_DATA. */
FRAM_API fram_status fram_evaluate(fram_handle h, fram_dtype dt, const void* A, const void* B, const void* F,
                                   const void* Ft, int64_t d, const int32_t* perm, void* stream, double out[4]);

/* ---- test entry points (parity harness) ----------------------------------------------------
 * fram_sdsn: one SDSN call (Alg.2) on a nonnegative n×n X.  p = FRAM_PREC_FP64: X and
 *   D_out are FP64; any other p: FP32.  Uses the handle's θ, γ_th, sdsn_max, sdsn_fixed and the
 *   FRAM_FLAG_NO_THETA_SCALE flag.  passes: host int32 out.  gamma_hist: host
 *   double[max(sdsn_max, sdsn_fixed)] (nullable) receives γ_j of every pass input.  Negative X → FRAM_ERR_DATA. */
FRAM_API fram_status fram_sdsn(fram_handle h, fram_precision p, const void* X, void* D_out,
                      int32_t* passes, double* gamma_hist, void* stream);

/* fram_gradient: preconditioning (Alg.1 steps 2-3) then G = A'·N·Ã' + λK' (step 5) for the given
 *   FP64 N.  G_out is FP64 for p = FRAM_PREC_FP64, else FP32.  c_out (host, nullable) = c. */
FRAM_API fram_status fram_gradient(fram_handle h, fram_dtype dt, const void* A, const void* B,
                          const void* K, const double* N, fram_precision p, void* stream,
                          void* G_out, double* c_out);

/* fram_lap: perm = argmax_π Σ_i N[i,π(i)] (Eq.(2); Alg.1 step 10) by the deterministic
 *   Hungarian of R17, bit-exact with the oracle's LAP given the same N (FP64).  N: host or device,
 *   n×n contiguous row-major (copied into the handle's workspace); perm_out: host or device
 *   int32[n]; returns after `stream` synchronizes.  One CTA for n ≤ 2048, a thread-block cluster
 *   above (4 CTAs to 8192, 8 CTAs to 16384), one CTA again up to 65536; a larger n fails to launch
 *   (FRAM_ERR_CUDA). */
FRAM_API fram_status fram_lap(fram_handle h, const double* N, int32_t* perm_out, void* stream);

/* Library/ABI version and the compile target ("sm_100a"). */
FRAM_API int         fram_abi_version(void);
FRAM_API const char* fram_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* FRAM_H */
