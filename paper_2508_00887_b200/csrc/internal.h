// internal.h — host-side launchers shared between the libfram translation units (not ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fram {

// ---- K4: SDSN (Alg. 2), persistent cooperative kernel, one launch per SDSN call ----
struct SdsnParams {
  void* Y;             // n×ld, T = float (mixed) or double (FP64); in: X (G), out: D, in place
  long n, ld;
  double theta, gamma_th;
  int sdsn_max, sdsn_fixed, scale;   // scale = 0 ⇒ skip Alg.2 step 1 (DSPFP)
  void* colpart;       // [grid][ld] T   per-CTA column partials
  double* Spart;       // [grid]         per-CTA Σ of its row sums
  double* Mpart;       // [grid]         per-CTA max
  double* cvec;        // [ld]           column sums c (FP64)
  unsigned* bar;       // [2]            grid barrier (zeroed before launch)
  int* passes_out;     // [1]
  double* gamma_hist;  // [sdsn_max] nullable: γ_j of every pass input
  double* sdsn_out;    // [4]: [0] γ of the last pass input, [1] max X, [2] S of last input
};
// f64: T=double; else T=float.  Returns the grid used via *grid_out.
cudaError_t launch_sdsn(const SdsnParams& p, bool f64, cudaStream_t st, int num_sms, int* grid_out);
// K4c: small n on one thread-block cluster (≤ 16 CTAs), iterate in shared memory, DSMEM all-reduce;
// uses Y, n, ld, theta, gamma_th, sdsn_max, sdsn_fixed, scale, passes_out, gamma_hist, sdsn_out only
bool sdsn_cluster_supported(long n, bool f64);
cudaError_t launch_sdsn_cluster(const SdsnParams& p, bool f64, cudaStream_t st);
int sdsn_grid_for(long n, int num_sms);
bool sdsn_supported(long n, bool f64);

// ---- K4r: SDSN with the iterate resident on chip (TMEM + shared memory), FP32, n ≤ ~4.2k ----
struct ResParams {
  float* Y;            // n×ld FP32: in X (G), out D (written back after the last pass)
  long n, ld;
  double theta, gamma_th;
  int sdsn_max, sdsn_fixed, scale;
  uint64_t* xchg;      // tagged exchange words (zeroed by the launcher), see sdsn_res_xchg_words
  unsigned* colpart;   // [grid][slots]   per-CTA column partials (slot layout), parity bit | fp32
  unsigned* bvec;      // [slots]         |b_j| = c_j/n (∞ on padding), parity bit | fp32
  uint64_t* Spart;     // [2][grid]       per-CTA Σ row sums (FP64, tag in the sign bit), by epoch parity
  uint64_t* Mpart;     // [grid]          per-CTA max (FP64, tag in the sign bit)
  int* passes_out;
  double* gamma_hist;  // nullable
  double* sdsn_out;    // [4] as SdsnParams
  int rs;              // rows per CTA held in shared memory (set by the launcher)
  int rmax;            // rows per CTA upper bound (set by the launcher)
  long long* dbg;      // dev-only (-DFRAM_DEV_RES_TIMING=1 builds): per-CTA phase times [grid][8]; null in the product
};
int sdsn_res_grid(long n, int num_sms);       // 0 ⇒ n not supported on chip
long sdsn_res_slots(long n);
size_t sdsn_res_xchg_words(long n, int num_sms);   // size of ResParams::xchg
cudaError_t launch_sdsn_resident(const ResParams& p, cudaStream_t st, int num_sms);

// ---- K4s: SDSN on a row block for the sharded solve (per-pass kernels + host NCCL all-reduce) ----
struct ShardSdsnState {
  int done, done_pending, passes, pass;   // `pass`: index of the next SDSN pass (advanced on the device,
                                          // so every pass is the same launch sequence: CUDA-graph friendly)
  double gamma_last, maxx, S_last;
};
struct ShardSdsnParams {
  void* Y;             // rows×ld, T (float mixed, double FP64), in place
  long rows, n, ld;
  double theta, gamma_th;
  int sdsn_max, sdsn_fixed, scale;
  void* colpart;       // [grid][ld] T
  double* rsum;        // [rows] local row sums of the current iterate (FP64)
  double* send;        // [n+1] local column sums, local mass (and [0] = local max in the max phase)
  double* recv;        // [n+1] all-reduced (sum; max in the max phase)
  double* gamma_hist;  // nullable, [sdsn_max]
  ShardSdsnState* state;
};
int sdsn_sh_grid(long rows, int num_sms, bool f64);
size_t sdsn_sh_smem(long ld, bool f64, long rows_max);
cudaError_t launch_sdsn_sh_max(const ShardSdsnParams& p, bool f64, cudaStream_t st, int num_sms);
// mode 0: scale sweep (after the max all-reduce), mode 1: the next pass (index state->pass, advanced
// on the device); both end with the local column/mass reduction into p.send (the caller all-reduces
// send → recv).  prepare_sdsn_sh sets the kernels' shared-memory limits (call before graph capture).
cudaError_t prepare_sdsn_sh(const ShardSdsnParams& p, bool f64, int num_sms);
cudaError_t launch_sdsn_sh_sweep(const ShardSdsnParams& p, bool f64, int mode, cudaStream_t st, int num_sms);

// ---- K1: preconditioning (Alg.1 steps 2-3) ------------------------------------
// in_dt: 0 f64, 1 f32, 2 bf16.  op: 0 f64, 1 tf32 (stored f32), 2 bf16, 3 fp16.
struct PrecondScan {        // device-side result of the validation / max scan
  double maxv[3];           // max A, max B, max K
  unsigned long long bad_nonfinite, bad_negative, bad_asym;
};
cudaError_t launch_precond_scan(const void* A, const void* B, const void* K, int in_dt, long n,
                                bool check_sym, PrecondScan* out_dev, double* blockbuf,
                                unsigned* counter, cudaStream_t st);
// accumulate max / non-finite / negative counts of the rows × n blocks A and K into *out_dev
// (no memset; no symmetry test — a row block cannot see its transpose)
cudaError_t launch_precond_scan_rows(const void* A, const void* K, int in_dt, long rows, long n,
                                     PrecondScan* out_dev, cudaStream_t st);
// A' = A/√c → op (row-major, ld), Bt' = (Ã/√c)ᵀ → op (row-major, ld), K' = K/c → kdst (f32 or f64);
// A and K have rows_a rows (n, or n/W for a shard), Ã is n × n
cudaError_t launch_precond_apply(const void* A, const void* B, const void* K, int in_dt, long n,
                                 long ld, const double* c_dev, int op, void* Aq, void* BqT,
                                 void* Kq, bool k_f64, cudaStream_t st, long rows_a = -1);

// ---- K2/K3: gradient GEMMs ------------------------------------------------------------------
// D[M×N] = Aop[M×K] · Bop[N×K]ᵀ (both row-major, K contiguous, leading dim ld).
// epi 0: OutT[j*ldo + i] = round_op(D[i][j])  (transposed store in the operand format)
// epi 1: G[i*ldo + j] = D[i][j] + lam*Kq[i*ldo + j]  (FP32 G; Kq nullable)
// kchunk > 0: Bop is K-blocked — K/kchunk chunks of (N × kchunk) row-major matrices, element (j, k)
// at Bop[(k / kchunk)·N·kchunk + j·kchunk + k % kchunk] (the all-gathered Uᵀ blocks of a sharded
// solve); kchunk must divide K and be a multiple of 64.
struct GemmArgs {
  const void* Aop; const void* Bop; long M, N, K, ld;
  int epi; void* out; long ldo; const void* Kq; double lam;
  long kchunk = 0;
};
cudaError_t launch_gemm_tc(const GemmArgs& g, int op, cudaStream_t st);     // tcgen05 (op 1,2,3)
cudaError_t launch_gemm_f64(const GemmArgs& g, cudaStream_t st);            // DMMA FP64

// ---- K5/K6: update N ← (1−α)N + αD, N_q, δ (Alg.1 steps 7-8) --------------------------------
// rows × n blocks (rows = n for a full solve; n/W for a shard)
cudaError_t launch_update(double* N, const void* D, bool d_f64, void* Nq, int op, long rows, long n, long ld,
                          double alpha, double* partials, unsigned* counter, double* out3,
                          cudaStream_t st, int num_sms);
cudaError_t launch_init_n(double* N, void* Nq, int op, const double* X0, long rows, long n, long ld,
                          cudaStream_t st);

// ---- K7: LAP (Alg.1 step 10, R17) --------------------------------------------------------------
cudaError_t launch_lap(const double* N, long n, long ld, int32_t* perm, void* work,
                       cudaStream_t st);
// ---- K9: evaluation of a matching (Eq.1, matching error P:379); part: [n][4] FP64 workspace,
// out (device): [Σ(A−MÃMᵀ)², Σ‖F−MF̃‖², Σ A∘MÃMᵀ, Σ⟨F, MF̃⟩]; *bad = 1 if perm is not in [0, n)
cudaError_t launch_evaluate(const void* A, const void* B, const void* F, const void* Ft, int dt, long n, long d,
                            const int32_t* perm, double* part, double* out, int* bad, cudaStream_t st);
size_t lap_work_bytes(long n);
size_t lap_err_offset(long n);     // byte offset of the LAP kernels' error word in the workspace (int, 0 = ok)

// ---- misc ---------------------------------------------------------------------------------------
cudaError_t launch_pad_convert(double* dst, long ldd, long drows, long dcols, const void* src, int dt, long lds,
                               long rows, long cols, cudaStream_t st);
cudaError_t launch_copy2d_f64(double* dst, long ldd, const double* src, long lds, long rows,
                              long cols, cudaStream_t st);
cudaError_t launch_scan_finite(const double* X, long count, unsigned long long* bad, cudaStream_t st);
cudaError_t launch_scan_nonneg(const void* X, bool f64, long n, unsigned long long* bad,
                               cudaStream_t st);

}  // namespace fram
