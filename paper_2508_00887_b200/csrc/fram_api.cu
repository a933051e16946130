// fram_api.cu — the C ABI of libfram.so (include/fram.h) and the host orchestrator of Alg. 1
// (PAPER.md P:322-342).  Host code only validates, stages, allocates and sequences kernels; every
// arithmetic step runs in the CUDA kernels of this library.  One host sync per outer iteration
// (to read δ and the SDSN pass count); the SDSN pass loop itself is device-resident.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/fram.h"
#include "internal.h"
#include "batched.h"
#include "sharded.h"

namespace {

thread_local std::string g_err;

fram_status fail(fram_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t b) {
    if (b <= bytes && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, b);
    if (e != cudaSuccess) { p = nullptr; return e; }
    bytes = b;
    // zero-filled before any caller stream (possibly non-blocking) can touch it: some kernels rely on
    // the zero (the update kernel's arrival counter, ld padding columns of the operand buffers)
    e = cudaMemset(p, 0, b);
    if (e != cudaSuccess) return e;
    return cudaDeviceSynchronize();
  }
  void release() { if (p) cudaFree(p); p = nullptr; bytes = 0; }
  template <typename T> T* as() const { return reinterpret_cast<T*>(p); }
};

size_t op_size(int op) { return op == 0 ? 8 : (op == 1 ? 4 : 2); }
size_t dt_size(int dt) { return dt == 0 ? 8 : (dt == 1 ? 4 : 2); }

}  // namespace

// NVTX ranges (header-only NVTX v3: no library, ~ns per range when no tool is attached) around a solve
// and its phases, for ncu --nvtx / nsys timelines.  Host-side: they mark when the work is enqueued.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct fram_ctx {
  int64_t n = 0;
  double lambda = 1.0;
  fram_schedule sched{};
  std::vector<int32_t> replay;
  int device = 0;
  int num_sms = 148;
  bool dev_checked = false;
  long ld = 0;
  // workspace
  DevBuf Aq, BqT, Kq, N, Nq, UT, Y, colpart, Spart, Mpart, cvec, bar, scal, ghist, upd, lapw, permd;
  DevBuf rcolpart, rbvec, rflags, rdbg;
  bool no_cluster = false;   // K4c could not be launched here once: use K4/K4r from then on
  DevBuf shUT, shUblk, shRsum, shSend, shRecv, shState, shNfull, shColpart, shScan;   // sharded solve
  DevBuf atA, atB, atK, atF, atFt, atPerm;                                           // attributed solve   // on-chip-resident SDSN (K4r)
  DevBuf stA, stB, stK, stX0, stX;
  DevBuf evPart, evOut, evPerm;                                                        // evaluation (K9)
  DevBuf scan;
  double* hscal = nullptr;          // pinned readback
  cudaEvent_t ev[8] = {};
  cudaStream_t side = nullptr;                 // X_out copy-out, concurrent with the LAP
  cudaEvent_t sev[2] = {};
  cudaEvent_t gev[3] = {};                     // queued-gradient timing pair (odd iterations), scalar readback
  int64_t launches = 0;
  // batched workspace
  fram::BatchedWs bws;
  // sharded
  fram::ShardCtx* shard = nullptr;
  // virtual-shard group (fram_create_sharded_virtual): W rank sub-handles on this GPU, one host thread
  // and stream each; this handle only dispatches
  std::vector<fram_ctx*> vsub;
  std::vector<cudaStream_t> vstreams;
  fram::VGroup* vgroup = nullptr;
  // sharded SDSN: a chunk of passes (pass kernel, reduce, all-reduce) captured once as a CUDA
  // graph and relaunched (NCCL communicators only; see sharded_solve)
  cudaGraphExec_t sh_graph = nullptr;
  cudaStream_t sh_cap_stream = nullptr;
  bool sh_graph_off = false;
  // batched solves with n > 64: worker sub-handles, one host thread and stream each
  std::vector<fram_ctx*> bsub;
  std::vector<cudaStream_t> bstreams;        // capture failed once here: plain launches from then on
  unsigned char sh_graph_key[sizeof(fram::ShardSdsnParams) + 8] = {};
};

namespace {

constexpr int kScalDoubles = 32;     // scal layout: [0..3] sdsn_out, [4..6] upd out3, [8] passes (int)

fram_status cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();
  if (e == cudaErrorMemoryAllocation) return fail(FRAM_ERR_OOM, std::string(what) + ": out of device memory");
  return fail(FRAM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(expr, what)                                 \
  do {                                                 \
    cudaError_t _e = (expr);                           \
    if (_e != cudaSuccess) return cuda_fail(_e, what); \
  } while (0)

fram_status check_schedule(const fram_schedule& s) {
  if (!(s.theta > 0) || !std::isfinite(s.theta)) return fail(FRAM_ERR_USAGE, "theta must be > 0");
  if (!(s.alpha > 0 && s.alpha <= 1)) return fail(FRAM_ERR_USAGE, "alpha must be in (0,1]");
  if (!(s.gamma_th > 0)) return fail(FRAM_ERR_USAGE, "gamma_th must be > 0");
  if (!(s.delta_th >= 0)) return fail(FRAM_ERR_USAGE, "delta_th must be >= 0");
  if (s.max_outer < 1 || s.sdsn_max < 1 || s.sdsn_fixed < 0) return fail(FRAM_ERR_USAGE, "bad caps");
  if (s.replay_len < 0 || (s.replay_len > 0 && !s.replay_passes)) return fail(FRAM_ERR_USAGE, "bad replay");
  if (s.replay_len > s.max_outer)
    return fail(FRAM_ERR_USAGE, "replay_len must be <= max_outer (the stats trace arrays hold max_outer entries)");
  for (int i = 0; i < s.replay_len; ++i)
    if (s.replay_passes[i] < 1) return fail(FRAM_ERR_USAGE, "replay pass counts must be >= 1");
  return FRAM_OK;
}

fram_schedule default_schedule() {
  fram_schedule s{};
  s.theta = 10.0;
  s.alpha = 0.95;
  s.gamma_th = 1e-3;
  s.delta_th = 1e-4;
  s.max_outer = 100;
  s.sdsn_max = 1000;
  s.sdsn_fixed = 0;
  s.flags = FRAM_FLAG_CHECK_SYMMETRY;
  return s;
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Returns a device pointer holding `bytes` of the caller's data (the pointer itself if on device).
fram_status stage_in(fram_ctx* h, DevBuf& buf, const void* src, size_t bytes, cudaStream_t st, const void** out) {
  if (!src) { *out = nullptr; return FRAM_OK; }
  if (is_device_ptr(src)) { *out = src; return FRAM_OK; }
  CK(buf.ensure(bytes), "staging alloc");
  CK(cudaMemcpyAsync(buf.p, src, bytes, cudaMemcpyHostToDevice, st), "H2D copy");
  (void)h;
  *out = buf.p;
  return FRAM_OK;
}

long ld_for(int64_t n) { return (long)((n + 15) / 16 * 16); }

int sdsn_cap(const fram_ctx* h) {
  int cap = std::max(h->sched.sdsn_max, h->sched.sdsn_fixed);
  for (int32_t r : h->replay) cap = std::max(cap, r);
  return cap + 1;
}

// Allocate the solve workspace for operand format `op`.
fram_status ensure_ws(fram_ctx* h, int op, bool withK) {
  const long n = h->n, ld = h->ld;
  const size_t nn = (size_t)n * ld;
  const bool f64 = (op == 0);
  const int G = fram::sdsn_grid_for(n, h->num_sms);
  CK(h->Aq.ensure(nn * op_size(op)), "alloc A'");
  CK(h->BqT.ensure(nn * op_size(op)), "alloc B'");
  if (withK) CK(h->Kq.ensure(nn * (f64 ? 8 : 4)), "alloc K'");
  CK(h->N.ensure(nn * 8), "alloc N");
  if (!f64) CK(h->Nq.ensure(nn * op_size(op)), "alloc Nq");
  CK(h->UT.ensure(nn * op_size(op)), "alloc U");
  CK(h->Y.ensure(nn * (f64 ? 8 : 4)), "alloc G/Y");
  CK(h->colpart.ensure((size_t)G * ld * (f64 ? 8 : 4)), "alloc colpart");
  CK(h->Spart.ensure(2 * (size_t)std::max(G, h->num_sms) * 8), "alloc Spart");   // [2][G] tagged (K4)
  CK(h->Mpart.ensure((size_t)std::max(G, h->num_sms) * 8), "alloc Mpart");
  if (!f64 && fram::sdsn_res_grid(n, h->num_sms) > 0) {
    CK(h->rcolpart.ensure(fram::sdsn_res_xchg_words(n, h->num_sms) * 8), "alloc resident exchange");
  }
  CK(h->cvec.ensure((size_t)ld * 8), "alloc cvec");
  CK(h->bar.ensure(64), "alloc bar");
  CK(h->scal.ensure(kScalDoubles * 8), "alloc scal");
  CK(h->ghist.ensure((size_t)sdsn_cap(h) * 8), "alloc ghist");
  CK(h->upd.ensure((size_t)(h->num_sms * 4 * 2 + 16) * 8), "alloc upd");
  CK(h->lapw.ensure(fram::lap_work_bytes(n)), "alloc lap");
  CK(h->permd.ensure((size_t)n * 4), "alloc perm");
  CK(h->scan.ensure(sizeof(fram::PrecondScan)), "alloc scan");
  if (!h->hscal) CK(cudaMallocHost((void**)&h->hscal, kScalDoubles * 8), "alloc pinned");
  for (auto& e : h->ev)
    if (!e) CK(cudaEventCreate(&e), "event create");
  if (!h->side) CK(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking), "side stream");
  for (auto& e : h->sev)
    if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
  if (!h->gev[0]) CK(cudaEventCreate(&h->gev[0]), "event create");
  if (!h->gev[1]) CK(cudaEventCreate(&h->gev[1]), "event create");
  if (!h->gev[2]) CK(cudaEventCreateWithFlags(&h->gev[2], cudaEventDisableTiming), "event create");
  return FRAM_OK;
}

fram_status set_device(fram_ctx* h) {
  if (h->dev_checked) {                      // properties are queried once per handle (the query costs ms)
    CK(cudaSetDevice(h->device), "cudaSetDevice");
    return FRAM_OK;
  }
  int cnt = 0;
  cudaError_t e = cudaGetDeviceCount(&cnt);
  if (e != cudaSuccess || cnt == 0) return cuda_fail(e == cudaSuccess ? cudaErrorNoDevice : e, "no CUDA device");
  CK(cudaSetDevice(h->device), "cudaSetDevice");
  int major = 0, sms = 0;
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, h->device), "device attribute");
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device), "device attribute");
  if (major != 10) return fail(FRAM_ERR_CUDA, "libfram is built for sm_100a (B200); device is sm_" +
                                                  std::to_string(major) + "x");
  h->num_sms = sms;
  h->dev_checked = true;
  return FRAM_OK;
}

// Preconditioning (K1): scan → host check → apply.  Returns c in *c_out.
fram_status precondition(fram_ctx* h, int dt, const void* A, const void* B, const void* K, int op, cudaStream_t st,
                         double* c_out) {
  const long n = h->n;
  fram::PrecondScan* sc = h->scan.as<fram::PrecondScan>();
  const bool sym = (h->sched.flags & FRAM_FLAG_CHECK_SYMMETRY) != 0;
  CK(fram::launch_precond_scan(A, B, K, dt, n, sym, sc, nullptr, nullptr, st), "precond scan");
  h->launches++;
  fram::PrecondScan hs;
  CK(cudaMemcpyAsync(&hs, sc, sizeof(hs), cudaMemcpyDeviceToHost, st), "scan readback");
  CK(cudaStreamSynchronize(st), "scan sync");
  if (hs.bad_nonfinite) return fail(FRAM_ERR_DATA, "non-finite entries in A, B or K");
  if (hs.bad_negative) return fail(FRAM_ERR_DATA, "negative entries in A, B or K (P:55)");
  if (hs.bad_asym) return fail(FRAM_ERR_DATA, "A or B is not symmetric (P:55, R28)");
  const double c = std::max(std::max(hs.maxv[0], hs.maxv[1]), hs.maxv[2]);
  if (!(c > 0)) return fail(FRAM_ERR_DATA, "c = max(A, B, K) = 0 (S:344)");
  if (c_out) *c_out = c;
  CK(fram::launch_precond_apply(A, B, K, dt, n, h->ld, sc->maxv, op, h->Aq.p, h->BqT.p, K ? h->Kq.p : nullptr,
                                op == 0, st),
     "precond apply");
  h->launches++;
  return FRAM_OK;
}

fram_status gradient(fram_ctx* h, int op, bool haveK, cudaStream_t st) {
  const long n = h->n, ld = h->ld;
  fram::GemmArgs g1{op == 0 ? h->N.p : h->Nq.p, h->BqT.p, n, n, n, ld, 0, h->UT.p, ld, nullptr, 0.0};
  fram::GemmArgs g2{h->Aq.p, h->UT.p, n, n, n, ld, 1, h->Y.p, ld, haveK ? h->Kq.p : nullptr, h->lambda};
  if (op == 0) {
    CK(fram::launch_gemm_f64(g1, st), "gemm1 f64");
    CK(fram::launch_gemm_f64(g2, st), "gemm2 f64");
  } else {
    CK(fram::launch_gemm_tc(g1, op, st), "gemm1 tcgen05");
    CK(fram::launch_gemm_tc(g2, op, st), "gemm2 tcgen05");
  }
  h->launches += 2;
  return FRAM_OK;
}

// SDSN kernel choice: 4 = K4c (one cluster; FP64 n ≤ ~600, FP32 n ≤ 160), 2 = K4r (FP32 on chip,
// n ≤ 4096), 1 = K4 (streaming).  Dev comparisons of the kernels build a variant library with
// -DFRAM_DEV_FORCE_STREAM=1 or -DFRAM_DEV_NOCLUSTER=1 (tools/build_variant.sh); the product has no
// run-time knobs.
#ifndef FRAM_DEV_FORCE_STREAM
#define FRAM_DEV_FORCE_STREAM 0
#endif
#ifndef FRAM_DEV_NOCLUSTER
#define FRAM_DEV_NOCLUSTER 0
#endif
#ifndef FRAM_DEV_RES_TIMING
#define FRAM_DEV_RES_TIMING 0
#endif
int sdsn_kind(const fram_ctx* h, bool f64) {
  if (FRAM_DEV_FORCE_STREAM) return 1;
  // K4c where it measured fastest (tools/sdsn_small_timing.py): FP64 up to its size limit (vs K4),
  // FP32 only for n ≤ 160 (with the mbarrier hand-off K4c and K4r tie at n = 256, K4r is faster above)
  if (!FRAM_DEV_NOCLUSTER && !h->no_cluster && fram::sdsn_cluster_supported(h->n, f64) && (f64 || h->n <= 160))
    return 4;
  if (!f64 && fram::sdsn_res_grid(h->n, h->num_sms) > 0) return 2;
  return 1;
}
bool use_resident(const fram_ctx* h, bool f64) { return sdsn_kind(h, f64) == 2; }

fram_status run_sdsn(fram_ctx* h, bool f64, int fixed, cudaStream_t st) {
  double* scal = h->scal.as<double>();
  if (sdsn_kind(h, f64) == 4) {
    fram::SdsnParams p{};
    p.Y = h->Y.p;
    p.n = h->n;
    p.ld = h->ld;
    p.theta = h->sched.theta;
    p.gamma_th = h->sched.gamma_th;
    p.sdsn_max = h->sched.sdsn_max;
    p.sdsn_fixed = fixed;
    p.scale = (h->sched.flags & FRAM_FLAG_NO_THETA_SCALE) ? 0 : 1;
    p.passes_out = reinterpret_cast<int*>(scal + 8);
    p.gamma_hist = h->ghist.as<double>();
    p.sdsn_out = scal;
    const cudaError_t ce = fram::launch_sdsn_cluster(p, f64, st);
    if (ce == cudaSuccess) {
      h->launches += 1;
      return FRAM_OK;
    }
    // a 16-CTA cluster may not be schedulable (e.g. on a partitioned GPU): clear the launch error and
    // take the kernel the size would use without K4c
    if (ce != cudaErrorInvalidClusterSize && ce != cudaErrorLaunchOutOfResources && ce != cudaErrorInvalidValue &&
        ce != cudaErrorNotSupported)
      CK(ce, "sdsn (cluster) launch");
    cudaGetLastError();
    h->no_cluster = true;
  }
  if (use_resident(h, f64)) {
    fram::ResParams r{};
    r.Y = h->Y.as<float>();
    r.n = h->n;
    r.ld = h->ld;
    r.theta = h->sched.theta;
    r.gamma_th = h->sched.gamma_th;
    r.sdsn_max = h->sched.sdsn_max;
    r.sdsn_fixed = fixed;
    r.scale = (h->sched.flags & FRAM_FLAG_NO_THETA_SCALE) ? 0 : 1;
    r.xchg = h->rcolpart.as<uint64_t>();
    r.passes_out = reinterpret_cast<int*>(scal + 8);
    r.gamma_hist = h->ghist.as<double>();
    r.sdsn_out = scal;
#if FRAM_DEV_RES_TIMING   // dev builds only (tools/build_variant.sh ... -DFRAM_DEV_RES_TIMING=1)
    {
      CK(h->rdbg.ensure((size_t)h->num_sms * 24 * 8), "alloc dbg");
      r.dbg = h->rdbg.as<long long>();
      CK(cudaMemsetAsync(r.dbg, 0, (size_t)h->num_sms * 24 * 8, st), "dbg memset");
    }
#endif
    CK(fram::launch_sdsn_resident(r, st, h->num_sms), "sdsn (on-chip) launch");
#if FRAM_DEV_RES_TIMING
    {
      std::vector<long long> d((size_t)h->num_sms * 24);
      CK(cudaMemcpyAsync(d.data(), r.dbg, d.size() * 8, cudaMemcpyDeviceToHost, st), "dbg");
      CK(cudaStreamSynchronize(st), "dbg sync");
      const int G = fram::sdsn_res_grid(h->n, h->num_sms);
      double mx[6] = {0};
      for (int bb = 0; bb < G; ++bb)
        for (int k = 0; k < 6; ++k) mx[k] = std::max(mx[k], (double)d[bb * 16 + k]);
      const double np = std::max(1.0, (double)(d[5] & 0xffff));
      fprintf(stderr, "[res timing] CTA0 load phase %.1f us, kernel start→loop end %.1f us\n", (d[5] >> 16) / 1e3, d[3] / 1e3);
      fprintf(stderr, "[res timing n=%ld G=%d passes=%.0f] ns/pass (CTA0): bload %.0f sweep %.0f [rows g0 %.0f g1 %.0f; spart %.0f stores %.0f srows %.0f sync %.0f] slice %.0f | max over CTAs: %.0f %.0f\n",
              (long)h->n, G, np, d[0] / np, d[1] / np, d[9] / np, d[10] / np, d[2] / np, d[4] / np, d[6] / np, d[7] / np,
              d[8] / np, mx[0] / np, mx[1] / np);
      {   // timeline of pass 500: per stamp, min / median / max over CTAs relative to the earliest pass start
        const long long* tl = d.data() + (size_t)G * 16;
        long long base = tl[0];
        for (int bb = 0; bb < G; ++bb) base = std::min(base, tl[bb * 8]);
        const char* names[6] = {"pass start", "b ready (g0)", "after sync", "sweep+epilogue end", "slice polls done", "slice end"};
        for (int k = 0; k < 6 && base > 0; ++k) {
          std::vector<long long> v;
          for (int bb = 0; bb < G; ++bb) v.push_back(tl[bb * 8 + k] - base);
          std::sort(v.begin(), v.end());
          fprintf(stderr, "[res timeline p500] %-20s min %6lld med %6lld max %6lld ns\n", names[k], v.front(), v[v.size() / 2], v.back());
        }
      }
      fprintf(stderr, "[res timing] rows cycles/pass g0 %.0f g1 %.0f -> SM clock %.0f / %.0f MHz\n", d[11] / np, d[12] / np,
              1e3 * d[11] / std::max(1.0, (double)d[9]), 1e3 * d[12] / std::max(1.0, (double)d[10]));
    }
#endif
    h->launches += 2;   // flag memset + kernel
    return FRAM_OK;
  }
  fram::SdsnParams p{};
  p.Y = h->Y.p;
  p.n = h->n;
  p.ld = h->ld;
  p.theta = h->sched.theta;
  p.gamma_th = h->sched.gamma_th;
  p.sdsn_max = h->sched.sdsn_max;
  p.sdsn_fixed = fixed;
  p.scale = (h->sched.flags & FRAM_FLAG_NO_THETA_SCALE) ? 0 : 1;
  p.colpart = h->colpart.p;
  p.Spart = h->Spart.as<double>();
  p.Mpart = h->Mpart.as<double>();
  p.cvec = h->cvec.as<double>();
  p.bar = h->bar.as<unsigned>();
  p.passes_out = reinterpret_cast<int*>(scal + 8);
  p.gamma_hist = h->ghist.as<double>();
  p.sdsn_out = scal;
  CK(fram::launch_sdsn(p, f64, st, h->num_sms, nullptr), "sdsn launch");
  h->launches += 2;   // barrier memset + kernel
  return FRAM_OK;
}

int prec_to_op(fram_precision p) { return (int)p; }   // 0 f64, 1 tf32, 2 bf16, 3 fp16

fram_status common_checks(fram_ctx* h, int dt, fram_precision p) {
  if (!h) return fail(FRAM_ERR_USAGE, "null handle");
  if (dt < 0 || dt > 2) return fail(FRAM_ERR_USAGE, "bad dtype");
  if ((int)p < 0 || (int)p > 3) return fail(FRAM_ERR_USAGE, "bad precision");
  return set_device(h);
}

// ---- row-sharded solve (config C5) ---------------------------------------------
// Rank r owns rows I_r = [r·m, (r+1)·m), m = n/W, of A, K, N and G; Ã is replicated.  Per outer
// iteration: GEMM1 U_rᵀ = (N_q,r·Ã')ᵀ (local) → all-gather of the U_rᵀ blocks → GEMM2
// G_r = A'_r·U + λK'_r (K-blocked operand) → SDSN on the row block (per-pass kernels, all-reduce of
// [column sums, mass]) → local update → all-reduce of (ΣΔ², ΣN²) → δ.  Finally N is all-gathered
// and every rank runs the same deterministic LAP (identical perm everywhere).
fram_status sharded_solve(fram_ctx* h, int dt, const void* A, const void* B, const void* K, const double* X0,
                          int op, cudaStream_t st, double* X_out, int32_t* perm_out, fram_stats* stats) {
  NvtxRange range_("sharded_solve");
  fram::ShardCtx* sh = h->shard;
  const int W = fram::shard_world(sh);
  const long n = h->n, m = n / W, ld = h->ld;
  const bool f64 = (op == 0);
  const size_t es = op_size(op), ts = f64 ? 8 : 4;
  std::string err;
  auto nck = [&](fram_status s) -> fram_status { if (s != FRAM_OK) g_err = err; return s; };
  if (!f64 && (m % 64 != 0)) return fail(FRAM_ERR_USAGE, "sharded mixed-precision solve needs (n/W) % 64 == 0");
  h->launches = 0;
  const bool timing = (h->sched.flags & FRAM_FLAG_TIME_PHASES) != 0;
  // workspace (local rows m, full Ã)
  CK(h->Aq.ensure((size_t)m * ld * es), "alloc A'");
  CK(h->BqT.ensure((size_t)n * ld * es), "alloc B'");
  if (K) CK(h->Kq.ensure((size_t)m * ld * ts), "alloc K'");
  CK(h->N.ensure((size_t)m * ld * 8), "alloc N");
  if (!f64) CK(h->Nq.ensure((size_t)m * ld * es), "alloc Nq");
  CK(h->shUT.ensure((size_t)n * m * es), "alloc U");
  CK(h->shUblk.ensure((size_t)n * n * es), "alloc U blocks");
  CK(h->Y.ensure((size_t)m * ld * ts), "alloc G/Y");
  const int G = fram::sdsn_sh_grid(m, h->num_sms, f64);
  CK(h->shColpart.ensure((size_t)G * ld * ts), "alloc colpart");
  CK(h->shRsum.ensure((size_t)m * 8), "alloc rsum");
  CK(h->shSend.ensure((size_t)(ld + 8) * 8), "alloc send");
  CK(h->shRecv.ensure((size_t)(ld + 8) * 8), "alloc recv");
  CK(h->shState.ensure(sizeof(fram::ShardSdsnState)), "alloc state");
  CK(h->ghist.ensure((size_t)sdsn_cap(h) * 8), "alloc ghist");
  CK(h->upd.ensure((size_t)(h->num_sms * 4 * 2 + 16) * 8), "alloc upd");
  CK(h->scal.ensure(kScalDoubles * 8), "alloc scal");
  CK(h->shNfull.ensure((size_t)n * ld * 8), "alloc N full");
  CK(h->lapw.ensure(fram::lap_work_bytes(n)), "alloc lap");
  CK(h->permd.ensure((size_t)n * 4), "alloc perm");
  CK(h->scan.ensure(sizeof(fram::PrecondScan)), "alloc scan");
  CK(h->shScan.ensure(sizeof(fram::PrecondScan)), "alloc scan (reduced)");
  if (!h->hscal) CK(cudaMallocHost((void**)&h->hscal, kScalDoubles * 8), "alloc pinned");
  for (auto& e : h->ev)
    if (!e) CK(cudaEventCreate(&e), "event create");
  if (timing) CK(cudaEventRecord(h->ev[0], st), "event");
  // stage inputs
  fram_status rs;
  const void *dA, *dB, *dK, *dX0;
  if ((rs = stage_in(h, h->stA, A, (size_t)m * n * dt_size(dt), st, &dA)) != FRAM_OK) return rs;
  if ((rs = stage_in(h, h->stB, B, (size_t)n * n * dt_size(dt), st, &dB)) != FRAM_OK) return rs;
  if ((rs = stage_in(h, h->stK, K, (size_t)m * n * dt_size(dt), st, &dK)) != FRAM_OK) return rs;
  if ((rs = stage_in(h, h->stX0, X0, (size_t)m * n * 8, st, &dX0)) != FRAM_OK) return rs;
  // K1: global c = max(A, Ã, K) and validation, all-reduced (max) over ranks
  fram::PrecondScan* sc = h->scan.as<fram::PrecondScan>();
  fram::PrecondScan* scr = h->shScan.as<fram::PrecondScan>();
  const bool sym = (h->sched.flags & FRAM_FLAG_CHECK_SYMMETRY) != 0;
  CK(fram::launch_precond_scan(nullptr, dB, nullptr, dt, n, sym, sc, nullptr, nullptr, st), "precond scan");
  CK(fram::launch_precond_scan_rows(dA, dK, dt, m, n, sc, st), "precond scan rows");
  h->launches += 2;
  if (nck(fram::shard_allreduce_f64(sh, sc->maxv, scr->maxv, 3, true, st, &err)) != FRAM_OK) return FRAM_ERR_NCCL;
  if (nck(fram::shard_allreduce_u64_max(sh, reinterpret_cast<const uint64_t*>(&sc->bad_nonfinite),
                                        reinterpret_cast<uint64_t*>(&scr->bad_nonfinite), 3, st, &err)) != FRAM_OK)
    return FRAM_ERR_NCCL;
  fram::PrecondScan hs;
  CK(cudaMemcpyAsync(&hs, scr, sizeof(hs), cudaMemcpyDeviceToHost, st), "scan readback");
  CK(cudaStreamSynchronize(st), "scan sync");
  if (hs.bad_nonfinite) return fail(FRAM_ERR_DATA, "non-finite entries in A, B or K");
  if (hs.bad_negative) return fail(FRAM_ERR_DATA, "negative entries in A, B or K (P:55)");
  if (hs.bad_asym) return fail(FRAM_ERR_DATA, "B is not symmetric (P:55, R28)");
  if (!(std::max(std::max(hs.maxv[0], hs.maxv[1]), hs.maxv[2]) > 0)) return fail(FRAM_ERR_DATA, "c = max(A, B, K) = 0 (S:344)");
  CK(fram::launch_precond_apply(dA, dB, dK, dt, n, ld, scr->maxv, op, h->Aq.p, h->BqT.p, dK ? h->Kq.p : nullptr,
                                f64, st, m),
     "precond apply");
  CK(fram::launch_init_n(h->N.as<double>(), h->Nq.p, op, (const double*)dX0, m, n, ld, st), "init N");
  h->launches += 2;
  if (timing) CK(cudaEventRecord(h->ev[1], st), "event");

  const fram_schedule& sch = h->sched;
  const bool replay = !h->replay.empty();
  const int T = replay ? (int)h->replay.size() : sch.max_outer;
  double* scal = h->scal.as<double>();
  double ms_gemm = 0, ms_sdsn = 0, ms_update = 0;
  int t = 0, capped = 0;
  int64_t total = 0;
  bool converged = false;
  fram::ShardSdsnParams sp{};
  sp.Y = h->Y.p; sp.rows = m; sp.n = n; sp.ld = ld;
  sp.theta = sch.theta; sp.gamma_th = sch.gamma_th; sp.sdsn_max = sch.sdsn_max;
  sp.scale = (sch.flags & FRAM_FLAG_NO_THETA_SCALE) ? 0 : 1;
  sp.colpart = h->shColpart.p; sp.rsum = h->shRsum.as<double>();
  sp.send = h->shSend.as<double>(); sp.recv = h->shRecv.as<double>();
  sp.gamma_hist = h->ghist.as<double>();
  sp.state = h->shState.as<fram::ShardSdsnState>();
  fram::ShardSdsnState hstate{};
  for (t = 1; t <= T; ++t) {
    if (timing) CK(cudaEventRecord(h->ev[2], st), "event");
    // gradient: U_rᵀ (n × m), all-gather, G_r = A'_r · U + λK'_r
    fram::GemmArgs g1{f64 ? h->N.p : h->Nq.p, h->BqT.p, m, n, n, ld, 0, h->shUT.p, m, nullptr, 0.0};
    if (f64) CK(fram::launch_gemm_f64(g1, st), "gemm1 f64"); else CK(fram::launch_gemm_tc(g1, op, st), "gemm1 tcgen05");
    if (nck(fram::shard_allgather_bytes(sh, h->shUT.p, h->shUblk.p, (size_t)n * m * es, st, &err)) != FRAM_OK)
      return FRAM_ERR_NCCL;
    fram::GemmArgs g2{h->Aq.p, h->shUblk.p, m, n, n, ld, 1, h->Y.p, ld, dK ? h->Kq.p : nullptr, h->lambda};
    g2.kchunk = m;
    if (f64) CK(fram::launch_gemm_f64(g2, st), "gemm2 f64"); else CK(fram::launch_gemm_tc(g2, op, st), "gemm2 tcgen05");
    h->launches += 2;
    if (timing) CK(cudaEventRecord(h->ev[3], st), "event");
    // SDSN on the row block
    sp.sdsn_fixed = replay ? h->replay[t - 1] : sch.sdsn_fixed;
    CK(cudaMemsetAsync(sp.state, 0, sizeof(fram::ShardSdsnState), st), "state reset");
    CK(fram::launch_sdsn_sh_max(sp, f64, st, h->num_sms), "sdsn max");
    if (nck(fram::shard_allreduce_f64(sh, sp.send, sp.recv, 1, true, st, &err)) != FRAM_OK) return FRAM_ERR_NCCL;
    CK(fram::prepare_sdsn_sh(sp, f64, h->num_sms), "sdsn prepare");
    CK(fram::launch_sdsn_sh_sweep(sp, f64, 0, st, h->num_sms), "sdsn scale");
    if (nck(fram::shard_allreduce_f64(sh, sp.send, sp.recv, n + 1, false, st, &err)) != FRAM_OK) return FRAM_ERR_NCCL;
    h->launches += 3;                                  // max, scale sweep, reduce
    const int cap = std::max(1, sp.sdsn_fixed > 0 ? sp.sdsn_fixed : sch.sdsn_max);
    // Passes are queued kChunk at a time between host polls of `done` (passes after the last are no-ops).
    // Every pass is the same launch sequence (the pass index lives on the device), so with an NCCL
    // communicator a chunk is captured once as a CUDA graph — kernels and ncclAllReduce — and relaunched:
    // one host call per chunk instead of 3 per pass.  Virtual shards synchronise their collectives on
    // the host and keep the plain launches.
    constexpr int kChunk = 16;
    bool use_graph = !fram::shard_is_virtual(sh) && !h->sh_graph_off;
    if (use_graph) {
      unsigned char key[sizeof(h->sh_graph_key)] = {};
      memcpy(key, &sp, sizeof(sp));
      key[sizeof(sp)] = f64 ? 1 : 2;
      if (!h->sh_graph || memcmp(key, h->sh_graph_key, sizeof(key)) != 0) {
        if (h->sh_graph) { cudaGraphExecDestroy(h->sh_graph); h->sh_graph = nullptr; }
        if (!h->sh_cap_stream) CK(cudaStreamCreateWithFlags(&h->sh_cap_stream, cudaStreamNonBlocking), "stream create");
        CK(fram::prepare_sdsn_sh(sp, f64, h->num_sms), "sdsn prepare");
        cudaGraph_t gr = nullptr;
        CK(cudaStreamBeginCapture(h->sh_cap_stream, cudaStreamCaptureModeThreadLocal), "graph capture begin");
        bool ok = true;
        for (int p = 0; p < kChunk && ok; ++p) {
          ok = fram::launch_sdsn_sh_sweep(sp, f64, 1, h->sh_cap_stream, h->num_sms) == cudaSuccess;
          ok = ok && fram::shard_allreduce_f64(sh, sp.send, sp.recv, n + 1, false, h->sh_cap_stream, &err) == FRAM_OK;
        }
        const cudaError_t ce = cudaStreamEndCapture(h->sh_cap_stream, &gr);
        cudaError_t ie = cudaErrorUnknown;
        if (ok && ce == cudaSuccess) ie = cudaGraphInstantiate(&h->sh_graph, gr, 0);
        if (gr) cudaGraphDestroy(gr);
        if (ie == cudaSuccess) {
          memcpy(h->sh_graph_key, key, sizeof(key));
        } else {                                       // e.g. a collective library that cannot be captured
          cudaGetLastError();
          h->sh_graph = nullptr;
          h->sh_graph_off = true;
          use_graph = false;
        }
      }
    }
    for (int p0 = 0; p0 < cap; p0 += kChunk) {
      if (use_graph) {
        CK(cudaGraphLaunch(h->sh_graph, st), "graph launch");
        h->launches += 2 * kChunk;
      } else {
        for (int p = p0; p < std::min(cap, p0 + kChunk); ++p) {
          CK(fram::launch_sdsn_sh_sweep(sp, f64, 1, st, h->num_sms), "sdsn pass");
          if (nck(fram::shard_allreduce_f64(sh, sp.send, sp.recv, n + 1, false, st, &err)) != FRAM_OK)
            return FRAM_ERR_NCCL;
          h->launches += 2;
        }
      }
      CK(cudaMemcpyAsync(&hstate, sp.state, sizeof(hstate), cudaMemcpyDeviceToHost, st), "state readback");
      CK(cudaStreamSynchronize(st), "state sync");
      if (hstate.done) break;
    }
    if (!hstate.done) return fail(FRAM_ERR_CUDA, "sharded SDSN did not finish");
    if (timing) CK(cudaEventRecord(h->ev[4], st), "event");
    CK(fram::launch_update(h->N.as<double>(), h->Y.p, f64, h->Nq.p, op, m, n, ld, sch.alpha, h->upd.as<double>(),
                           reinterpret_cast<unsigned*>(h->upd.as<double>() + h->num_sms * 8 + 8), scal + 4, st,
                           h->num_sms),
       "update");
    h->launches++;
    if (nck(fram::shard_allreduce_f64(sh, scal + 4, scal + 12, 2, false, st, &err)) != FRAM_OK) return FRAM_ERR_NCCL;
    if (timing) CK(cudaEventRecord(h->ev[5], st), "event");
    CK(cudaMemcpyAsync(h->hscal, scal, kScalDoubles * 8, cudaMemcpyDeviceToHost, st), "scalar readback");
    CK(cudaStreamSynchronize(st), "iteration sync");
    const int passes = hstate.passes;
    const double delta = std::sqrt(h->hscal[12]) / std::sqrt(h->hscal[13]);   // same formula as K5
    if (!std::isfinite(delta)) return fail(FRAM_ERR_DATA, "non-finite delta (overflow in the gradient?)");
    total += passes;
    if (sp.sdsn_fixed == 0 && passes >= sch.sdsn_max) ++capped;
    if (timing) {
      float a, b, cc;
      cudaEventElapsedTime(&a, h->ev[2], h->ev[3]);
      cudaEventElapsedTime(&b, h->ev[3], h->ev[4]);
      cudaEventElapsedTime(&cc, h->ev[4], h->ev[5]);
      ms_gemm += a; ms_sdsn += b; ms_update += cc;
    }
    if (stats && (sch.flags & FRAM_FLAG_TRACE)) {
      if (stats->passes_per_iter) stats->passes_per_iter[t - 1] = passes;
      if (stats->delta_trace) stats->delta_trace[t - 1] = delta;
      if (stats->gamma_last) stats->gamma_last[t - 1] = hstate.gamma_last;
    }
    if (delta <= sch.delta_th) {
      converged = true;
      if (!replay) break;
    } else if (replay) {
      converged = false;
    }
  }
  if (t > T) t = T;
  // discretisation: all ranks gather N and run the same deterministic LAP (R17)
  if (timing) CK(cudaEventRecord(h->ev[6], st), "event");
  if (nck(fram::shard_allgather_bytes(sh, h->N.p, h->shNfull.p, (size_t)m * ld * 8, st, &err)) != FRAM_OK)
    return FRAM_ERR_NCCL;
  CK(fram::launch_lap(h->shNfull.as<double>(), n, ld, h->permd.as<int32_t>(), h->lapw.p, st), "lap");
  h->launches++;
  if (timing) CK(cudaEventRecord(h->ev[7], st), "event");
  if (X_out) CK(cudaMemcpy2DAsync(X_out, n * 8, h->N.p, ld * 8, n * 8, m, cudaMemcpyDefault, st), "X_out copy");
  if (perm_out) CK(cudaMemcpyAsync(perm_out, h->permd.p, n * 4, cudaMemcpyDefault, st), "perm copy");
  CK(cudaStreamSynchronize(st), "final sync");
  if (stats) {
    stats->outer_iters = t;
    stats->converged = converged ? 1 : 0;
    stats->sdsn_capped_calls = capped;
    stats->total_passes = total;
    stats->kernel_launches = h->launches;
    stats->sdsn_kernel = 3;
    if (timing) {
      float a, b, cc;
      cudaEventElapsedTime(&a, h->ev[0], h->ev[1]);
      cudaEventElapsedTime(&b, h->ev[6], h->ev[7]);
      cudaEventElapsedTime(&cc, h->ev[0], h->ev[7]);
      stats->ms_precond = a; stats->ms_lap = b; stats->ms_total = cc;
      stats->ms_gemm = ms_gemm; stats->ms_sdsn = ms_sdsn; stats->ms_update = ms_update;
    }
  }
  if (!converged) {
    g_err = "max_outer reached without delta <= delta_th";
    return FRAM_NOT_CONVERGED;
  }
  return FRAM_OK;
}

// Virtual-shard group solve: rank r's thread runs the unchanged sharded_solve on row block r of the
// caller's full n×n inputs (A, K, X0 and X_out are sliced by rows; Ã is shared), with the collectives
// served by the group (sharded.cu).  Rank 0 writes perm_out and the stats.
fram_status group_solve(fram_ctx* g, int dt, const void* A, const void* B, const void* K, const double* X0, int op,
                        cudaStream_t caller, double* X_out, int32_t* perm_out, fram_stats* stats) {
  NvtxRange range_("group_solve");
  const int W = (int)g->vsub.size();
  const long n = g->n, m = n / W;
  CK(cudaStreamSynchronize(caller), "caller stream sync");        // inputs produced on the caller's stream
  fram::vgroup_reset(g->vgroup);                                  // a previous failed solve aborted it
  std::vector<fram_status> st(W, FRAM_OK);
  std::vector<std::string> msg(W);
  const size_t es = dt_size(dt);
  auto run = [&](int r) {
    fram_ctx* h = g->vsub[r];
    fram_status s0 = set_device(h);
    if (s0 == FRAM_OK) {
      const size_t off = (size_t)r * m * n;
      s0 = sharded_solve(h, dt, static_cast<const char*>(A) + off * es, B,
                         K ? static_cast<const char*>(K) + off * es : nullptr, X0 ? X0 + off : nullptr, op,
                         g->vstreams[r], X_out ? X_out + off : nullptr, r == 0 ? perm_out : nullptr,
                         r == 0 ? stats : nullptr);
    }
    st[r] = s0;
    if (s0 != FRAM_OK && s0 != FRAM_NOT_CONVERGED) {
      msg[r] = g_err;
      fram::vgroup_abort(g->vgroup);             // release ranks waiting in a collective
    }
  };
  std::vector<std::thread> th;
  for (int r = 1; r < W; ++r) th.emplace_back(run, r);
  run(0);
  for (auto& t : th) t.join();
  for (int r = 0; r < W; ++r)                    // the first rank's own error (not an abort it caused)
    if (st[r] != FRAM_OK && st[r] != FRAM_NOT_CONVERGED && st[r] != FRAM_ERR_NCCL) return fail(st[r], msg[r]);
  for (int r = 0; r < W; ++r)
    if (st[r] != FRAM_OK && st[r] != FRAM_NOT_CONVERGED) return fail(st[r], msg[r]);
  if (st[0] == FRAM_NOT_CONVERGED) g_err = "max_outer reached without delta <= delta_th";
  return st[0];
}

// Batched solves of instances larger than one CTA can hold (64 < n): P worker threads, each with its
// own sub-handle and non-blocking stream, take instances from a shared counter and run the single-
// instance solve on them (K4c one-cluster / K4r on-chip SDSN, LAP on one CTA or a cluster), so up to P
// instances occupy the GPU at once.  Per-instance status in status_out; the worst status is returned.
constexpr int kBatchWorkers = 4;
fram_status batched_multi(fram_ctx* h, int64_t batch, int dt, const void* A, const void* B, const void* K,
                          const double* X0, fram_precision p, cudaStream_t caller, double* X_out, int32_t* perm_out,
                          int32_t* status_out, fram_stats* stats) {
  const long n = h->n;
  if (batch == 0) return FRAM_OK;
  const int P = (int)std::min<int64_t>(kBatchWorkers, batch);
  while ((int)h->bsub.size() < P) {
    fram_handle sub = nullptr;
    fram_status s = fram_create(n, h->lambda, &h->sched, h->device, &sub);
    if (s != FRAM_OK) return s;
    sub->dev_checked = h->dev_checked;
    sub->num_sms = h->num_sms;
    h->bsub.push_back(sub);
    cudaStream_t cs = nullptr;
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "stream create");
    h->bstreams.push_back(cs);
  }
  for (int w = 0; w < P; ++w) fram_set_schedule(h->bsub[w], &h->sched);
  CK(cudaStreamSynchronize(caller), "caller stream sync");
  const size_t es = dt_size(dt), mat = (size_t)n * n;
  std::vector<int32_t> sts((size_t)batch, FRAM_OK);
  std::vector<fram_stats> ist((size_t)batch);
  std::vector<std::string> msg((size_t)batch);
  std::atomic<int64_t> next{0};
  auto work = [&](int w) {
    fram_ctx* sub = h->bsub[w];
    for (int64_t b = next++; b < batch; b = next++) {
      fram_stats& s = ist[b];
      s = fram_stats{};
      const fram_status r = fram_solve(sub, (fram_dtype)dt, static_cast<const char*>(A) + b * mat * es,
                                       static_cast<const char*>(B) + b * mat * es,
                                       K ? static_cast<const char*>(K) + b * mat * es : nullptr,
                                       X0 ? X0 + b * mat : nullptr, p, h->bstreams[w],
                                       X_out ? X_out + b * mat : nullptr, perm_out ? perm_out + b * n : nullptr, &s);
      sts[b] = r;
      if (r != FRAM_OK && r != FRAM_NOT_CONVERGED) msg[b] = g_err;
    }
  };
  std::vector<std::thread> th;
  for (int w = 1; w < P; ++w) th.emplace_back(work, w);
  work(0);
  for (auto& t : th) t.join();
  fram_status worst = FRAM_OK;
  std::string wmsg;
  int maxo = 0, allc = 1, capped = 0;
  int64_t tot = 0, launches = 0;
  for (int64_t b = 0; b < batch; ++b) {
    const fram_status s = (fram_status)sts[b];
    if (s != FRAM_OK && s != FRAM_NOT_CONVERGED) {
      if (worst == FRAM_OK || worst == FRAM_NOT_CONVERGED) { worst = s; wmsg = msg[b]; }
    } else if (s == FRAM_NOT_CONVERGED && worst == FRAM_OK) {
      worst = FRAM_NOT_CONVERGED;
    }
    maxo = std::max(maxo, ist[b].outer_iters);
    allc &= ist[b].converged;
    capped += ist[b].sdsn_capped_calls;
    tot += ist[b].total_passes;
    launches += ist[b].kernel_launches;
  }
  if (status_out) CK(cudaMemcpy(status_out, sts.data(), (size_t)batch * 4, cudaMemcpyDefault), "status copy");
  if (stats) {
    stats->outer_iters = maxo;
    stats->converged = allc;
    stats->sdsn_capped_calls = capped;
    stats->total_passes = tot;
    stats->kernel_launches = launches;
  }
  if (worst == FRAM_NOT_CONVERGED) g_err = "one or more instances did not converge (status_out)";
  else if (worst != FRAM_OK) g_err = "instance error (status_out): " + wmsg;
  return worst;
}

}  // namespace

extern "C" {

fram_status fram_create(int64_t n, double lambda, const fram_schedule* s, int device, fram_handle* out) {
  if (!out) return fail(FRAM_ERR_USAGE, "null out");
  *out = nullptr;
  if (n < 1) return fail(FRAM_ERR_USAGE, "n must be >= 1");
  if (!(lambda >= 0) || !std::isfinite(lambda)) return fail(FRAM_ERR_USAGE, "lambda must be >= 0");
  fram_schedule sc = s ? *s : default_schedule();
  fram_status st = check_schedule(sc);
  if (st != FRAM_OK) return st;
  fram_ctx* h = new fram_ctx();
  h->n = n;
  h->lambda = lambda;
  h->device = device;
  h->ld = ld_for(n);
  h->replay.assign(sc.replay_passes, sc.replay_passes + sc.replay_len);
  h->sched = sc;
  h->sched.replay_passes = h->replay.empty() ? nullptr : h->replay.data();
  *out = h;
  return FRAM_OK;
}

fram_status fram_set_schedule(fram_handle h, const fram_schedule* s) {
  if (!h || !s) return fail(FRAM_ERR_USAGE, "null argument");
  fram_status st = check_schedule(*s);
  if (st != FRAM_OK) return st;
  h->replay.assign(s->replay_passes, s->replay_passes + s->replay_len);
  h->sched = *s;
  h->sched.replay_passes = h->replay.empty() ? nullptr : h->replay.data();
  for (fram_ctx* sub : h->vsub) fram_set_schedule(sub, s);
  return FRAM_OK;
}

void fram_destroy(fram_handle h) {
  if (!h) return;
  cudaSetDevice(h->device);
  for (fram_ctx* sub : h->vsub) fram_destroy(sub);
  for (fram_ctx* sub : h->bsub) fram_destroy(sub);
  for (cudaStream_t s : h->bstreams) cudaStreamDestroy(s);
  for (cudaStream_t s : h->vstreams) cudaStreamDestroy(s);
  if (h->sh_graph) cudaGraphExecDestroy(h->sh_graph);
  if (h->sh_cap_stream) cudaStreamDestroy(h->sh_cap_stream);
  fram::vgroup_destroy(h->vgroup);
  DevBuf* bufs[] = {&h->Aq, &h->BqT, &h->Kq, &h->N, &h->Nq, &h->UT, &h->Y, &h->colpart, &h->Spart, &h->Mpart,
                    &h->cvec, &h->bar, &h->scal, &h->ghist, &h->upd, &h->lapw, &h->permd, &h->stA, &h->stB,
                    &h->stK, &h->stX0, &h->stX, &h->scan, &h->rcolpart, &h->rbvec, &h->rflags, &h->rdbg, &h->shUT, &h->shUblk, &h->shRsum,
                    &h->shSend, &h->shRecv, &h->shState, &h->shNfull, &h->shColpart, &h->shScan, &h->atA,
                    &h->atB, &h->atK, &h->atF, &h->atFt, &h->atPerm, &h->evPart, &h->evOut, &h->evPerm};
  for (DevBuf* b : bufs) b->release();
  if (h->hscal) cudaFreeHost(h->hscal);
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : h->sev)
    if (e) cudaEventDestroy(e);
  for (auto& e : h->gev)
    if (e) cudaEventDestroy(e);
  if (h->side) cudaStreamDestroy(h->side);
  fram::batched_release(h->bws);
  if (h->shard) fram::shard_destroy(h->shard);
  delete h;
}

const char* fram_last_error(void) { return g_err.c_str(); }
int fram_abi_version(void) { return FRAM_ABI_VERSION; }
const char* fram_build_info(void) { return "libfram sm_100a (tcgen05/TMEM/TMA GEMM, persistent SDSN, DMMA FP64, GPU Hungarian)"; }

fram_status fram_solve(fram_handle h, fram_dtype dt, const void* A, const void* B, const void* K, const double* X0,
                       fram_precision p, void* stream, double* X_out, int32_t* perm_out, fram_stats* stats) {
  NvtxRange range_solve("fram_solve");
  fram_status s0 = common_checks(h, (int)dt, p);
  if (s0 != FRAM_OK) return s0;
  if (!A || !B) return fail(FRAM_ERR_USAGE, "A and B are required");
  if (!h->vsub.empty())
    return group_solve(h, (int)dt, A, B, K, X0, (int)p, reinterpret_cast<cudaStream_t>(stream), X_out, perm_out,
                       stats);
  if (h->shard)
    return sharded_solve(h, (int)dt, A, B, K, X0, (int)p, reinterpret_cast<cudaStream_t>(stream), X_out, perm_out,
                         stats);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int op = prec_to_op(p);
  const bool f64 = (op == 0);
  const long n = h->n, ld = h->ld;
  if (!fram::sdsn_supported(n, f64)) return fail(FRAM_ERR_USAGE, "n too large for the SDSN kernel");
  h->launches = 0;
  const bool timing = (h->sched.flags & FRAM_FLAG_TIME_PHASES) != 0;
  fram_status rs = ensure_ws(h, op, K != nullptr);
  if (rs != FRAM_OK) return rs;
  if (timing) CK(cudaEventRecord(h->ev[0], st), "event");

  const size_t in_bytes = (size_t)n * n * dt_size(dt);
  const void *dA, *dB, *dK, *dX0;
  if ((rs = stage_in(h, h->stA, A, in_bytes, st, &dA)) != FRAM_OK) return rs;
  if ((rs = stage_in(h, h->stB, B, in_bytes, st, &dB)) != FRAM_OK) return rs;
  if ((rs = stage_in(h, h->stK, K, in_bytes, st, &dK)) != FRAM_OK) return rs;
  if ((rs = stage_in(h, h->stX0, X0, (size_t)n * n * 8, st, &dX0)) != FRAM_OK) return rs;

  double c = 0;
  {
    NvtxRange r_("precondition");
    if ((rs = precondition(h, (int)dt, dA, dB, dK, op, st, &c)) != FRAM_OK) return rs;
  }
  CK(fram::launch_init_n(h->N.as<double>(), h->Nq.p, op, (const double*)dX0, n, n, ld, st), "init N");
  h->launches++;
  if (timing) CK(cudaEventRecord(h->ev[1], st), "event");

  const fram_schedule& sc = h->sched;
  const bool replay = !h->replay.empty();
  const int T = replay ? (int)h->replay.size() : sc.max_outer;
  double* scal = h->scal.as<double>();
  double ms_gemm = 0, ms_sdsn = 0, ms_update = 0;
  int t = 0, capped = 0;
  int64_t total = 0;
  bool converged = false;
  // The gradient of iteration t+1 is queued before the host waits for iteration t's scalars (δ, passes):
  // it reads only N_q, written by update t in stream order, so the GPU runs it while the host reads δ
  // instead of idling between iterations.  After the last iteration one queued gradient is wasted
  // (it writes U and G only; the LAP reads N).  Its events alternate between two pairs.
  auto queue_gradient = [&](int par) -> fram_status {
    NvtxRange range_("gradient");
    if (timing) CK(cudaEventRecord(par ? h->gev[0] : h->ev[2], st), "event");
    fram_status r_ = gradient(h, op, dK != nullptr, st);
    if (r_ != FRAM_OK) return r_;
    if (timing) CK(cudaEventRecord(par ? h->gev[1] : h->ev[3], st), "event");
    return FRAM_OK;
  };
  if ((rs = queue_gradient(0)) != FRAM_OK) return rs;
  for (t = 1; t <= T; ++t) {
    NvtxRange r_outer("outer_iteration");
    const int par = (t - 1) & 1;
    const int fixed = replay ? h->replay[t - 1] : sc.sdsn_fixed;
    {
      NvtxRange r_("sdsn");
      if ((rs = run_sdsn(h, f64, fixed, st)) != FRAM_OK) return rs;
    }
    if (timing) CK(cudaEventRecord(h->ev[4], st), "event");
    CK(fram::launch_update(h->N.as<double>(), h->Y.p, f64, h->Nq.p, op, n, n, ld, sc.alpha, h->upd.as<double>(),
                           reinterpret_cast<unsigned*>(h->upd.as<double>() + h->num_sms * 8 + 8), scal + 4, st,
                           h->num_sms),
       "update");
    h->launches++;
    if (timing) CK(cudaEventRecord(h->ev[5], st), "event");
    CK(cudaMemcpyAsync(h->hscal, scal, kScalDoubles * 8, cudaMemcpyDeviceToHost, st), "scalar readback");
    CK(cudaEventRecord(h->gev[2], st), "event");
    if (t < T && (rs = queue_gradient(par ^ 1)) != FRAM_OK) return rs;
    CK(cudaEventSynchronize(h->gev[2]), "iteration sync");
    const int passes = *reinterpret_cast<int*>(h->hscal + 8);
    const double gam = h->hscal[0];
    const double delta = h->hscal[6];
    if (!std::isfinite(delta)) return fail(FRAM_ERR_DATA, "non-finite delta (overflow in the gradient?)");
    total += passes;
    if (fixed == 0 && passes >= sc.sdsn_max) ++capped;
    if (timing) {
      float a, b, cc;
      cudaEvent_t g0 = par ? h->gev[0] : h->ev[2], g1 = par ? h->gev[1] : h->ev[3];
      cudaEventElapsedTime(&a, g0, g1);
      cudaEventElapsedTime(&b, g1, h->ev[4]);
      cudaEventElapsedTime(&cc, h->ev[4], h->ev[5]);
      ms_gemm += a;
      ms_sdsn += b;
      ms_update += cc;
    }
    if (stats && (sc.flags & FRAM_FLAG_TRACE)) {
      if (stats->passes_per_iter) stats->passes_per_iter[t - 1] = passes;
      if (stats->delta_trace) stats->delta_trace[t - 1] = delta;
      if (stats->gamma_last) stats->gamma_last[t - 1] = gam;
    }
    if (delta <= sc.delta_th) {
      converged = true;
      if (!replay) break;
    } else if (replay) {
      converged = false;
    }
  }
  if (t > T) t = T;
  if (X_out) {                                // N is final: copy it out on the side stream while the LAP runs
    CK(cudaEventRecord(h->sev[0], st), "event");
    CK(cudaStreamWaitEvent(h->side, h->sev[0], 0), "side wait");
    CK(cudaMemcpy2DAsync(X_out, n * 8, h->N.p, ld * 8, n * 8, n, cudaMemcpyDefault, h->side), "X_out copy");
    CK(cudaEventRecord(h->sev[1], h->side), "event");
  }
  if (timing) CK(cudaEventRecord(h->ev[6], st), "event");
  NvtxRange r_lap("lap");
  const cudaError_t lap_e = fram::launch_lap(h->N.as<double>(), n, ld, h->permd.as<int32_t>(), h->lapw.p, st);
  // join the copy before any return: the next call on `st` rewrites N
  const cudaError_t join_e = X_out ? cudaStreamWaitEvent(st, h->sev[1], 0) : cudaSuccess;
  CK(lap_e, "lap");
  CK(join_e, "join X_out copy");
  h->launches++;
  if (timing) CK(cudaEventRecord(h->ev[7], st), "event");
  if (perm_out) CK(cudaMemcpyAsync(perm_out, h->permd.p, n * 4, cudaMemcpyDefault, st), "perm copy");
  CK(cudaStreamSynchronize(st), "final sync");
  if (stats) {
    stats->outer_iters = t;
    stats->converged = converged ? 1 : 0;
    stats->sdsn_capped_calls = capped;
    stats->total_passes = total;
    stats->kernel_launches = h->launches;
    stats->sdsn_kernel = sdsn_kind(h, f64);
    if (timing) {
      float a, b, cc;
      cudaEventElapsedTime(&a, h->ev[0], h->ev[1]);
      cudaEventElapsedTime(&b, h->ev[6], h->ev[7]);
      cudaEventElapsedTime(&cc, h->ev[0], h->ev[7]);
      stats->ms_precond = a;
      stats->ms_lap = b;
      stats->ms_total = cc;
      stats->ms_gemm = ms_gemm;
      stats->ms_sdsn = ms_sdsn;
      stats->ms_update = ms_update;
    }
  }
  (void)c;
  if (!converged) {
    g_err = "max_outer reached without delta <= delta_th";
    return FRAM_NOT_CONVERGED;
  }
  return FRAM_OK;
}

fram_status fram_sdsn(fram_handle h, fram_precision p, const void* X, void* D_out, int32_t* passes,
                      double* gamma_hist, void* stream) {
  fram_status s0 = common_checks(h, 0, p);
  if (s0 != FRAM_OK) return s0;
  if (h->shard || !h->vsub.empty()) return fail(FRAM_ERR_USAGE, "not available on a sharded handle");
  if (!X || !D_out || !passes) return fail(FRAM_ERR_USAGE, "X, D_out and passes are required");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool f64 = (p == FRAM_PREC_FP64);
  const long n = h->n, ld = h->ld;
  if (!fram::sdsn_supported(n, f64)) return fail(FRAM_ERR_USAGE, "n too large for the SDSN kernel");
  h->launches = 0;
  fram_status rs = ensure_ws(h, f64 ? 0 : 1, false);
  if (rs != FRAM_OK) return rs;
  const size_t es = f64 ? 8 : 4;
  const void* dX;
  if ((rs = stage_in(h, h->stX, X, (size_t)n * n * es, st, &dX)) != FRAM_OK) return rs;
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(h->scan.p);
  CK(fram::launch_scan_nonneg(dX, f64, n, bad, st), "scan");
  unsigned long long hbad = 0;
  CK(cudaMemcpyAsync(&hbad, bad, 8, cudaMemcpyDeviceToHost, st), "scan readback");
  CK(cudaStreamSynchronize(st), "scan sync");
  if (hbad) return fail(FRAM_ERR_DATA, "SDSN input must be finite and nonnegative (S:251)");
  CK(cudaMemcpy2DAsync(h->Y.p, ld * es, dX, n * es, n * es, n, cudaMemcpyDeviceToDevice, st), "X copy");
  if ((rs = run_sdsn(h, f64, h->sched.sdsn_fixed, st)) != FRAM_OK) return rs;
  CK(cudaMemcpyAsync(h->hscal, h->scal.p, kScalDoubles * 8, cudaMemcpyDeviceToHost, st), "readback");
  CK(cudaMemcpy2DAsync(D_out, n * es, h->Y.p, ld * es, n * es, n, cudaMemcpyDefault, st), "D copy");
  CK(cudaStreamSynchronize(st), "sync");
  const int k = *reinterpret_cast<int*>(h->hscal + 8);
  *passes = k;
  if (gamma_hist && k > 0)
    CK(cudaMemcpy(gamma_hist, h->ghist.p, (size_t)k * 8, cudaMemcpyDeviceToHost), "gamma readback");
  return FRAM_OK;
}

fram_status fram_gradient(fram_handle h, fram_dtype dt, const void* A, const void* B, const void* K,
                          const double* Nin, fram_precision p, void* stream, void* G_out, double* c_out) {
  fram_status s0 = common_checks(h, (int)dt, p);
  if (s0 != FRAM_OK) return s0;
  if (!A || !B || !Nin || !G_out) return fail(FRAM_ERR_USAGE, "A, B, N and G_out are required");
  if (h->shard || !h->vsub.empty()) return fail(FRAM_ERR_USAGE, "not available on a sharded handle");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int op = prec_to_op(p);
  const long n = h->n, ld = h->ld;
  h->launches = 0;
  fram_status rs = ensure_ws(h, op, K != nullptr);
  if (rs != FRAM_OK) return rs;
  const size_t in_bytes = (size_t)n * n * dt_size(dt);
  const void *dA, *dB, *dK, *dN;
  if ((rs = stage_in(h, h->stA, A, in_bytes, st, &dA)) != FRAM_OK) return rs;
  if ((rs = stage_in(h, h->stB, B, in_bytes, st, &dB)) != FRAM_OK) return rs;
  if ((rs = stage_in(h, h->stK, K, in_bytes, st, &dK)) != FRAM_OK) return rs;
  if ((rs = stage_in(h, h->stX0, Nin, (size_t)n * n * 8, st, &dN)) != FRAM_OK) return rs;
  double c = 0;
  if ((rs = precondition(h, (int)dt, dA, dB, dK, op, st, &c)) != FRAM_OK) return rs;
  CK(fram::launch_init_n(h->N.as<double>(), h->Nq.p, op, (const double*)dN, n, n, ld, st), "init N");
  if ((rs = gradient(h, op, dK != nullptr, st)) != FRAM_OK) return rs;
  const size_t es = op == 0 ? 8 : 4;
  CK(cudaMemcpy2DAsync(G_out, n * es, h->Y.p, ld * es, n * es, n, cudaMemcpyDefault, st), "G copy");
  CK(cudaStreamSynchronize(st), "sync");
  if (c_out) *c_out = c;
  return FRAM_OK;
}

fram_status fram_lap(fram_handle h, const double* Nin, int32_t* perm_out, void* stream) {
  fram_status s0 = common_checks(h, 0, FRAM_PREC_FP64);
  if (s0 != FRAM_OK) return s0;
  if (h->shard || !h->vsub.empty()) return fail(FRAM_ERR_USAGE, "not available on a sharded handle");
  if (!Nin || !perm_out) return fail(FRAM_ERR_USAGE, "N and perm_out are required");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const long n = h->n, ld = h->ld;
  CK(h->N.ensure((size_t)n * ld * 8), "alloc N");
  CK(h->lapw.ensure(fram::lap_work_bytes(n)), "alloc lap");
  CK(h->permd.ensure((size_t)n * 4), "alloc perm");
  CK(h->scan.ensure(sizeof(fram::PrecondScan)), "alloc scan");
  CK(cudaMemcpy2DAsync(h->N.p, ld * 8, Nin, n * 8, n * 8, n, cudaMemcpyDefault, st), "N copy");
  {   // a NaN would never win a comparison and leave the search without a column: reject non-finite N
    unsigned long long* bad = reinterpret_cast<unsigned long long*>(h->scan.p);
    CK(fram::launch_scan_finite(h->N.as<double>(), n * ld, bad, st), "scan");   // ld padding is zero
    unsigned long long hbad = 0;
    CK(cudaMemcpyAsync(&hbad, bad, 8, cudaMemcpyDeviceToHost, st), "scan readback");
    CK(cudaStreamSynchronize(st), "scan sync");
    if (hbad) return fail(FRAM_ERR_DATA, "N must be finite");
  }
  CK(fram::launch_lap(h->N.as<double>(), n, ld, h->permd.as<int32_t>(), h->lapw.p, st), "lap");
  int lap_err = 0;
  CK(cudaMemcpyAsync(&lap_err, static_cast<char*>(h->lapw.p) + fram::lap_err_offset(n), sizeof(int),
                     cudaMemcpyDeviceToHost, st), "lap status");
  CK(cudaStreamSynchronize(st), "sync");
  if (lap_err) return fail(FRAM_ERR_DATA, "LAP found no finite candidate column (non-finite N)");
  CK(cudaMemcpyAsync(perm_out, h->permd.p, n * 4, cudaMemcpyDefault, st), "perm copy");
  CK(cudaStreamSynchronize(st), "sync");
  return FRAM_OK;
}

fram_status fram_solve_batched(fram_handle h, int64_t batch, fram_dtype dt, const void* A, const void* B,
                               const void* K, const double* X0, fram_precision p, void* stream, double* X_out,
                               int32_t* perm_out, int32_t* status_out, fram_stats* stats) {
  NvtxRange range_("fram_solve_batched");
  fram_status s0 = common_checks(h, (int)dt, p);
  if (s0 != FRAM_OK) return s0;
  if (batch < 0 || !A || !B) return fail(FRAM_ERR_USAGE, "bad batch arguments");
  if (h->shard || !h->vsub.empty()) return fail(FRAM_ERR_USAGE, "not available on a sharded handle");
  if (h->n > 64)
    return batched_multi(h, batch, (int)dt, A, B, K, X0, p, reinterpret_cast<cudaStream_t>(stream), X_out, perm_out,
                         status_out, stats);
  std::string err;
  fram_status s = fram::batched_solve(h->bws, h->n, h->lambda, h->sched, batch, (int)dt, A, B, K, X0, (int)p,
                                      reinterpret_cast<cudaStream_t>(stream), X_out, perm_out, status_out, stats,
                                      h->num_sms, &err);
  if (s != FRAM_OK) g_err = err;
  return s;
}

fram_status fram_solve_attributed(fram_handle h, fram_dtype dt, int64_t n1, int64_t n2, int64_t d, const void* A,
                                  const void* B, const void* F, const void* Ft, fram_precision p, void* stream,
                                  double* X_out, int32_t* perm_out, fram_stats* stats) {
  fram_status s0 = common_checks(h, (int)dt, p);
  if (s0 != FRAM_OK) return s0;
  if (h->shard || !h->vsub.empty()) return fail(FRAM_ERR_USAGE, "not available on a sharded handle");
  const long m = h->n;
  if (!A || !B || n1 < 1 || n2 < 1 || n1 > m || n2 > m) return fail(FRAM_ERR_USAGE, "need 1 <= n1, n2 <= handle n");
  if ((F == nullptr) != (Ft == nullptr) || (F && d < 1)) return fail(FRAM_ERR_USAGE, "F and Ft go together, d >= 1");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t es = dt_size((int)dt);
  fram_status rs;
  const void *dA, *dB, *dF = nullptr, *dFt = nullptr;
  if ((rs = stage_in(h, h->stA, A, (size_t)n1 * n1 * es, st, &dA)) != FRAM_OK) return rs;
  if ((rs = stage_in(h, h->stB, B, (size_t)n2 * n2 * es, st, &dB)) != FRAM_OK) return rs;
  if (F) {
    if ((rs = stage_in(h, h->atF, F, (size_t)n1 * d * es, st, &dF)) != FRAM_OK) return rs;
    if ((rs = stage_in(h, h->atFt, Ft, (size_t)n2 * d * es, st, &dFt)) != FRAM_OK) return rs;
  }
  // R30: pad A, Ã to m×m (FP64) with isolated zero-attribute nodes; K = F F̃ᵀ in FP64, zero on padding
  CK(h->atA.ensure((size_t)m * m * 8), "alloc padded A");
  CK(h->atB.ensure((size_t)m * m * 8), "alloc padded B");
  CK(fram::launch_pad_convert(h->atA.as<double>(), m, m, m, dA, (int)dt, n1, n1, n1, st), "pad A");
  CK(fram::launch_pad_convert(h->atB.as<double>(), m, m, m, dB, (int)dt, n2, n2, n2, st), "pad B");
  h->launches += 2;
  const double* dK = nullptr;
  if (F) {
    const long ldd = (d + 1) / 2 * 2;                          // 16-byte rows for the DMMA loader
    CK(h->stX.ensure((size_t)2 * m * ldd * 8), "alloc features");
    double* Fq = h->stX.as<double>();
    double* Ftq = Fq + (size_t)m * ldd;
    CK(fram::launch_pad_convert(Fq, ldd, m, ldd, dF, (int)dt, d, n1, d, st), "pad F");
    CK(fram::launch_pad_convert(Ftq, ldd, m, ldd, dFt, (int)dt, d, n2, d, st), "pad Ft");
    CK(h->atK.ensure((size_t)m * m * 8), "alloc K");
    fram::GemmArgs gk{Fq, Ftq, m, m, d, ldd, 1, h->atK.p, m, nullptr, 0.0};   // K = F·F̃ᵀ (NT, FP64)
    CK(fram::launch_gemm_f64(gk, st), "K = F Ft^T");
    h->launches += 3;
    dK = h->atK.as<double>();
  }
  CK(h->atPerm.ensure((size_t)m * 4), "alloc perm");
  const int64_t launches_before = h->launches;
  fram_status so = fram_solve(h, FRAM_DT_F64, h->atA.p, h->atB.p, dK, nullptr, p, stream, X_out,
                              h->atPerm.as<int32_t>(), stats);
  if (so != FRAM_OK && so != FRAM_NOT_CONVERGED) return so;
  if (stats) stats->kernel_launches += launches_before;
  if (perm_out) {
    std::vector<int32_t> pm((size_t)m);
    CK(cudaMemcpy(pm.data(), h->atPerm.p, (size_t)m * 4, cudaMemcpyDeviceToHost), "perm readback");
    std::vector<int32_t> out((size_t)n1);
    for (long i = 0; i < n1; ++i) out[i] = pm[i] < n2 ? pm[i] : -1;
    CK(cudaMemcpyAsync(perm_out, out.data(), (size_t)n1 * 4, cudaMemcpyDefault, st), "perm copy");
    CK(cudaStreamSynchronize(st), "perm sync");
  }
  return so;
}

fram_status fram_create_sharded_virtual(int64_t n, double lambda, const fram_schedule* s, int world, int device,
                                        fram_handle* out) {
  if (!out) return fail(FRAM_ERR_USAGE, "null out");
  *out = nullptr;
  if (world < 1 || world > 16) return fail(FRAM_ERR_USAGE, "world must be in [1, 16]");
  if (n < 1 || n % world != 0) return fail(FRAM_ERR_USAGE, "n % world != 0");
  fram_status st = fram_create(n, lambda, s, device, out);
  if (st != FRAM_OK) return st;
  fram_handle g = *out;
  std::string err;
  st = set_device(g);
  if (st == FRAM_OK) {
    g->vgroup = fram::vgroup_create(world, &err);
    if (!g->vgroup) st = fail(FRAM_ERR_CUDA, err);
  }
  for (int r = 0; st == FRAM_OK && r < world; ++r) {
    fram_handle sub = nullptr;
    st = fram_create(n, lambda, s, device, &sub);
    if (st != FRAM_OK) break;
    g->vsub.push_back(sub);
    sub->dev_checked = g->dev_checked;
    sub->num_sms = g->num_sms;
    fram::shard_create_virtual(&sub->shard, g->vgroup, r);
    cudaStream_t cs = nullptr;
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) { st = fail(FRAM_ERR_CUDA, "stream create"); break; }
    g->vstreams.push_back(cs);
  }
  if (st != FRAM_OK) {
    fram_destroy(g);
    *out = nullptr;
  }
  return st;
}

fram_status fram_evaluate(fram_handle h, fram_dtype dt, const void* A, const void* B, const void* F, const void* Ft,
                          int64_t d, const int32_t* perm, void* stream, double out[4]) {
  fram_status s0 = common_checks(h, (int)dt, FRAM_PREC_FP64);
  if (s0 != FRAM_OK) return s0;
  if (!h->vsub.empty()) return fail(FRAM_ERR_USAGE, "not available on a virtual-shard group");
  if (!A || !B || !perm || !out) return fail(FRAM_ERR_USAGE, "A, B, perm and out are required");
  if ((F == nullptr) != (Ft == nullptr) || (F && d < 1)) return fail(FRAM_ERR_USAGE, "F and Ft go together, d >= 1");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const long n = h->n;
  const size_t es = dt_size((int)dt);
  fram_status rs;
  const void *dA, *dB, *dF = nullptr, *dFt = nullptr, *dP;
  if ((rs = stage_in(h, h->stA, A, (size_t)n * n * es, st, &dA)) != FRAM_OK) return rs;
  if ((rs = stage_in(h, h->stB, B, (size_t)n * n * es, st, &dB)) != FRAM_OK) return rs;
  if (F) {
    if ((rs = stage_in(h, h->atF, F, (size_t)n * d * es, st, &dF)) != FRAM_OK) return rs;
    if ((rs = stage_in(h, h->atFt, Ft, (size_t)n * d * es, st, &dFt)) != FRAM_OK) return rs;
  }
  if ((rs = stage_in(h, h->evPerm, perm, (size_t)n * 4, st, &dP)) != FRAM_OK) return rs;
  CK(h->evPart.ensure((size_t)n * 4 * 8), "alloc evaluation");
  CK(h->evOut.ensure(64), "alloc evaluation");
  double* dout = h->evOut.as<double>();
  int* bad = reinterpret_cast<int*>(dout + 4);
  CK(fram::launch_evaluate(dA, dB, dF, dFt, (int)dt, n, F ? d : 0, static_cast<const int32_t*>(dP),
                           h->evPart.as<double>(), dout, bad, st), "evaluate");
  double hv[5];
  CK(cudaMemcpyAsync(hv, dout, 5 * 8, cudaMemcpyDeviceToHost, st), "evaluation readback");
  CK(cudaStreamSynchronize(st), "sync");
  int hbad = 0;
  memcpy(&hbad, &hv[4], sizeof(int));
  if (hbad) return fail(FRAM_ERR_DATA, "perm entries must lie in [0, n)");
  const double e_edges = 0.5 * std::sqrt(hv[0]), e_feat = std::sqrt(hv[1]);
  out[0] = e_edges + e_feat;
  out[1] = e_edges;
  out[2] = e_feat;
  out[3] = 0.5 * hv[2] + h->lambda * hv[3];
  return FRAM_OK;
}

fram_status fram_get_unique_id(uint8_t id[128]) {
  std::string err;
  fram_status s = fram::shard_unique_id(id, &err);
  if (s != FRAM_OK) g_err = err;
  return s;
}

fram_status fram_create_sharded(int64_t n, double lambda, const fram_schedule* s, const uint8_t id[128], int rank,
                                int world, int device, fram_handle* out) {
  if (!out || !id) return fail(FRAM_ERR_USAGE, "null argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(FRAM_ERR_USAGE, "bad rank/world");
  if (n % world != 0) return fail(FRAM_ERR_USAGE, "n % world != 0");
  fram_status st = fram_create(n, lambda, s, device, out);
  if (st != FRAM_OK) return st;
  std::string err;
  fram_handle h = *out;
  st = set_device(h);
  if (st == FRAM_OK) st = fram::shard_create(&h->shard, id, rank, world, &err);
  if (st != FRAM_OK) {
    if (!err.empty()) g_err = err;
    fram_destroy(h);
    *out = nullptr;
  }
  return st;
}

}  // extern "C"
