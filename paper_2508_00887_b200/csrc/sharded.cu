// sharded.cu — NCCL plumbing for row-sharded solves.  NCCL is
// dlopen'ed (libnccl.so.2 — the one torch already loaded, if any) so that libfram loads on machines
// without it; only the sharded entry points need it.  nccl.h supplies the types only.
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>
#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>
#include "sharded.h"
#include <algorithm>

namespace fram {

// ---- virtual shards: W ranks of one process on one GPU (tests of the W > 1 path without W GPUs) ----
// Each rank runs the unchanged sharded solve on its own host thread and stream; a collective is
//   publish (send, recv) → event on my stream → host barrier → my stream waits for every rank's event →
//   fixed-order device sum / copies into MY recv → event → host barrier → my stream waits for every
//   rank's reduce (so no rank overwrites a send buffer another rank is still reading).
// Sums run in rank order 0..W−1 (deterministic).  A rank that fails aborts the group: every pending and
// later barrier returns false, so the other ranks leave their collectives with an error instead of
// waiting forever.
struct VGroup {
  int W = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  bool aborted = false;
  std::vector<const void*> send;
  std::vector<void*> recv;
  std::vector<cudaEvent_t> ev_ready, ev_done;
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) return false;
    const long g = gen;
    if (++arrived == W) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    cv.wait(lk, [&] { return gen != g || aborted; });
    return !aborted;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};

struct ShardCtx {
  VGroup* vg = nullptr;      // non-null: virtual rank of a one-GPU group (no NCCL)
  void* lib = nullptr;
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  ncclResult_t (*init)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allreduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allgather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  const char* (*errstr)(ncclResult_t) = nullptr;
};

namespace {
void* open_nccl(std::string* err) {
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    void* h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (h) return h;
  }
  *err = std::string("cannot dlopen libnccl.so.2: ") + (dlerror() ? dlerror() : "");
  return nullptr;
}
template <typename F>
bool sym(void* lib, const char* name, F* out) {
  *out = reinterpret_cast<F>(dlsym(lib, name));
  return *out != nullptr;
}
fram_status nccl_fail(ShardCtx* s, ncclResult_t r, const char* what, std::string* err) {
  *err = std::string(what) + ": " + (s->errstr ? s->errstr(r) : "nccl error");
  return FRAM_ERR_NCCL;
}
}  // namespace

fram_status shard_unique_id(uint8_t id[128], std::string* err) {
  void* lib = open_nccl(err);
  if (!lib) return FRAM_ERR_NCCL;
  ncclResult_t (*fn)(ncclUniqueId*) = nullptr;
  if (!sym(lib, "ncclGetUniqueId", &fn)) { *err = "ncclGetUniqueId not found"; return FRAM_ERR_NCCL; }
  ncclUniqueId uid;
  if (fn(&uid) != ncclSuccess) { *err = "ncclGetUniqueId failed"; return FRAM_ERR_NCCL; }
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id, &uid, 128);
  return FRAM_OK;
}

fram_status shard_create(ShardCtx** out, const uint8_t id[128], int rank, int world, std::string* err) {
  *out = nullptr;
  ShardCtx* s = new ShardCtx();
  s->rank = rank;
  s->world = world;
  s->lib = open_nccl(err);
  if (!s->lib) { delete s; return FRAM_ERR_NCCL; }
  if (!sym(s->lib, "ncclCommInitRank", &s->init) || !sym(s->lib, "ncclAllReduce", &s->allreduce) ||
      !sym(s->lib, "ncclAllGather", &s->allgather) || !sym(s->lib, "ncclCommDestroy", &s->destroy) ||
      !sym(s->lib, "ncclGetErrorString", &s->errstr)) {
    *err = "NCCL symbols not found";
    delete s;
    return FRAM_ERR_NCCL;
  }
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  ncclResult_t r = s->init(&s->comm, world, uid, rank);
  if (r != ncclSuccess) {
    fram_status st = nccl_fail(s, r, "ncclCommInitRank", err);
    delete s;
    return st;
  }
  *out = s;
  return FRAM_OK;
}

void shard_destroy(ShardCtx* s) {
  if (!s) return;
  if (s->comm && s->destroy) s->destroy(s->comm);
  delete s;
}

int shard_rank(const ShardCtx* s) { return s->rank; }
int shard_world(const ShardCtx* s) { return s->world; }
bool shard_is_virtual(const ShardCtx* s) { return s->vg != nullptr; }

namespace {
constexpr int kVMax = 16;
template <typename T>
struct VSrc { const T* p[kVMax]; };
template <typename T, bool MAX>
__global__ void vreduce_kernel(T* out, VSrc<T> src, int W, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    T acc = src.p[0][i];
    for (int k = 1; k < W; ++k) acc = MAX ? (src.p[k][i] > acc ? src.p[k][i] : acc) : acc + src.p[k][i];   // rank order
    out[i] = acc;
  }
}

template <typename Launch>
fram_status vcollective(ShardCtx* s, const void* send, void* recv, cudaStream_t st, std::string* err, Launch launch) {
  VGroup* g = s->vg;
  const int r = s->rank;
  g->send[r] = send;
  g->recv[r] = recv;
  cudaError_t e = cudaEventRecord(g->ev_ready[r], st);
  if (e != cudaSuccess || !g->barrier()) { g->abort(); *err = "virtual collective aborted"; return FRAM_ERR_NCCL; }
  for (int k = 0; k < g->W; ++k) cudaStreamWaitEvent(st, g->ev_ready[k], 0);
  launch();
  e = cudaEventRecord(g->ev_done[r], st);
  if (e != cudaSuccess || !g->barrier()) { g->abort(); *err = "virtual collective aborted"; return FRAM_ERR_NCCL; }
  for (int k = 0; k < g->W; ++k) cudaStreamWaitEvent(st, g->ev_done[k], 0);
  e = cudaGetLastError();
  if (e != cudaSuccess) { g->abort(); *err = std::string("virtual collective: ") + cudaGetErrorString(e); return FRAM_ERR_CUDA; }
  return FRAM_OK;
}

template <typename T>
fram_status vallreduce(ShardCtx* s, const T* send, T* recv, size_t count, bool max, cudaStream_t st, std::string* err) {
  return vcollective(s, send, recv, st, err, [&] {
    VSrc<T> src{};
    for (int k = 0; k < s->vg->W; ++k) src.p[k] = static_cast<const T*>(s->vg->send[k]);
    const unsigned blocks = (unsigned)std::min<size_t>((count + 255) / 256, 1024);
    if (max) vreduce_kernel<T, true><<<blocks, 256, 0, st>>>(recv, src, s->vg->W, count);
    else vreduce_kernel<T, false><<<blocks, 256, 0, st>>>(recv, src, s->vg->W, count);
  });
}
}  // namespace

VGroup* vgroup_create(int W, std::string* err) {
  if (W < 1 || W > kVMax) { *err = "virtual group size must be in [1, 16]"; return nullptr; }
  VGroup* g = new VGroup();
  g->W = W;
  g->send.assign(W, nullptr);
  g->recv.assign(W, nullptr);
  g->ev_ready.assign(W, nullptr);
  g->ev_done.assign(W, nullptr);
  for (int k = 0; k < W; ++k)
    if (cudaEventCreateWithFlags(&g->ev_ready[k], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->ev_done[k], cudaEventDisableTiming) != cudaSuccess) {
      *err = "event create failed";
      vgroup_destroy(g);
      return nullptr;
    }
  return g;
}

void vgroup_destroy(VGroup* g) {
  if (!g) return;
  for (auto e : g->ev_ready) if (e) cudaEventDestroy(e);
  for (auto e : g->ev_done) if (e) cudaEventDestroy(e);
  delete g;
}

void vgroup_abort(VGroup* g) { if (g) g->abort(); }

void vgroup_reset(VGroup* g) {                 // before a solve: no rank is inside a collective
  std::lock_guard<std::mutex> lk(g->mu);
  g->aborted = false;
  g->arrived = 0;
}

fram_status shard_create_virtual(ShardCtx** out, VGroup* g, int rank) {
  ShardCtx* s = new ShardCtx();
  s->vg = g;
  s->rank = rank;
  s->world = g->W;
  *out = s;
  return FRAM_OK;
}

fram_status shard_allreduce_f64(ShardCtx* s, const double* send, double* recv, size_t count, bool max,
                                cudaStream_t st, std::string* err) {
  if (s->vg) return vallreduce<double>(s, send, recv, count, max, st, err);
  ncclResult_t r = s->allreduce(send, recv, count, ncclFloat64, max ? ncclMax : ncclSum, s->comm, st);
  return r == ncclSuccess ? FRAM_OK : nccl_fail(s, r, "ncclAllReduce", err);
}

fram_status shard_allreduce_u64_max(ShardCtx* s, const uint64_t* send, uint64_t* recv, size_t count,
                                    cudaStream_t st, std::string* err) {
  if (s->vg) return vallreduce<unsigned long long>(s, reinterpret_cast<const unsigned long long*>(send),
                                                   reinterpret_cast<unsigned long long*>(recv), count, true, st, err);
  ncclResult_t r = s->allreduce(send, recv, count, ncclUint64, ncclMax, s->comm, st);
  return r == ncclSuccess ? FRAM_OK : nccl_fail(s, r, "ncclAllReduce", err);
}

fram_status shard_allgather_bytes(ShardCtx* s, const void* send, void* recv, size_t bytes_per_rank,
                                  cudaStream_t st, std::string* err) {
  if (s->vg)
    return vcollective(s, send, recv, st, err, [&] {       // rank k's block → recv[k·bytes, (k+1)·bytes)
      for (int k = 0; k < s->vg->W; ++k)
        cudaMemcpyAsync(static_cast<char*>(recv) + (size_t)k * bytes_per_rank, s->vg->send[k], bytes_per_rank,
                        cudaMemcpyDeviceToDevice, st);
    });
  ncclResult_t r = s->allgather(send, recv, bytes_per_rank, ncclUint8, s->comm, st);
  return r == ncclSuccess ? FRAM_OK : nccl_fail(s, r, "ncclAllGather", err);
}

}  // namespace fram
