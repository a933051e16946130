// sharded.cu — NCCL plumbing for row-sharded solves.  NCCL is
// dlopen'ed (libnccl.so.2 — the one torch already loaded, if any) so that libfram loads on machines
// without it; only the sharded entry points need it.  nccl.h supplies the types only.
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>
#include <string>
#include "sharded.h"

namespace fram {

struct ShardCtx {
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

fram_status shard_allreduce_f64(ShardCtx* s, const double* send, double* recv, size_t count, bool max,
                                cudaStream_t st, std::string* err) {
  ncclResult_t r = s->allreduce(send, recv, count, ncclFloat64, max ? ncclMax : ncclSum, s->comm, st);
  return r == ncclSuccess ? FRAM_OK : nccl_fail(s, r, "ncclAllReduce", err);
}

fram_status shard_allreduce_u64_max(ShardCtx* s, const uint64_t* send, uint64_t* recv, size_t count,
                                    cudaStream_t st, std::string* err) {
  ncclResult_t r = s->allreduce(send, recv, count, ncclUint64, ncclMax, s->comm, st);
  return r == ncclSuccess ? FRAM_OK : nccl_fail(s, r, "ncclAllReduce", err);
}

fram_status shard_allgather_bytes(ShardCtx* s, const void* send, void* recv, size_t bytes_per_rank,
                                  cudaStream_t st, std::string* err) {
  ncclResult_t r = s->allgather(send, recv, bytes_per_rank, ncclUint8, s->comm, st);
  return r == ncclSuccess ? FRAM_OK : nccl_fail(s, r, "ncclAllGather", err);
}

}  // namespace fram
