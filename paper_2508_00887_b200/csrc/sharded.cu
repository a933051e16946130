// sharded.cu — NCCL plumbing for row-sharded solves.  NCCL is dlopen'ed so that the
// library loads on machines without it; only the sharded entry points need it.
#include <dlfcn.h>
#include <string.h>
#include <string>
#include "sharded.h"

namespace fram {

struct ShardCtx {
  void* lib = nullptr;
  void* comm = nullptr;
  int rank = 0, world = 1;
};

namespace {
typedef int (*GetUniqueIdFn)(void*);
void* open_nccl(std::string* err) {
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    void* h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (h) return h;
  }
  *err = std::string("cannot dlopen libnccl.so.2: ") + (dlerror() ? dlerror() : "");
  return nullptr;
}
}  // namespace

fram_status shard_unique_id(uint8_t id[128], std::string* err) {
  void* lib = open_nccl(err);
  if (!lib) return FRAM_ERR_NCCL;
  auto fn = reinterpret_cast<GetUniqueIdFn>(dlsym(lib, "ncclGetUniqueId"));
  if (!fn) { *err = "ncclGetUniqueId not found"; return FRAM_ERR_NCCL; }
  if (fn(id) != 0) { *err = "ncclGetUniqueId failed"; return FRAM_ERR_NCCL; }
  return FRAM_OK;
}

fram_status shard_create(ShardCtx** out, const uint8_t id[128], int rank, int world, std::string* err) {
  (void)id; (void)rank; (void)world;
  *out = nullptr;
  *err = "sharded solves are not implemented in this build";
  return FRAM_ERR_USAGE;
}

void shard_destroy(ShardCtx* s) { delete s; }

}  // namespace fram
