// sharded.h — row-sharded FRAM over W GPUs with NCCL; NCCL loaded at run time.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>
#include <string>
#include "../../include/fram.h"

namespace fram {
struct ShardCtx;
struct VGroup;                       // virtual shards: W ranks of one process on one GPU (tests)
VGroup* vgroup_create(int W, std::string* err);
void vgroup_destroy(VGroup* g);
void vgroup_abort(VGroup* g);
void vgroup_reset(VGroup* g);
fram_status shard_create_virtual(ShardCtx** out, VGroup* g, int rank);
fram_status shard_unique_id(uint8_t id[128], std::string* err);
fram_status shard_create(ShardCtx** out, const uint8_t id[128], int rank, int world, std::string* err);
void shard_destroy(ShardCtx* s);
int shard_rank(const ShardCtx* s);
int shard_world(const ShardCtx* s);
bool shard_is_virtual(const ShardCtx* s);
// collectives on `st` (enqueued, not synchronized)
fram_status shard_allreduce_f64(ShardCtx* s, const double* send, double* recv, size_t count, bool max,
                                cudaStream_t st, std::string* err);
fram_status shard_allreduce_u64_max(ShardCtx* s, const uint64_t* send, uint64_t* recv, size_t count,
                                    cudaStream_t st, std::string* err);
fram_status shard_allgather_bytes(ShardCtx* s, const void* send, void* recv, size_t bytes_per_rank,
                                  cudaStream_t st, std::string* err);
}  // namespace fram
