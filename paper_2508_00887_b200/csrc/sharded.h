// sharded.h — row-sharded FRAM over W GPUs with NCCL; NCCL loaded at run time.
#pragma once
#include <stdint.h>
#include <string>
#include "../../include/fram.h"

namespace fram {
struct ShardCtx;
fram_status shard_unique_id(uint8_t id[128], std::string* err);
fram_status shard_create(ShardCtx** out, const uint8_t id[128], int rank, int world, std::string* err);
void shard_destroy(ShardCtx* s);
}  // namespace fram
