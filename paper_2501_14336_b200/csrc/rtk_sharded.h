// rtk_sharded.h — n-sharded single query over an NCCL communicator (rtk_sharded.cpp).
#pragma once
#include <cstdint>

#include "rtk_engine.h"

namespace rtk_b200 {

// per-handle buffers of the sharded path: send slot, gathered slots, gap-closed copy
struct ShardWork {
    DevBuf send_v, send_i, recv_v, recv_i, cat_v, cat_i;
    void release();
};

void nccl_unique_id(void* out128);
void* nccl_comm_init(int nranks, const void* id128, int rank, int device);
void nccl_comm_destroy(void* comm);
void topk_sharded(Engine* const* engines, ShardWork* const* work, void* const* comms, int L,
                  const void* const* d_shards, const uint64_t* shard_n, int world, uint64_t k, int dtype,
                  int esize, int order, void* const* d_out_vals, uint64_t* const* d_out_idx,
                  void* const* d_out_pivots, void* const* streams);

}  // namespace rtk_b200
