// rtk_sharded.cpp — one huge query split over the ranks of an NCCL communicator (SURVEY §8e,
// BASELINE C5): local top-k of every shard (the single-device pipeline), ncclAllGather of the k
// (value, local index) candidates of every rank, final select over the G·k candidates on every
// rank (rtk_merge_shards' rule), global u64 indices.
//
// NCCL is opened at run time (dlopen "libnccl.so.2"): the library has no link-time dependency on
// it, and inside a PyTorch process the loader returns the libnccl torch already mapped, so
// communicators made here and torch's share one NCCL. Types come from the system <nccl.h>.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rtk_c.h"
#include "rtk_engine.h"
#include "rtk_sharded.h"

namespace rtk_b200 {

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.error = std::string("NCCL not available: ") + dlerror();
            return;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn && api.error.empty()) api.error = std::string("NCCL symbol missing: ") + name;
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.CommCount, "ncclCommCount");
        sym(api.CommUserRank, "ncclCommUserRank");
        sym(api.AllGather, "ncclAllGather");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.GetErrorString, "ncclGetErrorString");
    });
    if (!api.error.empty()) throw Error{RTK_INVALID_ARGUMENT, api.error};
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Error{RTK_CUDA_ERROR, std::string(what) + ": " + nccl().GetErrorString(r)};
}

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error{RTK_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e)};
}

}  // namespace

void nccl_unique_id(void* out128) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
}

void* nccl_comm_init(int nranks, const void* id128, int rank, int device) {
    const NcclApi& api = nccl();
    DeviceGuard dg(device);
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm = nullptr;
    nccl_check(api.CommInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
    return comm;
}

void nccl_comm_destroy(void* comm) {
    if (comm) nccl_check(nccl().CommDestroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
}

// Per local rank i: engines[i] on its device, comms[i] of `world` ranks. All local ranks take part
// in one grouped all-gather (the single-process multi-GPU form needs the group; with one process
// per GPU it is a plain all-gather).
void topk_sharded(Engine* const* engines, ShardWork* const* work, void* const* comms, int L,
                  const void* const* d_shards, const uint64_t* shard_n, int world, uint64_t k, int dtype,
                  int esize, int order, void* const* d_out_vals, uint64_t* const* d_out_idx,
                  void* const* d_out_pivots, void* const* streams) {
    const NcclApi& api = nccl();
    std::vector<uint64_t> base(world), kk(world);
    uint64_t n_total = 0, S = 0;
    for (int g = 0; g < world; ++g) {
        base[g] = n_total;
        n_total += shard_n[g];
        kk[g] = std::min(k, shard_n[g]);
        S = std::max(S, kk[g]);
    }
    if (n_total == 0) throw Error{RTK_EMPTY_INPUT, "topk_sharded: empty input"};
    if (k == 0 || k > n_total) throw Error{RTK_RANK_OUT_OF_RANGE, "topk_sharded: k outside [1, n]"};
    std::vector<int> rank(L);
    for (int i = 0; i < L; ++i) {
        int cnt = 0;
        nccl_check(api.CommCount(static_cast<ncclComm_t>(comms[i]), &cnt), "ncclCommCount");
        nccl_check(api.CommUserRank(static_cast<ncclComm_t>(comms[i]), &rank[i]), "ncclCommUserRank");
        if (cnt != world) throw Error{RTK_INVALID_ARGUMENT, "topk_sharded: communicator size != number of shards"};
    }
    if (world == 1) {  // one rank: the shard is the query, its top-k the result (no exchange)
        DeviceGuard dg(engines[0]->device());
        engines[0]->run(static_cast<const uint32_t*>(d_shards[0]), dtype, order, false, 0.0f, false,
                        {RowReq{0, shard_n[0], k, 0}}, static_cast<uint32_t*>(d_out_vals[0]), d_out_idx[0],
                        static_cast<uint32_t*>(d_out_pivots ? d_out_pivots[0] : nullptr),
                        static_cast<cudaStream_t>(streams ? streams[0] : nullptr));
        return;
    }
    // 1. local top-k of every local shard into its send slot (values | u64 local indices)
    for (int i = 0; i < L; ++i) {
        const int r = rank[i];
        DeviceGuard dg(engines[i]->device());
        ShardWork& w = *work[i];
        w.send_v.ensure(esize * std::max<uint64_t>(S, 1));
        w.send_i.ensure(8 * std::max<uint64_t>(S, 1));
        w.recv_v.ensure(esize * S * world);
        w.recv_i.ensure(8 * S * world);
        w.cat_v.ensure(esize * S * world);
        w.cat_i.ensure(8 * S * world);
        cudaStream_t s = static_cast<cudaStream_t>(streams ? streams[i] : nullptr);
        if (kk[r] > 0)
            engines[i]->run(static_cast<const uint32_t*>(d_shards[i]), dtype, order, false, 0.0f, false,
                            {RowReq{0, shard_n[r], kk[r], 0}}, w.send_v.as<uint32_t>(), w.send_i.as<uint64_t>(),
                            nullptr, s);
    }
    // 2. all-gather of the fixed-size candidate slots (S per rank) over NCCL
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (int i = 0; i < L; ++i) {
        DeviceGuard dg(engines[i]->device());
        ShardWork& w = *work[i];
        cudaStream_t s = static_cast<cudaStream_t>(streams ? streams[i] : nullptr);
        ncclComm_t c = static_cast<ncclComm_t>(comms[i]);
        nccl_check(api.AllGather(w.send_v.p, w.recv_v.p, S * esize, ncclUint8, c, s), "ncclAllGather");
        nccl_check(api.AllGather(w.send_i.p, w.recv_i.p, S, ncclUint64, c, s), "ncclAllGather");
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
    // 3. the rtk_merge_shards rule on every local rank: blocks in rank (= index) order, the
    //    candidate's position as the tie-break index, then remap to global indices
    std::vector<uint64_t> start(world);
    uint64_t total = 0;
    for (int g = 0; g < world; ++g) {
        start[g] = total;
        total += kk[g];
    }
    for (int i = 0; i < L; ++i) {
        DeviceGuard dg(engines[i]->device());
        ShardWork& w = *work[i];
        cudaStream_t s = static_cast<cudaStream_t>(streams ? streams[i] : nullptr);
        const void* cv = w.recv_v.p;
        const uint64_t* ci = w.recv_i.as<uint64_t>();
        if (total != S * static_cast<uint64_t>(world)) {  // short shards: close the slot gaps
            for (int g = 0; g < world; ++g) {
                if (!kk[g]) continue;
                cuda_ok(cudaMemcpyAsync(w.cat_v.as<char>() + start[g] * esize, w.recv_v.as<char>() + g * S * esize,
                                        kk[g] * esize, cudaMemcpyDeviceToDevice, s), "compact");
                cuda_ok(cudaMemcpyAsync(w.cat_i.as<uint64_t>() + start[g], w.recv_i.as<uint64_t>() + g * S, kk[g] * 8,
                                        cudaMemcpyDeviceToDevice, s), "compact");
            }
            cv = w.cat_v.p;
            ci = w.cat_i.as<uint64_t>();
        }
        engines[i]->run(static_cast<const uint32_t*>(cv), dtype, order, false, 0.0f, false, {RowReq{0, total, k, 0}},
                        static_cast<uint32_t*>(d_out_vals[i]), d_out_idx[i],
                        static_cast<uint32_t*>(d_out_pivots ? d_out_pivots[i] : nullptr), s);
        engines[i]->remap(k, ci, start, base, d_out_idx[i], s);
    }
}

void ShardWork::release() {
    for (DevBuf* b : {&send_v, &send_i, &recv_v, &recv_i, &cat_v, &cat_i}) b->release();
}

}  // namespace rtk_b200
