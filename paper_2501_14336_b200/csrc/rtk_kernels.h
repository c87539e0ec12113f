// rtk_kernels.h — host-visible launchers of the sm_100a kernels (rtk_kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "rtk_device.cuh"

namespace rtk_b200 {

struct SortGroup {
    uint64_t off;        // element offset into SortGroups::buf
    uint32_t len;        // <= CAP
    uint32_t rid;        // state row
    uint64_t rank_base;  // output rank of the group's first element
};

struct SortGroups {
    const SortGroup* groups;
    const unsigned long long* buf;
    const uint64_t* row_k;
    const uint64_t* row_out_off;
    const uint64_t* row_in_off;   // gather mode only
    const uint32_t* in_base;      // gather mode only
    uint32_t* out_vals;
    uint64_t* out_idx;
    int gather;
    int dtype;
    int smallest;
};

void launch_init_sel(int R, const uint32_t* rid, const uint64_t* k, const uint64_t* target,
                     RowSel* sel, cudaStream_t s);
void launch_radix_pass(int src, uint64_t tiles, const Rows& rows, const InputSrc& in,
                       const uint64_t* buf, RowSel* sel, unsigned long long* ghist, cudaStream_t s);
void launch_sample_gather(uint64_t segments, const Rows& rows, const InputSrc& in,
                          const uint64_t* sample_off, const uint64_t* nseg_start, uint64_t* samples,
                          cudaStream_t s);
void launch_set_threshold(int R, const uint32_t* rid, const uint32_t* sampled, const RowSel* sel,
                          uint64_t* T, cudaStream_t s);
void launch_compact(uint64_t tiles, const Rows& rows, const InputSrc& in, const uint64_t* T,
                    uint64_t* cand, const uint64_t* cand_off, const uint64_t* cap,
                    unsigned long long* count, unsigned long long* kmin, unsigned long long* kmax,
                    cudaStream_t s);
void launch_seg_hist(uint64_t tiles, const Rows& segs, const uint32_t* pos, const uint64_t* src,
                     uint32_t* ghist, cudaStream_t s);
void launch_seg_scatter(uint64_t tiles, const Rows& segs, const uint32_t* pos, const uint64_t* src,
                        uint64_t* dst, const uint32_t* bstart, uint32_t* gcursor, cudaStream_t s);
void launch_sort_groups(int cap, int ngroups, const SortGroups& g, cudaStream_t s);
void launch_pivots(int R, const uint64_t* row_out_off, const uint64_t* row_k, const uint32_t* vals,
                   uint32_t* pivots, cudaStream_t s);
void launch_first_digit_hist(uint64_t tiles, const Rows& rows, const InputSrc& in, unsigned int d,
                             unsigned long long* ghist, cudaStream_t s);
void launch_remap_idx(uint64_t n, const uint64_t* cand_idx, uint32_t nblocks,
                      const uint64_t* block_start, const uint64_t* shard_base, uint64_t* idx,
                      cudaStream_t s);

}  // namespace rtk_b200
