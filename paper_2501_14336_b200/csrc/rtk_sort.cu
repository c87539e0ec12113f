// rtk_sort.cu — ordering and gather of the candidate sets (K5), planned on the device.
//
// After k_compact every row holds m >= k candidate composites K (all K >= T). The reference
// returns the k best in canonical order (normalize_result, engine.hpp:402-420). Here:
//
//   k_plan_rows    one thread per row: m <= kSortCap -> one sort group; m larger -> an MSD
//                  segment; count < k or overflow -> flag the row for the exact path.
//   k_seg_hist     2048-bin histogram of one 11-bit digit per active segment.
//   k_seg_plan     one CTA per segment: descending bucket offsets (block scan), the rank cut
//                  at k (buckets starting at rank >= k are dropped), buckets packed into
//                  CTA-sized sort groups, oversized buckets queued for a deeper level.
//   k_seg_scatter  moves kept elements into bucket order (one global atomic per
//                  (tile, bucket), slots handed out from shared memory).
//   k_sort_groups  persistent CTAs pull groups from a device work counter, bitonic-sort
//                  them in shared memory and write ranks < k as (value, u64 index).
//
// The host only reads two flags after the final synchronisation; deeper MSD levels and
// the exact path run only when a flag asks for them.
#include <cuda_runtime.h>

#include "rtk_device.cuh"
#include "rtk_kernels.h"
#include "rtk_plan.cuh"

namespace rtk_b200 {

// ---- k_seg_hist ---------------------------------------------------------------------------
// Tiles are laid out over per-slot UPPER BOUNDS (tile_start, host-known); each tile reads the
// slot's actual length from device memory and exits when past it.
__device__ __forceinline__ int slot_of_tile(const uint64_t* tile_start, int n, uint64_t t) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (tile_start[mid] <= t) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// ---- k_seg_plan ---------------------------------------------------------------------------
// One CTA (256 threads x 8 bins, thread 0 owns the top bins) per slot. Bucket classes, in
// descending digit order over the kept prefix (first rank < k):
//   big   (> kSortCap elements)              -> queued as a slot of the next MSD level
//   solo  (kGroupPack < c <= kSortCap)       -> its own sort group
//   small (<= kGroupPack)                    -> packed with its neighbours while their starts
//                                               stay in one kGroupPack quantum (group <= 2Q)
// A group ends at the next boundary (group start or big bucket) or at the kept end.
__device__ void seg_plan_block(int j, const SegSlot& sl, const SegPlanArgs& a) {
    constexpr int per = kBins / kThreads;
    constexpr uint32_t INF = 0xffffffffu;
    __shared__ unsigned long long s_warp[32];
    __shared__ uint32_t s_wmin[kThreads / 32];
    __shared__ uint32_t s_kept_end;
    if (sl.len == 0) return;  // block-uniform
    uint32_t* ghist = a.ghist;
    uint32_t* gcursor = a.gcursor;
    const uint64_t* row_k = a.row_k;
    uint32_t* bstart = a.bstart;
    const GroupList& groups = a.groups;
    const uint32_t dst_buf = a.dst_buf;
    const SlotList& next = a.next;
    uint32_t* flags = a.flags;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t* h = ghist + static_cast<uint64_t>(j) * kBins;
    uint32_t* bs = bstart + static_cast<uint64_t>(j) * kBins;
    uint32_t* gc = gcursor + static_cast<uint64_t>(j) * kBins;
    uint32_t c[per];
    uint32_t sum = 0;
#pragma unroll
    for (int i = 0; i < per; ++i) {
        const int b = kBins - 1 - (tid * per + i);
        c[i] = __ldcg(h + b);
        h[b] = 0;   // histogram is left zeroed for the next level / call
        gc[b] = 0;  // scatter cursors start at zero
        sum += c[i];
    }
    unsigned long long tot;
    const uint32_t before = static_cast<uint32_t>(block_excl_scan(sum, s_warp, &tot));
    const uint64_t kr = row_k[sl.rid];
    uint32_t start[per];
    uint8_t cls[per];  // 0 dropped/empty, 1 small, 2 solo, 3 big
    uint32_t s = before;
    uint32_t kept_end_local = 0;
#pragma unroll
    for (int i = 0; i < per; ++i) {
        start[i] = s;
        const bool kept = c[i] && sl.rank_base + s < kr;
        cls[i] = !kept ? 0 : (c[i] > kSortCap ? 3 : (c[i] > kGroupPack ? 2 : 1));
        if (kept) kept_end_local = s + c[i];
        s += c[i];
    }
    // previous kept bucket (start, solo-or-big) via an exclusive max-scan in bucket order
    unsigned long long last = 0;
#pragma unroll
    for (int i = 0; i < per; ++i)
        if (cls[i]) last = (static_cast<unsigned long long>(start[i]) + 1) << 1 | (cls[i] >= 2 ? 1 : 0);
    unsigned long long prev;
    {
        unsigned long long v = last;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long o = __shfl_up_sync(0xffffffffu, v, d);
            if (lane >= d) v = max(v, o);
        }
        const unsigned long long ex = __shfl_up_sync(0xffffffffu, v, 1);
        __syncthreads();
        if (lane == 31) s_warp[warp] = v;
        __syncthreads();
        unsigned long long wpre = 0;
        for (int w = 0; w < warp; ++w) wpre = max(wpre, s_warp[w]);
        prev = max(wpre, lane ? ex : 0ull);
    }
    // boundaries (group starts + big buckets) and the kept end
    bool bnd[per], gst[per];
    uint32_t first_bnd = INF;
    {
        unsigned long long pv = prev;
#pragma unroll
        for (int i = 0; i < per; ++i) {
            gst[i] = false;
            bnd[i] = false;
            if (!cls[i]) continue;
            const bool has_prev = pv != 0;
            const uint32_t pstart = has_prev ? static_cast<uint32_t>((pv >> 1) - 1) : 0;
            const bool pbreak = has_prev && (pv & 1);
            if (cls[i] == 3) {
                bnd[i] = true;
            } else if (cls[i] == 2 || !has_prev || pbreak || start[i] / kGroupPack != pstart / kGroupPack) {
                gst[i] = bnd[i] = true;
            }
            if (bnd[i] && first_bnd == INF) first_bnd = start[i];
            pv = (static_cast<unsigned long long>(start[i]) + 1) << 1 | (cls[i] >= 2 ? 1 : 0);
        }
    }
    // kept end = max over threads; next boundary after this thread = suffix-min of first_bnd
    uint32_t ke = kept_end_local, sm = first_bnd;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) ke = max(ke, __shfl_xor_sync(0xffffffffu, ke, d));
    uint32_t suf = sm;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_down_sync(0xffffffffu, suf, d);
        if (lane + d < 32) suf = min(suf, o);
    }
    const uint32_t suf_ex_lane = __shfl_down_sync(0xffffffffu, suf, 1);
    if (tid == 0) s_kept_end = 0;
    __syncthreads();
    if (lane == 0) s_wmin[warp] = suf;
    if (lane == 0) atomicMax(&s_kept_end, ke);
    __syncthreads();
    uint32_t after = lane < 31 ? suf_ex_lane : INF;
    for (int w = warp + 1; w < kThreads / 32; ++w) after = min(after, s_wmin[w]);
    const uint32_t kept_end = s_kept_end;

    // emit: bucket starts for the scatter, groups, next-level slots
#pragma unroll
    for (int i = 0; i < per; ++i) {
        const int b = kBins - 1 - (tid * per + i);
        bs[b] = cls[i] ? start[i] : ~0u;
        if (cls[i] == 3) {
            const uint32_t q = atomicAdd(next.count, 1u);
            if (q < next.cap)
                next.slots[q] = SegSlot{sl.off + start[i], c[i], sl.rank_base + start[i], sl.rid,
                                        sl.pos >= kDigit ? sl.pos - kDigit : 0u};
            atomicOr(flags, kFlagMore);
        } else if (gst[i]) {
            uint32_t end = INF;
#pragma unroll
            for (int i2 = 0; i2 < per; ++i2)
                if (i2 > i && bnd[i2] && end == INF) end = start[i2];
            if (end == INF) end = after;
            if (end == INF || end > kept_end) end = kept_end;
            const uint32_t g = atomicAdd(groups.count, 1u);
            if (g < groups.cap)
                groups.groups[g] = SortGroup{sl.off + start[i], end - start[i], sl.rid,
                                             dst_buf, 0, sl.rank_base + start[i]};
            else
                atomicOr(flags, kFlagOverflow);
        }
    }
}

__global__ void __launch_bounds__(kThreads) k_seg_hist(const SegSlot* slots, int nslots,
                                                       const uint64_t* tile_start,
                                                       const uint64_t* src, SegPlanArgs pa) {
    __shared__ uint32_t h[kBins];
    __shared__ int s_last;
    for (int b = threadIdx.x; b < kBins; b += kThreads) h[b] = 0;
    __syncthreads();
    const uint64_t ntiles = tile_start[nslots];
    int cur = -1;
    uint32_t mine = 0;
    SegSlot sl{};
    // flush this CTA's histogram of slot j; the CTA that completes the slot's last tile runs
    // the bucket plan for it (k_seg_plan fused: no extra launch, no host round trip)
    auto finish_slot = [&](int j) {
        __syncthreads();
        for (int b = threadIdx.x; b < kBins; b += kThreads)
            if (h[b]) { atomicAdd(pa.ghist + static_cast<uint64_t>(j) * kBins + b, h[b]); h[b] = 0; }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t tiles = static_cast<uint32_t>(tile_start[j + 1] - tile_start[j]);
            const uint32_t old = atomicAdd(pa.ticket + j, mine);
            s_last = old + mine == tiles;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            seg_plan_block(j, sl, pa);
        }
        __syncthreads();
    };
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int j = slot_of_tile(tile_start, nslots, t);
        if (j != cur) {
            if (cur >= 0) finish_slot(cur);
            cur = j;
            mine = 0;
            sl = slots[j];
        }
        ++mine;
        const uint32_t lead = static_cast<uint32_t>(sl.off & 3);
        const uint64_t span_len = sl.len ? sl.len + lead : 0;
        const uint64_t e0 = (t - tile_start[j]) * kTile64;
        if (e0 >= span_len) continue;
        uint64_t v[4][kVec64];
        load_u64_tile(src + sl.off - lead, span_len, lead, e0, v);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int i = 0; i < kVec64; ++i) {
                const uint64_t q = e0 + static_cast<uint64_t>(u * kThreads + threadIdx.x) * kVec64 + i;
                hist_add_spread(h, static_cast<uint32_t>(v[u][i] >> sl.pos) & (kBins - 1), q >= lead && q < span_len);
            }
    }
    if (cur >= 0) finish_slot(cur);
}

// ---- k_seg_scatter ------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_seg_scatter(const SegSlot* slots, int nslots,
                                                          const uint64_t* tile_start,
                                                          const uint64_t* src, uint64_t* dst,
                                                          const uint32_t* bstart, uint32_t* gcursor) {
    __shared__ uint32_t h[kBins];
    __shared__ uint32_t base[kBins];
    const uint64_t ntiles = tile_start[nslots];
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int j = slot_of_tile(tile_start, nslots, t);
        const SegSlot sl = slots[j];
        const uint32_t lead = static_cast<uint32_t>(sl.off & 3);
        const uint64_t span_len = sl.len ? sl.len + lead : 0;
        const uint64_t e0 = (t - tile_start[j]) * kTile64;
        if (e0 >= span_len) continue;  // uniform across the CTA
        const uint32_t* bs = bstart + static_cast<uint64_t>(j) * kBins;
        uint32_t* gc = gcursor + static_cast<uint64_t>(j) * kBins;
        for (int b = threadIdx.x; b < kBins; b += kThreads) h[b] = 0;
        __syncthreads();
        uint64_t v[4][kVec64];
        uint32_t slot[4][kVec64];
        load_u64_tile(src + sl.off - lead, span_len, lead, e0, v);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int i = 0; i < kVec64; ++i) {
                const uint64_t q = e0 + static_cast<uint64_t>(u * kThreads + threadIdx.x) * kVec64 + i;
                const uint32_t d = static_cast<uint32_t>(v[u][i] >> sl.pos) & (kBins - 1);
                slot[u][i] = (q >= lead && q < span_len && bs[d] != ~0u) ? atomicAdd(&h[d], 1u) : ~0u;
            }
        __syncthreads();
        for (int b = threadIdx.x; b < kBins; b += kThreads)
            if (h[b]) base[b] = bs[b] + atomicAdd(gc + b, h[b]);
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int i = 0; i < kVec64; ++i) {
                if (slot[u][i] != ~0u) {
                    const uint32_t d = static_cast<uint32_t>(v[u][i] >> sl.pos) & (kBins - 1);
                    dst[sl.off + base[d] + slot[u][i]] = v[u][i];
                }
            }
        __syncthreads();
    }
}

// ---- k_sort_groups ------------------------------------------------------------------------
// Persistent CTAs (512 threads) pull groups of <= 4096 composites from a device work counter
// and sort them descending with an in-smem LSD radix sort (8-bit digits) over only the bits
// that differ inside the group. Warp w owns sequence positions [256w, 256w+256) in warp-
// striped order (item j of lane l at 256w + 32j + l); each pass ranks digits stably with one
// __match_any_sync per item and per-warp digit counters, scans the 16x256 counters
// (digit-major) and scatters. Padding positions (>= len) carry the lowest digit in every pass
// and therefore stay last. Then the gather: rank = rank_base + position; ranks < k are
// written as value bits (decoded from the key, or re-read from the original input for scaled
// runs, scaling.hpp:74-75) and the u64 row-local index (engine.hpp:106).
constexpr int kSortThreads = 256;
constexpr int kSortItems = kSortCap / kSortThreads;  // 8
static_assert(kSortItems == 8, "sort layout");

__global__ void __launch_bounds__(kSortThreads, 4) k_sort_groups(SortArgs g) {
    extern __shared__ unsigned long long buf[];  // kSortCap entries (dynamic: > 48 KB static)
    __shared__ uint32_t cnt[kSortThreads / 32][256];
    __shared__ uint32_t s_scan[kSortThreads / 32];
    __shared__ unsigned long long s_or[kSortThreads / 32];
    __shared__ uint32_t s_g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned full = 0xffffffffu;
    const unsigned lt = (1u << lane) - 1u;
    for (;;) {
        if (tid == 0) s_g = atomicAdd(g.work, 1u);
        __syncthreads();
        const uint32_t gi = s_g;
        if (gi >= min(*g.groups.count, g.groups.cap)) break;
        const SortGroup grp = g.groups.groups[gi];
        const uint32_t len = grp.len;
        const unsigned long long* src = (grp.buf ? g.buf1 : g.buf0) + grp.off;
        unsigned long long key[kSortItems];
        const unsigned long long ref = src[0];
        unsigned long long orv = 0;
#pragma unroll
        for (int j = 0; j < kSortItems; ++j) {
            const uint32_t p = warp * 256 + j * 32 + lane;
            key[j] = p < len ? src[p] : 0ull;
            if (p < len) orv |= key[j] ^ ref;
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) orv |= __shfl_xor_sync(full, orv, d);
        if (lane == 0) s_or[warp] = orv;
        __syncthreads();
        orv = 0;
        for (int w = 0; w < kSortThreads / 32; ++w) orv |= s_or[w];
        const int nbits = orv ? 64 - __clzll(orv) : 0;

        for (int lo = 0; lo < nbits; lo += 8) {
            if (((orv >> lo) & 0xFFull) == 0) continue;  // digit constant across the group
        if (((orv >> lo) & 0xFFull) == 0) continue;  // digit constant across the group: no-op pass
            for (int i = tid; i < (kSortThreads / 32) * 256; i += kSortThreads) (&cnt[0][0])[i] = 0;
            __syncthreads();
            uint32_t dig[kSortItems], rk[kSortItems];
#pragma unroll
            for (int j = 0; j < kSortItems; ++j) {
                const uint32_t p = warp * 256 + j * 32 + lane;
                // descending: rank by 255 - digit; padding always takes the last digit
                dig[j] = p < len ? 255u - static_cast<uint32_t>((key[j] >> lo) & 0xFFu) : 255u;
                const unsigned peers = __match_any_sync(full, dig[j]);
                const uint32_t base = cnt[warp][dig[j]];
                rk[j] = base + __popc(peers & lt);
                __syncwarp();
                if ((peers & lt) == 0) cnt[warp][dig[j]] = base + __popc(peers);
                __syncwarp();
            }
            __syncthreads();
            // exclusive scan over counters in (digit, warp) order: thread t -> digit t, all 8 warps
            {
                constexpr int NW = kSortThreads / 32;
                const int d = tid, w0 = 0;
                uint32_t c[NW], sum = 0;
#pragma unroll
                for (int i = 0; i < NW; ++i) { c[i] = cnt[w0 + i][d]; sum += c[i]; }
                uint32_t inc = sum;
#pragma unroll
                for (int dd = 1; dd < 32; dd <<= 1) {
                    const uint32_t o = __shfl_up_sync(full, inc, dd);
                    if (lane >= dd) inc += o;
                }
                if (lane == 31) s_scan[warp] = inc;
                __syncthreads();
                uint32_t pre = inc - sum;
                for (int w = 0; w < warp; ++w) pre += s_scan[w];
#pragma unroll
                for (int i = 0; i < NW; ++i) { cnt[w0 + i][d] = pre; pre += c[i]; }
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < kSortItems; ++j) buf[cnt[warp][dig[j]] + rk[j]] = key[j];
            __syncthreads();
#pragma unroll
            for (int j = 0; j < kSortItems; ++j) key[j] = buf[warp * 256 + j * 32 + lane];
            __syncthreads();
        }

        const uint32_t r = grp.rid;
        const uint64_t kr = g.row_k[r];
        const uint64_t oo = g.row_out_off[r];
#pragma unroll
        for (int j = 0; j < kSortItems; ++j) {
            const uint32_t p = warp * 256 + j * 32 + lane;
            const uint64_t rank = grp.rank_base + p;
            if (p >= len || rank >= kr) continue;
            const unsigned long long K = key[j];
            const uint32_t kk = static_cast<uint32_t>(K >> 32);
            const uint32_t idx = ~static_cast<uint32_t>(K);
            uint32_t val;
            if (g.gather) val = __ldg(g.in_base + g.row_in_off[r] + idx);
            else if (g.dtype == kF32) val = decode_f32_bits(kk, g.smallest);
            else val = g.smallest ? ~kk : kk;
            g.out_vals[oo + rank] = val;
            g.out_idx[oo + rank] = idx;
            if (rank == kr - 1 && g.pivots) g.pivots[r] = val;  // engine.hpp:333
        }
        __syncthreads();
    }
}

// ---- launchers ----------------------------------------------------------------------------
void launch_seg_hist(uint64_t tiles, const SegSlot* slots, int nslots, const uint64_t* tile_start,
                     const uint64_t* src, const SegPlanArgs& pa, cudaStream_t s) {
    const int grid = persistent_grid(k_seg_hist, kThreads, 0, tiles);
    k_seg_hist<<<grid, kThreads, 0, s>>>(slots, nslots, tile_start, src, pa);
}

void launch_seg_scatter(uint64_t tiles, const SegSlot* slots, int nslots, const uint64_t* tile_start,
                        const uint64_t* src, uint64_t* dst, const uint32_t* bstart, uint32_t* gcursor,
                        cudaStream_t s) {
    const int grid = persistent_grid(k_seg_scatter, kThreads, 0, tiles);
    k_seg_scatter<<<grid, kThreads, 0, s>>>(slots, nslots, tile_start, src, dst, bstart, gcursor);
}

void launch_sort_groups(uint32_t max_groups, const SortArgs& g, cudaStream_t s) {
    if (max_groups == 0) return;
    constexpr size_t smem = kSortCap * sizeof(unsigned long long);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_sort_groups, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        configured = true;
    }
    const int grid = persistent_grid(k_sort_groups, kSortThreads, smem, max_groups);
    k_sort_groups<<<grid, kSortThreads, smem, s>>>(g);
}

}  // namespace rtk_b200
