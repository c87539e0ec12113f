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
#include <cooperative_groups.h>
#include <cstdlib>
#include <cstdio>
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
                                        sl.pos >= kDigit ? sl.pos - kDigit : 0u, kDigit, 0, 0, sl.base, sl.tz, sl.ib};
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
                hist_add_spread(h, static_cast<uint32_t>(slot_rel(sl, v[u][i]) >> sl.pos) & (kBins - 1), q >= lead && q < span_len);
            }
    }
    if (cur >= 0) finish_slot(cur);
}


// ---- level-0 MSD (upsweep / downsweep) -------------------------------------------------------
// One 2^bits-bin digit (11 or 13 bits) just below the common prefix of the row's candidates.
// k_msd_up: CTA (j, c) histograms chunk c of slot j in shared memory and stores it as row c of
// the slot's count matrix; the CTA that finishes the slot last turns the matrix columns into
// per-chunk offsets and plans the buckets (three sweeps over the totals in shared memory, block
// scans in between). k_msd_down: CTA (j, c) re-reads its chunk and scatters with shared-memory
// cursors seeded from its matrix row. No global atomics on the data path.
constexpr int kMsdThreads = 1024;
constexpr int kMsdWarps = kMsdThreads / 32;

// chunk c of G over m elements: [c*ch, min(m, (c+1)*ch)), ch a multiple of 4
__device__ __forceinline__ void msd_chunk(uint64_t m, uint32_t G, uint32_t c, uint64_t& e0, uint64_t& e1) {
    const uint64_t ch = ((m + G - 1) / G + 3) & ~uint64_t(3);
    e0 = min(m, c * ch);
    e1 = min(m, e0 + ch);
}

__device__ __forceinline__ unsigned long long msd_timer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Visit the composites of [e0, e1) (32-byte aligned start): f(K, valid) for every lane slot,
// 2 x 32-byte loads per thread in flight, block-uniform trip count (warp collectives allowed).
template <typename F>
__device__ __forceinline__ void msd_stream(const uint64_t* p, uint64_t e0, uint64_t e1, F f) {
    constexpr uint64_t step = 2ull * kMsdThreads * kVec64;
    for (uint64_t base = e0; base < e1; base += step) {
        uint64_t v[2][kVec64];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const uint64_t e = base + (static_cast<uint64_t>(u) * kMsdThreads + threadIdx.x) * kVec64;
            if (e + kVec64 <= e1) {
                ldg256_u64(p + e, v[u]);
            } else {
#pragma unroll
                for (int i = 0; i < kVec64; ++i) v[u][i] = e + i < e1 ? __ldcg(p + e + i) : 0ull;
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int i = 0; i < kVec64; ++i) {
                const uint64_t e = base + (static_cast<uint64_t>(u) * kMsdThreads + threadIdx.x) * kVec64 + i;
                f(v[u][i], e < e1);
            }
    }
}

__device__ __forceinline__ void grid_barrier(uint32_t* ctr, uint32_t target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        uint32_t v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            if (v < target) __nanosleep(100);
        } while (v < target);
        __threadfence();
    }
    __syncthreads();
}

// Plan of this CTA's bucket slice [s0, s0 + slice) (totals tot[0, slice), shared memory), whose
// first (highest) bucket starts at rank `off` of the slot. tot becomes the bucket starts (~0 for
// empty or dropped buckets). Every kept bucket is one group: <= kWarpGroupMax -> warp group,
// <= kSortCap -> CTA group, larger -> next-level slot. emit == false: starts only.
__device__ void msd_plan_slice(const SegSlot& sl, uint32_t* tot, uint32_t slice, uint32_t off, bool emit,
                               const FineArgs& a) {
    __shared__ uint32_t s_w[kMsdWarps];
    __shared__ unsigned long long s_c[kMsdWarps];
    __shared__ uint32_t s_base[3];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned full = 0xffffffffu;
    const uint32_t nt = slice < kMsdThreads ? slice : kMsdThreads;
    const uint32_t per = slice / nt;
    const bool act = static_cast<uint32_t>(tid) < nt;
    const uint32_t lo = act ? slice - (tid + 1) * per : 0;  // descending: thread 0 owns the top buckets
    const uint64_t kr = a.row_k[sl.rid];
    const uint64_t krel = kr > sl.rank_base ? kr - sl.rank_base : 0;
    uint32_t sum = 0;
    if (act)
        for (uint32_t i = 0; i < per; ++i) sum += tot[lo + i];
    uint32_t inc = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(full, inc, d);
        if (lane >= d) inc += o;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    uint32_t before = off + inc - sum;
    for (int w = 0; w < warp; ++w) before += s_w[w];
    const bool dbg = a.dbg && blockIdx.x == 0 && tid == 0;
    if (dbg) a.dbg[10] = msd_timer();
    // classes of the kept buckets -> list positions
    uint32_t nw = 0, nc = 0, nb = 0;
    if (act) {
        uint32_t st = before;
        for (uint32_t i = per; i-- > 0;) {
            const uint32_t c = tot[lo + i];
            if (c && st < krel) {
                if (c <= kWarpGroupMax) ++nw; else if (c <= kSortCap) ++nc; else ++nb;
            }
            st += c;
        }
    }
    const unsigned long long c3 = static_cast<unsigned long long>(nw) | static_cast<unsigned long long>(nc) << 21 |
                                  static_cast<unsigned long long>(nb) << 42;
    unsigned long long ci = c3;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long o = __shfl_up_sync(full, ci, d);
        if (lane >= d) ci += o;
    }
    if (lane == 31) s_c[warp] = ci;
    __syncthreads();
    unsigned long long cpre = ci - c3, ctot = 0;
    for (int w = 0; w < kMsdWarps; ++w) {
        if (w < warp) cpre += s_c[w];
        ctot += s_c[w];
    }
    if (tid == 0 && emit) {
        const uint32_t tw = static_cast<uint32_t>(ctot & 0x1FFFFF), tc = static_cast<uint32_t>((ctot >> 21) & 0x1FFFFF),
                       tb = static_cast<uint32_t>(ctot >> 42);
        s_base[0] = tw ? atomicAdd(a.wgroups.count, tw) : 0;
        s_base[1] = tc ? atomicAdd(a.groups.count, tc) : 0;
        s_base[2] = tb ? atomicAdd(a.next.count, tb) : 0;
        if (tb) atomicOr(a.flags, kFlagMore);
    }
    __syncthreads();
    if (dbg) a.dbg[11] = msd_timer();
    uint32_t iw = s_base[0] + static_cast<uint32_t>(cpre & 0x1FFFFF);
    uint32_t ic = s_base[1] + static_cast<uint32_t>((cpre >> 21) & 0x1FFFFF);
    uint32_t ib = s_base[2] + static_cast<uint32_t>(cpre >> 42);
    bool overflow = false;
    if (act) {
        uint32_t st = before;
        for (uint32_t i = per; i-- > 0;) {
            const uint32_t c = tot[lo + i];
            const bool kept = c && st < krel;
            tot[lo + i] = kept ? st : ~0u;
            if (kept && emit) {
                const SortGroup gr{sl.off + st, c, sl.rid, 1u, 0u, sl.rank_base + st};
                if (c <= kWarpGroupMax) {
                    if (iw < a.wgroups.cap) a.wgroups.groups[iw] = gr; else overflow = true;
                    ++iw;
                } else if (c <= kSortCap) {
                    if (ic < a.groups.cap) a.groups.groups[ic] = gr; else overflow = true;
                    ++ic;
                } else {
                    if (ib < a.next.cap)
                        a.next.slots[ib] = SegSlot{sl.off + st, c, sl.rank_base + st, sl.rid,
                                                   sl.pos >= kDigit ? sl.pos - kDigit : 0u, kDigit, 0, 0, sl.base, sl.tz, sl.ib};
                    else
                        overflow = true;
                    ++ib;
                }
            }
            st += c;
        }
    }
    if (overflow) atomicOr(a.flags, kFlagOverflow);
    if (dbg) a.dbg[12] = msd_timer();
    __syncthreads();
}

// Level-0 MSD of the slots, one cluster (or, fa.Q > 1, Q co-resident clusters) per slot:
//  1 chunk histograms (shared memory)           2 intra-cluster column scan over DSMEM
//  3 [Q > 1: cluster totals -> global, grid barrier, cross-cluster column scan]
//  4 each CTA plans its bucket slice (slice offsets exchanged over DSMEM; only cluster 0 emits)
//  5 cursors = bucket start + cross-cluster + intra-cluster offset; scatter of the chunk
// Input elements [e0, e1) of a dense row as composites (key transform fused, index = position),
// 4 loads in flight per thread, block-uniform trip count.
template <typename F>
__device__ __forceinline__ void msd_stream_in(const InputSrc& in, uint64_t row_in_off, uint64_t e0, uint64_t e1,
                                              F f) {
    for (uint64_t base = e0; base < e1; base += 4ull * kMsdThreads) {
        uint32_t raw[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t e = base + static_cast<uint64_t>(u) * kMsdThreads + threadIdx.x;
            raw[u] = e < e1 ? load_elem(in, row_in_off + e) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t e = base + static_cast<uint64_t>(u) * kMsdThreads + threadIdx.x;
            const bool valid = e < e1;
            f(valid ? composite(make_key(in, raw[u]), e) : 0ull, valid);
        }
    }
}

__global__ void __launch_bounds__(kMsdThreads, 1) k_msd_cluster(const SegSlot* slots, const uint64_t* src,
                                                                uint64_t* dst, FineArgs fa) {
    namespace cg = cooperative_groups;
    resolve_src(fa.in);
    cg::cluster_group cluster = cg::this_cluster();
    // [0,B): counts -> intra-cluster offsets -> cursors; [B, B+slice): slice totals -> starts;
    // [B+slice, B+2 slice): cross-cluster offsets (Q > 1)
    extern __shared__ __align__(16) uint32_t sm[];
    __shared__ uint32_t s_ssum[16];
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const uint32_t CS = cluster.num_blocks();
    const uint32_t r = cluster.block_rank();
    const uint32_t cid = blockIdx.x / CS;
    const uint32_t Q = fa.Q;
    const uint32_t j = Q > 1 ? 0 : cid, q = Q > 1 ? cid : 0;
    pdl_trigger();  // k_sort_groups may launch now (it waits in griddepcontrol.wait)
    const SegSlot sl = slots[j];
    if (sl.len == 0) return;  // uniform over the cluster (and over the grid when Q > 1)
    const uint32_t B = 1u << sl.bits, dmask = B - 1;
    const uint32_t slice = B / CS, s0 = r * slice;
    uint32_t* h = sm;
    uint32_t* tot = sm + B;
    uint32_t* qoff = sm + B + slice;
    const bool dbg = fa.dbg && blockIdx.x == 0 && threadIdx.x == 0;
    if (dbg) fa.dbg[0] = msd_timer();
    for (uint32_t b = threadIdx.x; b < B; b += kMsdThreads) h[b] = 0;
    __syncthreads();
    uint64_t e0, e1;
    msd_chunk(sl.len, Q * CS, q * CS + r, e0, e1);
    const uint64_t* p = src + sl.off;
    auto hist_one = [&](unsigned long long K, bool valid) {
        const uint32_t d = static_cast<uint32_t>(slot_rel(sl, K) >> sl.pos) & dmask;
        const uint32_t d0 = __shfl_sync(full, d, 0);
        if (__all_sync(full, valid && d == d0)) {
            if (lane == 0) atomicAdd(h + d0, 32u);  // tie-heavy rows: one atomic per warp
        } else if (valid) {
            atomicAdd(h + d, 1u);
        }
    };
    if (sl.src) msd_stream_in(fa.in, sl.in_off, e0, e1, hist_one);  // dense row: no compaction
    else msd_stream(p, e0, e1, hist_one);
    cluster.sync();
    if (dbg) fa.dbg[1] = msd_timer();
    // 2: intra-cluster column scan of this CTA's slice through DSMEM
    for (uint32_t i = threadIdx.x; i < slice; i += kMsdThreads) {
        const uint32_t b = s0 + i;
        uint32_t v[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = c < static_cast<int>(CS) ? *cluster.map_shared_rank(h + b, c) : 0u;
        uint32_t run = 0;
#pragma unroll
        for (int c = 0; c < 16; ++c)
            if (c < static_cast<int>(CS)) {
                *cluster.map_shared_rank(h + b, c) = run;
                run += v[c];
            }
        tot[i] = run;
        if (Q > 1) fa.ctot[static_cast<uint64_t>(q) * B + b] = run;
    }
    if (Q > 1) {
        // 3: cross-cluster column scan (redundant per cluster: no second barrier)
        grid_barrier(fa.bar, fa.bar_target);
        if (dbg) fa.dbg[2] = msd_timer();
        // two consecutive buckets per thread, up to 32 clusters' rows loaded before use
        for (uint32_t i = threadIdx.x * 2; i < slice; i += kMsdThreads * 2) {
            uint2 pre = make_uint2(0, 0), all = make_uint2(0, 0);
            for (uint32_t q0 = 0; q0 < Q; q0 += 16) {
                uint2 v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u)
                    v[u] = q0 + u < Q ? __ldcg(reinterpret_cast<const uint2*>(fa.ctot + static_cast<uint64_t>(q0 + u) * B + s0 + i))
                                      : make_uint2(0, 0);
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    if (q0 + u < q) { pre.x += v[u].x; pre.y += v[u].y; }
                    all.x += v[u].x;
                    all.y += v[u].y;
                }
            }
            qoff[i] = pre.x;
            qoff[i + 1] = pre.y;
            tot[i] = all.x;
            tot[i + 1] = all.y;
        }
    }
    __syncthreads();
    // 4: slice sums -> slice offsets (descending digits: higher slices first), plan the slice
    {
        uint32_t part = 0;
        for (uint32_t i = threadIdx.x; i < slice; i += kMsdThreads) part += tot[i];
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) part += __shfl_xor_sync(full, part, d);
        __shared__ uint32_t s_part[kMsdWarps];
        if (lane == 0) s_part[threadIdx.x >> 5] = part;
        __syncthreads();
        if (threadIdx.x < CS) {
            uint32_t ssum = 0;
            for (int w = 0; w < kMsdWarps; ++w) ssum += s_part[w];
            *cluster.map_shared_rank(s_ssum + r, threadIdx.x) = ssum;  // publish to every CTA
        }
    }
    cluster.sync();
    if (dbg) fa.dbg[3] = msd_timer();
    uint32_t off = 0;
    for (uint32_t r2 = r + 1; r2 < CS; ++r2) off += s_ssum[r2];
    msd_plan_slice(sl, tot, slice, off, q == 0, fa);
    cluster.sync();
    if (dbg) fa.dbg[4] = msd_timer();
    // 5: cursors from the owners' bucket starts (+ cross-cluster offsets), 16-byte DSMEM reads
    for (uint32_t b = threadIdx.x * 4; b < B; b += kMsdThreads * 4) {
        const uint32_t ow = b / slice, i = b - ow * slice;  // slice is a multiple of 4
        const uint4 st = *reinterpret_cast<const uint4*>(cluster.map_shared_rank(tot + i, ow));
        const uint4 qo = Q > 1 ? *reinterpret_cast<const uint4*>(cluster.map_shared_rank(qoff + i, ow))
                               : make_uint4(0, 0, 0, 0);
        uint4 c = *reinterpret_cast<uint4*>(h + b);
        c.x = st.x == ~0u ? ~0u : st.x + qo.x + c.x;
        c.y = st.y == ~0u ? ~0u : st.y + qo.y + c.y;
        c.z = st.z == ~0u ? ~0u : st.z + qo.z + c.z;
        c.w = st.w == ~0u ? ~0u : st.w + qo.w + c.w;
        *reinterpret_cast<uint4*>(h + b) = c;
    }
    cluster.sync();  // owners' shared memory is read by everyone before anyone exits
    if (dbg) fa.dbg[5] = msd_timer();
    uint64_t* qd = dst + sl.off;
    auto scatter_one = [&](unsigned long long K, bool valid) {
        const uint32_t d = static_cast<uint32_t>(slot_rel(sl, K) >> sl.pos) & dmask;
        const uint32_t d0 = __shfl_sync(full, d, 0);
        if (__all_sync(full, valid && d == d0)) {  // tie-heavy: one shared atomic per warp
            if (h[d0] != ~0u) {                     // warp-uniform (dropped buckets stay ~0)
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(h + d0, 32u);
                base = __shfl_sync(full, base, 0);
                qd[base + lane] = K;
            }
        } else if (valid) {
            if (h[d] != ~0u) qd[atomicAdd(h + d, 1u)] = K;
        }
    };
    if (sl.src) msd_stream_in(fa.in, sl.in_off, e0, e1, scatter_one);
    else msd_stream(p, e0, e1, scatter_one);
    if (dbg) { fa.dbg[6] = msd_timer(); fa.dbg[31] = 7; }
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
                const uint32_t d = static_cast<uint32_t>(slot_rel(sl, v[u][i]) >> sl.pos) & (kBins - 1);
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
                    const uint32_t d = static_cast<uint32_t>(slot_rel(sl, v[u][i]) >> sl.pos) & (kBins - 1);
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
// shared peer-mask atomic per item and per-warp digit counters, scans the 16x256 counters
// (digit-major) and scatters. Padding positions (>= len) carry the lowest digit in every pass
// and therefore stay last. Then the gather: rank = rank_base + position; ranks < k are
// written as value bits (decoded from the key, or re-read from the original input for scaled
// runs, scaling.hpp:74-75) and the u64 row-local index (engine.hpp:106).
constexpr int kSortThreads = 256;
constexpr int kSortItems = kSortCap / kSortThreads;  // 8
static_assert(kSortItems == 8, "sort layout");

// Bitonic network (descending) over one warp's registers: element p = lane * IPL + e; strides
// < IPL compare inside the lane, larger ones across lanes (shuffles).
template <int IPL, typename T>
__device__ __forceinline__ void warp_bitonic_desc(T (&a)[IPL], int lane) {
    constexpr uint32_t N = 32 * IPL;
    const unsigned full = 0xffffffffu;
#pragma unroll
    for (uint32_t kk = 2; kk <= N; kk <<= 1) {
#pragma unroll
        for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
            if (jj < IPL) {
#pragma unroll
                for (int e = 0; e < IPL; ++e) {
                    if (e & jj) continue;
                    const bool desc = ((lane * IPL + e) & kk) == 0;
                    const T x = a[e], y = a[e + jj];
                    const T hi = max(x, y), lo = min(x, y);
                    a[e] = desc ? hi : lo;
                    a[e + jj] = desc ? lo : hi;
                }
            } else {
                const int lm = static_cast<int>(jj / IPL);
                const bool lower = (lane & lm) == 0;
#pragma unroll
                for (int e = 0; e < IPL; ++e) {
                    const bool desc = ((lane * IPL + e) & kk) == 0;
                    const T o = __shfl_xor_sync(full, a[e], lm);
                    a[e] = (lower == desc) ? max(a[e], o) : min(a[e], o);
                }
            }
        }
    }
}

__device__ __forceinline__ void emit_rank(const SortArgs& g, uint32_t r, uint64_t kr, uint64_t oo, uint64_t rank,
                                          uint32_t key, uint32_t idx) {
    uint32_t val;
    if (g.gather) val = __ldg(g.in_base + g.row_in_off[r] + idx);
    else if (g.dtype == kF32) val = decode_f32_bits(key, g.smallest);
    else if (g.dtype == kF16) val = decode_f16_bits(key, g.smallest);
    else val = g.smallest ? ~key : key;
    store_val(g.out_vals, g.dtype, oo + rank, val);
    g.out_idx[oo + rank] = idx;
    if (rank == kr - 1 && g.pivots) store_val(g.pivots, g.dtype, r, val);  // engine.hpp:333
}

// Sort one group of <= 32*IPL composites by one warp and write ranks < k as (value bits, u64
// index). When the group's keys span < 2^(32 - b) values and its indices fit b bits, the
// composite is packed order-preserving into 32 bits, ((key - kmin) << b) | (2^b - 1 - idx) >= 1
// (padding = 0 sorts last), halving the network's shuffles and compares.
template <int IPL>
__device__ __forceinline__ void warp_sort_group(const SortGroup& grp, const SortArgs& g, int lane) {
    const unsigned full = 0xffffffffu;
    const unsigned long long* src = (grp.buf ? g.buf1 : g.buf0) + grp.off;
    unsigned long long a[IPL];
    uint32_t kmin = ~0u, kmax = 0, imax = 0;
#pragma unroll
    for (int e = 0; e < IPL; ++e) {
        const uint32_t p = lane * IPL + e;
        a[e] = p < grp.len ? __ldcg(src + p) : 0ull;
        if (p < grp.len) {
            const uint32_t key = static_cast<uint32_t>(a[e] >> 32), idx = ~static_cast<uint32_t>(a[e]);
            kmin = min(kmin, key);
            kmax = max(kmax, key);
            imax = max(imax, idx);
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(full, kmin, d));
        kmax = max(kmax, __shfl_xor_sync(full, kmax, d));
        imax = max(imax, __shfl_xor_sync(full, imax, d));
    }
    const uint32_t r = grp.rid;
    const uint64_t kr = g.row_k[r];
    const uint64_t oo = g.row_out_off[r];
    const int ib = imax >= 0x7fffffffu ? 32 : 32 - __clz(imax + 1);  // bits of imax + 1
    if (ib < 32 && (kmax - kmin) < (1u << (32 - ib)) >> 0 && (static_cast<uint64_t>(kmax - kmin) << ib) < (1ull << 32)) {
        const uint32_t mask = (1u << ib) - 1u;
        uint32_t q[IPL];
#pragma unroll
        for (int e = 0; e < IPL; ++e) {
            const uint32_t p = lane * IPL + e;
            q[e] = p < grp.len ? ((static_cast<uint32_t>(a[e] >> 32) - kmin) << ib) | (mask - ~static_cast<uint32_t>(a[e]))
                               : 0u;
        }
        warp_bitonic_desc<IPL>(q, lane);
#pragma unroll
        for (int e = 0; e < IPL; ++e) {
            const uint32_t p = lane * IPL + e;
            const uint64_t rank = grp.rank_base + p;
            if (p >= grp.len || rank >= kr) continue;
            emit_rank(g, r, kr, oo, rank, kmin + (q[e] >> ib), mask - (q[e] & mask));
        }
    } else {
        warp_bitonic_desc<IPL>(a, lane);
#pragma unroll
        for (int e = 0; e < IPL; ++e) {
            const uint32_t p = lane * IPL + e;
            const uint64_t rank = grp.rank_base + p;
            if (p >= grp.len || rank >= kr) continue;
            emit_rank(g, r, kr, oo, rank, static_cast<uint32_t>(a[e] >> 32), ~static_cast<uint32_t>(a[e]));
        }
    }
}

// One CTA group (<= 256 * IT composites): in-smem LSD radix sort (see k_sort_groups), IT items
// per thread so the work follows the group size (512 / 1024 / 2048 slots).
template <int IT>
__device__ __forceinline__ void cta_sort_group(const SortGroup& grp, const SortArgs& g, unsigned long long* buf,
                                               uint32_t (*cnt)[256], uint32_t* s_scan, unsigned long long* s_or,
                                               uint32_t (*pmask)[256]) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned full = 0xffffffffu;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t len = grp.len;
    const unsigned long long* src = (grp.buf ? g.buf1 : g.buf0) + grp.off;
    unsigned long long key[IT];
    const unsigned long long ref = src[0];
    unsigned long long orv = 0;
#pragma unroll
    for (int j = 0; j < IT; ++j) {
        const uint32_t p = warp * (32 * IT) + j * 32 + lane;
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

    auto lsd = [&](int lo0) {
    for (int lo = lo0; lo < nbits; lo += 8) {
        if (((orv >> lo) & 0xFFull) == 0) continue;  // digit constant across the group: no-op pass
        for (int i = tid; i < (kSortThreads / 32) * 256; i += kSortThreads) {
            (&cnt[0][0])[i] = 0;
            (&pmask[0][0])[i] = 0;
        }
        __syncthreads();
        uint32_t dig[IT], rk[IT];
#pragma unroll
        for (int j = 0; j < IT; ++j) {
            const uint32_t p = warp * (32 * IT) + j * 32 + lane;
            // descending: rank by 255 - digit; padding always takes the last digit
            dig[j] = p < len ? 255u - static_cast<uint32_t>((key[j] >> lo) & 0xFFu) : 255u;
            // peers: each lane ORs its bit into the (warp, digit) mask and reads it back (one
            // shared atomic; __match_any_sync and 8-ballot multisplits measured slower)
            atomicOr(&pmask[warp][dig[j]], 1u << lane);
            __syncwarp();
            const unsigned peers = pmask[warp][dig[j]];
            const uint32_t base = cnt[warp][dig[j]];
            rk[j] = base + __popc(peers & lt);
            __syncwarp();
            if ((peers & lt) == 0) {
                cnt[warp][dig[j]] = base + __popc(peers);
                pmask[warp][dig[j]] = 0u;
            }
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
        for (int j = 0; j < IT; ++j) buf[cnt[warp][dig[j]] + rk[j]] = key[j];
        __syncthreads();
#pragma unroll
        for (int j = 0; j < IT; ++j) key[j] = buf[warp * (32 * IT) + j * 32 + lane];
        __syncthreads();
    }
    };
    // Real keys rarely tie: rank by the KEY bits only (3 passes instead of ~5 with the index
    // bits), then put tied keys back in index order with an odd-even transposition restricted
    // to runs of equal keys (a run of length L settles in <= L rounds). Long runs (tie-heavy
    // groups) fall back to the full composite passes.
    // 16-bit keys tie in runs of tens (65536 values over ~10^5 elements): full composite passes
    const bool key_only = g.dtype != kF16 && (orv >> 32) != 0 && (orv & 0xffffffffull) != 0;
    lsd(key_only ? 32 : 0);
    if (key_only) {
        bool prev_sw = true, settled = false;
        for (int it = 0; it < 24; ++it) {
            bool sw = false;
            for (uint32_t q = tid; 2 * q + 1 < len; q += kSortThreads) {
                const uint32_t p = 2 * q + (it & 1);
                if (p + 1 < len) {
                    const unsigned long long x = buf[p], y = buf[p + 1];
                    if ((x >> 32) == (y >> 32) && x < y) { buf[p] = y; buf[p + 1] = x; sw = true; }
                }
            }
            const bool any = __syncthreads_or(sw);
            if (!any && !prev_sw) { settled = true; break; }
            prev_sw = any;
        }
#pragma unroll
        for (int j = 0; j < IT; ++j) key[j] = buf[warp * (32 * IT) + j * 32 + lane];
        __syncthreads();
        if (!settled) lsd(0);  // tie-heavy group: full composite order
    }

    const uint32_t r = grp.rid;
    const uint64_t kr = g.row_k[r];
    const uint64_t oo = g.row_out_off[r];
#pragma unroll
    for (int j = 0; j < IT; ++j) {
        const uint32_t p = warp * (32 * IT) + j * 32 + lane;
        const uint64_t rank = grp.rank_base + p;
        if (p >= len || rank >= kr) continue;
        const unsigned long long K = key[j];
        const uint32_t kk = static_cast<uint32_t>(K >> 32);
        const uint32_t idx = ~static_cast<uint32_t>(K);
        emit_rank(g, r, kr, oo, rank, kk, idx);
    }
}

__global__ void __launch_bounds__(kSortThreads, 4) k_sort_groups(SortArgs g) {
    extern __shared__ unsigned long long buf[];  // kSortCap entries (dynamic: > 48 KB static)
    __shared__ uint32_t cnt[kSortThreads / 32][256];
    __shared__ uint32_t pmask[kSortThreads / 32][256];
    __shared__ uint32_t s_scan[kSortThreads / 32];
    __shared__ unsigned long long s_or[kSortThreads / 32];
    __shared__ uint32_t s_g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    pdl_wait();  // launched early (PDL) while the MSD kernel finishes
    for (;;) {
        if (tid == 0) s_g = atomicAdd(g.work, 1u);
        __syncthreads();
        const uint32_t gi = s_g;
        if (gi >= min(*g.groups.count, g.groups.cap)) break;
        const SortGroup grp = g.groups.groups[gi];
        if (grp.len <= 512) cta_sort_group<2>(grp, g, buf, cnt, s_scan, s_or, pmask);
        else if (grp.len <= 1024) cta_sort_group<4>(grp, g, buf, cnt, s_scan, s_or, pmask);
        else cta_sort_group<8>(grp, g, buf, cnt, s_scan, s_or, pmask);
        __syncthreads();
    }
    // warp groups (<= kWarpGroupMax composites): one warp each, bitonic in registers, no shared
    // memory, no block barriers; 2, 4 or 8 items per lane by group size
    // static striding over the list (groups are similar-sized; a shared work counter would
    // serialise thousands of same-address atomics); *wwork = first group of this launch
    const uint32_t wend = min(*g.wgroups.count, g.wgroups.cap);
    const uint32_t nwarps = gridDim.x * (kSortThreads / 32);
    for (uint32_t gi = *g.wwork + blockIdx.x * (kSortThreads / 32) + warp; gi < wend; gi += nwarps) {
        const SortGroup grp = g.wgroups.groups[gi];
        if (grp.len <= 64) warp_sort_group<2>(grp, g, lane);
        else if (grp.len <= 128) warp_sort_group<4>(grp, g, lane);
        else warp_sort_group<8>(grp, g, lane);
    }
    call_tail(g.tail, &s_g);
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

static size_t msd_smem(int cs) {
    // counts (2^14) + slice totals + cross-cluster offsets (2 x 2^14 / cs)
    return ((size_t(1) << kMsdMaxBits) + 2 * ((size_t(1) << kMsdMaxBits) / cs)) * sizeof(uint32_t);
}

static void msd_configure() {
    static DeviceOnce configured;
    configured([&] {
        cudaFuncSetAttribute(k_msd_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        cudaFuncSetAttribute(k_msd_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    });
}

int msd_max_clusters(int cs) {
    static std::atomic<int> cache_all[64][17];  // per device
    if (cs < 1 || cs > 16) return 1;
    int dev = 0;
    cudaGetDevice(&dev);
    std::atomic<int>* cache = cache_all[dev & 63];
    if (!cache[cs].load()) {
        msd_configure();
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(kMsdThreads);
        cfg.dynamicSmemBytes = msd_smem(cs);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k_msd_cluster, &cfg) != cudaSuccess) {
            cudaGetLastError();
            n = 1;
        }
        cache[cs].store(n > 0 ? n : 1);
    }
    return cache[cs].load();
}

bool launch_msd_cluster(int nslots, int cs, const SegSlot* slots, const uint64_t* src, uint64_t* dst,
                        const FineArgs& fa, cudaStream_t s) {
    if (nslots <= 0) return true;
    const size_t smem = msd_smem(cs);
    msd_configure();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((fa.Q > 1 ? fa.Q : nslots) * cs);
    cfg.blockDim = dim3(kMsdThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = fa.Q > 1 ? 2 : 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k_msd_cluster, slots, src, dst, fa);
    if (e != cudaSuccess && fa.Q > 1) {
        cudaGetLastError();  // refused (co-residency): caller relaunches with Q = 1
        if (fa.dbg) {
            int ncl = 0;
            cfg.numAttrs = 1;
            cudaOccupancyMaxActiveClusters(&ncl, k_msd_cluster, &cfg);
            fprintf(stderr, "[rtk] multi-cluster MSD refused: %s (max active clusters %d)\n", cudaGetErrorString(e), ncl);
        }
        return false;
    }
    return true;
}

void launch_sort_groups(uint32_t max_groups, const SortArgs& g, cudaStream_t s) {
    if (max_groups == 0) return;
    constexpr size_t smem = kSortCap * sizeof(unsigned long long);
    static DeviceOnce configured;
    configured([&] {
        cudaFuncSetAttribute(k_sort_groups, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    });
    const int grid = persistent_grid(k_sort_groups, kSortThreads, smem, max_groups);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kSortThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    static const bool no_pdl = [] {
        const char* e = std::getenv("RTK_NO_PDL_SORT");
        return e && *e && *e != '0';
    }();
    cfg.numAttrs = no_pdl ? 0 : 1;
    cudaLaunchKernelEx(&cfg, k_sort_groups, g);
}

}  // namespace rtk_b200
