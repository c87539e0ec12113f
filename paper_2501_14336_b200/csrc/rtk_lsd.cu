// rtk_lsd.cu — dense rows (every general row unsampled with k >= n/2, e.g. LLM-vocab rows with
// k = vocab): the whole row is ordered, so the selection degenerates into a sort of
// (key desc, index asc) — normalize_result (engine.hpp:402-420) over all n elements. Here it is
// a segmented, stable, one-sweep LSD radix sort over all rows at once:
//
//   k_lsd_hist   one read of the input: per-row histograms of every 8-bit digit of the sort
//                key sk = ~key (ascending sk = descending key)
//   k_lsd_pass   per digit (4 for 32-bit keys, 2 for 16-bit keys, whose low half is constant):
//                4096-element tiles taken in row order from a tile counter; stable tile-local
//                ranks (ballot multisplit per warp), decoupled look-back over the row's earlier
//                tiles for the per-digit exclusive prefix, tile reordered by digit in shared
//                memory, coalesced write of each digit run. Pass 0 reads the input (key
//                transform fused, index = position); the last pass writes (value, u64 index) of
//                ranks < k straight into the output and the pivot.
//
// Stability + the initial index order give ties in ascending index order, the reference's
// tie rule. Stable warp ranks: each lane ORs its bit into a shared (warp, digit) mask and reads
// its peers back — one shared atomic per item instead of an 8-ballot multisplit (which measured
// 0.74 / 1.35 ms for bf16 / f32 C3 k = vocab against 0.66 / 1.21 ms). RTK_LSD=off selects the
// MSD + bucket-sort path (1.34 ms f32, 1.37 ms bf16), RTK_LSD=16 this path for 16-bit keys only.
// Traffic per element: 4 B (hist) + 4 B in / 8 B out (pass 0) + 16 B per middle pass + 8 B in /
// 12 B out (last pass) — against ~5 scattered passes of the MSD + bucket-sort path.
#include <cuda_runtime.h>

#include <algorithm>
#include <utility>

#include "rtk_device.cuh"
#include "rtk_kernels.h"

namespace rtk_b200 {

#ifndef RTK_LSD_THREADS
#define RTK_LSD_THREADS 256
#endif
constexpr int kLsdThreads = RTK_LSD_THREADS;  // >= 256: thread d < 256 owns digit d
constexpr int kLsdWarps = kLsdThreads / 32;
#ifndef RTK_LSD_ITEMS
#define RTK_LSD_ITEMS 16
#endif
#ifndef RTK_LSD_MINB
#define RTK_LSD_MINB 4
#endif
constexpr int kLsdItems = RTK_LSD_ITEMS;
constexpr int kLsdTile = kLsdThreads * kLsdItems;  // 4096 elements
constexpr int kLsdHistThreads = 512;
#ifndef RTK_LSD_LBW
#define RTK_LSD_LBW 1  // look-back window: predecessor words loaded per L2 round trip
#endif
#ifndef RTK_LSD_BALLOT
#define RTK_LSD_BALLOT 0
#endif
constexpr unsigned long long kLsdAgg = 1ull << 30, kLsdPrefix = 2ull << 30;

uint32_t lsd_tile() { return kLsdTile; }

__device__ __forceinline__ int lsd_row_of_tile(const LsdArgs& a, uint64_t t) {
    int lo = 0, hi = a.R - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.tile_start[mid] <= t) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Block-wide exclusive scan of one u32 per thread (kLsdThreads); *total = sum.
__device__ __forceinline__ uint32_t lsd_block_scan(uint32_t v, uint32_t* s_w, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    uint32_t pre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kLsdWarps; ++w) {
        const uint32_t x = s_w[w];
        if (w < warp) pre += x;
        tot += x;
    }
    __syncthreads();
    *total = tot;
    return pre + inc - v;
}

// ---- k_lsd_hist: CTA (j, c) histograms chunk c of row j for every pass digit -----------------
__global__ void __launch_bounds__(kLsdHistThreads) k_lsd_hist(LsdArgs a, uint32_t chunks) {
    __shared__ uint32_t h[4][kLsdHistThreads / 32 / 4][256];  // 4 digits x 4 warp groups
    resolve_src(a.in);
    const int j = blockIdx.x / chunks, c = blockIdx.x % chunks;
    const int warp = threadIdx.x >> 5;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(a.ctr + 4, 1u);  // this call's epoch
    for (int i = threadIdx.x; i < 4 * 4 * 256; i += kLsdHistThreads) (&h[0][0][0])[i] = 0;
    __syncthreads();
    const uint64_t n = a.len[j];
    const uint64_t e0 = n * c / chunks, e1 = n * (c + 1) / chunks;
    const uint64_t base = a.in_off[j];
    uint32_t* hg = &h[0][warp & 3][0];
    auto count = [&](uint32_t raw) {
        const uint32_t sk = ~make_key(a.in, raw);
#pragma unroll
        for (int p = 0; p < 4; ++p)
            if (p < a.npass) atomicAdd(hg + p * 4 * 256 + ((sk >> (a.shift0 + 8 * p)) & 255u), 1u);
    };
    // 16-byte loads over the aligned body (4 f32 / 8 half words each, 4 in flight per thread);
    // scalar head and tail
    const int EB = a.in.dtype == kF16 ? 2 : 4;
    const int VE = 16 / EB;
    const char* bytes = reinterpret_cast<const char*>(a.in.base) + (base + e0) * EB;
    const uint64_t mis = (reinterpret_cast<uintptr_t>(bytes) & 15) / EB;
    const uint64_t head = mis ? min(static_cast<uint64_t>(VE) - mis, e1 - e0) : 0;
    const uint64_t nvec = (e1 - e0 - head) / VE;
    for (uint64_t e = e0 + threadIdx.x; e < e0 + head; e += kLsdHistThreads) count(load_elem(a.in, base + e));
    const uint4* vp = reinterpret_cast<const uint4*>(bytes + head * EB);
    constexpr int U = 4;
    for (uint64_t v0 = 0; v0 < nvec; v0 += static_cast<uint64_t>(U) * kLsdHistThreads) {
        uint4 q[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t v = v0 + static_cast<uint64_t>(u) * kLsdHistThreads + threadIdx.x;
            if (v < nvec) q[u] = __ldcs(vp + v);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t v = v0 + static_cast<uint64_t>(u) * kLsdHistThreads + threadIdx.x;
            if (v >= nvec) continue;
            const uint32_t w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (EB == 2) {
                    count(w[i] & 0xFFFFu);
                    count(w[i] >> 16);
                } else {
                    count(w[i]);
                }
            }
        }
    }
    for (uint64_t e = e0 + head + nvec * VE + threadIdx.x; e < e1; e += kLsdHistThreads) count(load_elem(a.in, base + e));
    __syncthreads();
    for (int i = threadIdx.x; i < static_cast<int>(a.npass) * 256; i += kLsdHistThreads) {
        const int p = i >> 8, d = i & 255;
        const uint32_t v = h[p][0][d] + h[p][1][d] + h[p][2][d] + h[p][3][d];
        if (v) {
            if (chunks == 1) a.hist[j * 1024 + i] = v;
            else atomicAdd(a.hist + j * 1024 + i, v);
        }
    }
}

// ---- k_lsd_pass -----------------------------------------------------------------------------
// SH: the digit's shift in the sort key (compile-time: one byte extract per item); FIRST:
// pass 0 (reads the input); LAST: writes the output
template <int SH, bool FIRST, bool LAST>
__global__ void __launch_bounds__(kLsdThreads, RTK_LSD_MINB) k_lsd_pass(LsdArgs a, uint32_t pass) {
    extern __shared__ unsigned long long s_tile[];  // kLsdTile
    __shared__ uint32_t s_cnt[kLsdWarps][256];
#if !RTK_LSD_BALLOT
    // peer masks live in the tile buffer, which is only written after the ranking
    uint32_t (*s_match)[256] = reinterpret_cast<uint32_t (*)[256]>(s_tile);
#endif
    __shared__ uint32_t s_gbase[256];
    __shared__ uint32_t s_w[kLsdWarps];
    __shared__ uint32_t s_t;
    resolve_src(a.in);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned full = 0xffffffffu;
    const unsigned lt = (1u << lane) - 1u;
    unsigned long long t_start = 0;
    if (a.trace && tid == 0) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_start));
    if (tid == 0) s_t = atomicAdd(a.ctr + pass, 1u);
    for (int i = tid; i < kLsdWarps * 256; i += kLsdThreads) {
        (&s_cnt[0][0])[i] = 0;
#if !RTK_LSD_BALLOT
        (&s_match[0][0])[i] = 0;
#endif
    }
    __syncthreads();
    const uint64_t t = a.order ? a.order[s_t] : s_t;  // row-major tile id
    unsigned long long* tr = a.trace ? a.trace + (static_cast<uint64_t>(pass) * a.tile_start[a.R] + t) * 8 : nullptr;
    int ntr = 1;
    auto stamp = [&]() {
        if (tr && tid == 0) {
            unsigned long long x;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(x));
            tr[ntr++] = x;
        }
    };
    if (tr && tid == 0) {
        tr[0] = t_start;
        uint32_t sm;
        asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
        tr[7] = sm;
    }
    const int j = lsd_row_of_tile(a, t);
    const uint64_t t0 = a.tile_start[j];
    const uint64_t n = a.len[j];
    const uint64_t e0 = (t - t0) * kLsdTile;
    const uint32_t cnt = static_cast<uint32_t>(n - e0 < kLsdTile ? n - e0 : kLsdTile);
    const uint32_t epoch = *reinterpret_cast<volatile uint32_t*>(a.ctr + 4) * 4u + pass + 1u;
    const uint32_t hrow = tid < 256 ? __ldcg(a.hist + j * 1024 + pass * 256 + tid) : 0u;  // used after the look-back
    const bool full_tile = cnt == kLsdTile;
    (void)full_tile;
    (void)full;
    auto digit = [](unsigned long long K) { return (static_cast<uint32_t>(K >> 32) >> SH) & 255u; };

    // load: warp w owns tile elements [512w, 512w + 512), round i covers 32 consecutive ones
    unsigned long long c[kLsdItems];
    if (FIRST) {
        uint32_t raw[kLsdItems];
#pragma unroll
        for (int i = 0; i < kLsdItems; ++i) {
            const uint32_t e = warp * (kLsdItems * 32) + i * 32 + lane;
            raw[i] = e < cnt ? load_elem(a.in, a.in_off[j] + e0 + e) : 0u;
        }
#pragma unroll
        for (int i = 0; i < kLsdItems; ++i) {
            const uint32_t e = warp * (kLsdItems * 32) + i * 32 + lane;
            const uint32_t sk = ~make_key(a.in, raw[i]);
            c[i] = (static_cast<unsigned long long>(sk) << 32) | static_cast<uint32_t>(e0 + e);
        }
    } else {
        const unsigned long long* src = a.src + a.buf_off[j] + e0;
#pragma unroll
        for (int i = 0; i < kLsdItems; ++i) {
            const uint32_t e = warp * (kLsdItems * 32) + i * 32 + lane;
            c[i] = e < cnt ? __ldcs(src + e) : 0ull;
        }
    }
    // stable warp-local ranks in (round, lane) order
    uint32_t rk2[kLsdItems / 2];  // warp-local ranks (< 2^12), two per register
#pragma unroll
    for (int i = 0; i < kLsdItems; ++i) {
        const uint32_t e = warp * (kLsdItems * 32) + i * 32 + lane;
        const bool valid = e < cnt;
        const uint32_t d = digit(c[i]);
#if RTK_LSD_BALLOT == 1
        // ballot multisplit (8 ballots)
        unsigned peers = warp_peers8(d);
        if (!full_tile) peers &= __ballot_sync(full, valid);
#elif RTK_LSD_BALLOT == 2
        // one match.any per item (invalid lanes get unique keys)
        const unsigned peers = __match_any_sync(full, valid ? d : 256u + lane);
#else
        // peers through a shared-memory bitmask per (warp, digit): each lane ORs its bit in, reads
        // the mask back; the lowest peer clears it below (one shared atomic instead of 8 ballots)
        if (valid) atomicOr(&s_match[warp][d], 1u << lane);
        __syncwarp();
        const unsigned peers = valid ? s_match[warp][d] : 0u;
#endif
        const uint32_t b0 = s_cnt[warp][d];
        const uint32_t r = b0 + __popc(peers & lt);
        if (i & 1) rk2[i / 2] |= r << 16; else rk2[i / 2] = r;
        __syncwarp();
        if (valid && (peers & lt) == 0) {
            s_cnt[warp][d] = b0 + __popc(peers);
#if !RTK_LSD_BALLOT
            s_match[warp][d] = 0u;
#endif
        }
        __syncwarp();
    }
    __syncthreads();
    stamp();  // [1] loaded + ranked
    // thread d: warp offsets of digit d, the tile's count of d, look-back, bases
    const uint32_t d = tid;
    uint32_t tc = 0, excl = 0;
    if (kLsdThreads == 256 || d < 256) {
#pragma unroll
    for (int w = 0; w < kLsdWarps; ++w) {
        const uint32_t v = s_cnt[w][d];
        s_cnt[w][d] = tc;
        tc += v;
    }
    unsigned long long* st = a.status + t * 256 + d;
    const unsigned long long ep = static_cast<unsigned long long>(epoch) << 32;
    if (t == t0) {
        __stcg(st, ep | kLsdPrefix | tc);
    } else {
        __stcg(st, ep | kLsdAgg | tc);
        // windowed look-back: the next W predecessors' words are loaded at once (one L2 round
        // trip per window instead of per tile), then consumed nearest-first until a prefix
        constexpr int W = RTK_LSD_LBW;
        const long long first = static_cast<long long>(t0);
        long long q = static_cast<long long>(t) - 1;
        bool done = false;
        while (!done) {
            unsigned long long v[W];
#pragma unroll
            for (int w = 0; w < W; ++w)
                v[w] = q - w >= first ? *reinterpret_cast<volatile unsigned long long*>(a.status + (q - w) * 256 + d) : 0ull;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                if (done) continue;
                if (q - w < first) { done = true; continue; }
                while ((v[w] >> 32) != epoch)
                    v[w] = *reinterpret_cast<volatile unsigned long long*>(a.status + (q - w) * 256 + d);
                excl += static_cast<uint32_t>(v[w] & (kLsdAgg - 1));
                if (v[w] & kLsdPrefix) done = true;
            }
            q -= W;
        }
        __stcg(st, ep | kLsdPrefix | (excl + tc));  // flag and count in one 64-bit word: no fence
    }
    }
    if (tr && tid == 0) stamp();  // [2] own digit's look-back done (thread 0 = digit 0)
    uint32_t tot;
    const uint32_t rowbase = lsd_block_scan(hrow, s_w, &tot);
    const uint32_t dstart = lsd_block_scan(tc, s_w, &tot);
    // tile-sorted position q of digit d goes to row position q + (rowbase + excl - dstart)
    if (kLsdThreads == 256 || d < 256) {
        s_gbase[d] = rowbase + excl - dstart;
#pragma unroll
        for (int w = 0; w < kLsdWarps; ++w) s_cnt[w][d] += dstart;  // warp offsets -> tile positions
    }
    __syncthreads();
    stamp();  // [3] all look-backs + scans
    // reorder the tile by digit (stable) in shared memory
#pragma unroll
    for (int i = 0; i < kLsdItems; ++i) {
        const uint32_t e = warp * (kLsdItems * 32) + i * 32 + lane;
        if (e < cnt) {
            const uint32_t dd = digit(c[i]);
            s_tile[s_cnt[warp][dd] + ((rk2[i / 2] >> (16 * (i & 1))) & 0xFFFFu)] = c[i];
        }
    }
    __syncthreads();
    stamp();  // [4] reordered in smem
    // coalesced runs: tile-sorted position q -> row position gbase[d] + (q - dstart[d])
    if (!LAST) {
        unsigned long long* dst = a.dst + a.buf_off[j];
        for (uint32_t q = tid; q < cnt; q += kLsdThreads) {
            const unsigned long long K = s_tile[q];
            const uint32_t dd = digit(K);
            __stcs(dst + (s_gbase[dd] + q), K);
        }
        stamp();  // [5] stores issued
    } else {
        const uint64_t k = a.k[j], oo = a.out_off[j];
        for (uint32_t q = tid; q < cnt; q += kLsdThreads) {
            const unsigned long long K = s_tile[q];
            const uint32_t dd = digit(K);
            const uint64_t rank = s_gbase[dd] + q;
            if (rank >= k) continue;
            const uint32_t kv = ~static_cast<uint32_t>(K >> 32);
            const uint32_t idx = static_cast<uint32_t>(K);
            uint32_t val;
            if (a.in.scaled) val = load_elem(a.in, a.in_off[j] + idx);
            else if (a.in.dtype == kF32) val = decode_f32_bits(kv, a.in.smallest);
            else if (a.in.dtype == kF16) val = decode_f16_bits(kv, a.in.smallest);
            else val = a.in.smallest ? ~kv : kv;
            store_val(a.out_vals, a.in.dtype, oo + rank, val);
            a.out_idx[oo + rank] = idx;
            if (rank == k - 1 && a.pivots) store_val(a.pivots, a.in.dtype, a.rid[j], val);
        }
        call_tail(a.tail, &s_t);
    }
}

void launch_lsd(uint64_t tiles, const LsdArgs& a, cudaStream_t s) {
    const uint32_t chunks = static_cast<uint32_t>(
        std::max<int>(1, std::min<int>(64, (2 * num_sms() + a.R - 1) / a.R)));
    k_lsd_hist<<<a.R * chunks, kLsdHistThreads, 0, s>>>(a, chunks);
    for (uint32_t p = 0; p < a.npass; ++p) {
        LsdArgs b = a;
        if (p % 2 == 1) std::swap(b.src, b.dst);  // pass p reads what pass p-1 wrote
        if (p + 1 < a.npass) b.tail = CallTail{};
        const dim3 g(static_cast<unsigned>(tiles));
        const uint32_t sh = a.shift0 + 8 * p;
        const bool first = p == 0, last = p + 1 == a.npass;
        constexpr size_t sm = kLsdTile * sizeof(unsigned long long);
        static DeviceOnce configured;
        configured([&] {
            cudaFuncSetAttribute(k_lsd_pass<0, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
            cudaFuncSetAttribute(k_lsd_pass<8, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
            cudaFuncSetAttribute(k_lsd_pass<16, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
            cudaFuncSetAttribute(k_lsd_pass<16, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
            cudaFuncSetAttribute(k_lsd_pass<24, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
            cudaFuncSetAttribute(k_lsd_pass<24, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        });
        if (sh == 0) k_lsd_pass<0, true, false><<<g, kLsdThreads, sm, s>>>(b, p);
        else if (sh == 8) k_lsd_pass<8, false, false><<<g, kLsdThreads, sm, s>>>(b, p);
        else if (sh == 16 && first) k_lsd_pass<16, true, false><<<g, kLsdThreads, sm, s>>>(b, p);
        else if (sh == 16) k_lsd_pass<16, false, false><<<g, kLsdThreads, sm, s>>>(b, p);
        else if (last) k_lsd_pass<24, false, true><<<g, kLsdThreads, sm, s>>>(b, p);
        else k_lsd_pass<24, false, false><<<g, kLsdThreads, sm, s>>>(b, p);
    }
}

}  // namespace rtk_b200
