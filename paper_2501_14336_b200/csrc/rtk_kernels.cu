// rtk_kernels.cu — sm_100a kernels of the B200 radix top-k (no tensor cores: the path has
// no dense contraction; every kernel here is HBM/L2/SMEM-bandwidth or atomic bound).
//
//   k_sample_gather   stratified sample of each row -> composite buffer          (K6/K7 aid)
//   k_radix_pass      one MSD digit pass: fused key transform + prefix filter +   (K1+K2+K3)
//                     smem histogram + grid merge + last-CTA bin select / early stop
//   k_compact         ONE streaming read of the input: fused key transform +     (K1+K4)
//                     threshold filter + flush-efficient smem staging
//   k_seg_hist / k_seg_scatter   MSD partition of large candidate sets            (K5 sort)
//   k_sort_groups     in-smem bitonic sort + gather of values/indices            (K5)
//   k_first_digit_hist  the adaptive-scaling trigger histogram                   (K7)
//
// Reference mapping: count_bins engine.hpp:177-222, select_bin :231-241, select_candidates
// :245-284 (+ WriteBuffer :138-169), radix_select :293-312, filter :318-398,
// normalize_result :402-420, scaled_topk scaling.hpp:42-78.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "rtk_device.cuh"
#include "rtk_kernels.h"
#include "rtk_plan.cuh"

namespace rtk_b200 {

__host__ __device__ __forceinline__ unsigned int digit_hi(unsigned int pos) {
    return pos == 53 ? 64u : (pos == 0 ? 9u : pos + 11u);
}
__host__ __device__ __forceinline__ unsigned int next_pos(unsigned int pos) {
    return pos == 9 ? 0u : pos - 11u;
}

// ----------------------------------------------------------------------------------------
// k_init_sel: reset selection state of launch rows. k_rem[j] = rank to select, target[j].
// ----------------------------------------------------------------------------------------
__global__ void k_init_sel(int R, const uint32_t* rid, const uint64_t* k, const uint64_t* target,
                           RowSel* sel) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= R) return;
    RowSel s;
    s.prefix = 0;
    s.k_rem = k[j];
    s.above = 0;
    s.T = 0;
    s.count_ge = 0;
    s.target = target[j];
    s.pos = 53;
    s.status = 0;
    s.ticket = 0;
    s.passes = 0;
    sel[rid[j]] = s;
}

// ----------------------------------------------------------------------------------------
// Bin selection (select_bin, engine.hpp:231-241) over the merged 2048-bin histogram of one
// row, executed by the last CTA of the pass. Bins are walked from the top digit down; the
// first bin whose cumulative count reaches k_rem is the pivot bin. Early stop: the row is
// resolved as soon as #{K >= T} <= target (target = k means "bucket count equals the
// remaining k", the paper's early exit; larger targets stop at a small candidate set).
// ----------------------------------------------------------------------------------------
__device__ void select_in_block(RowSel* sp, unsigned long long* gh) {
    __shared__ unsigned long long s_warp[32];
    __shared__ unsigned long long s_res[4];
    constexpr int per = kBins / kThreads;  // 8 bins per thread, thread 0 owns the top bins
    const int tid = threadIdx.x;
    unsigned long long c[per];
    unsigned long long sum = 0;
#pragma unroll
    for (int i = 0; i < per; ++i) {
        const int b = kBins - 1 - (tid * per + i);
        c[i] = __ldcg(gh + b);
        gh[b] = 0;  // ready for the next pass
        sum += c[i];
    }
    unsigned long long total;
    const unsigned long long before = block_excl_scan(sum, s_warp, &total);
    const unsigned long long k_rem = sp->k_rem;
    if (tid == 0) s_res[0] = ~0ull;
    __syncthreads();
    if (k_rem >= 1 && k_rem <= total && before < k_rem && before + sum >= k_rem) {
        unsigned long long cum = before;
#pragma unroll
        for (int i = 0; i < per; ++i) {
            if (cum + c[i] >= k_rem) {
                s_res[0] = static_cast<unsigned long long>(kBins - 1 - (tid * per + i));
                s_res[1] = cum;  // elements above the pivot bin inside the range
                s_res[2] = c[i];
                break;
            }
            cum += c[i];
        }
    }
    __syncthreads();
    if (tid == 0) {
        if (s_res[0] == ~0ull) {
            sp->status = 2;  // rank outside histogram total (select_bin throws)
        } else {
            const unsigned int pos = sp->pos;
            const unsigned long long bin = s_res[0];
            ++sp->passes;
            sp->prefix |= bin << pos;
            sp->above += s_res[1];
            sp->k_rem = k_rem - s_res[1];
            sp->T = sp->prefix;
            sp->count_ge = sp->above + s_res[2];
            if (sp->count_ge <= sp->target || pos == 0) sp->status = 1;
            else sp->pos = next_pos(pos);
        }
    }
}

// ----------------------------------------------------------------------------------------
// k_radix_pass<SRC>: one digit pass over every active row of the launch.
// SRC 0: the input (fused encode / scale, composite with the element index);
// SRC 1: a u64 composite buffer (samples or candidates).
// Per CTA: 2048-bin smem histogram of elements matching the row's prefix; one global merge
// per (CTA, row) (hierarchical atomics, engine.hpp:195-197); a per-row ticket elects the
// last CTA, which runs select_in_block — no host round trip between passes.
// ----------------------------------------------------------------------------------------
template <int SRC>
__global__ void __launch_bounds__(kThreads) k_radix_pass(Rows rows, InputSrc in,
                                                         const uint64_t* buf, RowSel* sel,
                                                         unsigned long long* ghist) {
    __shared__ uint32_t h[kBins];
    __shared__ int s_last;
    resolve_src(in);
    for (int b = threadIdx.x; b < kBins; b += kThreads) h[b] = 0;
    __syncthreads();

    const uint64_t ntiles = rows.tile_start[rows.R];
    int cur = -1;
    uint32_t cur_tiles = 0;
    bool active = false;
    unsigned long long prefix = 0;
    unsigned int pos = 0, hi = 64;
    uint64_t off = 0, len = 0;
    uint32_t lead = 0;

    auto finish_row = [&](int j) {
        __syncthreads();
        unsigned long long* gh = ghist + static_cast<uint64_t>(j) * kBins;
        for (int b = threadIdx.x; b < kBins; b += kThreads) {
            uint32_t c = h[b];
            if (c) {
                atomicAdd(gh + b, static_cast<unsigned long long>(c));
                h[b] = 0;
            }
        }
        __threadfence();
        __syncthreads();
        RowSel* sp = sel + rows.rid[j];
        if (threadIdx.x == 0) {
            const uint64_t mine = cur_tiles;
            const uint64_t tiles = rows.tile_start[j + 1] - rows.tile_start[j];
            const unsigned int old = atomicAdd(&sp->ticket, static_cast<unsigned int>(mine));
            s_last = (static_cast<uint64_t>(old) + mine == tiles);
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            if (active) select_in_block(sp, gh);
            if (threadIdx.x == 0) sp->ticket = 0;
        }
        __syncthreads();
    };

    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int j = row_of_tile(rows, t);
        if (j != cur) {
            if (cur >= 0) finish_row(cur);
            cur = j;
            cur_tiles = 0;
            const RowSel* sp = sel + rows.rid[j];
            active = (*(volatile const unsigned int*)&sp->status) == 0;
            prefix = sp->prefix;
            pos = sp->pos;
            hi = digit_hi(pos);
            off = rows.off[j];
            len = rows.len[j];
            lead = rows.lead[j];
        }
        ++cur_tiles;
        if (!active) continue;
        const uint64_t tt = t - rows.tile_start[j];
        const unsigned long long pmask = hi >= 64 ? 0ull : (prefix >> hi);
        const uint32_t dmask = (1u << (hi - pos)) - 1u;
        if (SRC == 0) {
            uint32_t v[kUnroll][kVec];
            const uint64_t span0 = tt * kTile;
            const uint64_t span_len = len + lead;
            load_input_tile_any(in, off, span_len, lead, span0, v);
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const uint64_t p = span0 + static_cast<uint64_t>(u * kThreads + threadIdx.x) * kVec;
#pragma unroll
                for (int i = 0; i < kVec; ++i) {
                    const uint64_t q = p + i;
                    const bool valid = q >= lead && q < span_len;
                    const unsigned long long K = composite(make_key(in, v[u][i]), q - lead);
                    const bool match = valid && (hi >= 64 || (K >> hi) == pmask);
                    hist_add(h, static_cast<uint32_t>(K >> pos) & dmask, match);
                }
            }
        } else {
            uint64_t v[4][kVec64];
            const uint64_t e0 = tt * kTile64;
            const uint64_t span_len = len + lead;
            load_u64_tile(buf + off - lead, span_len, lead, e0, v);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t p = e0 + static_cast<uint64_t>(u * kThreads + threadIdx.x) * kVec64;
#pragma unroll
                for (int i = 0; i < kVec64; ++i) {
                    const unsigned long long K = v[u][i];
                    const bool valid = p + i >= lead && p + i < span_len;
                    const bool match = valid && (hi >= 64 || (K >> hi) == pmask);
                    hist_add(h, static_cast<uint32_t>(K >> pos) & dmask, match);
                }
            }
        }
    }
    if (cur >= 0) finish_row(cur);
}

// k_init_call: reset every per-call counter in one launch.
__global__ void k_init_call(int R, unsigned long long* count, unsigned long long* kmin,
                            unsigned long long* kmax, uint32_t* kor, uint64_t* T, uint32_t* row_fail, uint32_t* ctl,
                            uint32_t* seg_hist, uint32_t* done, uint32_t* seg_ticket) {
    const uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = i0; i < static_cast<uint64_t>(R); i += stride) {
        count[i] = 0;
        kmin[i] = ~0ull;
        kmax[i] = 0;
        kor[i] = 0;
        T[i] = 0;
        row_fail[i] = 0;
        done[i] = 0;
        seg_ticket[i] = 0;
    }
    if (i0 < 16) ctl[i0] = 0;
    for (uint64_t i = i0; i < static_cast<uint64_t>(R) * kBins; i += stride) seg_hist[i] = 0;
}

// ----------------------------------------------------------------------------------------
// k_sample_select: the sampled threshold of each row in ONE kernel. A thread-block cluster of
// CS CTAs owns one row: the CTAs gather a stratified sample (nseg segments of 32 contiguous
// elements spread evenly over the row) into shared memory as composites, then run radix
// select passes over it (2048-bin digits, MSD first). Per pass every CTA histograms its part,
// the cluster barriers, and every CTA sums all CS histograms through distributed shared
// memory (DSMEM) and takes the same bin decision — no global atomics, no extra launches.
// The loop stops once #{sample K >= T} <= target (or the composite is exhausted), so heavy
// key ties in the sample are split by index inside the same loop. T[rid] = that composite.
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(1024) k_sample_select(SampleRows sr, InputSrc in, uint64_t* T) {
    pdl_trigger();  // k_compact may launch now (it waits for T in griddepcontrol.wait)
    resolve_src(in);
    unsigned long long* dbg = sr.dbg;
    int ndbg = 0;
    auto stamp = [&]() {
        if (dbg && blockIdx.x == 0 && threadIdx.x == 0 && ndbg < 30) dbg[ndbg++] = gtimer();
    };
    stamp();
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ unsigned long long smp[];
    // double-buffered by pass parity: a pass never rewrites what another CTA may still read from
    // the previous pass, so each pass needs two cluster barriers instead of three
    __shared__ __align__(16) uint32_t hist2[2][kBins];
    __shared__ __align__(16) uint32_t hred2[2][kBins];  // this CTA's reduced slice (first SL bins)
    __shared__ uint32_t s_wsum[32];
    __shared__ unsigned long long s_res[3];
    const unsigned CS = cluster.num_blocks();
    const unsigned crank = cluster.block_rank();
    const int j = blockIdx.x / CS;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t n = sr.len[j], off = sr.off[j];
    const uint64_t nseg = sr.nseg[j];
    const uint64_t s0 = crank * nseg / CS, s1 = (crank + 1) * nseg / CS;
    // segment start = floor(sg * (n - 32) / (nseg - 1)) in 16.16-style fixed point
    const uint64_t stride_fp = ((n - 32) << 16) / (nseg > 1 ? nseg - 1 : 1);
    // gather: element e of this CTA's share = lane (e % 32) of segment s0 + e / 32; each
    // thread issues all of its loads before the first use (memory-level parallelism)
    uint32_t local = static_cast<uint32_t>((s1 - s0) * 32);
    constexpr int kG = 8;  // per_cta <= 8192 = 8 x 1024 (double-buffered: 2 x 64 KB)
    unsigned long long* cur = smp;
    unsigned long long* alt = smp + kG * 1024;
    uint32_t* hsub = reinterpret_cast<uint32_t*>(smp + 2 * kG * 1024);  // 4 x kBins sub-histograms
    __shared__ uint32_t s_cnt;
    uint32_t raw[kG];
#pragma unroll
    for (int q = 0; q < kG; ++q) {
        const uint32_t e = q * 1024u + tid;
        if (e < local) {
            const uint64_t sg = s0 + e / 32;
            raw[q] = load_elem(in, off + ((sg * stride_fp) >> 16) + (e & 31));
        }
    }
#pragma unroll
    for (int q = 0; q < kG; ++q) {
        const uint32_t e = q * 1024u + tid;
        if (e < local) {
            const uint64_t sg = s0 + e / 32;
            cur[e] = composite(make_key(in, raw[q]), ((sg * stride_fp) >> 16) + (e & 31));
        }
    }
    __syncthreads();
    stamp();

    unsigned long long prefix = 0, k_rem = sr.k[j], above = 0;
    const unsigned long long target = sr.target[j];
    unsigned int pos = 53;
    for (uint32_t ps = 0;; ++ps) {
        uint32_t* hist = hist2[ps & 1];
        uint32_t* hred = hred2[ps & 1];
        for (int b = tid; b < 4 * kBins; b += blockDim.x) hsub[b] = 0;
        for (int b = tid; b < kBins; b += blockDim.x) hred[b] = 0;
        __syncthreads();
        const unsigned int hi = digit_hi(pos);
        const uint32_t dmask = (1u << (hi - pos)) - 1u;
        // samples outside the selected prefix are skipped in place (no compaction between
        // passes: <= 8 samples per thread); four warp-interleaved sub-histograms: the clustered
        // top digit of real data hits few bins
        uint32_t* hmine = hsub + (warp & 3) * kBins;
        const unsigned long long pm = hi >= 64 ? 0ull : (prefix >> hi);
        for (uint32_t i = tid; i < ((local + 31) & ~31u); i += blockDim.x) {
            const bool in_range = i < local;
            const unsigned long long K = in_range ? cur[i] : 0ull;
            if (in_range && (hi >= 64 || (K >> hi) == pm)) atomicAdd(hmine + (static_cast<uint32_t>(K >> pos) & dmask), 1u);
        }
        __syncthreads();
        for (int b = tid; b < kBins; b += blockDim.x)
            hist[b] = hsub[b] + hsub[kBins + b] + hsub[2 * kBins + b] + hsub[3 * kBins + b];
        stamp();
        cluster.sync();
        stamp();
        // cluster reduction of the CS histograms in two vectorised DSMEM rounds:
        //  A) CTA c sums bin slice [c*SL, (c+1)*SL) over all ranks (uint4 loads) into hred;
        //  B) every thread fetches the reduced counts of its two bins from the slice owner.
        const uint32_t SL = kBins / CS;
        if (tid < static_cast<int>(CS * SL / 4) && tid < 1024) {
            const unsigned rk = tid / (SL / 4);
            const uint32_t b4 = crank * SL + (tid % (SL / 4)) * 4;
            const uint4 v4 = *reinterpret_cast<const uint4*>(cluster.map_shared_rank(hist, rk) + b4);
            const uint32_t o = b4 - crank * SL;
            if (v4.x) atomicAdd(&hred[o], v4.x);
            if (v4.y) atomicAdd(&hred[o + 1], v4.y);
            if (v4.z) atomicAdd(&hred[o + 2], v4.z);
            if (v4.w) atomicAdd(&hred[o + 3], v4.w);
        }
        cluster.sync();
        stamp();
        uint32_t c0, c1;
        const int b0 = kBins - 1 - 2 * tid, b1 = b0 - 1;
        {
            const unsigned owner = b1 / SL;
            const uint2 v2 = *reinterpret_cast<const uint2*>(cluster.map_shared_rank(hred, owner) + (b1 - owner * SL));
            c1 = v2.x;
            c0 = v2.y;
        }
        // block exclusive scan of (c0 + c1) in descending-bin order
        const uint32_t v = c0 + c1;
        uint32_t inc = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += o;
        }
        if (lane == 31) s_wsum[warp] = inc;
        __syncthreads();
        uint32_t wpre = 0;
        for (int w = 0; w < warp; ++w) wpre += s_wsum[w];
        const uint64_t before = wpre + inc - v;
        if (tid == 0) s_res[0] = ~0ull;
        __syncthreads();
        if (before < k_rem && before + v >= k_rem) {
            if (before + c0 >= k_rem) { s_res[0] = b0; s_res[1] = before; s_res[2] = c0; }
            else { s_res[0] = b1; s_res[1] = before + c0; s_res[2] = c1; }
        }
        stamp();
        __syncthreads();  // s_res read by every thread before it changes
        stamp();
        if (s_res[0] == ~0ull) break;  // rank outside sample (cannot happen: k <= sample size)
        prefix |= s_res[0] << pos;
        above += s_res[1];
        k_rem -= s_res[1];
        const unsigned long long count_ge = above + s_res[2];
        if (count_ge <= target || pos == 0) break;
        stamp();
        pos = pos == 9 ? 0u : pos - 11u;
    }
    cluster.sync();  // no CTA leaves while another may still read its shared memory
    if (crank == 0 && tid == 0) T[sr.rid[j]] = prefix;
    stamp();
    if (dbg && blockIdx.x == 0 && threadIdx.x == 0) dbg[31] = ndbg;
}

// ----------------------------------------------------------------------------------------
// k_compact<KM>: the single streaming pass over the input. Keeps K >= T[rid] (fused key
// transform, compile-time per dtype/order/scale) into the row's candidate region.
//
// Flush-efficient buffering (engine.hpp:138-169), made warp-private: each
// warp owns a kWarpStage-entry slice of shared memory and a warp-uniform cursor. A hit slot is
// appended with one ballot + popc (no atomics); when the slice is nearly full the warp claims
// a contiguous range of the row's candidate region with ONE global cursor atomic and copies
// the slice out. No block-wide barrier in the streaming loop — only at row boundaries.
// Per element on the common (no-hit) path: key transform (2 ops) + compare + mask bit.
// Counts are exact even past `cap` (writes beyond cap are dropped -> host falls back).
// ----------------------------------------------------------------------------------------
constexpr int kWarpStage = 512;
#ifndef RTK_COMPACT_MINB
#define RTK_COMPACT_MINB 3
#endif

template <int KM>
__global__ void __launch_bounds__(kThreads, RTK_COMPACT_MINB) k_compact(Rows rows, InputSrc in, const uint64_t* T,
                                                         uint64_t* cand, const uint64_t* cand_off,
                                                         const uint64_t* cap,
                                                         unsigned long long* count,
                                                         unsigned long long* kmin,
                                                         unsigned long long* kmax, PlanArgs pa) {
    __shared__ unsigned long long stage_all[kThreads / 32][kWarpStage];
    __shared__ int s_last;
    const uint64_t ntiles = rows.tile_start[rows.R];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned full = 0xffffffffu;
    const unsigned lt_mask = (1u << lane) - 1u;
    unsigned long long* stage = stage_all[warp];

    // CTA-uniform state of the current row that the streaming loop does not touch lives in
    // shared memory (register pressure: the loop holds 32 input words per thread)
    struct RowState {
        uint64_t coff, ccap, len;
        uint32_t r, j;
    };
    __shared__ RowState s_row;
    bool have_row = false;
    unsigned long long mn = ~0ull, mx = 0;
    uint32_t ko = 0;  // OR of (key ^ T.hi) over this thread's hits of the current row
    uint32_t thi = 0, tlo = 0, wcur = 0;
    uint64_t base_el = 0, span_len = 0, tile0 = 0, tile1 = 0;  // base_el = row offset - lead
    uint32_t lead = 0, mine_tiles = 0;

    // PDL: this grid may start while k_sample_select still runs. The input does not depend on
    // it: each CTA pulls its first tiles into L2 with TMA bulk prefetches (<= ~96 MB in total,
    // inside the 126 MB L2), then waits for the thresholds.
    if (threadIdx.x < 8) {
        const uint64_t budget = (static_cast<uint64_t>(pa.prefetch_mb) << 20) / (static_cast<uint64_t>(gridDim.x) * kTile * 4);
        const uint64_t t = pa.contig ? blockIdx.x * ((ntiles + gridDim.x - 1) / gridDim.x) + threadIdx.x
                                     : blockIdx.x + threadIdx.x * static_cast<uint64_t>(gridDim.x);
        if (threadIdx.x < budget && t < ntiles) {
            const int j0 = row_of_tile(rows, t);
            const uint64_t sp0 = (t - rows.tile_start[j0]) * kTile;
            const uint64_t span_len0 = rows.len[j0] + rows.lead[j0];
            if (sp0 + kTile <= span_len0) {
                constexpr int EB = km_is16<KM>() ? 2 : 4;
                const char* tp0 = reinterpret_cast<const char*>(in.base) + (rows.off[j0] - rows.lead[j0] + sp0) * EB;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(tp0), "r"(kTile * EB) : "memory");
            }
        }
    }
    pdl_wait();
    resolve_src(in);  // scaled_topk decided on the device (k_scale_decide / k_scale_guess)
    // speculative Adaptive trigger (k_scale_guess): count the unscaled first-window digits
    // above / at the guessed bin over every element of the row (main path only)
    constexpr bool kAdapt = KM == kKmF32LAdapt || KM == kKmF32SAdapt;
    uint32_t g_bin = 0, g_shift = 32, c_gt = 0, c_eq = 0;
    if constexpr (kAdapt) {
        if (pa.trig) {
            g_bin = __ldcg(in.adapt + 2);
            g_shift = __ldcg(in.adapt + 3);
        }
    }

    auto warp_flush = [&]() {  // warp-uniform
        if (wcur == 0) return;
        __syncwarp();
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(count + s_row.r, static_cast<unsigned long long>(wcur));
        base = __shfl_sync(full, base, 0);
        const uint64_t coff = s_row.coff, ccap = s_row.ccap;
        for (uint32_t i = lane; i < wcur; i += 32) {
            const unsigned long long K = stage[i];
            mn = min(mn, K);
            mx = max(mx, K);
            ko |= static_cast<uint32_t>(K >> 32) ^ thi;
            if (base + i < ccap) cand[coff + base + i] = K;
        }
        __syncwarp();
        wcur = 0;
    };
    auto finish_row = [&]() {
        warp_flush();
        unsigned long long a = mn, b = mx;
        uint32_t o = ko;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            a = min(a, __shfl_xor_sync(full, a, d));
            b = max(b, __shfl_xor_sync(full, b, d));
            o |= __shfl_xor_sync(full, o, d);
        }
        const uint32_t r = s_row.r;
        if (lane == 0 && a <= b) {
            atomicMin(kmin + r, a);
            atomicMax(kmax + r, b);
            if (pa.kor && o) atomicOr(pa.kor + r, o);
        }
        mn = ~0ull;
        mx = 0;
        ko = 0;
        // the CTA that finishes the row's last tile plans its ordering (k_plan_rows fused)
        if (pa.done) {
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) {
                const uint32_t tiles = static_cast<uint32_t>(tile1 - tile0);
                const uint32_t old = atomicAdd(pa.done + r, mine_tiles);
                s_last = old + mine_tiles == tiles;
                if (s_last) {
                    __threadfence();
                    plan_row(static_cast<int>(s_row.j), r, pa, s_row.len);
                }
            }
            __syncthreads();
        }
    };

    // interleaved tile order (CTA b: tiles b, b+G, ...): measured ~12% faster streaming on B200
    // than contiguous runs per CTA, at the price of a row switch per tile in many-row batches
    // many-row batches: contiguous tile runs per CTA (one row switch per run instead of per tile)
    const uint64_t per = pa.contig ? (ntiles + gridDim.x - 1) / gridDim.x : 1;
    const uint64_t t_begin = pa.contig ? blockIdx.x * per : blockIdx.x;
    const uint64_t t_end = pa.contig ? min(ntiles, t_begin + per) : ntiles;
    const uint64_t t_step = pa.contig ? 1 : gridDim.x;
    uint32_t v[kUnroll][kVec];
    auto load_tile = [&](uint64_t tt) {
        const uint64_t sp = (tt - tile0) * kTile;
        const uint32_t lo = sp >= lead ? 0u : static_cast<uint32_t>(lead - sp);
        const uint32_t hi = static_cast<uint32_t>(span_len - sp < kTile ? span_len - sp : kTile);
        if constexpr (km_is16<KM>())
            load_tile_local16(reinterpret_cast<const unsigned short*>(in.base) + base_el + sp, lo, hi, v);
        else
            load_tile_local(in.base + base_el + sp, lo, hi, v);
    };
    // interleaved mode: the last `dyn` tiles are handed out from a counter, so CTAs that start
    // late (PDL launch next to the sample kernel's cluster) do not leave a tail
    __shared__ uint64_t s_next;
    const uint64_t dyn_want = static_cast<uint64_t>(gridDim.x) * pa.dyn_per_cta;
    const uint64_t dyn = (!pa.contig && pa.dyn_ctr) ? (dyn_want < ntiles ? dyn_want : ntiles) : 0;
    const uint64_t ns = ntiles - dyn;
    auto grab = [&]() -> uint64_t {  // block-collective
        __syncthreads();
        if (threadIdx.x == 0) s_next = ns + atomicAdd(pa.dyn_ctr, 1u);
        __syncthreads();
        return s_next;
    };
    auto next_tile = [&](uint64_t tt) -> uint64_t {
        if (dyn == 0 || tt + t_step < ns) return tt + t_step;
        return grab();
    };
    const uint64_t t_first = (dyn != 0 && t_begin >= ns) ? grab() : t_begin;
    for (uint64_t t = t_first; t < t_end; t = next_tile(t)) {
        if (t >= tile1 || !have_row) {  // CTA-uniform
            if (have_row) finish_row();
            have_row = true;
            const int j = row_of_tile(rows, t);
            const uint32_t r = rows.rid[j];
            const unsigned long long thr = T[r];
            thi = static_cast<uint32_t>(thr >> 32);
            tlo = static_cast<uint32_t>(thr);
            lead = rows.lead[j];
            const uint64_t len = rows.len[j];
            base_el = rows.off[j] - lead;
            span_len = len + lead;
            tile0 = rows.tile_start[j];
            tile1 = rows.tile_start[j + 1];
            mine_tiles = 0;
            __syncthreads();  // every warp is done with the previous row's shared state
            if (threadIdx.x == 0) s_row = RowState{cand_off[r], cap[r], len, r, static_cast<uint32_t>(j)};
            __syncthreads();
        }
        ++mine_tiles;
        const uint64_t span0 = (t - tile0) * kTile;
        // validity window of this tile in tile-local positions (32-bit math from here on)
        const uint32_t vlo = span0 >= lead ? 0u : static_cast<uint32_t>(lead - span0);
        const uint32_t vhi = static_cast<uint32_t>(span_len - span0 < kTile ? span_len - span0 : kTile);
        const uint32_t idx0 = static_cast<uint32_t>(span0 - lead);  // low 32 bits of the row index
        load_tile(t);

        // K >= T with T = (T.hi, T.lo): key > T.hi, or key == T.hi and index <= ~T.lo. T.lo != 0
        // when ties at the threshold key were split by index (tie-heavy inputs, the exact path).
        // The index condition is decided per TILE: a tile whose valid indices all lie at or below
        // ~T.lo keeps equal keys (compare with T.hi), one wholly above drops them (compare with
        // T.hi + 1); only the one tile straddling ~T.lo compares element by element.
        uint32_t tthr = thi;
        bool straddle = false;
        if (tlo != 0) {
            const uint32_t tidx = ~tlo, first = idx0 + vlo, last = idx0 + vhi - 1;
            if (last <= tidx) {
            } else if (first > tidx && thi != 0xFFFFFFFFu) {
                tthr = thi + 1;
            } else {
                straddle = true;
            }
        }
        if constexpr (kAdapt) {
            if (g_shift < 32) {  // digit >= b  <=>  key >= b << shift;  digit > b  <=>  key > ((b + 1) << shift) - 1
                const uint32_t lo = g_bin << g_shift, hm1 = ((g_bin + 1) << g_shift) - 1u;  // top bin: hm1 = ~0
                uint32_t ge = 0, gt = 0;
                if (vlo == 0 && vhi == kTile) {
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                        for (int i = 0; i < kVec; ++i) {
                            const uint32_t ku = encode_f32_bits(v[u][i], KM == kKmF32SAdapt);
                            // two compares + two predicated increments per element
                            asm("{\n.reg .pred p, q;\nsetp.ge.u32 p, %2, %3;\nsetp.gt.u32 q, %2, %4;\n"
                                "@p add.u32 %0, %0, 1;\n@q add.u32 %1, %1, 1;\n}"
                                : "+r"(ge), "+r"(gt) : "r"(ku), "r"(lo), "r"(hm1));
                        }
                } else {
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                        for (int i = 0; i < kVec; ++i) {
                            const uint32_t l = (u * kThreads + threadIdx.x) * kVec + i;
                            const uint32_t ku = encode_f32_bits(v[u][i], KM == kKmF32SAdapt);
                            const bool ok = l >= vlo && l < vhi;
                            ge += ok && ku >= lo;
                            gt += ok && ku > hm1;
                        }
                }
                c_gt += gt;
                c_eq += ge - gt;
            }
        }
        // pass 1: key transform + per-thread hit mask (bit u*8+i). Scaled keys (y = x - a_s): a
        // plain fp32 subtraction per element and one NaN flag per thread; only a thread that
        // produced a NaN re-derives those keys with the x86 NaN rule of sub_x86 (the element
        // re-read from L2), instead of a NaN test per element
        constexpr bool kSub = KM == kKmF32LScaled || KM == kKmF32SScaled || kAdapt;
        constexpr bool kSm = KM == kKmF32SScaled || KM == kKmF32SAdapt;
        uint32_t mask = 0;
        if constexpr (kSub) {
            if (!kAdapt || in.scaled) {
                bool anynan = false;
#pragma unroll
                for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                    for (int i = 0; i < kVec; ++i) {
                        const float y = __fsub_rn(__uint_as_float(v[u][i]), in.a_s);
                        anynan |= y != y;
                        // the bits through an opaque move: otherwise the sign-flip encode is
                        // rewritten as float negation (FADD -|y|), which canonicalises NaNs
                        uint32_t yb;
                        asm("mov.b32 %0, %1;" : "=r"(yb) : "f"(y));
                        v[u][i] = encode_f32_bits(yb, kSm);
                    }
                if (anynan) {
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                        for (int i = 0; i < kVec; ++i) {
                            const uint32_t e = kSm ? ~v[u][i] : v[u][i];  // encode(y) -> y
                            const uint32_t yb = (e & 0x80000000u) ? (e ^ 0x80000000u) : ~e;
                            const uint32_t l = (u * kThreads + threadIdx.x) * kVec + i;
                            if ((yb & 0x7fffffffu) > 0x7f800000u && l >= vlo && l < vhi)
                                v[u][i] = encode_f32_bits(sub_x86(__ldg(in.base + base_el + span0 + l), in.a_s), kSm);
                        }
                }
            } else {
#pragma unroll
                for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                    for (int i = 0; i < kVec; ++i) v[u][i] = encode_f32_bits(v[u][i], kSm);
            }
            if (vlo == 0 && vhi == kTile) {
#pragma unroll
                for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                    for (int i = 0; i < kVec; ++i) mask |= static_cast<uint32_t>(v[u][i] >= tthr) << (u * kVec + i);
            } else {
#pragma unroll
                for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                    for (int i = 0; i < kVec; ++i) {
                        const uint32_t l = (u * kThreads + threadIdx.x) * kVec + i;
                        mask |= static_cast<uint32_t>(v[u][i] >= tthr && l >= vlo && l < vhi) << (u * kVec + i);
                    }
            }
        } else if (vlo == 0 && vhi == kTile) {
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                for (int i = 0; i < kVec; ++i) {
                    const uint32_t key = key_of<KM>(v[u][i], in);
                    v[u][i] = key;
                    mask |= static_cast<uint32_t>(key >= tthr) << (u * kVec + i);
                }
        } else {
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                for (int i = 0; i < kVec; ++i) {
                    const uint32_t key = key_of<KM>(v[u][i], in);
                    v[u][i] = key;
                    const uint32_t l = (u * kThreads + threadIdx.x) * kVec + i;
                    mask |= static_cast<uint32_t>(key >= tthr && l >= vlo && l < vhi) << (u * kVec + i);
                }
        }
        if (straddle) {
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                for (int i = 0; i < kVec; ++i) {
                    const uint32_t l = (u * kThreads + threadIdx.x) * kVec + i;
                    if (v[u][i] == thi && ~(idx0 + l) < tlo) mask &= ~(1u << (u * kVec + i));
                }
        }
        if (!__any_sync(full, mask)) continue;

        // pass 2 (tiles with hits only): each thread appends its hits as one contiguous run
        const uint32_t c = __popc(mask);
        uint32_t incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(full, incl, d);
            if (lane >= d) incl += o;
        }
        const uint32_t wtot = __shfl_sync(full, incl, 31);
        if (wcur + wtot > kWarpStage) warp_flush();
        const uint32_t nidx0 = ~idx0;  // ~(idx0 + l) == nidx0 - l
        if (wtot <= pa.sparse_max) {
            // sparse hits (the common case): visit only the set bits; the element is re-read
            // from L2 (its tile was just streamed) instead of indexing registers dynamically
            const uint64_t tp = base_el + span0;  // element offset of the tile
            uint32_t o = wcur + incl - c;
            uint32_t m = mask;
            if (pa.sparse_sel) {
                // the hit's key from registers through a 31-SEL tree (static register indices;
                // no L2 re-read stalling the warp before its next tile's loads)
                while (m) {
                    const uint32_t b = __ffs(m) - 1;
                    m &= m - 1;
                    uint32_t t[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) t[j] = (b & 1) ? v[(2 * j + 1) >> 3][(2 * j + 1) & 7] : v[(2 * j) >> 3][(2 * j) & 7];
#pragma unroll
                    for (int w = 8; w >= 1; w >>= 1) {
                        const uint32_t bit = 16u / w;  // 2, 4, 8, 16
#pragma unroll
                        for (int j = 0; j < w; ++j) t[j] = (b & bit) ? t[2 * j + 1] : t[2 * j];
                    }
                    const uint32_t l = ((b >> 3) * kThreads + threadIdx.x) * kVec + (b & 7);
                    stage[o++] = (static_cast<unsigned long long>(t[0]) << 32) | (nidx0 - l);
                }
                m = 0;
            }
            while (m) {
                const uint32_t b = __ffs(m) - 1;
                m &= m - 1;
                const uint32_t l = ((b >> 3) * kThreads + threadIdx.x) * kVec + (b & 7);
                uint32_t raw;
                if constexpr (km_is16<KM>())
                    raw = __ldg(reinterpret_cast<const unsigned short*>(in.base) + tp + l);
                else
                    raw = __ldg(in.base + tp + l);
                const uint32_t key = key_of<KM>(raw, in);
                stage[o++] = (static_cast<unsigned long long>(key) << 32) | (nidx0 - l);
            }
            wcur += wtot;
        } else if (wtot <= kWarpStage) {
            uint32_t o = wcur + incl - c;
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                for (int i = 0; i < kVec; ++i) {
                    if ((mask >> (u * kVec + i)) & 1u) {
                        const uint32_t l = (u * kThreads + threadIdx.x) * kVec + i;
                        stage[o++] = (static_cast<unsigned long long>(v[u][i]) << 32) | (nidx0 - l);
                    }
                }
            wcur += wtot;
        } else {  // dense hits (k close to n): straight to global with one cursor atomic
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(count + s_row.r, static_cast<unsigned long long>(wtot));
            base = __shfl_sync(full, base, 0) + (incl - c);
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                for (int i = 0; i < kVec; ++i) {
                    if ((mask >> (u * kVec + i)) & 1u) {
                        const uint32_t l = (u * kThreads + threadIdx.x) * kVec + i;
                        const unsigned long long K = (static_cast<unsigned long long>(v[u][i]) << 32) | (nidx0 - l);
                        mn = min(mn, K);
                        mx = max(mx, K);
                        ko |= v[u][i] ^ thi;  // same per-row OR as warp_flush (plan_row's tz)
                        if (base < s_row.ccap) cand[s_row.coff + base] = K;
                        ++base;
                    }
                }
        }
    }
    if (have_row) finish_row();
    if constexpr (kAdapt) {
        if (g_shift < 32) {  // warp totals -> ctl[10..11] (#{digit > b}), ctl[12..13] (#{digit == b})
            unsigned long long a = c_gt, b = c_eq;
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                a += __shfl_xor_sync(full, a, d);
                b += __shfl_xor_sync(full, b, d);
            }
            if (lane == 0) {
                atomicAdd(reinterpret_cast<unsigned long long*>(pa.flags + 10), a);
                atomicAdd(reinterpret_cast<unsigned long long*>(pa.flags + 12), b);
            }
        }
    }
    if (dyn) {  // the last CTA out resets the tile counters for the next launch
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(pa.dyn_ctr + 1, 1u) == gridDim.x - 1) {
                pa.dyn_ctr[0] = 0;
                pa.dyn_ctr[1] = 0;
            }
        }
    }
}

// pivot[r] = values[k-1] of each row (engine.hpp:333 / scaling.hpp:76).
__global__ void k_pivots(int R, const uint64_t* row_out_off, const uint64_t* row_k,
                         const uint32_t* vals, uint32_t* pivots) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < R) pivots[j] = vals[row_out_off[j] + row_k[j] - 1];
}

// Shard-merge remap: out_idx[i] holds a position j in the concatenated candidate blocks;
// replace it by the shard-local index stored there plus the shard's global base.
__global__ void k_remap_idx(uint64_t n, const uint64_t* cand_idx, uint32_t nblocks,
                            const uint64_t* block_start, const uint64_t* shard_base, uint64_t* idx) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t j = idx[i];
        uint32_t lo = 0, hi = nblocks - 1;
        while (lo < hi) {
            uint32_t mid = (lo + hi + 1) >> 1;
            if (block_start[mid] <= j) lo = mid; else hi = mid - 1;
        }
        idx[i] = cand_idx[j] + shard_base[lo];
    }
}

// ----------------------------------------------------------------------------------------
// k_first_digit_hist: exact histogram of the first d-bit window of the UNSCALED keys
// (scaled_topk's adaptive trigger, scaling.hpp:50-58). d <= 13 uses smem; wider digits go
// straight to global u64 atomics.
// ----------------------------------------------------------------------------------------
template <int KM>
__global__ void __launch_bounds__(kThreads) k_first_digit_hist(Rows rows, InputSrc in, unsigned int d,
                                                               unsigned long long* ghist) {
    extern __shared__ uint32_t hs[];
    const uint32_t nb = 1u << d;
    const bool use_smem = d <= 13;
    if (use_smem) {
        for (uint32_t b = threadIdx.x; b < nb; b += kThreads) hs[b] = 0;
        __syncthreads();
    }
    const uint64_t ntiles = rows.tile_start[rows.R];
    const uint64_t off = rows.off[0], len = rows.len[0];
    const uint32_t lead = rows.lead[0];
    const uint64_t span_len = len + lead;
    const unsigned full = 0xffffffffu;
    // warp-uniform tiles (the adversarial inputs this trigger exists for put every key in ONE
    // bin) accumulate in a register: one shared atomic per run, not one per warp and element
    uint32_t run_d = 0, run_c = 0;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t span0 = t * kTile;
        const uint32_t vlo = span0 >= lead ? 0u : static_cast<uint32_t>(lead - span0);
        const uint32_t vhi = static_cast<uint32_t>(span_len - span0 < kTile ? span_len - span0 : kTile);
        uint32_t v[kUnroll][kVec];
        load_tile_local(in.base + off - lead + span0, vlo, vhi, v);
        const bool whole = vlo == 0 && vhi == kTile;
        uint32_t d0 = 0;
        bool same = whole;
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
#pragma unroll
            for (int i = 0; i < kVec; ++i) {
                v[u][i] = key_of<KM>(v[u][i], in) >> (32 - d);
                if (u == 0 && i == 0) d0 = v[0][0];
                same &= v[u][i] == d0;
            }
        const uint32_t w0 = __shfl_sync(full, d0, 0);
        if (use_smem && __all_sync(full, same && d0 == w0)) {
            if (w0 != run_d) {
                if (run_c && (threadIdx.x & 31) == 0) atomicAdd(&hs[run_d], run_c);
                run_d = w0;
                run_c = 0;
            }
            run_c += 32 * kUnroll * kVec;
            continue;
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
#pragma unroll
            for (int i = 0; i < kVec; ++i) {
                const uint32_t l = (u * kThreads + threadIdx.x) * kVec + i;
                const bool valid = l >= vlo && l < vhi;
                if (use_smem) hist_add(hs, v[u][i], valid);
                else if (valid) atomicAdd(ghist + v[u][i], 1ull);
            }
    }
    if (use_smem) {
        if (run_c && (threadIdx.x & 31) == 0) atomicAdd(&hs[run_d], run_c);
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < nb; b += kThreads)
            if (hs[b]) atomicAdd(ghist + b, static_cast<unsigned long long>(hs[b]));
    }
}

// ----------------------------------------------------------------------------------------
// k_scale_decide: scaled_topk's decision on the device (scaling.hpp:47-67) — no host round trip.
// mode 1 (Always): scale. mode 2 (Adaptive): select_bin on the exact first-window histogram
// (engine.hpp:231-241: first bin from the top whose cumulative count reaches k) and scale iff
// that bin holds more than tau * n keys. a_s = x[a_index] (the index is drawn on the host with
// mt19937_64(seed) exactly as draw_scale does). out = {flag, a_s bits}; host_out (mapped, may be
// null) receives {flag, a_s bits} for ScaleInfo.
// ----------------------------------------------------------------------------------------
__global__ void k_scale_decide(int mode, const unsigned long long* hist, uint32_t nbins, uint64_t n, uint64_t k,
                               double tau, const uint32_t* x, uint64_t a_index, uint32_t* out,
                               volatile uint32_t* host_out) {
    __shared__ unsigned long long s_warp[32];
    __shared__ int s_fat;
    const int tid = threadIdx.x;
    if (tid == 0) s_fat = mode == 1;
    __syncthreads();
    if (mode == 2) {
        // descending cumulative scan over nbins (<= 65536) with 1024 threads
        const uint32_t per = (nbins + blockDim.x - 1) / blockDim.x;
        unsigned long long sum = 0;
        for (uint32_t i = 0; i < per; ++i) {
            const uint32_t b = tid * per + i;  // b-th bin from the top
            if (b < nbins) sum += hist[nbins - 1 - b];
        }
        unsigned long long tot;
        const unsigned long long before = block_excl_scan(sum, s_warp, &tot);
        if (before < k && before + sum >= k) {
            unsigned long long cum = before;
            for (uint32_t i = 0; i < per; ++i) {
                const uint32_t b = tid * per + i;
                if (b >= nbins) break;
                const unsigned long long c = hist[nbins - 1 - b];
                if (cum + c >= k) {
                    s_fat = static_cast<double>(c) > tau * static_cast<double>(n);
                    break;
                }
                cum += c;
            }
        }
        __syncthreads();
    }
    if (tid == 0) {
        const uint32_t fat = s_fat ? 1u : 0u;
        const uint32_t a = fat ? __ldg(x + a_index) : 0u;
        out[0] = fat;
        out[1] = a;
        if (host_out) {
            host_out[0] = fat;
            host_out[1] = a;
            __threadfence_system();
        }
    }
}

// k_scale_guess: Adaptive scaled_topk without the extra counting pass. One CTA samples the
// unscaled keys (kGuessSeg segments of 32 consecutive elements spread over the row), takes
// select_bin of their first d-bit window at the sample rank of k, and GUESSES the trigger
// (sample fraction of that bin > tau). out = {flag, a_s bits, bin b, 32 - d}; the selection then
// runs in the guessed mode while k_compact counts, over ALL n elements, #{digit > b} and
// #{digit == b} of the unscaled keys (ctl[10..13]). The host accepts the run only if those
// counts prove b is the exact select_bin bin (#{> b} < k <= #{>= b}) and reproduce the decision
// hist[b] > tau * n of scaling.hpp:50-58; otherwise it reruns with the exact trigger pass.
constexpr int kGuessSeg = 512;
__global__ void __launch_bounds__(1024) k_scale_guess(const uint32_t* x, uint64_t n, uint64_t k, uint32_t d,
                                                      int smallest, double tau, uint64_t a_index, uint32_t* out,
                                                      volatile uint32_t* host_out) {
    extern __shared__ uint32_t h[];  // 2^d bins (d <= 14)
    __shared__ unsigned long long s_warp[32];
    __shared__ uint32_t s_bin, s_cnt;
    const int tid = threadIdx.x;
    const uint32_t nb = 1u << d;
    for (uint32_t b = tid; b < nb; b += blockDim.x) h[b] = 0;
    if (tid == 0) {
        s_bin = 0;
        s_cnt = 0;
    }
    __syncthreads();
    const uint64_t segs = n >= 32ull * kGuessSeg ? kGuessSeg : (n + 31) / 32;
    const uint64_t stride = segs > 1 ? (n - 32) / (segs - 1) : 0;
    uint32_t S = 0;
    // warp-aggregated (the adversarial case puts every sample in ONE bin: 16K same-address
    // shared atomics would serialise); the trip count is warp-uniform (blockDim | 32 * segs)
    // all 16 loads per thread in flight before the first use (one DRAM round trip, not 16)
    constexpr int kPer = kGuessSeg * 32 / 1024;
    uint32_t raw[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const uint32_t e = q * 1024 + tid;
        const uint64_t i = (e / 32) * stride + (e & 31);
        raw[q] = e < segs * 32 && i < n ? __ldg(x + i) : 0u;
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const uint32_t e = q * 1024 + tid;
        const uint64_t i = (e / 32) * stride + (e & 31);
        const bool valid = e < segs * 32 && i < n;
        const uint32_t dg = valid ? encode_f32_bits(raw[q], smallest != 0) >> (32 - d) : 0xFFFFFFFFu;
        const unsigned peers = __match_any_sync(0xffffffffu, dg);
        if (valid && (tid & 31) == __ffs(peers) - 1) atomicAdd(h + dg, static_cast<uint32_t>(__popc(peers)));
    }
    S = static_cast<uint32_t>(n < segs * 32 ? n : segs * 32);
    __syncthreads();
    // sample rank of k: ceil(k * S / n), then select_bin (descending cumulative scan)
    const uint64_t ks0 = (k * S + n - 1) / n;
    const uint64_t ks = ks0 > 0 ? ks0 : 1;
    const uint32_t per = (nb + blockDim.x - 1) / blockDim.x;
    unsigned long long sum = 0;
    for (uint32_t i = 0; i < per; ++i) {
        const uint32_t b = tid * per + i;
        if (b < nb) sum += h[nb - 1 - b];
    }
    unsigned long long tot;
    const unsigned long long before = block_excl_scan(sum, s_warp, &tot);
    if (before < ks && before + sum >= ks) {
        unsigned long long cum = before;
        for (uint32_t i = 0; i < per; ++i) {
            const uint32_t b = tid * per + i;
            if (b >= nb) break;
            const uint32_t c = h[nb - 1 - b];
            if (cum + c >= ks) {
                s_bin = nb - 1 - b;
                s_cnt = c;
                break;
            }
            cum += c;
        }
    }
    __syncthreads();
    if (tid == 0) {
        const uint32_t fat = static_cast<double>(s_cnt) > tau * static_cast<double>(S) ? 1u : 0u;
        const uint32_t a = fat ? __ldg(x + a_index) : 0u;
        out[0] = fat;
        out[1] = a;
        out[2] = s_bin;
        out[3] = 32 - d;
        if (host_out) {
            host_out[0] = fat;
            host_out[1] = a;
            __threadfence_system();
        }
    }
}

void launch_scale_guess(const uint32_t* x, uint64_t n, uint64_t k, uint32_t d, int smallest, double tau,
                        uint64_t a_index, uint32_t* out, volatile uint32_t* host_out, cudaStream_t s) {
    const size_t smem = (size_t(1) << d) * sizeof(uint32_t);
    static DeviceOnce configured;
    configured([&] {
        cudaFuncSetAttribute(k_scale_guess, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    });
    k_scale_guess<<<1, 1024, smem, s>>>(x, n, k, d, smallest, tau, a_index, out, host_out);
}

// ----------------------------------------------------------------------------------------
// Launchers. Streaming kernels run as persistent grids: resident CTAs per SM (occupancy API)
// x SM count, capped by the tile count.
// ----------------------------------------------------------------------------------------
void launch_init_sel(int R, const uint32_t* rid, const uint64_t* k, const uint64_t* target,
                     RowSel* sel, cudaStream_t s) {
    if (R > 0) k_init_sel<<<(R + 255) / 256, 256, 0, s>>>(R, rid, k, target, sel);
}

void launch_radix_pass(int src, uint64_t tiles, const Rows& rows, const InputSrc& in,
                       const uint64_t* buf, RowSel* sel, unsigned long long* ghist, cudaStream_t s) {
    if (src == 0) {
        const int grid = persistent_grid(k_radix_pass<0>, kThreads, 0, tiles);
        k_radix_pass<0><<<grid, kThreads, 0, s>>>(rows, in, buf, sel, ghist);
    } else {
        const int grid = persistent_grid(k_radix_pass<1>, kThreads, 0, tiles);
        k_radix_pass<1><<<grid, kThreads, 0, s>>>(rows, in, buf, sel, ghist);
    }
}

void launch_init_call(int R, unsigned long long* count, unsigned long long* kmin, unsigned long long* kmax,
                      uint32_t* kor, uint64_t* T, uint32_t* row_fail, uint32_t* ctl, uint32_t* seg_hist, uint32_t* done,
                      uint32_t* seg_ticket, cudaStream_t s) {
    const uint64_t work = static_cast<uint64_t>(R) * kBins;
    const int grid = static_cast<int>(std::min<uint64_t>((work + 255) / 256, 1024));
    k_init_call<<<grid, 256, 0, s>>>(R, count, kmin, kmax, kor, T, row_fail, ctl, seg_hist, done, seg_ticket);
}

void launch_sample_select(int rows, int cs, uint32_t per_cta, const SampleRows& sr, const InputSrc& in,
                          uint64_t* T, cudaStream_t s) {
    if (rows <= 0) return;
    // double buffer (per_cta <= 8192) + 4 sub-histograms
    const size_t smem = 2 * 8192 * sizeof(unsigned long long) + 4 * kBins * sizeof(uint32_t);
    (void)per_cta;
    static DeviceOnce configured;
    configured([&] {
        cudaFuncSetAttribute(k_sample_select, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        cudaFuncSetAttribute(k_sample_select, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    });
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(rows * cs);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_sample_select, sr, in, T);
}

template <int KM>
static void compact_km(uint64_t tiles, const Rows& rows, const InputSrc& in, const uint64_t* T,
                       uint64_t* cand, const uint64_t* cand_off, const uint64_t* cap,
                       unsigned long long* count, unsigned long long* kmin, unsigned long long* kmax,
                       const PlanArgs& pa, cudaStream_t s) {
    const int grid = persistent_grid(k_compact<KM>, kThreads, 0, tiles);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    // PDL (RTK_PDL_COMPACT=1): compaction CTAs launch while the sample kernel runs (L2 prefetch
    // prologue, then griddepcontrol.wait); those that cannot fit next to the sample's cluster
    // start late. Off by default: with the static split it measured +14 us at k = 256 (tail);
    // with the dynamic tail (pa.dyn_ctr, 12 tiles per CTA) it is neutral at k = 256 and +5 us at
    // k = 2^20, while the dynamic tail alone gains 4 / 7 us (C2 k = 256 / 2^20).
    static const bool env_off = [] {
        const char* e = std::getenv("RTK_PDL_COMPACT");
        return !(e && *e && *e != '0');
    }();
    const bool no_pdl = env_off || pa.dyn_ctr == nullptr || pa.contig;
    cfg.numAttrs = no_pdl ? 0 : 1;
    cudaLaunchKernelEx(&cfg, k_compact<KM>, rows, in, T, cand, cand_off, cap, count, kmin, kmax, pa);
}

void launch_compact(uint64_t tiles, const Rows& rows, const InputSrc& in, const uint64_t* T,
                    uint64_t* cand, const uint64_t* cand_off, const uint64_t* cap,
                    unsigned long long* count, unsigned long long* kmin, unsigned long long* kmax,
                    const PlanArgs& pa, cudaStream_t s) {
    switch (key_mode(in.dtype, in.smallest, in.scaled, in.adapt)) {
        case kKmF32L: compact_km<kKmF32L>(tiles, rows, in, T, cand, cand_off, cap, count, kmin, kmax, pa, s); break;
        case kKmF32S: compact_km<kKmF32S>(tiles, rows, in, T, cand, cand_off, cap, count, kmin, kmax, pa, s); break;
        case kKmF32LScaled: compact_km<kKmF32LScaled>(tiles, rows, in, T, cand, cand_off, cap, count, kmin, kmax, pa, s); break;
        case kKmF32SScaled: compact_km<kKmF32SScaled>(tiles, rows, in, T, cand, cand_off, cap, count, kmin, kmax, pa, s); break;
        case kKmU32L: compact_km<kKmU32L>(tiles, rows, in, T, cand, cand_off, cap, count, kmin, kmax, pa, s); break;
        case kKmF16L: compact_km<kKmF16L>(tiles, rows, in, T, cand, cand_off, cap, count, kmin, kmax, pa, s); break;
        case kKmF32LAdapt: compact_km<kKmF32LAdapt>(tiles, rows, in, T, cand, cand_off, cap, count, kmin, kmax, pa, s); break;
        case kKmF32SAdapt: compact_km<kKmF32SAdapt>(tiles, rows, in, T, cand, cand_off, cap, count, kmin, kmax, pa, s); break;
        case kKmF16S: compact_km<kKmF16S>(tiles, rows, in, T, cand, cand_off, cap, count, kmin, kmax, pa, s); break;
        default: compact_km<kKmU32S>(tiles, rows, in, T, cand, cand_off, cap, count, kmin, kmax, pa, s); break;
    }
}

void launch_pivots(int R, const uint64_t* row_out_off, const uint64_t* row_k, const uint32_t* vals,
                   uint32_t* pivots, cudaStream_t s) {
    if (R > 0) k_pivots<<<(R + 255) / 256, 256, 0, s>>>(R, row_out_off, row_k, vals, pivots);
}

void launch_first_digit_hist(uint64_t tiles, const Rows& rows, const InputSrc& in, unsigned int d,
                             unsigned long long* ghist, cudaStream_t s) {
    const size_t smem = d <= 13 ? (static_cast<size_t>(1) << d) * sizeof(uint32_t) : 0;
    // the trigger always histograms the UNSCALED f32 keys (scaling.hpp:50-58)
    if (in.smallest) {
        const int grid = persistent_grid(k_first_digit_hist<kKmF32S>, kThreads, smem, tiles);
        k_first_digit_hist<kKmF32S><<<grid, kThreads, smem, s>>>(rows, in, d, ghist);
    } else {
        const int grid = persistent_grid(k_first_digit_hist<kKmF32L>, kThreads, smem, tiles);
        k_first_digit_hist<kKmF32L><<<grid, kThreads, smem, s>>>(rows, in, d, ghist);
    }
}

void launch_scale_decide(int mode, const unsigned long long* hist, uint32_t nbins, uint64_t n, uint64_t k,
                         double tau, const uint32_t* x, uint64_t a_index, uint32_t* out,
                         volatile uint32_t* host_out, cudaStream_t s) {
    k_scale_decide<<<1, 1024, 0, s>>>(mode, hist, nbins, n, k, tau, x, a_index, out, host_out);
}

void launch_remap_idx(uint64_t n, const uint64_t* cand_idx, uint32_t nblocks,
                      const uint64_t* block_start, const uint64_t* shard_base, uint64_t* idx,
                      cudaStream_t s) {
    if (n == 0) return;
    const uint64_t blocks = (n + 255) / 256;
    k_remap_idx<<<static_cast<int>(blocks < 8192 ? blocks : 8192), 256, 0, s>>>(
        n, cand_idx, nblocks, block_start, shard_base, idx);
}

}  // namespace rtk_b200
