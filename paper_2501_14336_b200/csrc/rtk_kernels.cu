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
#include <cuda_runtime.h>

#include "rtk_device.cuh"
#include "rtk_kernels.h"

namespace rtk_b200 {

__host__ __device__ __forceinline__ unsigned int digit_hi(unsigned int pos) {
    return pos == 53 ? 64u : (pos == 0 ? 9u : pos + 11u);
}
__host__ __device__ __forceinline__ unsigned int next_pos(unsigned int pos) {
    return pos == 9 ? 0u : pos - 11u;
}

// ----------------------------------------------------------------------------------------
// Block-wide helpers (kThreads = 256 = 8 warps)
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long warp_incl_scan(unsigned long long v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        unsigned long long o = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += o;
    }
    return v;
}

// Exclusive scan across the block; returns this thread's exclusive prefix, *total = sum.
__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v,
                                                              unsigned long long* s_warp,
                                                              unsigned long long* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned long long inc = warp_incl_scan(v);
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    unsigned long long wbase = 0, tot = 0;
    for (int w = 0; w < nw; ++w) {
        unsigned long long x = s_warp[w];
        if (w < warp) wbase += x;
        tot += x;
    }
    __syncthreads();
    *total = tot;
    return wbase + inc - v;
}

// ----------------------------------------------------------------------------------------
// Input tile loading: 4 x 32-byte loads per thread, scalar head/tail. Element (u, i) of a
// thread sits at span position p_u + i, p_u = span0 + (u * kThreads + tid) * 8; the row's
// element index is span position - lead.
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ void load_input_tile(const uint32_t* row_ptr, uint64_t span_len,
                                                uint32_t lead, uint64_t span0,
                                                uint32_t (&v)[kUnroll][kVec]) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
        const uint64_t p = span0 + static_cast<uint64_t>(u * kThreads + threadIdx.x) * kVec;
        if (p >= lead && p + kVec <= span_len) {
            ldg256(row_ptr + p, v[u]);
        } else {
#pragma unroll
            for (int i = 0; i < kVec; ++i) {
                const uint64_t q = p + i;
                v[u][i] = (q >= lead && q < span_len) ? __ldg(row_ptr + q) : 0u;
            }
        }
    }
}

// u64 tiles use the same span convention: ptr is 32-byte aligned, element e of the row sits
// at span position e + lead (lead = row start's offset inside its 32-byte sector).
// Same as load_input_tile, but addressed from the tile's own (32-byte aligned) start with the
// tile-local validity window [vlo, vhi): 32-bit index math only.
__device__ __forceinline__ void load_tile_local(const uint32_t* tile_ptr, uint32_t vlo, uint32_t vhi,
                                                uint32_t (&v)[kUnroll][kVec]) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
        const uint32_t l = (u * kThreads + threadIdx.x) * kVec;
        if (l >= vlo && l + kVec <= vhi) {
            ldg256(tile_ptr + l, v[u]);
        } else {
#pragma unroll
            for (int i = 0; i < kVec; ++i)
                v[u][i] = (l + i >= vlo && l + i < vhi) ? __ldg(tile_ptr + l + i) : 0u;
        }
    }
}

__device__ __forceinline__ void load_u64_tile(const uint64_t* ptr, uint64_t span_len, uint32_t lead,
                                              uint64_t e0, uint64_t (&v)[4][kVec64]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const uint64_t p = e0 + static_cast<uint64_t>(u * kThreads + threadIdx.x) * kVec64;
        if (p >= lead && p + kVec64 <= span_len) {
            ldg256_u64(ptr + p, v[u]);
        } else {
#pragma unroll
            for (int i = 0; i < kVec64; ++i) {
                const uint64_t q = p + i;
                v[u][i] = (q >= lead && q < span_len) ? __ldg(ptr + q) : 0ull;
            }
        }
    }
}

// smem histogram increment with a whole-warp fast path: adversarial inputs put every
// element of a warp into one bin (engine_test.cpp:45-56, C4), which would otherwise
// serialise 32 same-address shared atomics.
__device__ __forceinline__ void hist_add(uint32_t* h, uint32_t digit, bool valid) {
    const unsigned full = 0xffffffffu;
    const uint32_t d0 = __shfl_sync(full, digit, 0);
    const bool v0 = __shfl_sync(full, valid ? 1 : 0, 0);
    if (__all_sync(full, valid && digit == d0) && v0) {
        if ((threadIdx.x & 31) == 0) atomicAdd(&h[d0], 32u);
    } else {
        // clustered digits (e.g. the top digit of Uniform[0,1) keys lands in ~8 bins): one
        // shared atomic per distinct digit of the warp instead of one per lane
        const unsigned act = __ballot_sync(full, valid);
        if (valid) {
            const unsigned peers = __match_any_sync(act, digit);
            if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[digit], __popc(peers));
        }
    }
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
    s.pad = 0;
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
            load_input_tile(in.base + off - lead, span_len, lead, span0, v);
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

// ----------------------------------------------------------------------------------------
// k_sample_gather: stratified sample. Row j contributes nseg[j] segments of 32 contiguous
// elements spread evenly over the row; one warp per segment writes 32 composites.
// ----------------------------------------------------------------------------------------
__global__ void k_sample_gather(Rows rows, InputSrc in, const uint64_t* sample_off,
                                const uint64_t* nseg_start, uint64_t* samples) {
    const uint64_t total = nseg_start[rows.R];
    const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
    const int lane = threadIdx.x & 31;
    for (uint64_t g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < total; g += warps) {
        int lo = 0, hi = rows.R - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (nseg_start[mid] <= g) lo = mid; else hi = mid - 1;
        }
        const int j = lo;
        const uint64_t s = g - nseg_start[j];
        const uint64_t nseg = nseg_start[j + 1] - nseg_start[j];
        const uint64_t n = rows.len[j];
        const uint64_t start = (s * (n - 32)) / (nseg > 1 ? nseg - 1 : 1);
        const uint64_t idx = start + lane;
        const uint32_t raw = __ldg(in.base + rows.off[j] + idx);
        samples[sample_off[j] + s * 32 + lane] = composite(make_key(in, raw), idx);
    }
}

// T[rid] = key-level threshold from the resolved sample selection (or 0 = take all).
__global__ void k_set_threshold(int R, const uint32_t* rid, const uint32_t* sampled,
                                const RowSel* sel, uint64_t* T) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= R) return;
    const uint32_t r = rid[j];
    T[r] = sampled[j] ? (sel[r].T & 0xFFFFFFFF00000000ull) : 0ull;
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

template <int KM>
__global__ void __launch_bounds__(kThreads, 4) k_compact(Rows rows, InputSrc in, const uint64_t* T,
                                                         uint64_t* cand, const uint64_t* cand_off,
                                                         const uint64_t* cap,
                                                         unsigned long long* count,
                                                         unsigned long long* kmin,
                                                         unsigned long long* kmax) {
    __shared__ unsigned long long stage_all[kThreads / 32][kWarpStage];
    const uint64_t ntiles = rows.tile_start[rows.R];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned full = 0xffffffffu;
    const unsigned lt_mask = (1u << lane) - 1u;
    unsigned long long* stage = stage_all[warp];

    int cur = -1;
    unsigned long long thr = 0, mn = ~0ull, mx = 0;
    uint32_t thi = 0, tlo = 0, wcur = 0;
    uint64_t off = 0, len = 0, coff = 0, ccap = 0, tile0 = 0, tile1 = 0;
    uint32_t lead = 0, r = 0;

    auto warp_flush = [&]() {  // warp-uniform
        if (wcur == 0) return;
        __syncwarp();
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(count + r, static_cast<unsigned long long>(wcur));
        base = __shfl_sync(full, base, 0);
        for (uint32_t i = lane; i < wcur; i += 32) {
            const unsigned long long K = stage[i];
            mn = min(mn, K);
            mx = max(mx, K);
            if (base + i < ccap) cand[coff + base + i] = K;
        }
        __syncwarp();
        wcur = 0;
    };
    auto finish_row = [&]() {
        warp_flush();
        unsigned long long a = mn, b = mx;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            a = min(a, __shfl_xor_sync(full, a, d));
            b = max(b, __shfl_xor_sync(full, b, d));
        }
        if (lane == 0 && a <= b) { atomicMin(kmin + r, a); atomicMax(kmax + r, b); }
        mn = ~0ull;
        mx = 0;
    };

    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        if (t >= tile1 || cur < 0) {
            if (cur >= 0) finish_row();
            const int j = row_of_tile(rows, t);
            cur = j;
            r = rows.rid[j];
            thr = T[r];
            thi = static_cast<uint32_t>(thr >> 32);
            tlo = static_cast<uint32_t>(thr);
            off = rows.off[j];
            len = rows.len[j];
            lead = rows.lead[j];
            coff = cand_off[r];
            ccap = cap[r];
            tile0 = rows.tile_start[j];
            tile1 = rows.tile_start[j + 1];
        }
        const uint64_t span0 = (t - tile0) * kTile;
        const uint64_t span_len = len + lead;
        // validity window of this tile in tile-local positions (32-bit math from here on)
        const uint32_t vlo = span0 >= lead ? 0u : static_cast<uint32_t>(lead - span0);
        const uint32_t vhi = static_cast<uint32_t>(span_len - span0 < kTile ? span_len - span0 : kTile);
        const uint32_t idx0 = static_cast<uint32_t>(span0 - lead);  // low 32 bits of the row index
        uint32_t v[kUnroll][kVec];
        load_tile_local(in.base + off - lead + span0, vlo, vhi, v);

        // pass 1: key transform + per-thread hit mask (bit u*8+i)
        uint32_t mask = 0;
        if (vlo == 0 && vhi == kTile) {
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                for (int i = 0; i < kVec; ++i) {
                    const uint32_t key = key_of<KM>(v[u][i], in.a_s);
                    v[u][i] = key;
                    mask |= static_cast<uint32_t>(key >= thi) << (u * kVec + i);
                }
        } else {
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                for (int i = 0; i < kVec; ++i) {
                    const uint32_t key = key_of<KM>(v[u][i], in.a_s);
                    v[u][i] = key;
                    const uint32_t l = (u * kThreads + threadIdx.x) * kVec + i;
                    mask |= static_cast<uint32_t>(key >= thi && l >= vlo && l < vhi) << (u * kVec + i);
                }
        }
        // exact composite compare: only differs from key >= T.hi when T.lo != 0 (exact path)
        if (tlo != 0) {
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
        if (wtot <= kWarpStage) {
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
            if (lane == 0) base = atomicAdd(count + r, static_cast<unsigned long long>(wtot));
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
                        if (base < ccap) cand[coff + base] = K;
                        ++base;
                    }
                }
        }
    }
    if (cur >= 0) finish_row();
}

// ----------------------------------------------------------------------------------------
// MSD partition (for candidate sets larger than one CTA's smem sort):
// k_seg_hist:    2048-bin histogram of digit (K >> pos[s]) & 2047 per segment.
// k_seg_scatter: writes every element whose bucket is kept (bstart != ~0u) to
//                dst[off + bstart[b] + slot]; slots are reserved per (tile, bucket) with one
//                global atomic each, then handed out from smem (warp/CTA aggregated).
// ----------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_seg_hist(Rows segs, const uint32_t* pos,
                                                       const uint64_t* src, uint32_t* ghist) {
    __shared__ uint32_t h[kBins];
    for (int b = threadIdx.x; b < kBins; b += kThreads) h[b] = 0;
    __syncthreads();
    const uint64_t ntiles = segs.tile_start[segs.R];
    int cur = -1;
    uint64_t off = 0, len = 0;
    uint32_t lead = 0;
    unsigned int p = 0;
    auto flush = [&](int j) {
        __syncthreads();
        for (int b = threadIdx.x; b < kBins; b += kThreads) {
            if (h[b]) { atomicAdd(ghist + static_cast<uint64_t>(j) * kBins + b, h[b]); h[b] = 0; }
        }
        __syncthreads();
    };
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int j = row_of_tile(segs, t);
        if (j != cur) {
            if (cur >= 0) flush(cur);
            cur = j;
            off = segs.off[j];
            len = segs.len[j];
            lead = segs.lead[j];
            p = pos[j];
        }
        const uint64_t e0 = (t - segs.tile_start[j]) * kTile64;
        const uint64_t span_len = len + lead;
        uint64_t v[4][kVec64];
        load_u64_tile(src + off - lead, span_len, lead, e0, v);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int i = 0; i < kVec64; ++i) {
                const uint64_t q = e0 + static_cast<uint64_t>(u * kThreads + threadIdx.x) * kVec64 + i;
                hist_add(h, static_cast<uint32_t>(v[u][i] >> p) & (kBins - 1), q >= lead && q < span_len);
            }
    }
    if (cur >= 0) flush(cur);
}

__global__ void __launch_bounds__(kThreads) k_seg_scatter(Rows segs, const uint32_t* pos,
                                                          const uint64_t* src, uint64_t* dst,
                                                          const uint32_t* bstart,
                                                          uint32_t* gcursor) {
    __shared__ uint32_t h[kBins];
    __shared__ uint32_t base[kBins];
    const uint64_t ntiles = segs.tile_start[segs.R];
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int j = row_of_tile(segs, t);
        const uint64_t off = segs.off[j], len = segs.len[j];
        const uint32_t lead = segs.lead[j];
        const uint64_t span_len = len + lead;
        const unsigned int p = pos[j];
        const uint32_t* bs = bstart + static_cast<uint64_t>(j) * kBins;
        uint32_t* gc = gcursor + static_cast<uint64_t>(j) * kBins;
        for (int b = threadIdx.x; b < kBins; b += kThreads) h[b] = 0;
        __syncthreads();
        const uint64_t e0 = (t - segs.tile_start[j]) * kTile64;
        uint64_t v[4][kVec64];
        uint32_t slot[4][kVec64];
        load_u64_tile(src + off - lead, span_len, lead, e0, v);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int i = 0; i < kVec64; ++i) {
                const uint64_t q = e0 + static_cast<uint64_t>(u * kThreads + threadIdx.x) * kVec64 + i;
                const uint32_t d = static_cast<uint32_t>(v[u][i] >> p) & (kBins - 1);
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
                    const uint32_t d = static_cast<uint32_t>(v[u][i] >> p) & (kBins - 1);
                    dst[off + base[d] + slot[u][i]] = v[u][i];
                }
            }
        __syncthreads();
    }
}

// ----------------------------------------------------------------------------------------
// k_sort_groups<CAP>: one CTA per group of <= CAP composites. Bitonic sort (descending) in
// shared memory, then the gather: rank = rank_base + position; ranks < k are written as
// value bits (decoded from the key, or re-read from the original input for scaled runs,
// scaling.hpp:74-75) and the u64 row-local index (engine.hpp:106).
// ----------------------------------------------------------------------------------------
template <int CAP, int NT>
__global__ void __launch_bounds__(NT) k_sort_groups(SortGroups g) {
    extern __shared__ unsigned long long sk[];
    const SortGroup grp = g.groups[blockIdx.x];
    const uint32_t len = grp.len;
    const unsigned long long* src = g.buf + grp.off;
    int n2 = 1;
    while (n2 < static_cast<int>(len)) n2 <<= 1;
    for (int i = threadIdx.x; i < n2; i += NT) sk[i] = i < static_cast<int>(len) ? src[i] : 0ull;
    __syncthreads();
    for (int k = 2; k <= n2; k <<= 1) {
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int i = threadIdx.x; i < (n2 >> 1); i += NT) {
                const int lo = ((i & ~(jj - 1)) << 1) | (i & (jj - 1));
                const int hi = lo + jj;
                const unsigned long long a = sk[lo], b = sk[hi];
                const bool desc = (lo & k) == 0;
                if (desc ? (a < b) : (a > b)) { sk[lo] = b; sk[hi] = a; }
            }
            __syncthreads();
        }
    }
    const uint32_t r = grp.rid;
    const uint64_t kr = g.row_k[r];
    const uint64_t oo = g.row_out_off[r];
    for (int i = threadIdx.x; i < static_cast<int>(len); i += NT) {
        const uint64_t rank = grp.rank_base + i;
        if (rank >= kr) continue;
        const unsigned long long K = sk[i];
        const uint32_t key = static_cast<uint32_t>(K >> 32);
        const uint32_t idx = ~static_cast<uint32_t>(K);
        uint32_t val;
        if (g.gather) val = __ldg(g.in_base + g.row_in_off[r] + idx);
        else if (g.dtype == kF32) val = decode_f32_bits(key, g.smallest);
        else val = g.smallest ? ~key : key;
        g.out_vals[oo + rank] = val;
        g.out_idx[oo + rank] = idx;
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
__global__ void __launch_bounds__(kThreads) k_first_digit_hist(Rows rows, InputSrc in,
                                                               unsigned int d,
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
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        uint32_t v[kUnroll][kVec];
        const uint64_t span0 = t * kTile, span_len = len + lead;
        load_input_tile(in.base + off - lead, span_len, lead, span0, v);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
#pragma unroll
            for (int i = 0; i < kVec; ++i) {
                const uint64_t q = span0 + static_cast<uint64_t>(u * kThreads + threadIdx.x) * kVec + i;
                const bool valid = q >= lead && q < span_len;
                const uint32_t dig = make_key(in, v[u][i]) >> (32 - d);
                if (use_smem) hist_add(hs, dig, valid);
                else if (valid) atomicAdd(ghist + dig, 1ull);
            }
    }
    if (use_smem) {
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < nb; b += kThreads)
            if (hs[b]) atomicAdd(ghist + b, static_cast<unsigned long long>(hs[b]));
    }
}

// ----------------------------------------------------------------------------------------
// Launchers. Streaming kernels run as persistent grids: resident CTAs per SM (occupancy API)
// x SM count, capped by the tile count.
// ----------------------------------------------------------------------------------------
static int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

template <typename K>
static int persistent_grid(K kernel, int threads, size_t smem, uint64_t tiles) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
    if (occ <= 0) occ = 1;
    const uint64_t g = static_cast<uint64_t>(occ) * num_sms();
    return static_cast<int>(tiles < g ? (tiles ? tiles : 1) : g);
}

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

void launch_sample_gather(uint64_t segments, const Rows& rows, const InputSrc& in,
                          const uint64_t* sample_off, const uint64_t* nseg_start, uint64_t* samples,
                          cudaStream_t s) {
    const uint64_t blocks = (segments + 7) / 8;  // 8 warps per CTA, one segment per warp
    const int grid = static_cast<int>(blocks < 4096 ? (blocks ? blocks : 1) : 4096);
    k_sample_gather<<<grid, 256, 0, s>>>(rows, in, sample_off, nseg_start, samples);
}

void launch_set_threshold(int R, const uint32_t* rid, const uint32_t* sampled, const RowSel* sel,
                          uint64_t* T, cudaStream_t s) {
    if (R > 0) k_set_threshold<<<(R + 255) / 256, 256, 0, s>>>(R, rid, sampled, sel, T);
}

template <int KM>
static void compact_km(uint64_t tiles, const Rows& rows, const InputSrc& in, const uint64_t* T,
                       uint64_t* cand, const uint64_t* cand_off, const uint64_t* cap,
                       unsigned long long* count, unsigned long long* kmin, unsigned long long* kmax,
                       cudaStream_t s) {
    const int grid = persistent_grid(k_compact<KM>, kThreads, 0, tiles);
    k_compact<KM><<<grid, kThreads, 0, s>>>(rows, in, T, cand, cand_off, cap, count, kmin, kmax);
}

void launch_compact(uint64_t tiles, const Rows& rows, const InputSrc& in, const uint64_t* T,
                    uint64_t* cand, const uint64_t* cand_off, const uint64_t* cap,
                    unsigned long long* count, unsigned long long* kmin, unsigned long long* kmax,
                    cudaStream_t s) {
    switch (key_mode(in.dtype, in.smallest, in.scaled)) {
        case kKmF32L: compact_km<kKmF32L>(tiles, rows, in, T, cand, cand_off, cap, count, kmin, kmax, s); break;
        case kKmF32S: compact_km<kKmF32S>(tiles, rows, in, T, cand, cand_off, cap, count, kmin, kmax, s); break;
        case kKmF32LScaled: compact_km<kKmF32LScaled>(tiles, rows, in, T, cand, cand_off, cap, count, kmin, kmax, s); break;
        case kKmF32SScaled: compact_km<kKmF32SScaled>(tiles, rows, in, T, cand, cand_off, cap, count, kmin, kmax, s); break;
        case kKmU32L: compact_km<kKmU32L>(tiles, rows, in, T, cand, cand_off, cap, count, kmin, kmax, s); break;
        default: compact_km<kKmU32S>(tiles, rows, in, T, cand, cand_off, cap, count, kmin, kmax, s); break;
    }
}

void launch_seg_hist(uint64_t tiles, const Rows& segs, const uint32_t* pos, const uint64_t* src,
                     uint32_t* ghist, cudaStream_t s) {
    const int grid = persistent_grid(k_seg_hist, kThreads, 0, tiles);
    k_seg_hist<<<grid, kThreads, 0, s>>>(segs, pos, src, ghist);
}

void launch_seg_scatter(uint64_t tiles, const Rows& segs, const uint32_t* pos, const uint64_t* src,
                        uint64_t* dst, const uint32_t* bstart, uint32_t* gcursor, cudaStream_t s) {
    const int grid = persistent_grid(k_seg_scatter, kThreads, 0, tiles);
    k_seg_scatter<<<grid, kThreads, 0, s>>>(segs, pos, src, dst, bstart, gcursor);
}

template <int CAP, int NT>
static void sort_groups_cap(int ngroups, const SortGroups& g, cudaStream_t s) {
    constexpr size_t smem = static_cast<size_t>(CAP) * sizeof(unsigned long long);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_sort_groups<CAP, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        configured = true;
    }
    k_sort_groups<CAP, NT><<<ngroups, NT, smem, s>>>(g);
}

void launch_sort_groups(int cap, int ngroups, const SortGroups& g, cudaStream_t s) {
    if (ngroups <= 0) return;
    if (cap <= 1024) sort_groups_cap<1024, 256>(ngroups, g, s);
    else if (cap <= 2048) sort_groups_cap<2048, 256>(ngroups, g, s);
    else if (cap <= 4096) sort_groups_cap<4096, 512>(ngroups, g, s);
    else if (cap <= 8192) sort_groups_cap<8192, 1024>(ngroups, g, s);
    else sort_groups_cap<16384, 1024>(ngroups, g, s);
}

void launch_pivots(int R, const uint64_t* row_out_off, const uint64_t* row_k, const uint32_t* vals,
                   uint32_t* pivots, cudaStream_t s) {
    if (R > 0) k_pivots<<<(R + 255) / 256, 256, 0, s>>>(R, row_out_off, row_k, vals, pivots);
}

void launch_first_digit_hist(uint64_t tiles, const Rows& rows, const InputSrc& in, unsigned int d,
                             unsigned long long* ghist, cudaStream_t s) {
    const size_t smem = d <= 13 ? (static_cast<size_t>(1) << d) * sizeof(uint32_t) : 0;
    const int grid = persistent_grid(k_first_digit_hist, kThreads, smem, tiles);
    k_first_digit_hist<<<grid, kThreads, smem, s>>>(rows, in, d, ghist);
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
