// rtk_rows.cu — K6 fast path: one CTA owns one short row (LLM-vocab sampling, small k) and
// finishes it in ONE kernel, entirely in shared memory after a single HBM read of the row.
//
//   1. threshold: stratified 2048-element sample -> in-CTA radix select -> T (composite)
//      (rows with n <= kRowCand skip the sample: T = 0)
//   2. stream the row once (32-byte loads, fused key transform), append K >= T to smem
//   3. exact in-CTA radix select on the candidates: the k-th composite T2, #{K >= T2} == k
//   4. keep exactly k, LSD radix sort them (descending) in smem, write (value, u64 index),
//      pivot
// A row whose sample threshold missed (count < k) or whose candidates overflow the smem
// buffer is flagged and rerun by the host on the general multi-CTA path; correctness never
// depends on the sample. The reference's per-task semantics (batch.hpp:284-291: each task
// equals rtk::topk on its view) hold row by row.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "rtk_device.cuh"
#include "rtk_kernels.h"

namespace rtk_b200 {

constexpr int kRowThreads = 512;
constexpr int kRowWarps = kRowThreads / 32;
constexpr int kRowCand = 8192;    // smem candidate capacity (u64), large-k variant
constexpr int kRowKMax = 4096;    // largest k finished in the CTA
constexpr int kRowCandS = 2048;   // small-k variant (k <= kRowKMaxS): smaller buffer, deeper ring
constexpr int kRowKMaxS = 512;
constexpr int kRowSampleS = 2048;  // sample size of the small variant (64 segments x 32)
constexpr int kRowSampleL = 4096;  // large variant
constexpr int kRowChunk = 2048;   // elements per TMA bulk chunk (8 KB)
#ifndef RTK_ROWS_U
#define RTK_ROWS_U 4
#endif
#ifndef RTK_ROWS_SS
#define RTK_ROWS_SS 2
#endif
#ifndef RTK_ROWS_SL
#define RTK_ROWS_SL 1
#endif
constexpr int kRowU = RTK_ROWS_U;    // 2048-element chunks per ring stage (one TMA copy each)
constexpr int kRowStU = RTK_ROWS_SS; // stages of the small-k variant
constexpr int kRowStLU = RTK_ROWS_SL;  // stages of the large-k variant
#ifndef RTK_ROWS_UL
#define RTK_ROWS_UL RTK_ROWS_U
#endif
constexpr int kRowUL = RTK_ROWS_UL;  // 2048-element chunks per stage, large-k variant
#ifndef RTK_ROWS_SFIRST
#define RTK_ROWS_SFIRST 1
#endif

__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
                 "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// TMA 1-D bulk copy global -> shared, completion signalled on `bar` (expect_tx armed here)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
        "l"(src), "r"(bytes), "r"(b)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(b),
        "r"(parity)
        : "memory");
}

__host__ __device__ __forceinline__ unsigned int rows_digit_hi(unsigned int pos) {
    return pos == 53 ? 64u : (pos == 0 ? 9u : pos + 11u);
}

// Block-wide exclusive scan (kRowThreads) of a u32; *total = sum.
__device__ __forceinline__ uint32_t row_block_scan(uint32_t v, uint32_t* s_w, uint32_t* total) {
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
    for (int w = 0; w < kRowWarps; ++w) {
        const uint32_t x = s_w[w];
        if (w < warp) pre += x;
        tot += x;
    }
    __syncthreads();
    *total = tot;
    return pre + inc - v;
}

// In-CTA radix select over buf[0, m): the composite prefix T such that #{K >= T} ends in
// [k, target] (target == k: exact k-th element). Returns T; *count_ge = #{K >= T}.
// Early stop exactly as select_bin + radix_select (engine.hpp:231-241, 293-312).
__device__ unsigned long long cta_radix_select(const unsigned long long* buf, uint32_t m, uint64_t k,
                                               uint64_t target, uint32_t* hist, uint32_t* s_w,
                                               unsigned long long* s_res, uint64_t* count_ge,
                                               bool skip_const = false) {
    constexpr int per = kBins / kRowThreads;  // 4 bins per thread, thread 0 owns the top bins
    const int tid = threadIdx.x;
    unsigned long long prefix = 0;
    uint64_t k_rem = k, above = 0;
    unsigned int pos = 53;
    // bits where the elements differ: digit windows without any are skipped (their bits are
    // common to all, so they join the prefix as is). 16-bit keys leave bits 32-47 zero and small
    // rows leave the high index bits constant: up to two wasted passes otherwise.
    // (16-bit keys only: for f32 rows the extra reduction measured +1-2.5 us and nothing skips)
    unsigned long long dif = ~0ull;
    const unsigned long long ref = buf[0];
    if (skip_const) {
        dif = 0;
        for (uint32_t i = tid; i < m; i += kRowThreads) dif |= buf[i] ^ ref;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) dif |= __shfl_xor_sync(0xffffffffu, dif, d);
        if (tid == 0) s_res[0] = 0;
        __syncthreads();
        if ((tid & 31) == 0 && dif) atomicOr(&s_res[0], dif);
        __syncthreads();
        dif = s_res[0];
        __syncthreads();
    }
    for (;;) {
        while (pos > 0) {  // skip constant windows
            const unsigned int h = rows_digit_hi(pos);
            const unsigned long long wmask = (h >= 64 ? ~0ull : ((1ull << h) - 1)) & ~((1ull << pos) - 1);
            if (dif & wmask) break;
            prefix |= ref & wmask;
            pos = pos == 9 ? 0u : pos - 11u;
        }
        for (int b = tid; b < kBins; b += kRowThreads) hist[b] = 0;
        __syncthreads();
        const unsigned int hi = rows_digit_hi(pos);
        const unsigned long long pm = hi >= 64 ? 0ull : (prefix >> hi);
        const uint32_t dmask = (1u << (hi - pos)) - 1u;
        for (uint32_t i = tid; i < ((m + 31) & ~31u); i += kRowThreads) {
            const bool in = i < m;
            const unsigned long long K = in ? buf[i] : 0ull;
            // plain shared atomics (+ a whole-warp fast path for tie-heavy rows): __match_any_sync
            // costs more than the conflicts it saves on these mostly spread digits
            const bool v = in && (hi >= 64 || (K >> hi) == pm);
            const uint32_t d = static_cast<uint32_t>(K >> pos) & dmask;
            const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
            if (__all_sync(0xffffffffu, v && d == d0)) {
                if ((threadIdx.x & 31) == 0) atomicAdd(&hist[d0], 32u);
            } else if (v) {
                atomicAdd(&hist[d], 1u);
            }
        }
        __syncthreads();
        uint32_t c[per], sum = 0;
#pragma unroll
        for (int i = 0; i < per; ++i) {
            c[i] = hist[kBins - 1 - (tid * per + i)];
            sum += c[i];
        }
        uint32_t tot;
        const uint32_t before = row_block_scan(sum, s_w, &tot);
        if (tid == 0) s_res[0] = ~0ull;
        __syncthreads();
        if (before < k_rem && before + sum >= k_rem) {
            uint32_t cum = before;
#pragma unroll
            for (int i = 0; i < per; ++i) {
                if (cum + c[i] >= k_rem) {
                    s_res[0] = kBins - 1 - (tid * per + i);
                    s_res[1] = cum;
                    s_res[2] = c[i];
                    break;
                }
                cum += c[i];
            }
        }
        __syncthreads();
        const unsigned long long bin = s_res[0], ab = s_res[1], cb = s_res[2];
        __syncthreads();
        if (bin == ~0ull) {  // cannot happen for k <= m
            *count_ge = 0;
            return 0;
        }
        prefix |= bin << pos;
        above += ab;
        k_rem -= ab;
        const uint64_t cge = above + cb;
        if (cge <= target || pos == 0) {
            *count_ge = cge;
            return prefix;
        }
        pos = pos == 9 ? 0u : pos - 11u;
    }
}

// Warp 0 sorts buf[0, 32*IPL) descending in registers (element lane*IPL + i in x[i]): compare-
// exchanges inside a lane for strides < IPL, shuffles above; no block barrier per stage.
template <int IPL>
__device__ __forceinline__ void warp_bitonic_desc_smem(unsigned long long* buf) {
    const int lane = threadIdx.x & 31;
    constexpr int N = 32 * IPL;
    unsigned long long x[IPL];
#pragma unroll
    for (int i = 0; i < IPL; ++i) x[i] = buf[lane * IPL + i];
#pragma unroll
    for (int kk = 2; kk <= N; kk <<= 1) {
#pragma unroll
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
            if (jj < IPL) {
#pragma unroll
                for (int i = 0; i < IPL; ++i) {
                    if (i & jj) continue;
                    const bool desc = ((lane * IPL + i) & kk) == 0;
                    const unsigned long long u = x[i], v = x[i | jj];
                    const bool sw = desc ? (u < v) : (u > v);
                    x[i] = sw ? v : u;
                    x[i | jj] = sw ? u : v;
                }
            } else {
                const int lm = jj / IPL;
                const bool lo = (lane & lm) == 0;
#pragma unroll
                for (int i = 0; i < IPL; ++i) {
                    const bool desc = ((lane * IPL + i) & kk) == 0;
                    const unsigned long long y = __shfl_xor_sync(0xffffffffu, x[i], lm);
                    x[i] = (desc == lo) ? (x[i] > y ? x[i] : y) : (x[i] < y ? x[i] : y);
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < IPL; ++i) buf[lane * IPL + i] = x[i];
}

// small-k sort: n2 (a power of two) <= 512 composites by one warp in registers
__device__ __forceinline__ void small_sort_desc(unsigned long long* buf, int n2) {
    if (threadIdx.x < 32) {
        if (n2 <= 32) warp_bitonic_desc_smem<1>(buf);
        else if (n2 == 64) warp_bitonic_desc_smem<2>(buf);
        else if (n2 == 128) warp_bitonic_desc_smem<4>(buf);
        else if (n2 == 256) warp_bitonic_desc_smem<8>(buf);
        else warp_bitonic_desc_smem<16>(buf);
    }
    __syncthreads();
}

template <int KM, int CAND, int STAGES, int SAMPLE, int UU>
__device__ __forceinline__ void rows_fused_body(const RowsFusedArgs& a);

template <int KM, int CAND, int STAGES, int SAMPLE, int UU>
__global__ void __launch_bounds__(kRowThreads, 2) k_rows_fused(RowsFusedArgs a) {
    __shared__ uint32_t s_tail;
    resolve_src(a.in);
    rows_fused_body<KM, CAND, STAGES, SAMPLE, UU>(a);
    call_tail(a.tail, &s_tail);  // only when this is the call's last kernel
}

template <int KM, int CAND, int STAGES, int SAMPLE, int UU>
__device__ __forceinline__ void rows_fused_body(const RowsFusedArgs& a) {
    constexpr int kRowCand = CAND;
    constexpr int kRowStages = STAGES;
#ifndef RTK_ROWS_LANE_HITS
#define RTK_ROWS_LANE_HITS 1
#endif
    constexpr bool kLaneHits = RTK_ROWS_LANE_HITS;  // per-lane appends (0: warp-aggregated, for A/B)
    constexpr int kRowSample = SAMPLE;
    extern __shared__ unsigned long long cand[];  // kRowCand entries
    __shared__ uint32_t hist[kBins];
    __shared__ uint32_t s_w[kRowWarps];
    __shared__ unsigned long long s_res[3];
    __shared__ uint32_t s_m;
    __shared__ unsigned long long bar[STAGES];
    __shared__ uint32_t s_empty[STAGES];
    const int j = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned full = 0xffffffffu;
    const uint32_t r = a.rid[j];
    const uint64_t n = a.len[j], off = a.off[j], k = a.k[j];
    constexpr int EB = km_is16<KM>() ? 2 : 4;  // input element bytes
    const char* rowb = reinterpret_cast<const char*>(a.in.base) + off * EB;
    const uint32_t* row = reinterpret_cast<const uint32_t*>(rowb);  // 32-bit element rows only
    auto ld = [&](uint64_t i) -> uint32_t {
        if constexpr (EB == 2) return __ldg(reinterpret_cast<const unsigned short*>(rowb) + i);
        else return __ldg(row + i);
    };
    unsigned long long* dbg = a.dbg;
    int ndbg = 0;
    int ntr = 0;
    auto stamp = [&]() {
        if ((dbg && blockIdx.x == 0 || a.trace) && threadIdx.x == 0 && ndbg < 30) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            if (dbg && blockIdx.x == 0) dbg[ndbg++] = t;
            if (a.trace && ntr < 15) a.trace[blockIdx.x * 16ull + ntr++] = t;
        }
    };
    if (a.trace && threadIdx.x == 0) {
        uint32_t sm;
        asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
        a.trace[blockIdx.x * 16ull + 15] = sm;
    }
    stamp();

    // ---- sample loads first: issued ahead of the ring's bulk copies so they do not queue behind
    // them in the memory system (the threshold is the critical path of the CTA's start)
    constexpr int SQ = kRowSample / kRowThreads;
    const bool sampled = n > static_cast<uint64_t>(kRowCand);
    const uint64_t stride_fp = sampled ? ((n - 32) << 16) / (kRowSample / 32 - 1) : 0;
    uint32_t raw[SQ];
#if RTK_ROWS_SFIRST
    if (sampled) {
#pragma unroll
        for (int q = 0; q < SQ; ++q) {
            const int e = q * kRowThreads + tid;
            raw[q] = ld(((static_cast<uint64_t>(e / 32) * stride_fp) >> 16) + (e & 31));
        }
    }
#endif

    // ---- streaming ring: TMA 1-D bulk copies (cp.async.bulk) of 8 KB chunks into a 4-stage
    // shared-memory ring with mbarrier completion; the first stages are in flight while the
    // threshold is being selected.
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(rowb);
    // elements before 16-byte alignment (a row shorter than that is all head)
    const uint32_t head = static_cast<uint32_t>(min(static_cast<uint64_t>(((16 - (a0 & 15)) & 15) / EB), n));
    const uint64_t body = n > head ? n - head : 0;
    constexpr int U = km_is16<KM>() ? 2 * UU : UU;  // same stage BYTES for 16-bit rows
    constexpr uint32_t kChunk = static_cast<uint32_t>(U) * kRowChunk;  // elements per ring stage
    const uint64_t nchunks = body / kChunk;
    const char* bsrc = rowb + head * EB;
    char* ring = reinterpret_cast<char*>(cand + kRowCand);
    constexpr uint32_t kChunkBytes = kChunk * EB;
    if (tid == 0) {
        for (int st = 0; st < kRowStages; ++st) {
            mbar_init(&bar[st], 1);
            s_empty[st] = 0;
        }
        fence_mbar_init();
    }
    __syncthreads();
    // L2 prefetch `pf` chunks beyond the ring: bytes in flight per SM without shared memory
    auto prefetch = [&](uint64_t c) {
        if (c < nchunks)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(bsrc + c * kChunkBytes),
                         "r"(kChunkBytes) : "memory");
    };
    if (tid == 0) {
        for (uint64_t c = 0; c < nchunks && c < static_cast<uint64_t>(kRowStages); ++c)
            bulk_g2s(ring + c * kChunkBytes, bsrc + c * kChunkBytes, kChunkBytes, &bar[c]);
        // a.pf: L2 prefetch distance kept while streaming; a.pf >> 16: chunks beyond the ring
        // pulled into L2 once at the start (HBM is otherwise idle while the threshold is selected)
        for (uint32_t p = 0; p < (a.pf & 0xFFFFu) + (a.pf >> 16); ++p) prefetch(kRowStages + p);
    }

    // ---- 1. threshold -------------------------------------------------------------------
    stamp();
    unsigned long long T = 0;
    if (sampled) {
#if !RTK_ROWS_SFIRST
        // every sample load issued before the first is used (one memory round trip)
#pragma unroll
        for (int q = 0; q < SQ; ++q) {
            const int e = q * kRowThreads + tid;
            raw[q] = ld(((static_cast<uint64_t>(e / 32) * stride_fp) >> 16) + (e & 31));
        }
#endif
#pragma unroll
        for (int q = 0; q < SQ; ++q) {
            const int e = q * kRowThreads + tid;
            const uint64_t idx = ((static_cast<uint64_t>(e / 32) * stride_fp) >> 16) + (e & 31);
            cand[e] = composite(make_key(a.in, raw[q]), idx);
        }
        __syncthreads();
        const double rr = static_cast<double>(k) * kRowSample / static_cast<double>(n);
        const uint64_t rp = static_cast<uint64_t>(ceil(rr + 4.0 * sqrt(rr) + 3.0));
        uint64_t cge;
        // exact rp-th sample composite: keeps the candidate count (and its spread) minimal
        const uint64_t rpc = rp < kRowSample ? rp : kRowSample;
        T = cta_radix_select(cand, kRowSample, rpc, rpc, hist, s_w, s_res, &cge, km_is16<KM>());
    }
    if (tid == 0) s_m = 0;
    __syncthreads();
    stamp();
    const uint32_t Thi = static_cast<uint32_t>(T >> 32);

    // ---- 2. one streaming read of the row --------------------------------------------------
    auto append = [&](uint32_t mask, const uint32_t* keys, uint32_t (*idx_of)(uint32_t, const void*),
                      const void* ctx) {};
    (void)append;
    // appends up to 4 hits per thread (bit i of mask = element i) with one warp-aggregated
    // shared atomic; idx = ibase + i
    auto push4 = [&](uint32_t mask, const uint32_t (&key)[4], uint32_t ibase) {
        if (!__any_sync(full, mask)) return;
        const uint32_t c = __popc(mask);
        uint32_t inc = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(full, inc, d);
            if (lane >= d) inc += o;
        }
        const uint32_t wtot = __shfl_sync(full, inc, 31);
        uint32_t wbase = 0;
        if (lane == 31) wbase = atomicAdd(&s_m, wtot);
        wbase = __shfl_sync(full, wbase, 31);
        uint32_t o = wbase + inc - c;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if ((mask >> i) & 1u) {
                if (o < kRowCand)
                    cand[o] = (static_cast<unsigned long long>(key[i]) << 32) | ~(ibase + i);
                ++o;
            }
    };
    auto test4 = [&](uint32_t (&key)[4], uint32_t ibase, uint32_t valid) {
        // branch-free 64-bit composite compare (K >= T): two predicated compares per element
        uint32_t mask = 0;
        const uint32_t nb = ~ibase;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            key[i] = key_of<KM>(key[i], a.in);
            const unsigned long long K = (static_cast<unsigned long long>(key[i]) << 32) | (nb - i);
            mask |= static_cast<uint32_t>(K >= T) << i;
        }
        return mask & valid;
    };
    // consume the ring without block barriers: a warp that has read its slice of stage st
    // arrives on the stage's empty counter; the LAST warp to arrive refills the stage (TMA)
    // and re-arms the counter. Warps drift apart by up to the ring depth instead of meeting
    // at a __syncthreads per group. A stage holds U chunks of 2048 elements: 4*U independent
    // elements per thread between two waits (latency hiding with only 16 warps per CTA).
    constexpr int G = U / UU;  // 16-bit rows: the stage is consumed in G groups of UU sub-chunks
    for (uint64_t c = 0; c < nchunks; ++c) {
        const int st = static_cast<int>(c % kRowStages);
        if (a.trace && tid == 0) {  // RTK_ROWS_TRACE: thread 0's time waiting for ring stages
            unsigned long long t0w, t1w;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0w));
            mbar_wait(&bar[st], static_cast<uint32_t>((c / kRowStages) & 1));
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1w));
            a.trace[blockIdx.x * 16ull + 14] += t1w - t0w;
        } else {
            mbar_wait(&bar[st], static_cast<uint32_t>((c / kRowStages) & 1));
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
            uint32_t key[4 * UU];
#pragma unroll
            for (int u = 0; u < UU; ++u) {
                const int su = g * UU + u;
                if constexpr (EB == 2) {
                    const uint2 q = reinterpret_cast<const uint2*>(ring + st * kChunkBytes)[su * kRowThreads + tid];
                    key[4 * u] = q.x & 0xFFFFu; key[4 * u + 1] = q.x >> 16;
                    key[4 * u + 2] = q.y & 0xFFFFu; key[4 * u + 3] = q.y >> 16;
                } else {
                    const uint4 q = reinterpret_cast<const uint4*>(ring + st * kChunkBytes)[su * kRowThreads + tid];
                    key[4 * u] = q.x; key[4 * u + 1] = q.y; key[4 * u + 2] = q.z; key[4 * u + 3] = q.w;
                }
            }
            if (g == G - 1) {  // this warp is done reading the stage
                __syncwarp();
                if (lane == 0) {
                    __threadfence_block();
                    if (atomicAdd(&s_empty[st], 1u) == kRowWarps - 1) {
                        s_empty[st] = 0;
                        __threadfence_block();
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        if (c + kRowStages < nchunks)
                            bulk_g2s(ring + st * kChunkBytes, bsrc + (c + kRowStages) * kChunkBytes, kChunkBytes,
                                     &bar[st]);
                        if (a.pf & 0xFFFFu) prefetch(c + kRowStages + (a.pf & 0xFFFFu) + (a.pf >> 16));
                    }
                }
            }
            // 32-bit pre-filter (key >= T.hi: a superset of K >= T, one compare per element);
            // the exact composite mask only for warps where some element passes it
            bool maybe = false;
#pragma unroll
            for (int e = 0; e < 4 * UU; ++e) {
                key[e] = key_of<KM>(key[e], a.in);
                maybe |= key[e] >= Thi;
            }
            if constexpr (kLaneHits) {
                // a 512-element warp group holds ~2 candidates at k = 50 (~22 at k = 4096), so the
                // warp-aggregated append below ran for nearly every group; here only the lanes
                // that pass the pre-filter compute their composite mask and append with their own
                // shared atomic (no shuffles, no warp-wide work). Measured: C3 k = 50 f32 / bf16
                // -2 / -4 us, k = 4096 -1.5 / -5 us
                if (!maybe) continue;
                uint32_t mask = 0;
#pragma unroll
                for (int u = 0; u < UU; ++u) {
                    const uint32_t nb = ~(head + static_cast<uint32_t>(c * kChunk + (g * UU + u) * 2048) + tid * 4);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const unsigned long long K = (static_cast<unsigned long long>(key[4 * u + i]) << 32) | (nb - i);
                        mask |= static_cast<uint32_t>(K >= T) << (4 * u + i);
                    }
                }
                if (!mask) continue;
                uint32_t o = atomicAdd(&s_m, static_cast<uint32_t>(__popc(mask)));
#pragma unroll
                for (int u = 0; u < UU; ++u) {
                    const uint32_t nb = ~(head + static_cast<uint32_t>(c * kChunk + (g * UU + u) * 2048) + tid * 4);
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if ((mask >> (4 * u + i)) & 1u) {
                            if (o < kRowCand) cand[o] = (static_cast<unsigned long long>(key[4 * u + i]) << 32) | (nb - i);
                            ++o;
                        }
                }
                continue;
            }
            if (!__any_sync(full, maybe)) continue;
            uint32_t mask = 0;
#pragma unroll
            for (int u = 0; u < UU; ++u) {
                const uint32_t nb = ~(head + static_cast<uint32_t>(c * kChunk + (g * UU + u) * 2048) + tid * 4);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const unsigned long long K = (static_cast<unsigned long long>(key[4 * u + i]) << 32) | (nb - i);
                    mask |= static_cast<uint32_t>(K >= T) << (4 * u + i);
                }
            }
            if (__any_sync(full, mask)) {
                const uint32_t cnt = __popc(mask);
                uint32_t inc = cnt;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t o = __shfl_up_sync(full, inc, d);
                    if (lane >= d) inc += o;
                }
                const uint32_t wtot = __shfl_sync(full, inc, 31);
                uint32_t wbase = 0;
                if (lane == 31) wbase = atomicAdd(&s_m, wtot);
                wbase = __shfl_sync(full, wbase, 31);
                uint32_t o = wbase + inc - cnt;
#pragma unroll
                for (int u = 0; u < UU; ++u) {
                    const uint32_t nb = ~(head + static_cast<uint32_t>(c * kChunk + (g * UU + u) * 2048) + tid * 4);
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if ((mask >> (4 * u + i)) & 1u) {
                            if (o < kRowCand) cand[o] = (static_cast<unsigned long long>(key[4 * u + i]) << 32) | (nb - i);
                            ++o;
                        }
                }
            }
        }
    }
    // head (< 4 elements before 16-byte alignment) and tail (< one chunk) with plain loads
    {
        const uint64_t t0 = head + nchunks * kChunk;
        const uint64_t rest = n - t0;  // < kRowChunk + ...
        for (uint64_t b0 = 0; b0 < rest + head; b0 += 4 * kRowThreads) {
            uint32_t key[4];
            uint32_t valid = 0;
            uint32_t ib = 0;
            const uint64_t e = b0 + tid * 4;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                // positions [0, head) then [t0, n)
                const uint64_t g = e + i;
                uint64_t idx = g < head ? g : t0 + (g - head);
                const bool ok = g < head ? true : (g - head) < rest;
                key[i] = ok ? ld(idx) : 0u;
                valid |= static_cast<uint32_t>(ok) << i;
                if (i == 0) ib = static_cast<uint32_t>(idx);
            }
            // indices are not contiguous across the head/tail seam: push one element at a time
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint64_t g = e + i;
                const uint32_t idx = static_cast<uint32_t>(g < head ? g : t0 + (g - head));
                uint32_t one[4] = {key[i], 0u, 0u, 0u};
                const uint32_t m1 = test4(one, idx, (valid >> i) & 1u);
                push4(m1, one, idx);
            }
            (void)ib;
        }
    }
    __syncthreads();
    stamp();
    const uint32_t m = s_m;
    if (m < k || m > static_cast<uint32_t>(kRowCand)) {  // sample missed / overflow: general path
        if (tid == 0) {
            a.row_fail[r] = 1;
            atomicOr(a.flags, kFlagFail);
        }
        return;
    }

    // ---- 3. exact k-th composite among the candidates, keep exactly k ----------------------
    if (m > k) {
        uint64_t cge;
        const unsigned long long T2 = cta_radix_select(cand, m, k, k, hist, s_w, s_res, &cge, km_is16<KM>());
        // compaction to cand[0, k): read everything first, then write
        constexpr int PT = kRowCand / kRowThreads;  // 16
        unsigned long long keep[PT];
        uint32_t km = 0;
#pragma unroll
        for (int q = 0; q < PT; ++q) {
            const uint32_t i = q * kRowThreads + tid;
            keep[q] = (i < m) ? cand[i] : 0ull;
            km |= static_cast<uint32_t>(i < m && keep[q] >= T2) << q;
        }
        if (tid == 0) s_m = 0;
        __syncthreads();
        const uint32_t c = __popc(km);
        uint32_t inc = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o2 = __shfl_up_sync(full, inc, d);
            if (lane >= d) inc += o2;
        }
        const uint32_t wtot = __shfl_sync(full, inc, 31);
        uint32_t wbase = 0;
        if (lane == 31 && wtot) wbase = atomicAdd(&s_m, wtot);
        wbase = __shfl_sync(full, wbase, 31);
        uint32_t o = wbase + inc - c;
#pragma unroll
        for (int q = 0; q < PT; ++q)
            if ((km >> q) & 1u) cand[o++] = keep[q];
        __syncthreads();
    }
    const uint32_t kk = static_cast<uint32_t>(k);
    stamp();

    if (kk <= static_cast<uint32_t>(kRowKMaxS)) {
        // ---- 4'. small k: bitonic sort in smem (pad with 0 = smallest composite) ------------
        int n2 = 32;  // one warp sorts in registers (>= 32 slots)
        while (n2 < static_cast<int>(kk)) n2 <<= 1;
        for (int i = kk + tid; i < n2; i += kRowThreads) cand[i] = 0ull;
        __syncthreads();
        small_sort_desc(cand, n2);
        const uint64_t oo = a.row_out_off[r];
        for (uint32_t p = tid; p < kk; p += kRowThreads) {
            const unsigned long long K = cand[p];
            const uint32_t kv = static_cast<uint32_t>(K >> 32);
            const uint32_t idx = ~static_cast<uint32_t>(K);
            uint32_t val;
            if (a.in.scaled) val = __ldg(row + idx);
            else if (a.in.dtype == kF32) val = decode_f32_bits(kv, a.in.smallest);
            else if (a.in.dtype == kF16) val = decode_f16_bits(kv, a.in.smallest);
            else val = a.in.smallest ? ~kv : kv;
            store_val(a.out_vals, a.in.dtype, oo + p, val);
            a.out_idx[oo + p] = idx;
            if (p == kk - 1 && a.pivots) store_val(a.pivots, a.in.dtype, r, val);
        }
        stamp();
        if (dbg && blockIdx.x == 0 && threadIdx.x == 0) dbg[31] = ndbg;
        return;
    }
    // ---- 4. LSD radix sort of the k survivors (descending), 8 items per thread -------------
    // warp w owns positions [256w, 256w+256); item q of lane l is 256w + 32q + l.
    constexpr int IT = kRowKMax / kRowThreads;  // 8
    unsigned long long key[IT];
    unsigned long long orv = 0;
    // keys relative to the smallest survivor key (order-preserving): the range of the top-k keys
    // of real rows spans fewer bytes than the keys themselves (N(0,1) top 4096 of 128256: 3 of 4)
    uint32_t kmin = 0xFFFFFFFFu;
#pragma unroll
    for (int q = 0; q < IT; ++q) {
        const uint32_t p = warp * 256 + q * 32 + lane;
        key[q] = p < kk ? cand[p] : 0ull;
        if (p < kk) kmin = min(kmin, static_cast<uint32_t>(key[q] >> 32));
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) kmin = min(kmin, __shfl_xor_sync(full, kmin, d));
    __syncthreads();
    if (tid == 0) {
        s_res[0] = 0;
        s_res[1] = 0xFFFFFFFFull;
    }
    __syncthreads();
    if (lane == 0) atomicMin(&s_res[1], static_cast<unsigned long long>(kmin));
    __syncthreads();
    kmin = static_cast<uint32_t>(s_res[1]);
    const unsigned long long kbase = static_cast<unsigned long long>(kmin) << 32;
    const unsigned long long ref = cand[0] - kbase;  // digits equal to ref's everywhere: no-op passes
#pragma unroll
    for (int q = 0; q < IT; ++q) {
        const uint32_t p = warp * 256 + q * 32 + lane;
        if (p < kk) {
            key[q] -= kbase;
            orv |= key[q] ^ ref;
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) orv |= __shfl_xor_sync(full, orv, d);
    if (lane == 0) atomicOr(&s_res[0], orv);
    __syncthreads();
    orv = s_res[0];
    const int nbits = orv ? 64 - __clzll(orv) : 0;
    unsigned long long* tmp = cand + kRowKMax;
    // per-warp digit counters live in the (now idle) streaming ring
    uint32_t (*cnt)[256] = reinterpret_cast<uint32_t (*)[256]>(cand + kRowCand);
    // per-warp peer masks right after them (the large variant's ring holds exactly both)
    uint32_t (*pmask)[256] = cnt + kRowWarps;
    static_assert(STAGES * UU * kRowChunk * sizeof(uint32_t) >= 2 * kRowWarps * 256 * sizeof(uint32_t),
                  "the streaming ring must hold the sort's counters and peer masks");
    const unsigned lt = (1u << lane) - 1u;
    auto lsd = [&](int lo0) {
    for (int lo = lo0; lo < nbits; lo += 8) {
        if (((orv >> lo) & 0xFFull) == 0) continue;  // digit constant across the group: no-op pass
        for (int i = tid; i < kRowWarps * 256; i += kRowThreads) {
            (&cnt[0][0])[i] = 0;
            (&pmask[0][0])[i] = 0;
        }
        __syncthreads();
        uint32_t dig[IT], rk[IT];
#pragma unroll
        for (int q = 0; q < IT; ++q) {
            const uint32_t p = warp * 256 + q * 32 + lane;
            dig[q] = p < kk ? 255u - static_cast<uint32_t>((key[q] >> lo) & 0xFFu) : 255u;
            // peers: each lane ORs its bit into the (warp, digit) mask and reads it back (one
            // shared atomic instead of an 8-ballot multisplit); the lowest peer clears it
            atomicOr(&pmask[warp][dig[q]], 1u << lane);
            __syncwarp();
            const unsigned peers = pmask[warp][dig[q]];
            const uint32_t b0 = cnt[warp][dig[q]];
            rk[q] = b0 + __popc(peers & lt);
            __syncwarp();
            if ((peers & lt) == 0) {
                cnt[warp][dig[q]] = b0 + __popc(peers);
                pmask[warp][dig[q]] = 0u;
            }
            __syncwarp();
        }
        __syncthreads();
        {
            // exclusive scan over (digit, warp): thread t < 256 handles digit t, all warps
            uint32_t cs[kRowWarps], sum = 0;
            if (tid < 256) {
#pragma unroll
                for (int w = 0; w < kRowWarps; ++w) { cs[w] = cnt[w][tid]; sum += cs[w]; }
            }
            uint32_t tot;
            uint32_t pre = row_block_scan(tid < 256 ? sum : 0u, s_w, &tot);
            if (tid < 256) {
#pragma unroll
                for (int w = 0; w < kRowWarps; ++w) { cnt[w][tid] = pre; pre += cs[w]; }
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < IT; ++q) tmp[cnt[warp][dig[q]] + rk[q]] = key[q];
        __syncthreads();
#pragma unroll
        for (int q = 0; q < IT; ++q) key[q] = tmp[warp * 256 + q * 32 + lane];
        __syncthreads();
    }

    };
    // Real keys rarely tie: rank by the KEY bits only, then restore index order inside runs of
    // equal keys with an odd-even transposition (a run of length L settles in <= L rounds);
    // tie-heavy rows fall back to the full composite passes (as cta_sort_group, rtk_sort.cu).
    // 16-bit keys tie in runs of tens (65536 values over ~10^5 elements): full composite passes
    const bool key_only = !km_is16<KM>() && (orv >> 32) != 0 && (orv & 0xffffffffull) != 0;
    lsd(key_only ? 32 : 0);
    if (key_only) {
#pragma unroll
        for (int q = 0; q < IT; ++q) cand[warp * 256 + q * 32 + lane] = key[q];
        __syncthreads();
        bool prev_sw = true, settled = false;
        for (int it = 0; it < 24; ++it) {
            bool sw = false;
            for (uint32_t q = tid; 2 * q + 1 < kk; q += kRowThreads) {
                const uint32_t p = 2 * q + (it & 1);
                if (p + 1 < kk) {
                    const unsigned long long x = cand[p], y = cand[p + 1];
                    if ((x >> 32) == (y >> 32) && x < y) { cand[p] = y; cand[p + 1] = x; sw = true; }
                }
            }
            const bool any = __syncthreads_or(sw);
            if (!any && !prev_sw) { settled = true; break; }
            prev_sw = any;
        }
#pragma unroll
        for (int q = 0; q < IT; ++q) key[q] = cand[warp * 256 + q * 32 + lane];
        __syncthreads();
        if (!settled) lsd(0);  // tie-heavy row: full composite order
    }

    stamp();
    // ---- 5. gather ------------------------------------------------------------------------
    const uint64_t oo = a.row_out_off[r];
#pragma unroll
    for (int q = 0; q < IT; ++q) {
        const uint32_t p = warp * 256 + q * 32 + lane;
        if (p >= kk) continue;
        const unsigned long long K = key[q] + kbase;
        const uint32_t kv = static_cast<uint32_t>(K >> 32);
        const uint32_t idx = ~static_cast<uint32_t>(K);
        uint32_t val;
        if (a.in.scaled) val = __ldg(row + idx);
        else if (a.in.dtype == kF32) val = decode_f32_bits(kv, a.in.smallest);
        else if (a.in.dtype == kF16) val = decode_f16_bits(kv, a.in.smallest);
        else val = a.in.smallest ? ~kv : kv;
        store_val(a.out_vals, a.in.dtype, oo + p, val);
        a.out_idx[oo + p] = idx;
        if (p == kk - 1 && a.pivots) store_val(a.pivots, a.in.dtype, r, val);
    }
    stamp();
    if (dbg && blockIdx.x == 0 && threadIdx.x == 0) dbg[31] = ndbg;
}

template <int KM, int CAND, int STAGES, int SAMPLE, int UU>
static void rows_km(int R, const RowsFusedArgs& a, cudaStream_t s) {
    constexpr size_t smem = CAND * sizeof(unsigned long long) + STAGES * UU * kRowChunk * sizeof(uint32_t);
    static DeviceOnce configured;
    configured([&] {
        cudaFuncSetAttribute(k_rows_fused<KM, CAND, STAGES, SAMPLE, UU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    });
    k_rows_fused<KM, CAND, STAGES, SAMPLE, UU><<<R, kRowThreads, smem, s>>>(a);
}

template <int CAND, int STAGES, int SAMPLE, int UU>
static void rows_variant(int R, const RowsFusedArgs& a, cudaStream_t s) {
    switch (key_mode(a.in.dtype, a.in.smallest, a.in.scaled, a.in.adapt)) {
        case kKmF32L: rows_km<kKmF32L, CAND, STAGES, SAMPLE, UU>(R, a, s); break;
        case kKmF32S: rows_km<kKmF32S, CAND, STAGES, SAMPLE, UU>(R, a, s); break;
        case kKmF32LScaled: rows_km<kKmF32LScaled, CAND, STAGES, SAMPLE, UU>(R, a, s); break;
        case kKmF32SScaled: rows_km<kKmF32SScaled, CAND, STAGES, SAMPLE, UU>(R, a, s); break;
        case kKmU32L: rows_km<kKmU32L, CAND, STAGES, SAMPLE, UU>(R, a, s); break;
        case kKmF16L: rows_km<kKmF16L, CAND, STAGES, SAMPLE, UU>(R, a, s); break;
        case kKmF32LAdapt: rows_km<kKmF32LAdapt, CAND, STAGES, SAMPLE, UU>(R, a, s); break;
        case kKmF32SAdapt: rows_km<kKmF32SAdapt, CAND, STAGES, SAMPLE, UU>(R, a, s); break;
        case kKmF16S: rows_km<kKmF16S, CAND, STAGES, SAMPLE, UU>(R, a, s); break;
        default: rows_km<kKmU32S, CAND, STAGES, SAMPLE, UU>(R, a, s); break;
    }
}

// ---- one long row on a cluster (K6 for single queries, BASELINE C1) ----------------------------
// A single query with 2^18 < n <= 2^21 and k <= 512 is owned by ONE thread-block cluster of
// kRcCs CTAs instead of the four-kernel general path (sample, compaction, MSD, sort): CTA 0
// selects the sample threshold T (the one-CTA kernel's stratified sample + in-CTA radix select)
// while the other CTAs pull their contiguous slices into L2; after a cluster barrier every CTA
// streams its slice once and appends K >= T to CTA 0's shared candidate buffer through
// distributed shared memory (one remote atomic per warp, remote stores of the hits); after a
// second barrier CTA 0 selects exactly k (in-CTA radix select) and sorts them (one warp, in
// registers). A missed sample or an overflow flags the row for the exact path, as k_rows_fused.
// Sorts buf[0, m) (m <= kRowThreads, distinct composites) descending into out[0, m) by rank:
// element i lands at #{j : buf[j] > buf[i]}. P = kRowThreads / pow2ceil(m) threads share one
// element, each counting over j = part (mod P) — consecutive words, no bank conflicts — and
// combine by shuffles. One smem broadcast read per comparison, no barrier per stage.
__device__ __forceinline__ void rank_sort_desc(const unsigned long long* buf, uint32_t m,
                                               unsigned long long* out) {
    uint32_t n2 = 1;
    while (n2 < m) n2 <<= 1;
    const uint32_t P = n2 >= kRowThreads ? 1u : kRowThreads / n2;  // <= 512, power of two
    const uint32_t Pw = P > 32 ? 32u : P;                           // lanes combined per element
    const uint32_t tid = threadIdx.x;
    const uint32_t i = tid / Pw, part = tid % Pw;
    const unsigned long long me = i < m ? buf[i] : 0ull;
    uint32_t cnt = 0;
    if (i < m) {
        uint32_t j = part;
        for (; j + 7 * Pw < m; j += 8 * Pw) {
            unsigned long long b[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) b[q] = buf[j + q * Pw];
#pragma unroll
            for (int q = 0; q < 8; ++q) cnt += b[q] > me;
        }
        for (; j < m; j += Pw) cnt += buf[j] > me;
    }
    for (uint32_t d = 1; d < Pw; d <<= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
    if (i < m && part == 0) out[cnt] = me;
    __syncthreads();
}

constexpr int kRcCs = 16;
constexpr int kRcCand = 8192;
constexpr int kRcSample = 4096;

template <int KM>
__global__ void __cluster_dims__(kRcCs, 1, 1) __launch_bounds__(kRowThreads, 1) k_row_cluster(RowsFusedArgs a) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ unsigned long long cand[];  // kRcCand; CTA 0's is the row's candidate buffer
    __shared__ uint32_t hist[kBins];
    __shared__ uint32_t s_w[kRowWarps];
    __shared__ unsigned long long s_res[3];
    __shared__ uint32_t s_m;
    __shared__ unsigned long long s_T;
    __shared__ uint32_t s_tail;
    resolve_src(a.in);
    const uint32_t crank = cluster.block_rank();
    int ntr = 0;
    auto stamp = [&]() {  // RTK_ROWS_TRACE: CTA 0's phase ends (globaltimer)
        if (a.trace && crank == 0 && threadIdx.x == 0 && ntr < 15) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            a.trace[ntr++] = t;
        }
    };
    stamp();
    const int tid = threadIdx.x, lane = tid & 31;
    const unsigned full = 0xffffffffu;
    const uint32_t r = a.rid[0];
    const uint64_t n = a.len[0], off = a.off[0], k = a.k[0];
    constexpr int EB = km_is16<KM>() ? 2 : 4;
    const char* rowb = reinterpret_cast<const char*>(a.in.base) + off * EB;
    auto ld = [&](uint64_t i) -> uint32_t {
        if constexpr (EB == 2) return __ldg(reinterpret_cast<const unsigned short*>(rowb) + i);
        else return __ldg(reinterpret_cast<const uint32_t*>(rowb) + i);
    };
    // 16-byte vectors over the aligned body [a0, a1) of the row, split evenly over the CTAs; the
    // < VE elements before a0 and after a1 go to the last CTA's first threads
    constexpr int VE = 16 / EB;
    const uintptr_t rb = reinterpret_cast<uintptr_t>(rowb);
    const uint64_t a0 = min(n, static_cast<uint64_t>(((16 - (rb & 15)) & 15) / EB));
    const uint64_t nv = (n - a0) / VE;
    const uint64_t a1 = a0 + nv * VE;
    const uint64_t vper = (nv + kRcCs - 1) / kRcCs;
    const uint64_t v0 = min(nv, crank * vper), v1 = min(nv, v0 + vper);
    const uint4* vrow = reinterpret_cast<const uint4*>(rowb + a0 * EB);
    if (tid == 0) s_m = 0;
    if (tid < 64) {  // L2 prefetch of this CTA's slice: 64 threads x 16 KB bulk prefetches
        const uintptr_t lo = reinterpret_cast<uintptr_t>(vrow + v0), hi = reinterpret_cast<uintptr_t>(vrow + v1);
        for (uintptr_t p = lo + static_cast<uintptr_t>(tid) * 16384; p < hi; p += 64 * 16384) {
            const uint32_t bytes = static_cast<uint32_t>(hi - p < 16384 ? hi - p : 16384);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
        }
    }
    // ---- 1. threshold on CTA 0 (stratified sample, in-CTA radix select of the r'-th) ----------
    if (crank == 0) {
        const uint64_t nseg = kRcSample / 32;
        const uint64_t stride_fp = ((n - 32) << 16) / (nseg - 1);
        uint32_t raw[kRcSample / kRowThreads];
#pragma unroll
        for (int q = 0; q < kRcSample / kRowThreads; ++q) {
            const int e = q * kRowThreads + tid;
            raw[q] = ld(((static_cast<uint64_t>(e / 32) * stride_fp) >> 16) + (e & 31));
        }
#pragma unroll
        for (int q = 0; q < kRcSample / kRowThreads; ++q) {
            const int e = q * kRowThreads + tid;
            const uint64_t idx = ((static_cast<uint64_t>(e / 32) * stride_fp) >> 16) + (e & 31);
            cand[e] = composite(key_of<KM>(raw[q], a.in), idx);
        }
        __syncthreads();
        const double rr = static_cast<double>(k) * kRcSample / static_cast<double>(n);
        const uint64_t rp = static_cast<uint64_t>(ceil(rr + 4.0 * sqrt(rr) + 3.0));
        uint64_t cge;
        const uint64_t rpc = rp < kRcSample ? rp : kRcSample;
        const unsigned long long T = cta_radix_select(cand, kRcSample, rpc, rpc, hist, s_w, s_res, &cge, km_is16<KM>());
        if (tid == 0) s_T = T;
        stamp();
    }
    cluster.sync();
    stamp();
    // ---- 2. stream the slice, hits to CTA 0 through DSMEM ------------------------------------
    const unsigned long long T = *cluster.map_shared_rank(&s_T, 0);
    const uint32_t thi = static_cast<uint32_t>(T >> 32);
    const uint64_t eT = ~static_cast<uint32_t>(T);  // T's element index
    uint32_t* m0 = cluster.map_shared_rank(&s_m, 0);
    unsigned long long* cand0 = cluster.map_shared_rank(cand, 0);
    // one warp's hits (bit i of mask: element e_of(i) with key[i]) appended to CTA 0's buffer
    auto append = [&](const auto& key, uint32_t mask, auto e_of) {
        constexpr int NK = sizeof(key) / sizeof(key[0]);
        const uint32_t c = __popc(mask);
        uint32_t inc = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(full, inc, d);
            if (lane >= d) inc += o;
        }
        const uint32_t wtot = __shfl_sync(full, inc, 31);
        uint32_t wbase = 0;
        if (lane == 31) wbase = atomicAdd(m0, wtot);
        wbase = __shfl_sync(full, wbase, 31);
        uint32_t o = wbase + inc - c;
#pragma unroll
        for (int i = 0; i < NK; ++i)
            if ((mask >> i) & 1u) {
                if (o < static_cast<uint32_t>(kRcCand)) cand0[o] = composite(key[i], e_of(i));
                ++o;
            }
    };
    // 32 elements per thread per step (one 32-bit hit mask): 8 vectors of 4 f32/u32, 4 of 8 halves
    constexpr int RU = 32 / VE;
    constexpr int NE = RU * VE;
    for (uint64_t vb = v0; vb < v1; vb += static_cast<uint64_t>(RU) * kRowThreads) {
        uint4 w[RU];
#pragma unroll
        for (int u = 0; u < RU; ++u) {
            const uint64_t v = vb + static_cast<uint64_t>(u) * kRowThreads + tid;
            w[u] = v < v1 ? __ldg(vrow + v) : make_uint4(0u, 0u, 0u, 0u);
        }
        uint32_t key[NE];
        uint32_t mask = 0;
        // ties at T's key (index eT) are hits iff their index <= eT: decided once for the whole
        // step unless the step's index range straddles eT (at most one step per row)
        const uint64_t lo_e = a0 + vb * VE, hi_e = a0 + (vb + static_cast<uint64_t>(RU) * kRowThreads) * VE - 1;
        if (hi_e <= eT || lo_e > eT) {
            const bool tie_in = hi_e <= eT;
            if (!tie_in && thi == 0xffffffffu) continue;  // nothing above T's key
            const uint32_t ge = tie_in ? thi : thi + 1;
#pragma unroll
            for (int u = 0; u < RU; ++u) {
                const bool ok = vb + static_cast<uint64_t>(u) * kRowThreads + tid < v1;
                const uint32_t wd[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
#pragma unroll
                for (int j = 0; j < VE; ++j) {
                    const uint32_t rawk = EB == 2 ? (wd[j / 2] >> (16 * (j & 1))) & 0xffffu : wd[j];
                    const int i = u * VE + j;
                    key[i] = key_of<KM>(rawk, a.in);
                    mask |= static_cast<uint32_t>(ok && key[i] >= ge) << i;
                }
            }
        } else {
#pragma unroll
            for (int u = 0; u < RU; ++u) {
                const uint64_t v = vb + static_cast<uint64_t>(u) * kRowThreads + tid;
                const uint32_t wd[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
#pragma unroll
                for (int j = 0; j < VE; ++j) {
                    const uint32_t rawk = EB == 2 ? (wd[j / 2] >> (16 * (j & 1))) & 0xffffu : wd[j];
                    const int i = u * VE + j;
                    key[i] = key_of<KM>(rawk, a.in);
                    mask |= static_cast<uint32_t>(v < v1 && composite(key[i], a0 + v * VE + j) >= T) << i;
                }
            }
        }
        if (!__any_sync(full, mask)) continue;
        append(key, mask, [&](int i) {
            return a0 + (vb + static_cast<uint64_t>(i / VE) * kRowThreads + tid) * VE + (i % VE);
        });
    }
    if (crank == kRcCs - 1 && tid < 32) {  // head [0, a0) and tail [a1, n): < 2 VE elements
        const uint64_t nh = a0, nt = n - a1;
        const bool in = static_cast<uint64_t>(lane) < nh + nt;
        const uint64_t e = lane < nh ? lane : a1 + (lane - nh);
        uint32_t key[1];
        key[0] = in ? key_of<KM>(ld(e), a.in) : 0u;
        const uint32_t mask = static_cast<uint32_t>(in && composite(key[0], e) >= T);
        if (__any_sync(full, mask)) append(key, mask, [&](int) { return e; });
    }
    stamp();
    cluster.sync();
    stamp();
    // ---- 3. CTA 0: exactly k, sorted, written -------------------------------------------------
    if (crank == 0) {
        const uint32_t m = s_m;
        if (m < k || m > static_cast<uint32_t>(kRcCand)) {  // sample missed / overflow: exact path
            if (tid == 0) {
                a.row_fail[r] = 1;
                atomicOr(a.flags, kFlagFail);
            }
        } else {
            if (m > k) {
                uint64_t cge;
                // the candidates of one long query span a narrow key range: skip constant windows
                const unsigned long long T2 = cta_radix_select(cand, m, k, k, hist, s_w, s_res, &cge, true);
                constexpr int PT = kRcCand / kRowThreads;
                unsigned long long keep[PT];
                uint32_t km = 0;
#pragma unroll
                for (int q = 0; q < PT; ++q) {
                    const uint32_t i = q * kRowThreads + tid;
                    keep[q] = i < m ? cand[i] : 0ull;
                    km |= static_cast<uint32_t>(i < m && keep[q] >= T2) << q;
                }
                if (tid == 0) s_m = 0;
                __syncthreads();
                const uint32_t c = __popc(km);
                uint32_t inc = c;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t o2 = __shfl_up_sync(full, inc, d);
                    if (lane >= d) inc += o2;
                }
                const uint32_t wtot = __shfl_sync(full, inc, 31);
                uint32_t wbase = 0;
                if (lane == 31 && wtot) wbase = atomicAdd(&s_m, wtot);
                wbase = __shfl_sync(full, wbase, 31);
                uint32_t o = wbase + inc - c;
#pragma unroll
                for (int q = 0; q < PT; ++q)
                    if ((km >> q) & 1u) cand[o++] = keep[q];
                __syncthreads();
            }
            stamp();
            const uint32_t kk = static_cast<uint32_t>(k);
            unsigned long long* sorted = cand + kRcCand / 2;
            rank_sort_desc(cand, kk, sorted);
            stamp();
            const uint64_t oo = a.row_out_off[r];
            for (uint32_t p = tid; p < kk; p += kRowThreads) {
                const unsigned long long K = sorted[p];
                const uint32_t kv = static_cast<uint32_t>(K >> 32);
                const uint32_t idx = ~static_cast<uint32_t>(K);
                uint32_t val;
                if (a.in.scaled) val = ld(idx);
                else if (a.in.dtype == kF32) val = decode_f32_bits(kv, a.in.smallest);
                else if (a.in.dtype == kF16) val = decode_f16_bits(kv, a.in.smallest);
                else val = a.in.smallest ? ~kv : kv;
                store_val(a.out_vals, a.in.dtype, oo + p, val);
                a.out_idx[oo + p] = idx;
                if (p == kk - 1 && a.pivots) store_val(a.pivots, a.in.dtype, r, val);
            }
        }
    }
    stamp();
    if (a.trace && crank == 0 && threadIdx.x == 0) {
        uint32_t sm;
        asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
        a.trace[15] = sm;
    }
    call_tail(a.tail, &s_tail);
}

template <int KM>
static void row_cluster_km(const RowsFusedArgs& a, cudaStream_t s) {
    constexpr size_t smem = kRcCand * sizeof(unsigned long long);
    static DeviceOnce configured;
    configured([&] {
        cudaFuncSetAttribute(k_row_cluster<KM>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        cudaFuncSetAttribute(k_row_cluster<KM>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    });
    k_row_cluster<KM><<<kRcCs, kRowThreads, smem, s>>>(a);
}

void launch_row_cluster(const RowsFusedArgs& a, cudaStream_t s) {
    switch (key_mode(a.in.dtype, a.in.smallest, a.in.scaled, a.in.adapt)) {
        case kKmF32L: row_cluster_km<kKmF32L>(a, s); break;
        case kKmF32S: row_cluster_km<kKmF32S>(a, s); break;
        case kKmF32LScaled: row_cluster_km<kKmF32LScaled>(a, s); break;
        case kKmF32SScaled: row_cluster_km<kKmF32SScaled>(a, s); break;
        case kKmU32L: row_cluster_km<kKmU32L>(a, s); break;
        case kKmF16L: row_cluster_km<kKmF16L>(a, s); break;
        case kKmF32LAdapt: row_cluster_km<kKmF32LAdapt>(a, s); break;
        case kKmF32SAdapt: row_cluster_km<kKmF32SAdapt>(a, s); break;
        case kKmF16S: row_cluster_km<kKmF16S>(a, s); break;
        default: row_cluster_km<kKmU32S>(a, s); break;
    }
}

uint32_t row_cluster_kmax() { return kRowKMaxS; }

// small = rows whose k and expected candidate count fit the small-buffer variant
void launch_rows_fused(int R, const RowsFusedArgs& a, bool small, cudaStream_t s) {
    if (R <= 0) return;
    if (small) rows_variant<kRowCandS, kRowStU, kRowSampleS, kRowU>(R, a, s);
    else rows_variant<kRowCand, kRowStLU, kRowSampleL, kRowUL>(R, a, s);
}

uint32_t rows_fused_kmax(bool small) { return small ? kRowKMaxS : kRowKMax; }
uint32_t rows_fused_cand(bool small) { return small ? kRowCandS : kRowCand; }
uint32_t rows_fused_sample(bool small) { return small ? kRowSampleS : kRowSampleL; }

}  // namespace rtk_b200
