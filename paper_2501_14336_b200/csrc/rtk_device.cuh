// rtk_device.cuh — device-side types shared by the sm_100a radix top-k kernels.
//
// Every selection runs on a 64-bit COMPOSITE key
//     K(i) = (u64)encode(x_i) << 32 | (u32)~i          (i = row-local index, n <= 2^32)
// encode() is the reference's order-preserving map (keycodec.hpp:55-81). Sorting K
// descending is exactly the reference's canonical order (key desc, index asc;
// engine.hpp:402-411), and K is unique per element, so "the k largest K" is exactly the
// reference result including its tie rule (pivot-equal elements by ascending index,
// engine.hpp:387-396) — no separate tie pass exists anywhere in this design.
#pragma once
#include <cstdint>

namespace rtk_b200 {

constexpr int kThreads = 256;          // streaming kernels
constexpr int kVec = 8;                // 8 x u32 = one 32-byte LDG.256
constexpr int kUnroll = 4;             // 4 loads in flight per thread per tile
constexpr int kTile = kThreads * kVec * kUnroll;  // 8192 input elements per tile
constexpr int kVec64 = 4;              // 4 x u64 = 32 bytes
constexpr int kTile64 = kThreads * kVec64 * 4;    // 4096 composites per tile
constexpr int kDigit = 11;             // radix digit width for the 64-bit composite
constexpr int kBins = 1 << kDigit;
constexpr int kStageCap = 4096;        // compaction staging buffer (u64), 32 KB smem

// kF16: any 16-bit IEEE-style float (f16 or bf16 — the order-preserving map is the same bit
// manipulation); its 16-bit key sits in the HIGH half of the 32-bit key, so every selection /
// ordering stage works on the same 32-bit keys and 64-bit composites as for f32.
enum : int { kF32 = 0, kU32 = 1, kF16 = 2 };

__host__ __device__ __forceinline__ int elem_bytes(int dtype) { return dtype == kF16 ? 2 : 4; }

// Selection state of one row (one query, one sample, or one MSD segment).
// Digits are examined MSD-first at bit positions 53, 42, 31, 20, 9, 0 of K.
struct RowSel {
    unsigned long long prefix;   // selected composite bits above `pos`
    unsigned long long k_rem;    // rank still to place inside the current range
    unsigned long long above;    // elements strictly above the current range
    unsigned long long T;        // threshold: candidates are K >= T
    unsigned long long count_ge; // #{K >= T}
    unsigned long long target;   // resolve once count_ge <= target
    unsigned int pos;            // low bit of the next digit
    unsigned int status;         // 0 active, 1 resolved, 2 rank error
    unsigned int ticket;         // CTAs that finished this pass
    unsigned int passes;         // digit passes this row took
};

// Per-launch row list (device arrays). Launch row j maps to state row rid[j].
struct Rows {
    int R;
    const uint32_t* rid;
    const uint64_t* off;         // element offset (input words or u64 buffer)
    const uint64_t* len;         // elements
    const uint32_t* lead;        // input only: elements before `off` in the first 32-B sector
    const uint64_t* tile_start;  // R+1 exclusive prefix of tiles
};

struct InputSrc {
    const uint32_t* base;
    int dtype;
    int smallest;
    int scaled;
    float a_s;
    // scaled_topk decided on the device (ScaleMode::Adaptive / Always): {scale flag, a_s bits},
    // written by k_scale_decide; every kernel resolves it once at its start (resolve_src)
    const uint32_t* adapt;
};

#ifdef __CUDACC__
__device__ __forceinline__ void resolve_src(InputSrc& s) {
    if (s.adapt) {
        s.scaled = static_cast<int>(__ldcg(s.adapt));
        s.a_s = __uint_as_float(__ldcg(s.adapt + 1));
    }
}
#endif

__device__ __forceinline__ uint32_t encode_f32_bits(uint32_t raw, bool smallest) {
    // KeyCodec<float>::encode, keycodec.hpp:57-62
    uint32_t bits = (raw & 0x80000000u) ? ~raw : (raw | 0x80000000u);
    return smallest ? ~bits : bits;
}

__device__ __forceinline__ uint32_t decode_f32_bits(uint32_t bits, bool smallest) {
    // KeyCodec<float>::decode, keycodec.hpp:64-69
    if (smallest) bits = ~bits;
    return (bits & 0x80000000u) ? (bits ^ 0x80000000u) : ~bits;
}

// KeyCodec for 16-bit floats (the f32 map, keycodec.hpp:57-62, on 16 bits), placed in the high half
__device__ __forceinline__ uint32_t encode_f16_key(uint32_t raw16, bool smallest) {
    uint32_t bits = (raw16 & 0x8000u) ? (~raw16 & 0xFFFFu) : (raw16 | 0x8000u);
    if (smallest) bits = ~bits & 0xFFFFu;
    return bits << 16;
}

__device__ __forceinline__ uint32_t decode_f16_bits(uint32_t key, bool smallest) {
    uint32_t bits = key >> 16;
    if (smallest) bits = ~bits & 0xFFFFu;
    return (bits & 0x8000u) ? (bits ^ 0x8000u) : (~bits & 0xFFFFu);
}

// output value (16-bit dtypes write 16-bit words)
__device__ __forceinline__ void store_val(uint32_t* out, int dtype, uint64_t i, uint32_t v) {
    if (dtype == kF16) reinterpret_cast<unsigned short*>(out)[i] = static_cast<unsigned short>(v);
    else out[i] = v;
}

// element i of an input row (runtime element size; the hot kernels use compile-time paths)
__device__ __forceinline__ uint32_t load_elem(const InputSrc& s, uint64_t i) {
    if (s.dtype == kF16) return __ldg(reinterpret_cast<const unsigned short*>(s.base) + i);
    return __ldg(s.base + i);
}

// y = x - a_s as the reference computes it on x86-64 (scaling.hpp:69-70, SSE subss): IEEE fp32
// round-to-nearest with denormals kept (the library is built without -use_fast_math / -ftz);
// a NaN result follows the x86 rule instead of the GPU's canonical 0x7FFFFFFF — the first NaN
// operand quieted (x, then a_s, sign and payload kept), else the default NaN 0xFFC00000
// (inf - inf). The NaN's sign decides whether it ranks above +inf or below -inf.
__device__ __forceinline__ uint32_t sub_x86(uint32_t xb, float a) {
    const float y = __fsub_rn(__uint_as_float(xb), a);
    if (y == y) return __float_as_uint(y);
    const uint32_t ab = __float_as_uint(a);
    if ((xb & 0x7fffffffu) > 0x7f800000u) return xb | 0x00400000u;
    if ((ab & 0x7fffffffu) > 0x7f800000u) return ab | 0x00400000u;
    return 0xFFC00000u;
}

__device__ __forceinline__ uint32_t make_key(const InputSrc& s, uint32_t raw) {
    if (s.dtype == kF16) return encode_f16_key(raw, s.smallest);
    if (s.dtype == kF32) {
        if (s.scaled) raw = sub_x86(raw, s.a_s);
        return encode_f32_bits(raw, s.smallest);
    }
    return s.smallest ? ~raw : raw;  // KeyCodec<u32>, keycodec.hpp:72-81
}

// Compile-time key transforms for the streaming kernels (KM = key mode).
enum : int { kKmF32L = 0, kKmF32S = 1, kKmF32LScaled = 2, kKmF32SScaled = 3, kKmU32L = 4, kKmU32S = 5,
             kKmF16L = 6, kKmF16S = 7, kKmF32LAdapt = 8, kKmF32SAdapt = 9 };

inline int key_mode(int dtype, int smallest, int scaled, const uint32_t* adapt = nullptr) {
    if (dtype == kF16) return smallest ? kKmF16S : kKmF16L;
    if (dtype != kF32) return smallest ? kKmU32S : kKmU32L;
    if (adapt) return smallest ? kKmF32SAdapt : kKmF32LAdapt;
    return (scaled ? 2 : 0) + (smallest ? 1 : 0);
}

template <int KM>
__host__ __device__ constexpr bool km_is16() { return KM == kKmF16L || KM == kKmF16S; }

template <int KM>
__device__ __forceinline__ uint32_t key_of(uint32_t raw, const InputSrc& in) {
    const float a_s = in.a_s;
    if (KM == kKmF32LAdapt || KM == kKmF32SAdapt) {  // decided on the device: kernel-uniform branch
        if (in.scaled) raw = sub_x86(raw, a_s);
        const uint32_t m = static_cast<uint32_t>(static_cast<int32_t>(raw) >> 31) | 0x80000000u;
        const uint32_t bits = raw ^ m;
        return KM == kKmF32SAdapt ? ~bits : bits;
    }
    if (KM == kKmF16L || KM == kKmF16S) {
        // raw = zero-extended 16-bit word; sign-flip map as mask arithmetic, key in the high half
        const uint32_t m = ((raw & 0x8000u) ? 0xFFFFu : 0x8000u);
        const uint32_t bits = (raw ^ m) << 16;
        return KM == kKmF16S ? ~bits & 0xFFFF0000u : bits;
    }
    if (KM == kKmU32L) return raw;
    if (KM == kKmU32S) return ~raw;
    if (KM == kKmF32LScaled || KM == kKmF32SScaled)
        raw = sub_x86(raw, a_s);
    // sign-flip map as mask arithmetic: negative -> ~raw, positive -> raw | sign
    const uint32_t m = static_cast<uint32_t>(static_cast<int32_t>(raw) >> 31) | 0x80000000u;
    const uint32_t bits = raw ^ m;
    return (KM == kKmF32S || KM == kKmF32SScaled) ? ~bits : bits;
}

__device__ __forceinline__ uint64_t composite(uint32_t key, uint64_t idx) {
    return (static_cast<uint64_t>(key) << 32) | static_cast<uint32_t>(~static_cast<uint32_t>(idx));
}

__device__ __forceinline__ void ldg256(const uint32_t* p, uint32_t (&r)[8]) {
    asm volatile(
        "ld.global.nc.L1::no_allocate.L2::256B.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7])
        : "l"(p));
}

__device__ __forceinline__ void ldg256_u64(const uint64_t* p, uint64_t (&r)[4]) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.b64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(r[0]), "=l"(r[1]), "=l"(r[2]), "=l"(r[3])
                 : "l"(p));
}

// Programmatic dependent launch (PDL): a dependent kernel may start while its predecessor
// runs; it must wait before touching the predecessor's outputs. Both are no-ops when the
// kernel was launched without the programmatic-serialization attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Launch row owning flat tile t (tile_start is an exclusive prefix, R+1 entries).
__device__ __forceinline__ int row_of_tile(const Rows& rows, uint64_t t) {
    int lo = 0, hi = rows.R - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (rows.tile_start[mid] <= t) lo = mid; else hi = mid - 1;
    }
    return lo;
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

// load_input_tile for any element size (rare paths: exact radix passes, trigger histogram)
__device__ __forceinline__ void load_input_tile_any(const InputSrc& in, uint64_t row_off, uint64_t span_len,
                                                    uint32_t lead, uint64_t span0, uint32_t (&v)[kUnroll][kVec]) {
    if (in.dtype != kF16) {
        load_input_tile(in.base + row_off - lead, span_len, lead, span0, v);
        return;
    }
    const unsigned short* rp = reinterpret_cast<const unsigned short*>(in.base) + row_off - lead;
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
        const uint64_t p = span0 + static_cast<uint64_t>(u * kThreads + threadIdx.x) * kVec;
#pragma unroll
        for (int i = 0; i < kVec; ++i) {
            const uint64_t q = p + i;
            v[u][i] = (q >= lead && q < span_len) ? static_cast<uint32_t>(__ldg(rp + q)) : 0u;
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

// 16-bit elements: the same (u, tid, i) layout, 8 halves = one 16-byte load per (u, tid)
__device__ __forceinline__ void load_tile_local16(const unsigned short* tile_ptr, uint32_t vlo, uint32_t vhi,
                                                  uint32_t (&v)[kUnroll][kVec]) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
        const uint32_t l = (u * kThreads + threadIdx.x) * kVec;
        if (l >= vlo && l + kVec <= vhi) {
            uint32_t w0, w1, w2, w3;
            asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                         : "l"(tile_ptr + l));
            v[u][0] = w0 & 0xFFFFu; v[u][1] = w0 >> 16;
            v[u][2] = w1 & 0xFFFFu; v[u][3] = w1 >> 16;
            v[u][4] = w2 & 0xFFFFu; v[u][5] = w2 >> 16;
            v[u][6] = w3 & 0xFFFFu; v[u][7] = w3 >> 16;
        } else {
#pragma unroll
            for (int i = 0; i < kVec; ++i)
                v[u][i] = (l + i >= vlo && l + i < vhi) ? static_cast<uint32_t>(__ldg(tile_ptr + l + i)) : 0u;
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

// Lanes of the (full) warp whose 8-bit digit equals this lane's: the ballot multisplit (one
// ballot per digit bit, AND of the matching masks) — cheaper than __match_any_sync.
__device__ __forceinline__ unsigned warp_peers8(uint32_t d) {
    unsigned m = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const unsigned bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        m &= ((d >> b) & 1u) ? bal : ~bal;
    }
    return m;
}

// smem histogram increment with a whole-warp fast path: adversarial inputs put every
// element of a warp into one bin (engine_test.cpp:45-56, C4), which would otherwise
// serialise 32 same-address shared atomics.
// Spread digits (MSD levels over candidates): plain shared atomics, conflicts are rare.
__device__ __forceinline__ void hist_add_spread(uint32_t* h, uint32_t digit, bool valid) {
    if (valid) atomicAdd(&h[digit], 1u);
}

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

}  // namespace rtk_b200
