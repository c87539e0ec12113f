// rtk_philox.h — Philox4x32-10 counter-based generator (Salmon, Moraes, Dror, Shaw, SC'11),
// shared by the device generator (rtk_gen.cu) and its host twin (rtk_host.cpp), so both produce
// bit-identical streams. Element i of a stream with key `seed` is word (i & 3) of the Philox
// block with counter (i >> 2, 0); uniform floats in [a, b) are u = (w >> 8) * 2^-24 (exact) and
// x = a + u * (b - a) in fp32 round-to-nearest without contraction — x = u exactly for [0, 1).
// Used for the C5 configuration (n = 2^32 over 8 GPUs): every shard generates its own elements
// on its device from its global index range, and the host verifier regenerates any element.
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define RTK_HD __host__ __device__ __forceinline__
#else
#define RTK_HD inline
#endif

namespace rtk_b200 {

RTK_HD void philox4x32_10(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c[0];
        const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c[2];
        const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
        const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// the 4 words of block b (elements 4b .. 4b+3)
RTK_HD void philox_block(uint64_t seed, uint64_t b, uint32_t (&w)[4]) {
    w[0] = static_cast<uint32_t>(b);
    w[1] = static_cast<uint32_t>(b >> 32);
    w[2] = 0;
    w[3] = 0;
    philox4x32_10(w, static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
}

RTK_HD float philox_uniform(uint32_t w, float a, float span) {
    const float u = static_cast<float>(w >> 8) * 5.9604644775390625e-08f;  // exact: 24 bits * 2^-24
#ifdef __CUDA_ARCH__
    return __fadd_rn(a, __fmul_rn(u, span));
#else
    volatile float t = u * span;  // two roundings, as on the device (no fused multiply-add)
    return a + t;
#endif
}

}  // namespace rtk_b200
