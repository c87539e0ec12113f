// rtk_sample.cu — LLM sampling consumer of the batched top-k (the paper's
// motivating caller): softmax over each row's top-k logits, top-p
// (nucleus) cut, and one inverse-CDF draw per row.
//
// Input per row: the top-k (value, index) pairs the selection kernels just wrote, in canonical
// order (value descending, index ascending), still in L2. Definition (fp32 throughout):
//   z_j = (v_j - v_0) / T,  e_j = expf(z_j)        (v_0 is the row maximum, so e_0 = 1)
//   m   = min { m : sum_{j<m} e_j >= top_p * sum_{j<k} e_j }   (>= 1; top_p = 1 keeps all k)
//   token = idx[j*],  j* = min { j < m : sum_{i<=j} e_i > u * sum_{i<m} e_i }  (m - 1 if none)
//   probs_j = e_j / sum_{i<m} e_i for j < m, 0 otherwise (optional output)
// One CTA per row; the row is walked in 2048-element chunks (8 consecutive elements per thread,
// one block scan per chunk), stopping as soon as the cut / the draw is located.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "rtk_device.cuh"
#include "rtk_kernels.h"

namespace rtk_b200 {

constexpr int kSmpThreads = 256;
constexpr int kSmpPer = 8;
constexpr int kSmpChunk = kSmpThreads * kSmpPer;

__device__ __forceinline__ float to_f32(const void* vals, int fmt, uint64_t i) {
    if (fmt == 0) return __ldg(static_cast<const float*>(vals) + i);
    const unsigned short h = __ldg(static_cast<const unsigned short*>(vals) + i);
    if (fmt == 2) return __half2float(__ushort_as_half(h));
    return __uint_as_float(static_cast<uint32_t>(h) << 16);  // bf16
}

// block-wide exclusive scan of one float per thread; *total = block sum
__device__ __forceinline__ float smp_scan(float v, float* s_w, float* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const float o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    float pre = 0.f, tot = 0.f;
#pragma unroll
    for (int w = 0; w < kSmpThreads / 32; ++w) {
        const float x = s_w[w];
        if (w < warp) pre += x;
        tot += x;
    }
    __syncthreads();
    *total = tot;
    return pre + inc - v;
}

__global__ void __launch_bounds__(kSmpThreads) k_sample_rows(const void* vals, int fmt, const uint64_t* idx,
                                                             uint64_t k, float top_p, float temperature,
                                                             const float* uniform, uint64_t* token,
                                                             float* probs) {
    __shared__ float s_w[kSmpThreads / 32];
    __shared__ float s_red[kSmpThreads / 32];
    __shared__ int s_hit;
    __shared__ float s_hitv;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t r = blockIdx.x;
    const uint64_t base = r * k;
    const float v0 = to_f32(vals, fmt, base);
    auto e_of = [&](uint64_t j) { return expf(__fdiv_rn(__fsub_rn(to_f32(vals, fmt, base + j), v0), temperature)); };

    // 1. total mass (coalesced, order-free)
    float acc = 0.f;
    for (uint64_t j = tid; j < k; j += kSmpThreads) acc += e_of(j);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
    if (lane == 0) s_red[warp] = acc;
    __syncthreads();
    float S = 0.f;
#pragma unroll
    for (int w = 0; w < kSmpThreads / 32; ++w) S += s_red[w];

    // 2. cut m: first prefix whose mass reaches top_p * S; 3. draw inside [0, m)
    const float want = top_p >= 1.f ? INFINITY : top_p * S;
    uint64_t m = k;
    float Em = S;
    for (int pass = 0; pass < 2; ++pass) {
        const float thr = pass == 0 ? want : uniform[r] * Em;
        const uint64_t lim = pass == 0 ? k : m;
        if (pass == 0 && !(want < INFINITY)) continue;  // top_p = 1: keep all k
        float carry = 0.f;
        uint64_t hit = lim;
        float hitv = 0.f;
        for (uint64_t c0 = 0; c0 < lim; c0 += kSmpChunk) {
            float e[kSmpPer], t = 0.f;
#pragma unroll
            for (int i = 0; i < kSmpPer; ++i) {
                const uint64_t j = c0 + static_cast<uint64_t>(tid) * kSmpPer + i;
                e[i] = j < lim ? e_of(j) : 0.f;
                t += e[i];
            }
            float tot;
            float run = carry + smp_scan(t, s_w, &tot);
            if (tid == 0) s_hit = 0x7fffffff;
            __syncthreads();
            int mine = 0x7fffffff;
            float mine_v = 0.f;
#pragma unroll
            for (int i = 0; i < kSmpPer; ++i) {
                const uint64_t j = c0 + static_cast<uint64_t>(tid) * kSmpPer + i;
                run += e[i];
                const bool cross = pass == 0 ? run >= thr : run > thr;
                if (j < lim && cross && mine == 0x7fffffff) {
                    mine = tid * kSmpPer + i;
                    mine_v = run;
                }
            }
            if (mine != 0x7fffffff) atomicMin(&s_hit, mine);
            __syncthreads();
            const int h = s_hit;
            if (h != 0x7fffffff) {
                if (tid * kSmpPer <= h && h < (tid + 1) * kSmpPer) s_hitv = mine_v;
                __syncthreads();
                hit = c0 + static_cast<uint64_t>(h);
                hitv = s_hitv;
                break;
            }
            carry += tot;
            __syncthreads();
        }
        if (pass == 0) {
            if (hit < k) {
                m = hit + 1;
                Em = hitv;
            }
        } else {
            const uint64_t js = hit < m ? hit : m - 1;
            if (tid == 0) token[r] = idx[base + js];
        }
    }
    if (probs) {
        const float inv = 1.f / Em;
        for (uint64_t j = tid; j < k; j += kSmpThreads) probs[base + j] = j < m ? e_of(j) * inv : 0.f;
    }
}

void launch_sample_rows(uint64_t rows, const void* vals, int fmt, const uint64_t* idx, uint64_t k, float top_p,
                        float temperature, const float* uniform, uint64_t* token, float* probs, cudaStream_t s) {
    if (rows == 0) return;
    k_sample_rows<<<static_cast<unsigned>(rows), kSmpThreads, 0, s>>>(vals, fmt, idx, k, top_p, temperature,
                                                                     uniform, token, probs);
}

}  // namespace rtk_b200
