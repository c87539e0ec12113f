// rtk_gen.cu — on-device Philox input generator (rtk_philox.h) for the C5 configuration: each
// rank writes its shard of one huge query straight into HBM from its global index range, so a
// 2^32-element query never passes through host memory. Write-bound: 4 B per element.
#include <cuda_runtime.h>

#include "rtk_kernels.h"
#include "rtk_philox.h"

namespace rtk_b200 {

// one Philox block (4 elements) per thread and iteration; element j of the output is global
// element offset + j. Aligned shards (offset and pointer multiples of 4 elements) store float4.
__global__ void __launch_bounds__(256) k_philox_uniform(float* out, uint64_t n, uint64_t seed, uint64_t offset,
                                                        float a, float span) {
    const uint64_t first = offset >> 2, last = (offset + n + 3) >> 2;
    const bool vec = (offset & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    for (uint64_t b = first + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; b < last;
         b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t w[4];
        philox_block(seed, b, w);
        const uint64_t g0 = b << 2;
        if (vec && g0 + 4 <= offset + n) {
            float4 v = make_float4(philox_uniform(w[0], a, span), philox_uniform(w[1], a, span),
                                   philox_uniform(w[2], a, span), philox_uniform(w[3], a, span));
            __stcs(reinterpret_cast<float4*>(out + (g0 - offset)), v);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint64_t g = g0 + j;
                if (g >= offset && g < offset + n) out[g - offset] = philox_uniform(w[j], a, span);
            }
        }
    }
}

void launch_philox_uniform(float* out, uint64_t n, uint64_t seed, uint64_t offset, float a, float b,
                           cudaStream_t s) {
    if (n == 0) return;
    const uint64_t blocks = ((offset + n + 3) >> 2) - (offset >> 2);
    const uint64_t want = (blocks + 255) / 256;
    const unsigned grid = static_cast<unsigned>(want < 148ull * 16 ? want : 148ull * 16);
    k_philox_uniform<<<grid, 256, 0, s>>>(out, n, seed, offset, a, b - a);
}

}  // namespace rtk_b200
