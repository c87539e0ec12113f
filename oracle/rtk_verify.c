/*
 * rtk_verify.c — streaming top-k verifier for queries too large for a host-side oracle
 * (TEST INFRASTRUCTURE, like the rest of oracle/, BASELINE C5 n = 2^32).
 *
 * The input is the Philox4x32-10 uniform stream of include/rtk_c.h (rtk_generate_philox),
 * restated here independently in plain C (Salmon et al., SC'11; the Random123 round function:
 * multipliers 0xD2511F53 / 0xCD9E8D57, Weyl key increments 0x9E3779B9 / 0xBB67AE85, 10 rounds).
 * Any element can be regenerated from its index, so the check needs O(k) memory:
 *
 *   P      = key of the returned pivot values[k-1] (KeyCodec, keycodec.hpp:55-62)
 *   order  : returned (key, index) strictly in (key desc, index asc) order (engine.hpp:402-420)
 *   values : values[i] == x[indices[i]] bit for bit
 *   set    : #{x: key > P} == #{returned: key > P}          (all strictly-greater elements)
 *            #{x: key == P, index <= indices[k-1]} == k - #{returned: key > P}
 *                                                           (ties filled by lowest index,
 *                                                            engine.hpp:387-396)
 * One streaming pass over the regenerated input, split over `threads` pthreads.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0, n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1, n3 = (uint32_t)p0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

static float uniform(uint32_t w, float a, float span) {
    volatile float t = (float)(w >> 8) * 5.9604644775390625e-08f * span;
    return a + t;
}

static uint32_t f32_bits(float f) { uint32_t b; memcpy(&b, &f, 4); return b; }

static uint32_t key_of(uint32_t raw, int order) {
    uint32_t k = (raw & 0x80000000u) ? ~raw : (raw | 0x80000000u);
    return order ? ~k : k;
}

/* element g of the stream (raw f32 bits) */
uint32_t rtkv_philox_elem(uint64_t seed, uint64_t g, float a, float b) {
    uint32_t c[4] = {(uint32_t)(g >> 2), (uint32_t)(g >> 34), 0, 0};
    philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    return f32_bits(uniform(c[g & 3], a, b - a));
}

/* n consecutive elements from global index `offset` (raw bits) */
void rtkv_philox_fill(uint64_t seed, uint64_t offset, uint64_t n, float a, float b, uint32_t* out) {
    const float span = b - a;
    uint64_t g = offset;
    for (uint64_t j = 0; j < n;) {
        uint32_t c[4] = {(uint32_t)(g >> 2), (uint32_t)(g >> 34), 0, 0};
        philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
        for (uint32_t q = (uint32_t)(g & 3); q < 4 && j < n; ++q, ++j, ++g) out[j] = f32_bits(uniform(c[q], a, span));
    }
}

typedef struct {
    uint64_t seed, b0, b1, m;
    float a, span;
    uint32_t P;
    int order;
    uint64_t gt, eq, eq_le_m;
} part_t;

static void* scan(void* arg) {
    part_t* p = (part_t*)arg;
    uint64_t gt = 0, eq = 0, le = 0;
    for (uint64_t blk = p->b0; blk < p->b1; ++blk) {
        uint32_t c[4] = {(uint32_t)blk, (uint32_t)(blk >> 32), 0, 0};
        philox(c, (uint32_t)p->seed, (uint32_t)(p->seed >> 32));
        for (int q = 0; q < 4; ++q) {
            const uint32_t kk = key_of(f32_bits(uniform(c[q], p->a, p->span)), p->order);
            if (kk > p->P) ++gt;
            else if (kk == p->P) {
                ++eq;
                if ((blk << 2) + (uint64_t)q <= p->m) ++le;
            }
        }
    }
    p->gt = gt;
    p->eq = eq;
    p->eq_le_m = le;
    return NULL;
}

/* 0 = verified; otherwise 1 and a message. n must be a multiple of 4 (whole Philox blocks).
 * stats (nullable, 3 entries): #{key > P}, #{key == P}, #{key == P, index <= indices[k-1]}. */
int rtkv_verify_philox_topk(uint64_t seed, uint64_t n, float a, float b, int order, uint64_t k,
                            const uint32_t* vals, const uint64_t* idx, int threads, uint64_t* stats,
                            char* msg, int msglen) {
    if (k == 0 || k > n || (n & 3)) { snprintf(msg, msglen, "bad arguments"); return 1; }
    const uint32_t P = key_of(vals[k - 1], order);
    uint64_t ret_gt = 0;
    for (uint64_t i = 0; i < k; ++i) {
        if (idx[i] >= n) { snprintf(msg, msglen, "rank %llu: index out of range", (unsigned long long)i); return 1; }
        if (rtkv_philox_elem(seed, idx[i], a, b) != vals[i]) {
            snprintf(msg, msglen, "rank %llu: value is not x[%llu]", (unsigned long long)i, (unsigned long long)idx[i]);
            return 1;
        }
        const uint32_t ki = key_of(vals[i], order);
        if (i) {
            const uint32_t kp = key_of(vals[i - 1], order);
            if (!(kp > ki || (kp == ki && idx[i - 1] < idx[i]))) {
                snprintf(msg, msglen, "rank %llu: not in (key desc, index asc) order", (unsigned long long)i);
                return 1;
            }
        }
        if (ki > P) ++ret_gt;
    }
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    part_t parts[256];
    pthread_t tid[256];
    const uint64_t blocks = n >> 2, per = (blocks + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        part_t* p = &parts[t];
        p->seed = seed;
        p->b0 = (uint64_t)t * per < blocks ? (uint64_t)t * per : blocks;
        p->b1 = p->b0 + per < blocks ? p->b0 + per : blocks;
        p->m = idx[k - 1];
        p->a = a;
        p->span = b - a;
        p->P = P;
        p->order = order;
        pthread_create(&tid[t], NULL, scan, p);
    }
    uint64_t gt = 0, eq = 0, le = 0;
    for (int t = 0; t < threads; ++t) {
        pthread_join(tid[t], NULL);
        gt += parts[t].gt;
        eq += parts[t].eq;
        le += parts[t].eq_le_m;
    }
    if (stats) { stats[0] = gt; stats[1] = eq; stats[2] = le; }
    if (gt != ret_gt) {
        snprintf(msg, msglen, "%llu elements above the pivot, %llu returned", (unsigned long long)gt,
                 (unsigned long long)ret_gt);
        return 1;
    }
    if (le != k - ret_gt) {
        snprintf(msg, msglen, "pivot ties: %llu with index <= %llu, %llu returned", (unsigned long long)le,
                 (unsigned long long)idx[k - 1], (unsigned long long)(k - ret_gt));
        return 1;
    }
    if (!(gt < k && k <= gt + eq)) { snprintf(msg, msglen, "pivot rank inconsistent"); return 1; }
    return 0;
}
