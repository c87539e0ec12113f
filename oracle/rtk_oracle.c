/*
 * rtk_oracle.c — CPU restatement of the reference radix top-k (TEST INFRASTRUCTURE).
 *
 * This file is the parity oracle for the B200 path. It is NOT part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it. The product library (paper_2501_14336_b200/librtk_b200.so) never
 * links or calls it.
 *
 * It restates, in plain sequential C, the algorithm of the reference artifact
 * (/root/reference/proj/include/rtk/*.hpp). Each function cites the file:line it follows.
 * Parity of this restatement is pinned in tests/test_oracle.py against
 *   (1) the reference's own known-answer tests (keycodec_test.cpp, engine_test.cpp,
 *       batch_test.cpp, scaling_test.cpp), restated there, and
 *   (2) tests/golden/*.npz, produced by the reference compiled from its own headers
 *       (oracle/_ref, built by oracle/Makefile; generator tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { RTKO_OK = 0, RTKO_EMPTY_INPUT = 1, RTKO_RANK_OUT_OF_RANGE = 2,
       RTKO_INVARIANT_VIOLATION = 3, RTKO_INVALID_ARGUMENT = 4, RTKO_NOMEM = 6 };
enum { RTKO_F32 = 0, RTKO_U32 = 1 };
enum { RTKO_LARGEST = 0, RTKO_SMALLEST = 1 };

/* ---- key codec: keycodec.hpp:55-91 ---------------------------------------------- */

/* KeyCodec<float>::encode (keycodec.hpp:57-62) */
uint32_t rtko_encode_f32_bits(uint32_t raw, int order) {
    uint32_t bits = (raw & 0x80000000u) ? ~raw : (raw | 0x80000000u);
    if (order == RTKO_SMALLEST) bits = ~bits;
    return bits;
}

/* KeyCodec<float>::decode (keycodec.hpp:64-69) */
uint32_t rtko_decode_f32_bits(uint32_t bits, int order) {
    if (order == RTKO_SMALLEST) bits = ~bits;
    return (bits & 0x80000000u) ? (bits ^ 0x80000000u) : ~bits;
}

/* KeyCodec<u32> (keycodec.hpp:72-81) */
uint32_t rtko_encode_u32(uint32_t v, int order) { return order == RTKO_LARGEST ? v : ~v; }

static uint32_t encode_any(const void* in, uint64_t i, int dtype, int order) {
    uint32_t raw = ((const uint32_t*)in)[i];
    return dtype == RTKO_F32 ? rtko_encode_f32_bits(raw, order) : rtko_encode_u32(raw, order);
}

/* DigitWindow::first / next (keycodec.hpp:39-45) and extract_digit (:48-50) */
typedef struct { unsigned low, high; } window_t;
static window_t window_first(unsigned d) { window_t w = {32 > d ? 32 - d : 0, 32}; return w; }
static window_t window_next(window_t w, unsigned d) {
    window_t r = {w.low > d ? w.low - d : 0, w.low};
    return r;
}
uint32_t rtko_extract_digit(uint32_t key, unsigned low, unsigned high) {
    unsigned width = high - low;
    return (key >> low) & (width >= 32 ? 0xFFFFFFFFu : ((1u << width) - 1u));
}

/* ---- count_bins (engine.hpp:177-222): sequential, same counts ------------------- */
void rtko_count_bins(const uint32_t* keys, uint64_t m, unsigned low, unsigned high,
                     uint64_t* hist /* 2^(high-low) */) {
    uint64_t nb = (uint64_t)1 << (high - low);
    memset(hist, 0, nb * sizeof(uint64_t));
    for (uint64_t i = 0; i < m; ++i) ++hist[rtko_extract_digit(keys[i], low, high)];
}

/* ---- select_bin (engine.hpp:231-241) -------------------------------------------- */
int rtko_select_bin(const uint64_t* hist, uint64_t nbins, uint64_t k, uint32_t* bin,
                    uint64_t* k_new) {
    uint64_t total = 0;
    for (uint64_t b = 0; b < nbins; ++b) total += hist[b];
    if (k == 0 || k > total) return RTKO_RANK_OUT_OF_RANGE;
    uint64_t cum = 0;
    for (uint64_t b = nbins; b-- > 0;) {
        cum += hist[b];
        if (cum >= k) {
            *bin = (uint32_t)b;
            *k_new = k - (cum - hist[b]);
            return RTKO_OK;
        }
    }
    return RTKO_RANK_OUT_OF_RANGE;
}

/* ---- radix_select (engine.hpp:293-312) with select_candidates (:245-284) -------- */
int rtko_radix_select(const uint32_t* keys, uint64_t n, uint64_t k, unsigned d,
                      uint32_t* pivot_key, uint64_t* k_at_pivot, uint64_t* passes) {
    if (d < 1 || d > 16) return RTKO_INVALID_ARGUMENT;
    if (k == 0 || k > n) return RTKO_RANK_OUT_OF_RANGE;
    uint32_t* cand = (uint32_t*)malloc(n * sizeof(uint32_t));
    uint64_t* hist = (uint64_t*)malloc(((size_t)1 << d) * sizeof(uint64_t));
    if (!cand || !hist) { free(cand); free(hist); return RTKO_NOMEM; }
    memcpy(cand, keys, n * sizeof(uint32_t));
    uint64_t m = n, k_rem = k, p = 0;
    window_t w = window_first(d);
    while (m > 1 && w.high != 0) {
        uint64_t nb = (uint64_t)1 << (w.high - w.low);
        rtko_count_bins(cand, m, w.low, w.high, hist);
        uint32_t bin;
        uint64_t k_new;
        int st = rtko_select_bin(hist, nb, k_rem, &bin, &k_new);
        if (st) { free(cand); free(hist); return st; }
        k_rem = k_new;
        uint64_t out = 0; /* in-place compaction: order is unspecified in the reference */
        for (uint64_t i = 0; i < m; ++i)
            if (rtko_extract_digit(cand[i], w.low, w.high) == bin) cand[out++] = cand[i];
        m = out;
        w = window_next(w, d);
        ++p;
    }
    *pivot_key = cand[0];
    *k_at_pivot = k_rem;
    if (passes) *passes = p;
    free(cand);
    free(hist);
    return RTKO_OK;
}

/* ---- normalize_result (engine.hpp:402-420): sort by (key desc, index asc) -------- */
typedef struct { uint32_t key; uint32_t raw; uint64_t idx; } item_t;
static int cmp_item(const void* a, const void* b) {
    const item_t* x = (const item_t*)a;
    const item_t* y = (const item_t*)b;
    if (x->key != y->key) return x->key > y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* ---- filter (engine.hpp:318-398) + normalize (402-420) ---------------------------- */
static int filter_and_normalize(const void* in, uint64_t n, uint32_t pivot, uint64_t k,
                                int dtype, int order, uint32_t* out_vals, uint64_t* out_idx,
                                uint32_t* out_pivot_raw) {
    item_t* items = (item_t*)malloc(k * sizeof(item_t));
    uint64_t* ties = (uint64_t*)malloc(n * sizeof(uint64_t));
    if (!items || !ties) { free(items); free(ties); return RTKO_NOMEM; }
    uint64_t greater = 0, nties = 0;
    const uint32_t* raw = (const uint32_t*)in;
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t key = encode_any(in, i, dtype, order);
        if (key > pivot) {
            if (greater == k) { free(items); free(ties); return RTKO_INVARIANT_VIOLATION; }
            items[greater].key = key;
            items[greater].raw = raw[i];
            items[greater].idx = i;
            ++greater;
        } else if (key == pivot) {
            ties[nties++] = i; /* already ascending: sequential scan (:387-396 sorts) */
        }
    }
    uint64_t need = k - greater;
    if (nties < need) { free(items); free(ties); return RTKO_INVARIANT_VIOLATION; }
    for (uint64_t j = 0; j < need; ++j) {
        item_t* it = &items[greater + j];
        it->key = pivot;
        it->raw = raw[ties[j]];
        it->idx = ties[j];
    }
    qsort(items, k, sizeof(item_t), cmp_item);
    for (uint64_t j = 0; j < k; ++j) {
        out_vals[j] = items[j].raw;
        out_idx[j] = items[j].idx;
    }
    /* result.pivot = decode_key(pivot_key) (engine.hpp:333) */
    *out_pivot_raw = dtype == RTKO_F32 ? rtko_decode_f32_bits(pivot, order)
                                       : (order == RTKO_LARGEST ? pivot : ~pivot);
    free(items);
    free(ties);
    return RTKO_OK;
}

/* ---- topk (engine.hpp:422-443) ---------------------------------------------------- */
int rtko_topk(const void* in, uint64_t n, uint64_t k, int dtype, int order, unsigned d,
              uint32_t* out_vals, uint64_t* out_idx, uint32_t* out_pivot_raw,
              uint64_t* passes) {
    if (n == 0) return RTKO_EMPTY_INPUT;
    if (k == 0 || k > n) return RTKO_RANK_OUT_OF_RANGE;
    uint32_t* keys = (uint32_t*)malloc(n * sizeof(uint32_t));
    if (!keys) return RTKO_NOMEM;
    for (uint64_t i = 0; i < n; ++i) keys[i] = encode_any(in, i, dtype, order);
    uint32_t pivot;
    uint64_t k_at;
    int st = rtko_radix_select(keys, n, k, d, &pivot, &k_at, passes);
    free(keys);
    if (st) return st;
    return filter_and_normalize(in, n, pivot, k, dtype, order, out_vals, out_idx,
                                out_pivot_raw);
}

/* ---- oracle_topk (oracle.hpp:19-39): stable sort by key desc, take k ------------- */
int rtko_oracle_topk(const void* in, uint64_t n, uint64_t k, int dtype, int order,
                     uint32_t* out_vals, uint64_t* out_idx, uint32_t* out_pivot_raw) {
    if (n == 0) return RTKO_EMPTY_INPUT;
    if (k == 0 || k > n) return RTKO_RANK_OUT_OF_RANGE;
    item_t* items = (item_t*)malloc(n * sizeof(item_t));
    if (!items) return RTKO_NOMEM;
    const uint32_t* raw = (const uint32_t*)in;
    for (uint64_t i = 0; i < n; ++i) {
        items[i].key = encode_any(in, i, dtype, order);
        items[i].raw = raw[i];
        items[i].idx = i;
    }
    /* (key desc, idx asc) == stable_sort by key desc over the identity permutation */
    qsort(items, n, sizeof(item_t), cmp_item);
    for (uint64_t j = 0; j < k; ++j) {
        out_vals[j] = items[j].raw;
        out_idx[j] = items[j].idx;
    }
    *out_pivot_raw = items[k - 1].raw;
    free(items);
    return RTKO_OK;
}

/* ---- batch_topk (batch.hpp:261-367): results equal per-task topk (:284-291) ------ */
/* BatchInput::validate (batch.hpp:40-53). Returns the failing task in *bad_task. */
int rtko_batch_validate(uint64_t data_len, const uint64_t* offsets, const uint64_t* lengths,
                        const uint64_t* ks, uint64_t B, uint64_t* bad_task) {
    if (B == 0) return RTKO_INVALID_ARGUMENT;
    for (uint64_t t = 0; t < B; ++t) {
        uint64_t next = t + 1 < B ? offsets[t + 1] : data_len;
        *bad_task = t;
        if (offsets[t] + lengths[t] > next) return RTKO_INVALID_ARGUMENT;
        if (ks[t] == 0 || ks[t] > lengths[t]) return RTKO_INVALID_ARGUMENT;
    }
    return RTKO_OK;
}

int rtko_batch_topk(const void* data, uint64_t data_len, const uint64_t* offsets,
                    const uint64_t* lengths, const uint64_t* ks, uint64_t B, int dtype,
                    int order, unsigned d, uint32_t* out_vals, uint64_t* out_idx,
                    const uint64_t* out_offsets, uint32_t* out_pivots, uint64_t* bad_task) {
    int st = rtko_batch_validate(data_len, offsets, lengths, ks, B, bad_task);
    if (st) return st;
    for (uint64_t t = 0; t < B; ++t) {
        *bad_task = t;
        st = rtko_topk((const uint32_t*)data + offsets[t], lengths[t], ks[t], dtype, order, d,
                       out_vals + out_offsets[t], out_idx + out_offsets[t], &out_pivots[t],
                       NULL);
        if (st) return st;
    }
    return RTKO_OK;
}

/* ---- mt19937_64 (the engine scaling.hpp:65 seeds; std::mersenne_twister_engine) -- */
typedef struct { uint64_t mt[312]; int i; } mt64_t;
static void mt64_seed(mt64_t* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->i = 312;
}
static uint64_t mt64_next(mt64_t* s) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (s->i >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (s->mt[i] & UM) | (s->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->i = 0;
    }
    uint64_t x = s->mt[s->i++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}
uint64_t rtko_mt19937_64_first(uint64_t seed) {
    mt64_t s;
    mt64_seed(&s, seed);
    return mt64_next(&s);
}

/* ---- scaled_topk (scaling.hpp:42-78) ---------------------------------------------
 * mode 0 Off, 1 Always, 2 Adaptive. info[0]=scaled, info[1]=a_s bits, info[2]=a_index. */
int rtko_scaled_topk(const float* in, uint64_t n, uint64_t k, int order, unsigned d, int mode,
                     double tau, uint64_t seed, uint32_t* out_vals, uint64_t* out_idx,
                     uint32_t* out_pivot_raw, uint64_t* info) {
    if (n == 0) return RTKO_EMPTY_INPUT;
    if (k == 0 || k > n) return RTKO_RANK_OUT_OF_RANGE;
    int scale = mode == 1;
    if (mode == 2) { /* adaptive trigger (:50-58) */
        if (d < 1 || d > 16) return RTKO_INVALID_ARGUMENT;
        uint32_t* keys = (uint32_t*)malloc(n * sizeof(uint32_t));
        uint64_t nb = (uint64_t)1 << d;
        uint64_t* hist = (uint64_t*)malloc(nb * sizeof(uint64_t));
        if (!keys || !hist) { free(keys); free(hist); return RTKO_NOMEM; }
        for (uint64_t i = 0; i < n; ++i) keys[i] = encode_any(in, i, RTKO_F32, order);
        window_t w = window_first(d);
        rtko_count_bins(keys, n, w.low, w.high, hist);
        uint32_t bin;
        uint64_t k_new;
        int st = rtko_select_bin(hist, nb, k, &bin, &k_new);
        if (!st) scale = (double)hist[bin] > tau * (double)n;
        free(keys);
        free(hist);
        if (st) return st;
    }
    info[0] = info[1] = info[2] = 0;
    if (!scale)
        return rtko_topk(in, n, k, RTKO_F32, order, d, out_vals, out_idx, out_pivot_raw, NULL);
    /* draw_scale (:35-40): index = mt19937_64(seed)() % n */
    uint64_t a_index = rtko_mt19937_64_first(seed) % n;
    float a_s = in[a_index];
    info[0] = 1;
    memcpy(&info[1], &a_s, sizeof(float));
    info[1] &= 0xFFFFFFFFULL;
    info[2] = a_index;
    float* shifted = (float*)malloc(n * sizeof(float));
    if (!shifted) return RTKO_NOMEM;
    for (uint64_t i = 0; i < n; ++i) shifted[i] = in[i] - a_s; /* fp32 RN (:69-70) */
    int st = rtko_topk(shifted, n, k, RTKO_F32, order, d, out_vals, out_idx, out_pivot_raw,
                       NULL);
    free(shifted);
    if (st) return st;
    /* values re-read from the original input by index; pivot = values.back() (:74-76) */
    const uint32_t* raw = (const uint32_t*)in;
    for (uint64_t j = 0; j < k; ++j) out_vals[j] = raw[out_idx[j]];
    *out_pivot_raw = out_vals[k - 1];
    return RTKO_OK;
}
