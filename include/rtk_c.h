/*
 * rtk_c.h — C-ABI of the B200-native radix top-k (librtk_b200.so).
 *
 * This is the drop-in boundary for the reference's top-k entry points
 * (/root/reference/proj/include/rtk/). Plain pointers and sizes only; no torch or C++
 * types. Each entry point names the reference interface it replaces:
 *
 *   rtk_topk / rtk_topk_host                 <- rtk::topk            engine.hpp:422-443
 *   rtk_topk_batched / rtk_topk_batched_host <- rtk::batch_topk      batch.hpp:261-367
 *   rtk_topk_scaled / rtk_topk_scaled_host   <- rtk::scaled_topk     scaling.hpp:42-86
 *   rtk_cfg + rtk_cfg_validate               <- rtk::EngineConfig    engine.hpp:48-68
 *   rtk_batch_opts                           <- rtk::BatchOptions    batch.hpp:133-136
 *   rtk_scale_info                           <- rtk::ScaleInfo       scaling.hpp:29-33
 *   status codes                             <- rtk::empty_input_error / rank_out_of_range /
 *                                               invariant_violation (engine.hpp:31-41),
 *                                               std::invalid_argument (EngineConfig::validate
 *                                               :61-67, BatchInput::validate batch.hpp:40-53)
 *   rtk_merge_shards                         <- (new) final select of the n-sharded multi-GPU
 *                                               query after the NCCL allgather
 *   rtk_topk_sharded (+ rtk_nccl_*)          <- (new) the n-sharded query itself: local top-k,
 *                                               ncclAllGather, final select
 *
 * Result semantics are the reference's (engine.hpp:402-420, oracle.hpp:19-39): the k
 * selected elements sorted by (encoded key descending, index ascending); ties at the pivot
 * take the lowest indices; values[i] == input[indices[i]] bit for bit; pivot = values[k-1].
 * Indices are u64 and row-local (engine.hpp:106, batch.hpp:36-38).
 *
 * rtk_topk* take DEVICE pointers and run on `stream` (a cudaStream_t, NULL = legacy
 * default stream). The call returns once the device has signalled completion through mapped
 * host memory (no stream synchronisation; rare paths — exact recomputation, deeper MSD
 * levels — add host round trips). rtk_*_host take HOST pointers and include the copies.
 *
 * Limits: n <= 2^32 elements per row on one device (the composite key carries a 32-bit
 * row-local index); dtype F32 or U32; scaled mode is F32 only (as in the reference).
 */
#ifndef RTK_C_H
#define RTK_C_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define RTK_OK 0
#define RTK_EMPTY_INPUT 1          /* rtk::empty_input_error   (std::invalid_argument) */
#define RTK_RANK_OUT_OF_RANGE 2    /* rtk::rank_out_of_range   (std::out_of_range)      */
#define RTK_INVARIANT_VIOLATION 3  /* rtk::invariant_violation (std::logic_error)       */
#define RTK_INVALID_ARGUMENT 4     /* std::invalid_argument (config / batch validation) */
#define RTK_CUDA_ERROR 5
#define RTK_OUT_OF_MEMORY 6
#define RTK_INTERNAL 7
#define RTK_IO_ERROR 8             /* std::runtime_error from the RTK1/RTKB readers (io.cpp) */

/* dtypes (io.hpp:19 codes 0/1) and selection order (keycodec.hpp:19) */
#define RTK_F32 0
#define RTK_U32 1
/* 16-bit floats (io.hpp:3 declares dtype code 2 = f16; the reference build rejects it, io.cpp:71-72).
 * Order and tie rule as for f32 (the same sign-flip KeyCodec on 16 bits); values come back as
 * 16-bit words. The result equals rtk::topk on the exactly widened f32 input. */
#define RTK_F16 2
#define RTK_BF16 3
#define RTK_LARGEST 0
#define RTK_SMALLEST 1

/* scale modes (scaling.hpp:20) */
#define RTK_SCALE_OFF 0
#define RTK_SCALE_ALWAYS 1
#define RTK_SCALE_ADAPTIVE 2

/* mirrors rtk::EngineConfig (engine.hpp:48-68). On the GPU these are tuning hints only:
 * results never depend on them (engine_test.cpp:305-322); d additionally selects the
 * adaptive-scaling trigger window exactly as the reference does (scaling.hpp:53). */
typedef struct rtk_cfg {
    uint32_t d;                      /* digit width, [1,16], default 12 */
    uint64_t block_size;             /* >= 1, default 1024 */
    uint32_t grid_size;              /* >= 1, default 4 */
    int32_t buffer_policy;           /* 0 Naive, 1 FlushEfficient (default) */
    uint64_t pack_size;              /* power of two >= 4, default 16 */
    int32_t hierarchical_atomics;    /* default 1 */
    uint64_t filter_fixed_ceiling;   /* default 4096 */
} rtk_cfg;

/* mirrors rtk::BatchOptions (batch.hpp:133-136); results are identical for all settings */
typedef struct rtk_batch_opts {
    int32_t rescheduling;
    int32_t padding;
} rtk_batch_opts;

/* mirrors rtk::ScaleInfo (scaling.hpp:29-33) */
typedef struct rtk_scale_info {
    int32_t scaled;
    float a_s;
    uint64_t a_index;
} rtk_scale_info;

/* work counters of the last call on a handle (cf. rtk::Instrumentation engine.hpp:74-101) */
typedef struct rtk_stats {
    uint64_t passes;             /* digit passes over the full input (fallback/trigger)   */
    uint64_t elements_scanned;   /* elements read from the input (incl. samples)          */
    uint64_t candidates;         /* sum over rows of the candidate-set size              */
    uint64_t fallback_rows;      /* rows whose sampled threshold had to be recomputed    */
    uint64_t kernel_launches;    /* kernels launched by the call                          */
    float compact_ms;            /* device time of the streaming k_compact launch (events) */
    float total_ms;              /* device time of the whole call on its stream (events)   */
    uint64_t deep_levels;        /* host-driven deeper MSD levels (buckets > 2048 after     */
                                 /* level 0; the GPU analogue of BatchRunInfo::phase_b_rounds) */
} rtk_stats;

typedef struct rtk_handle_s* rtk_handle;

/* mirrors rtk::DistributionSpec (datagen.hpp:18-48); kinds in DistKind order */
#define RTK_DIST_UNIFORM 0
#define RTK_DIST_NORMAL 1
#define RTK_DIST_ZIPF 2
#define RTK_DIST_PEAKED 3
typedef struct rtk_dist {
    int32_t kind;
    double a;          /* Uniform lower / Normal mean       (default 0)   */
    double b;          /* Uniform upper / Normal stddev     (default 1)   */
    double s;          /* Zipf skewness                     (default 1.1) */
    double mass;       /* Peaked: probability mass on modes (default 0.8) */
    uint32_t modes;    /* Peaked: number of modes           (default 1)   */
    uint64_t seed;
    uint64_t n;
} rtk_dist;

/* library / handle */
const char* rtk_version(void);
const char* rtk_last_error(void);             /* thread-local message of the last failure */
int rtk_handle_create(rtk_handle* out, int device);
int rtk_handle_destroy(rtk_handle h);
int rtk_get_stats(rtk_handle h, rtk_stats* out);
/* timing mode (on != 0): calls are never replayed from a CUDA graph and k_compact is bracketed
 * by CUDA events on the call's stream, so rtk_stats.compact_ms is measured for every call. Off
 * (default): repeated identical calls replay one graph with no events inside (kernel-to-kernel
 * programmatic launch edges stay intact); compact_ms is then only set for non-replayed calls. */
int rtk_set_timing(rtk_handle h, int on);

/* Benchmark helper: `warmup` untimed then `steps` timed back-to-back rtk_topk calls issued from C
 * (the reference's own call sites are C++ loops over rtk::topk, rtk_cli.cpp:398). Per step:
 * step_ms[i] (nullable) = device time between CUDA events the engine records on `stream` right
 * before its first and after its last device operation of the call (host planning and the
 * completion wait excluded); step_host_ms[i] (nullable) = host wall time of the rtk_topk call
 * (steady_clock; the call returns after the device's completion signal); *mean_ms = mean of
 * step_ms. When flush_bytes > 0, d_flush is overwritten before every step OUTSIDE both clocks
 * (evicts the input from L2). Same arguments and errors as rtk_topk. */
int rtk_bench_topk(rtk_handle h, const void* d_in, uint64_t n, uint64_t k, int dtype, int order,
                   void* d_out_vals, uint64_t* d_out_idx, void* d_out_pivot, const rtk_cfg* cfg,
                   void* stream, void* d_flush, uint64_t flush_bytes, int warmup, int steps, float* step_ms,
                   float* step_host_ms, float* mean_ms);
/* Scaled counterpart (rtk_topk_scaled per step; the start event precedes the scale decision's
 * kernels). Same arguments and errors as rtk_topk_scaled. */
int rtk_bench_scaled(rtk_handle h, const float* d_in, uint64_t n, uint64_t k, int order, int mode,
                     double trigger_fraction, uint64_t seed, float* d_out_vals, uint64_t* d_out_idx,
                     float* d_out_pivot, const rtk_cfg* cfg, void* stream, void* d_flush, uint64_t flush_bytes,
                     int warmup, int steps, float* step_ms, float* step_host_ms, float* mean_ms);
/* Batched counterpart (rtk_topk_batched per step). */
int rtk_bench_batched(rtk_handle h, const void* d_data, uint64_t data_len, const uint64_t* offsets,
                      const uint64_t* lengths, const uint64_t* ks, uint64_t B, int dtype, int order,
                      void* d_out_vals, uint64_t* d_out_idx, const uint64_t* out_offsets,
                      void* d_out_pivots, const rtk_cfg* cfg, void* stream, void* d_flush,
                      uint64_t flush_bytes, int warmup, int steps, float* step_ms, float* step_host_ms,
                      float* mean_ms);
/* Test / diagnostic switches of a handle (not tuning: results never change). name:
 *   "force_exact"  value != 0: every row takes the exact path (the radix passes of
 *                  radix_select, engine.hpp:293-312, with the early stop) as if its sampled
 *                  threshold had missed; short rows skip the one-CTA kernel, dense rows the
 *                  LSD sort. rtk_stats.fallback_rows reports the rows that took it.
 *   "force_deep"   value != 0: the level-0 MSD digit is cut to 6 bits, so buckets larger than
 *                  one CTA sort take the host-driven deeper levels (rtk_stats.deep_levels).
 * Also read from the environment at handle creation (RTK_FORCE_EXACT=1, RTK_FORCE_DEEP=1).
 * Unknown names -> RTK_INVALID_ARGUMENT. */
int rtk_set_option(rtk_handle h, const char* name, int64_t value);
/* rtk::BatchRunInfo (batch.hpp:138-141) of the last call on the handle: task_passes[t] = full
 * reads of task t's input (1 on the single-read sampled path; + the exact path's digit passes
 * and its re-compaction when the sampled threshold missed); *phase_b_rounds = deeper MSD levels
 * run over the live buckets of all tasks (rtk_stats.deep_levels). task_passes may be NULL;
 * B must not exceed the last call's row count. */
int rtk_get_batch_info(rtk_handle h, uint64_t* task_passes, uint64_t B, uint64_t* phase_b_rounds);
void rtk_cfg_default(rtk_cfg* cfg);
int rtk_cfg_validate(const rtk_cfg* cfg);

/* single query, device pointers. out_pivot may be NULL. */
int rtk_topk(rtk_handle h, const void* d_in, uint64_t n, uint64_t k, int dtype, int order,
             void* d_out_vals, uint64_t* d_out_idx, void* d_out_pivot, const rtk_cfg* cfg,
             void* stream);

/* batch of B (ragged) rows, device data + HOST descriptors (offsets/lengths/ks in elements,
 * data_len = elements in d_data). Row t's outputs start at out_offsets[t] (NULL = exclusive
 * prefix of ks). d_out_pivots (B values) may be NULL. On a task error the message carries
 * "task N: ..." (batch.hpp:274-280). */
int rtk_topk_batched(rtk_handle h, const void* d_data, uint64_t data_len,
                     const uint64_t* offsets, const uint64_t* lengths, const uint64_t* ks,
                     uint64_t B, int dtype, int order, void* d_out_vals, uint64_t* d_out_idx,
                     const uint64_t* out_offsets, void* d_out_pivots, const rtk_cfg* cfg,
                     const rtk_batch_opts* opts, void* stream);

/* adaptive scaling (f32 only). a_s is drawn exactly as the reference draws it:
 * index = std::mt19937_64(seed)() % n (scaling.hpp:35-40, 65-66). info may be NULL. */
int rtk_topk_scaled(rtk_handle h, const float* d_in, uint64_t n, uint64_t k, int order,
                    int mode, double trigger_fraction, uint64_t seed, float* d_out_vals,
                    uint64_t* d_out_idx, float* d_out_pivot, rtk_scale_info* info,
                    const rtk_cfg* cfg, void* stream);

/* host-pointer variants: same contracts, host buffers, copies included */
int rtk_topk_host(rtk_handle h, const void* in, uint64_t n, uint64_t k, int dtype, int order,
                  void* out_vals, uint64_t* out_idx, void* out_pivot, const rtk_cfg* cfg);
int rtk_topk_batched_host(rtk_handle h, const void* data, uint64_t data_len,
                          const uint64_t* offsets, const uint64_t* lengths, const uint64_t* ks,
                          uint64_t B, int dtype, int order, void* out_vals, uint64_t* out_idx,
                          const uint64_t* out_offsets, void* out_pivots, const rtk_cfg* cfg,
                          const rtk_batch_opts* opts);
int rtk_topk_scaled_host(rtk_handle h, const float* in, uint64_t n, uint64_t k, int order,
                         int mode, double trigger_fraction, uint64_t seed, float* out_vals,
                         uint64_t* out_idx, float* out_pivot, rtk_scale_info* info,
                         const rtk_cfg* cfg);

/* Final select of an n-sharded query. d_cand_vals/d_cand_idx hold G blocks of
 * kk = min(k, shard_n[g]) results, each block already in canonical order for its shard
 * (the output of rtk_topk on that shard), concatenated in shard order; shard_base[g] is the
 * global index of shard g's element 0 (host array). Writes the global top-k (values, global
 * u64 indices, pivot) in canonical order. */
int rtk_merge_shards(rtk_handle h, const void* d_cand_vals, const uint64_t* d_cand_idx,
                     const uint64_t* block_len, const uint64_t* shard_base, uint32_t G,
                     uint64_t k, int dtype, int order, void* d_out_vals, uint64_t* d_out_idx,
                     void* d_out_pivot, void* stream);

/* ---- one huge query over several GPUs (BASELINE C5) ------------------------
 * The query is split by contiguous index ranges over the `world` ranks of an NCCL communicator:
 * rank r holds shard_n[r] elements whose global indices start at sum_{g<r} shard_n[g]
 * (shard_n: host array of `world` entries, rank order). The call drives L >= 1 local ranks:
 * handles[i] (on the rank's device), comms[i] (ncclComm_t), d_shards[i], streams[i] and the
 * outputs of local rank i — L = 1 with one process per GPU, L = world in the single-process
 * multi-GPU form. Per rank: local top-k of the shard (rtk_topk, canonical order) ->
 * ncclAllGather of the min(k, shard_n[g]) (value, local u64 index) candidates of every rank ->
 * the rtk_merge_shards select over the gathered candidates -> every local rank receives the
 * global top-k (values, GLOBAL u64 indices, pivot), identical to rtk_topk on the whole query.
 * NCCL is loaded at run time (libnccl.so.2); without it the call fails with
 * RTK_INVALID_ARGUMENT. d_out_pivots and streams may be NULL. */
int rtk_nccl_get_unique_id(void* id_out /* 128 bytes (ncclUniqueId) */);
int rtk_nccl_comm_init_rank(void** comm_out, int nranks, const void* id /* 128 bytes */, int rank, int device);
int rtk_nccl_comm_destroy(void* comm);
int rtk_topk_sharded(const rtk_handle* handles, void* const* comms, int L, const void* const* d_shards,
                     const uint64_t* shard_n, int world, uint64_t k, int dtype, int order,
                     void* const* d_out_vals, uint64_t* const* d_out_idx, void* const* d_out_pivots,
                     void* const* streams);

/* LLM sampling consumer: top-k of B logit rows (row b at
 * d_logits + b*row_stride elements, V elements, dtype F32/F16/BF16), then per row, in fp32:
 *   e_j = expf((v_j - v_0) / temperature) over the top-k in canonical order (v_0 = row max);
 *   m = shortest prefix with sum_{j<m} e_j >= top_p * sum_j e_j (top_p = 1 keeps all k);
 *   token = index of the first j < m with sum_{i<=j} e_i > u_b * sum_{i<m} e_i (u_b = d_uniform[b],
 *   in [0, 1)); d_probs (nullable, B*k) = e_j / sum_{i<m} e_i for j < m, else 0.
 * d_topk_vals / d_topk_idx (nullable, B*k) receive the top-k itself (handle workspace if NULL).
 * Device pointers, stream-ordered. Tokens are row-local u64 indices. */
int rtk_topk_sample(rtk_handle h, const void* d_logits, uint64_t B, uint64_t V, uint64_t row_stride, int dtype,
                    uint64_t k, float top_p, float temperature, const float* d_uniform, uint64_t* d_token,
                    float* d_probs, void* d_topk_vals, uint64_t* d_topk_idx, void* stream);

/* ---- harness utilities (host only) -----------------------------------
 * rtk_generate        <- rtk::generate<float|uint32_t>     datagen.hpp:68-140 (same mt19937_64
 *                        streams and libstdc++ distributions, so inputs are bit-identical)
 * rtk_result_checksum <- result_checksum                   rtk_cli.cpp:100-115 (FNV-1a over
 *                        value bits then the u64 index, element by element)
 * rtk_write_dataset / rtk_read_dataset <- rtk::write_dataset / read_dataset  io.cpp:38-80 (RTK1;
 *                        dtype codes 0 f32, 1 u32, 2 f16 — accepted here — and 3 bf16)
 * rtk_write_batch / rtk_read_batch     <- rtk::write_batch / read_batch      io.cpp:82-110 (RTKB)
 * Readers are two-call: pass NULL outputs to query the sizes first. */
int rtk_generate(const rtk_dist* spec, int dtype, void* out);
/* Counter-based uniform f32 generator for queries too large for host memory (BASELINE C5,
 * n = 2^32 over 8 GPUs): element j of the output is element offset + j of
 * the Philox4x32-10 stream keyed by seed (word (g & 3) of block g >> 2), mapped to [a, b) as
 * a + ((w >> 8) * 2^-24) * (b - a) in fp32 round-to-nearest (exactly (w >> 8) * 2^-24 for [0, 1)).
 * rtk_generate_philox writes DEVICE memory on `stream`; rtk_generate_philox_host is the
 * bit-identical host twin (any index range, e.g. single elements for verification). */
int rtk_generate_philox(float* d_out, uint64_t n, uint64_t seed, uint64_t offset, float a, float b, void* stream);
int rtk_generate_philox_host(float* out, uint64_t n, uint64_t seed, uint64_t offset, float a, float b);
uint64_t rtk_result_checksum(const void* values, int dtype, const uint64_t* indices, uint64_t k);
int rtk_write_dataset(const char* path, int dtype, const void* data, uint64_t n);
int rtk_read_dataset(const char* path, int* dtype, uint64_t* n, void* out, uint64_t capacity);
int rtk_write_batch(const char* path, const uint64_t* lengths, uint32_t tasks, const void* payload,
                    uint64_t payload_bytes);
int rtk_read_batch(const char* path, uint32_t* tasks, uint64_t* payload_bytes, uint64_t* lengths,
                   void* payload);

#ifdef __cplusplus
}
#endif

#endif /* RTK_C_H */
