// rtk_capi.cpp — the extern "C" boundary (include/rtk_c.h). Validation mirrors the
// reference's exceptions one-to-one (engine.hpp:31-41, 61-67, 425-426; batch.hpp:40-53,
// 274-280; scaling.hpp:47-48) as status codes + a thread-local message.
#include <cuda_runtime.h>

#include <chrono>
#include <cstring>
#include <mutex>
#include <new>
#include <random>
#include <string>
#include <vector>

#include "../../include/rtk_c.h"
#include "rtk_engine.h"
#include "rtk_guard.h"
#include "rtk_sharded.h"

using rtk_b200::Engine;
using rtk_b200::Error;
using rtk_b200::RowReq;

struct rtk_handle_s {
    // one caller at a time per handle: the engine's workspace, pinned staging, graph cache and
    // signal words are shared state (recursive: the bench helpers call the entry points)
    std::recursive_mutex mu;
    Engine engine;
    rtk_b200::DevBuf smp_vals, smp_idx;  // top-k workspace of rtk_topk_sample (when not supplied)
    rtk_b200::ShardWork shard;           // candidate slots of rtk_topk_sharded
    explicit rtk_handle_s(int dev) : engine(dev) {}
    ~rtk_handle_s() {
        smp_vals.release();
        smp_idx.release();
        shard.release();
    }
};

thread_local std::string rtk_b200::g_last_error;
using rtk_b200::fail;
using rtk_b200::g_last_error;
using rtk_b200::guarded;

namespace {

// every entry point taking a handle: status codes, the handle's lock, its device made current
// (and the caller's restored)
template <typename F>
int on_handle(rtk_handle h, F&& f) {
    return guarded([&] {
        if (!h) throw Error{RTK_INVALID_ARGUMENT, "null handle"};
        std::lock_guard<std::recursive_mutex> lock(h->mu);
        rtk_b200::DeviceGuard dg(h->engine.device());
        f();
    });
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error{RTK_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e)};
}

// Step timing of the rtk_bench_* helpers: per step a start/end CUDA event pair (recorded by the
// engine on the call's stream around its device work) and the host wall time of the call
// (steady_clock around the C entry point, which returns after the device's completion signal).
// An optional L2 flush (memset of > L2 bytes) runs before each step, outside both clocks.
class BenchSteps {
public:
    BenchSteps(int steps, cudaStream_t s, void* flush, uint64_t flush_bytes)
        : ev_(2 * steps), host_(steps), s_(s), flush_(flush), flush_bytes_(flush_bytes) {
        for (auto& e : ev_) cuda_check(cudaEventCreate(&e), "event");
        cuda_check(cudaStreamSynchronize(s_), "sync");
    }
    ~BenchSteps() {
        for (auto& e : ev_) cudaEventDestroy(e);
    }
    cudaEvent_t start(int i) const { return ev_[2 * i]; }
    cudaEvent_t end(int i) const { return ev_[2 * i + 1]; }
    void before(int i) {
        if (flush_ && flush_bytes_) {
            cuda_check(cudaMemsetAsync(flush_, i & 0xff, flush_bytes_, s_), "flush");
            cuda_check(cudaStreamSynchronize(s_), "flush sync");
        }
        t0_ = std::chrono::steady_clock::now();
    }
    void after(int i) {
        host_[i] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count();
    }
    void finish(float* step_ms, float* step_host_ms, float* mean_ms) {
        cuda_check(cudaStreamSynchronize(s_), "sync");
        double sum = 0;
        for (size_t i = 0; i < host_.size(); ++i) {
            float ms = 0;
            cuda_check(cudaEventElapsedTime(&ms, ev_[2 * i], ev_[2 * i + 1]), "elapsed");
            if (step_ms) step_ms[i] = ms;
            if (step_host_ms) step_host_ms[i] = static_cast<float>(host_[i]);
            sum += ms;
        }
        if (mean_ms) *mean_ms = static_cast<float>(sum / host_.size());
    }

private:
    std::vector<cudaEvent_t> ev_;
    std::vector<double> host_;
    cudaStream_t s_;
    void* flush_;
    uint64_t flush_bytes_;
    std::chrono::steady_clock::time_point t0_;
};

rtk_cfg default_cfg() {
    rtk_cfg c;
    rtk_cfg_default(&c);
    return c;
}

// EngineConfig::validate (engine.hpp:61-67)
void validate_cfg(const rtk_cfg& c) {
    if (c.d < 1 || c.d > 16) throw Error{RTK_INVALID_ARGUMENT, "digit width must be in [1, 16]"};
    if (c.block_size < 1) throw Error{RTK_INVALID_ARGUMENT, "block_size must be >= 1"};
    if (c.grid_size < 1) throw Error{RTK_INVALID_ARGUMENT, "grid_size must be >= 1"};
    if (c.pack_size < 4 || (c.pack_size & (c.pack_size - 1)) != 0)
        throw Error{RTK_INVALID_ARGUMENT, "pack_size must be a power of two >= element width"};
}

bool dtype_ok(int d) { return d == RTK_F32 || d == RTK_U32 || d == RTK_F16 || d == RTK_BF16; }
int eng_dtype(int d) { return d == RTK_BF16 ? rtk_b200::kF16 : d; }  // f16 and bf16 share the map
size_t esize(int d) { return (d == RTK_F16 || d == RTK_BF16) ? 2 : 4; }

void check_common(const void* ptr, uint64_t n, uint64_t k, int dtype, int order, const rtk_cfg& cfg,
                  const char* who) {
    // topk: empty -> empty_input_error, k outside [1,n] -> rank_out_of_range (engine.hpp:425-426);
    // radix_select then validates the config (:296)
    if (n == 0) throw Error{RTK_EMPTY_INPUT, std::string(who) + ": empty input"};
    if (k == 0 || k > n) throw Error{RTK_RANK_OUT_OF_RANGE, std::string(who) + ": k outside [1, n]"};
    validate_cfg(cfg);
    if (!dtype_ok(dtype)) throw Error{RTK_INVALID_ARGUMENT, "dtype must be F32, U32, F16 or BF16"};
    if (order != RTK_LARGEST && order != RTK_SMALLEST) throw Error{RTK_INVALID_ARGUMENT, "bad order"};
    if (n > (uint64_t(1) << 32)) throw Error{RTK_INVALID_ARGUMENT, "n > 2^32 per device row is not supported"};
    if (!ptr) throw Error{RTK_INVALID_ARGUMENT, "null input"};
}

// BatchInput::validate (batch.hpp:40-53)
void validate_batch(uint64_t data_len, const uint64_t* offsets, const uint64_t* lengths,
                    const uint64_t* ks, uint64_t B) {
    if (B == 0) throw Error{RTK_INVALID_ARGUMENT, "batch: no tasks"};
    if (!offsets || !lengths || !ks) throw Error{RTK_INVALID_ARGUMENT, "batch: descriptor arrays disagree"};
    for (uint64_t i = 0; i < B; ++i) {
        const uint64_t next = i + 1 < B ? offsets[i + 1] : data_len;
        if (offsets[i] + lengths[i] > next)
            throw Error{RTK_INVALID_ARGUMENT, "batch: task " + std::to_string(i) + " overlaps its successor"};
        if (ks[i] == 0 || ks[i] > lengths[i])
            throw Error{RTK_INVALID_ARGUMENT, "batch: task " + std::to_string(i) + " has k outside [1, n]"};
        if (lengths[i] > (uint64_t(1) << 32))
            throw Error{RTK_INVALID_ARGUMENT, "batch: task " + std::to_string(i) + " longer than 2^32"};
    }
}

std::vector<uint64_t> packed_out_offsets(const uint64_t* ks, uint64_t B) {
    std::vector<uint64_t> o(B);
    uint64_t acc = 0;
    for (uint64_t i = 0; i < B; ++i) {
        o[i] = acc;
        acc += ks[i];
    }
    return o;
}

// scaled_topk (scaling.hpp:47-79). The decision is taken on the device: Adaptive runs the
// exact first-window histogram and a one-CTA select_bin/trigger kernel; Always only fetches
// a_s. Every pipeline kernel reads {flag, a_s} at its start, so no host round trip separates
// the trigger pass from the selection. a_index = mt19937_64(seed)() % n (draw_scale) is drawn
// on the host; values are re-read from the input by index (scaling.hpp:74-75).
void run_scaled(Engine& e, const float* d_in, uint64_t n, uint64_t k, int order, int mode, double tau,
                uint64_t seed, float* d_vals, uint64_t* d_idx, float* d_piv, rtk_scale_info* info,
                const rtk_cfg& cfg, cudaStream_t s) {
    if (mode != RTK_SCALE_OFF && mode != RTK_SCALE_ALWAYS && mode != RTK_SCALE_ADAPTIVE)
        throw Error{RTK_INVALID_ARGUMENT, "bad scale mode"};
    if (mode == RTK_SCALE_OFF) {
        e.run(reinterpret_cast<const uint32_t*>(d_in), RTK_F32, order, false, 0.0f, false, {RowReq{0, n, k, 0}},
              reinterpret_cast<uint32_t*>(d_vals), d_idx, reinterpret_cast<uint32_t*>(d_piv), s);
        if (info) *info = rtk_scale_info{0, 0.0f, 0};
        return;
    }
    std::mt19937_64 rng(seed);
    const uint64_t a_index = rng() % n;
    auto select = [&](bool count_trigger) {
        e.set_adapt(e.device_scale());
        e.set_trigger_count(count_trigger);
        try {
            e.run(reinterpret_cast<const uint32_t*>(d_in), RTK_F32, order, false, 0.0f, /*gather=*/true,
                  {RowReq{0, n, k, 0}}, reinterpret_cast<uint32_t*>(d_vals), d_idx,
                  reinterpret_cast<uint32_t*>(d_piv), s);
        } catch (...) {
            e.set_adapt(nullptr);
            e.set_trigger_count(false);
            throw;
        }
        e.set_adapt(nullptr);
        e.set_trigger_count(false);
    };
    // Adaptive on a row that streams through k_compact (not a one-CTA row, not a dense k >= n/2
    // row): speculate on a sampled trigger and verify it with the exact counts of the same pass
    const bool speculate = mode == RTK_SCALE_ADAPTIVE && cfg.d <= 14 && n > (uint64_t(1) << 18) && 2 * k < n;
    bool exact_trigger = mode == RTK_SCALE_ADAPTIVE && !speculate;
    if (speculate) {
        e.enqueue_scale_guess(reinterpret_cast<const uint32_t*>(d_in), n, k, cfg.d, order, tau, a_index, s);
        select(true);
        uint64_t gt = 0, eq = 0;
        e.trigger_counts(&gt, &eq);
        bool guessed = false;
        float unused = 0.0f;
        e.scale_result(&guessed, &unused);
        // gt < k <= gt + eq: the guessed bin IS select_bin's bin (engine.hpp:231-241), eq its count
        const bool bin_ok = gt < k && k <= gt + eq;
        const bool fat = static_cast<double>(eq) > tau * static_cast<double>(n);
        if (!bin_ok || fat != guessed) exact_trigger = true;  // wrong guess: the exact trigger, rerun
    }
    if (mode == RTK_SCALE_ALWAYS || exact_trigger) {
        e.enqueue_scale_decide(reinterpret_cast<const uint32_t*>(d_in), n, k, cfg.d, order,
                               mode == RTK_SCALE_ALWAYS ? 1 : 2, tau, a_index, s);
        select(false);
    }
    if (exact_trigger) {
        e.stats.passes += 1;
        e.stats.elements_scanned += n;
    }
    if (info) {
        bool sc = false;
        float a = 0.0f;
        e.scale_result(&sc, &a);
        info->scaled = sc ? 1 : 0;
        info->a_s = sc ? a : 0.0f;
        info->a_index = sc ? a_index : 0;
    }
}

}  // namespace

extern "C" {

const char* rtk_version(void) { return "rtk-b200 0.1 (sm_100a)"; }

const char* rtk_last_error(void) { return g_last_error.c_str(); }

void rtk_cfg_default(rtk_cfg* c) {
    if (!c) return;
    c->d = 12;
    c->block_size = 1024;
    c->grid_size = 4;
    c->buffer_policy = 1;
    c->pack_size = 16;
    c->hierarchical_atomics = 1;
    c->filter_fixed_ceiling = 4096;
}

int rtk_cfg_validate(const rtk_cfg* c) {
    return guarded([&] {
        if (!c) throw Error{RTK_INVALID_ARGUMENT, "null config"};
        validate_cfg(*c);
    });
}

int rtk_handle_create(rtk_handle* out, int device) {
    return guarded([&] {
        if (!out) throw Error{RTK_INVALID_ARGUMENT, "null handle pointer"};
        int count = 0;
        cuda_check(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
        if (device < 0 || device >= count) throw Error{RTK_INVALID_ARGUMENT, "no such CUDA device"};
        rtk_b200::DeviceGuard dg(device);
        *out = new rtk_handle_s(device);
    });
}

int rtk_handle_destroy(rtk_handle h) {
    return guarded([&] {
        if (!h) return;
        rtk_b200::DeviceGuard dg(h->engine.device());
        delete h;
    });
}

int rtk_set_timing(rtk_handle h, int on) {
    return on_handle(h, [&] {
        h->engine.set_timing(on != 0);
    });
}

int rtk_set_option(rtk_handle h, const char* name, int64_t value) {
    return on_handle(h, [&] {
        if (!name || !h->engine.set_option(name, value))
            throw Error{RTK_INVALID_ARGUMENT, std::string("unknown option: ") + (name ? name : "(null)")};
    });
}

int rtk_get_batch_info(rtk_handle h, uint64_t* task_passes, uint64_t B, uint64_t* phase_b_rounds) {
    return on_handle(h, [&] {
        const std::vector<uint64_t>& p = h->engine.row_passes();
        if (task_passes && B > p.size()) throw Error{RTK_INVALID_ARGUMENT, "batch info: more tasks than the last call had"};
        if (task_passes)
            for (uint64_t t = 0; t < B; ++t) task_passes[t] = p[t];
        if (phase_b_rounds) *phase_b_rounds = h->engine.last_stats().deep_levels;
    });
}

int rtk_get_stats(rtk_handle h, rtk_stats* out) {
    return on_handle(h, [&] {
        if (!out) throw Error{RTK_INVALID_ARGUMENT, "null argument"};
        *out = h->engine.last_stats();
    });
}

int rtk_topk(rtk_handle h, const void* d_in, uint64_t n, uint64_t k, int dtype, int order,
             void* d_out_vals, uint64_t* d_out_idx, void* d_out_pivot, const rtk_cfg* cfg,
             void* stream) {
    return on_handle(h, [&] {
        const rtk_cfg c = cfg ? *cfg : default_cfg();
        check_common(d_in, n, k, dtype, order, c, "topk");
        h->engine.run(static_cast<const uint32_t*>(d_in), eng_dtype(dtype), order, false, 0.0f, false,
                      {RowReq{0, n, k, 0}}, static_cast<uint32_t*>(d_out_vals), d_out_idx,
                      static_cast<uint32_t*>(d_out_pivot), static_cast<cudaStream_t>(stream));
    });
}

int rtk_bench_topk(rtk_handle h, const void* d_in, uint64_t n, uint64_t k, int dtype, int order,
                   void* d_out_vals, uint64_t* d_out_idx, void* d_out_pivot, const rtk_cfg* cfg,
                   void* stream, void* d_flush, uint64_t flush_bytes, int warmup, int steps, float* step_ms,
                   float* step_host_ms, float* mean_ms) {
    return on_handle(h, [&] {
        if (steps < 1 || warmup < 0) throw Error{RTK_INVALID_ARGUMENT, "bench: bad arguments"};
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        for (int i = 0; i < warmup; ++i) {
            const int st = rtk_topk(h, d_in, n, k, dtype, order, d_out_vals, d_out_idx, d_out_pivot, cfg, stream);
            if (st != RTK_OK) throw Error{st, g_last_error};
        }
        // per step: events the engine records right before its first and after its last device
        // operation of the call (host planning and the host's completion wait excluded)
        BenchSteps b(steps, s, d_flush, flush_bytes);
        for (int i = 0; i < steps; ++i) {
            b.before(i);
            h->engine.set_call_events(b.start(i), b.end(i));
            const int st = rtk_topk(h, d_in, n, k, dtype, order, d_out_vals, d_out_idx, d_out_pivot, cfg, stream);
            h->engine.set_call_events(nullptr, nullptr);
            if (st != RTK_OK) throw Error{st, g_last_error};
            b.after(i);
        }
        b.finish(step_ms, step_host_ms, mean_ms);
    });
}

int rtk_bench_scaled(rtk_handle h, const float* d_in, uint64_t n, uint64_t k, int order, int mode,
                     double trigger_fraction, uint64_t seed, float* d_out_vals, uint64_t* d_out_idx,
                     float* d_out_pivot, const rtk_cfg* cfg, void* stream, void* d_flush, uint64_t flush_bytes,
                     int warmup, int steps, float* step_ms, float* step_host_ms, float* mean_ms) {
    return on_handle(h, [&] {
        if (steps < 1 || warmup < 0) throw Error{RTK_INVALID_ARGUMENT, "bench: bad arguments"};
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        auto one = [&] {
            const int st = rtk_topk_scaled(h, d_in, n, k, order, mode, trigger_fraction, seed, d_out_vals, d_out_idx,
                                           d_out_pivot, nullptr, cfg, stream);
            if (st != RTK_OK) throw Error{st, g_last_error};
        };
        for (int i = 0; i < warmup; ++i) one();
        BenchSteps b(steps, s, d_flush, flush_bytes);
        for (int i = 0; i < steps; ++i) {
            b.before(i);
            cuda_check(cudaEventRecord(b.start(i), s), "event");  // before the scale decision's kernels
            h->engine.set_call_events(nullptr, b.end(i));
            try {
                one();
            } catch (...) {
                h->engine.set_call_events(nullptr, nullptr);
                throw;
            }
            h->engine.set_call_events(nullptr, nullptr);
            b.after(i);
        }
        b.finish(step_ms, step_host_ms, mean_ms);
    });
}

int rtk_bench_batched(rtk_handle h, const void* d_data, uint64_t data_len, const uint64_t* offsets,
                      const uint64_t* lengths, const uint64_t* ks, uint64_t B, int dtype, int order,
                      void* d_out_vals, uint64_t* d_out_idx, const uint64_t* out_offsets,
                      void* d_out_pivots, const rtk_cfg* cfg, void* stream, void* d_flush,
                      uint64_t flush_bytes, int warmup, int steps, float* step_ms, float* step_host_ms,
                      float* mean_ms) {
    return on_handle(h, [&] {
        if (steps < 1 || warmup < 0) throw Error{RTK_INVALID_ARGUMENT, "bench: bad arguments"};
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        auto one = [&] {
            const int st = rtk_topk_batched(h, d_data, data_len, offsets, lengths, ks, B, dtype, order, d_out_vals,
                                            d_out_idx, out_offsets, d_out_pivots, cfg, nullptr, stream);
            if (st != RTK_OK) throw Error{st, g_last_error};
        };
        for (int i = 0; i < warmup; ++i) one();
        BenchSteps b(steps, s, d_flush, flush_bytes);
        for (int i = 0; i < steps; ++i) {
            b.before(i);
            h->engine.set_call_events(b.start(i), b.end(i));
            try {
                one();
            } catch (...) {
                h->engine.set_call_events(nullptr, nullptr);
                throw;
            }
            h->engine.set_call_events(nullptr, nullptr);
            b.after(i);
        }
        b.finish(step_ms, step_host_ms, mean_ms);
    });
}

int rtk_topk_batched(rtk_handle h, const void* d_data, uint64_t data_len, const uint64_t* offsets,
                     const uint64_t* lengths, const uint64_t* ks, uint64_t B, int dtype, int order,
                     void* d_out_vals, uint64_t* d_out_idx, const uint64_t* out_offsets,
                     void* d_out_pivots, const rtk_cfg* cfg, const rtk_batch_opts* opts,
                     void* stream) {
    (void)opts;  // rescheduling / padding change the schedule only, never the results
    return on_handle(h, [&] {
        validate_batch(data_len, offsets, lengths, ks, B);
        const rtk_cfg c = cfg ? *cfg : default_cfg();
        validate_cfg(c);
        if (!dtype_ok(dtype)) throw Error{RTK_INVALID_ARGUMENT, "dtype must be F32, U32, F16 or BF16"};
        if (order != RTK_LARGEST && order != RTK_SMALLEST) throw Error{RTK_INVALID_ARGUMENT, "bad order"};
        if (!d_data) throw Error{RTK_INVALID_ARGUMENT, "null input"};
        std::vector<uint64_t> oo = out_offsets ? std::vector<uint64_t>(out_offsets, out_offsets + B)
                                               : packed_out_offsets(ks, B);
        std::vector<RowReq> rows(B);
        for (uint64_t t = 0; t < B; ++t) rows[t] = RowReq{offsets[t], lengths[t], ks[t], oo[t]};
        h->engine.run(static_cast<const uint32_t*>(d_data), eng_dtype(dtype), order, false, 0.0f, false, rows,
                      static_cast<uint32_t*>(d_out_vals), d_out_idx, static_cast<uint32_t*>(d_out_pivots),
                      static_cast<cudaStream_t>(stream));
    });
}

int rtk_topk_scaled(rtk_handle h, const float* d_in, uint64_t n, uint64_t k, int order, int mode,
                    double trigger_fraction, uint64_t seed, float* d_out_vals, uint64_t* d_out_idx,
                    float* d_out_pivot, rtk_scale_info* info, const rtk_cfg* cfg, void* stream) {
    return on_handle(h, [&] {
        const rtk_cfg c = cfg ? *cfg : default_cfg();
        if (n == 0) throw Error{RTK_EMPTY_INPUT, "scaled_topk: empty input"};
        if (k == 0 || k > n) throw Error{RTK_RANK_OUT_OF_RANGE, "scaled_topk: k outside [1, n]"};
        check_common(d_in, n, k, RTK_F32, order, c, "scaled_topk");
        run_scaled(h->engine, d_in, n, k, order, mode, trigger_fraction, seed, d_out_vals, d_out_idx,
                   d_out_pivot, info, c, static_cast<cudaStream_t>(stream));
    });
}

// LLM sampling consumer: batched top-k of B logit rows, then softmax /
// top-p / one inverse-CDF draw per row (rtk_sample.cu) on the same stream.
int rtk_topk_sample(rtk_handle h, const void* d_logits, uint64_t B, uint64_t V, uint64_t row_stride, int dtype,
                    uint64_t k, float top_p, float temperature, const float* d_uniform, uint64_t* d_token,
                    float* d_probs, void* d_topk_vals, uint64_t* d_topk_idx, void* stream) {
    return on_handle(h, [&] {
        if (B == 0) throw Error{RTK_INVALID_ARGUMENT, "sample: no rows"};
        if (V == 0) throw Error{RTK_EMPTY_INPUT, "sample: empty rows"};
        if (k == 0 || k > V) throw Error{RTK_RANK_OUT_OF_RANGE, "sample: k outside [1, V]"};
        if (row_stride < V) throw Error{RTK_INVALID_ARGUMENT, "sample: row_stride < V"};
        if (dtype != RTK_F32 && dtype != RTK_F16 && dtype != RTK_BF16)
            throw Error{RTK_INVALID_ARGUMENT, "sample: logits must be F32, F16 or BF16"};
        if (!(top_p > 0.f && top_p <= 1.f)) throw Error{RTK_INVALID_ARGUMENT, "sample: top_p must be in (0, 1]"};
        if (!(temperature > 0.f)) throw Error{RTK_INVALID_ARGUMENT, "sample: temperature must be > 0"};
        if (!d_logits || !d_uniform || !d_token) throw Error{RTK_INVALID_ARGUMENT, "sample: null argument"};
        if (V > (uint64_t(1) << 32)) throw Error{RTK_INVALID_ARGUMENT, "sample: V > 2^32"};
        Engine& e = h->engine;
        rtk_b200::DeviceGuard dg(e.device());
        void* tv = d_topk_vals;
        uint64_t* ti = d_topk_idx;
        if (!tv) {
            h->smp_vals.ensure(esize(dtype) * B * k);
            tv = h->smp_vals.p;
        }
        if (!ti) {
            h->smp_idx.ensure(8 * B * k);
            ti = h->smp_idx.as<uint64_t>();
        }
        std::vector<RowReq> rows(B);
        for (uint64_t b = 0; b < B; ++b) rows[b] = RowReq{b * row_stride, V, k, b * k};
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        e.run(static_cast<const uint32_t*>(d_logits), eng_dtype(dtype), RTK_LARGEST, false, 0.0f, false, rows,
              static_cast<uint32_t*>(tv), ti, nullptr, s);
        const int fmt = dtype == RTK_F32 ? 0 : (dtype == RTK_F16 ? 2 : 3);
        rtk_b200::launch_sample_rows(B, tv, fmt, ti, k, top_p, temperature, d_uniform, d_token, d_probs, s);
        cuda_check(cudaGetLastError(), "sample launch");
    });
}

// ---- host-pointer variants ----------------------------------------------------------------

int rtk_topk_host(rtk_handle h, const void* in, uint64_t n, uint64_t k, int dtype, int order,
                  void* out_vals, uint64_t* out_idx, void* out_pivot, const rtk_cfg* cfg) {
    return on_handle(h, [&] {
        const rtk_cfg c = cfg ? *cfg : default_cfg();
        check_common(in, n, k, dtype, order, c, "topk");
        Engine& e = h->engine;
        rtk_b200::DeviceGuard dg(e.device());
        e.io_in.ensure(esize(dtype) * n);
        e.io_vals.ensure(esize(dtype) * k);
        e.io_idx.ensure(8 * k);
        e.io_piv.ensure(4);
        cudaStream_t s = nullptr;
        cuda_check(cudaMemcpyAsync(e.io_in.p, in, esize(dtype) * n, cudaMemcpyHostToDevice, s), "h2d");
        e.run(e.io_in.as<uint32_t>(), eng_dtype(dtype), order, false, 0.0f, false, {RowReq{0, n, k, 0}},
              e.io_vals.as<uint32_t>(), e.io_idx.as<uint64_t>(), e.io_piv.as<uint32_t>(), s);
        cuda_check(cudaMemcpyAsync(out_vals, e.io_vals.p, esize(dtype) * k, cudaMemcpyDeviceToHost, s), "d2h");
        cuda_check(cudaMemcpyAsync(out_idx, e.io_idx.p, 8 * k, cudaMemcpyDeviceToHost, s), "d2h");
        if (out_pivot) cuda_check(cudaMemcpyAsync(out_pivot, e.io_piv.p, esize(dtype), cudaMemcpyDeviceToHost, s), "d2h");
        cuda_check(cudaStreamSynchronize(s), "sync");
    });
}

int rtk_topk_batched_host(rtk_handle h, const void* data, uint64_t data_len, const uint64_t* offsets,
                          const uint64_t* lengths, const uint64_t* ks, uint64_t B, int dtype, int order,
                          void* out_vals, uint64_t* out_idx, const uint64_t* out_offsets, void* out_pivots,
                          const rtk_cfg* cfg, const rtk_batch_opts* opts) {
    return on_handle(h, [&] {
        validate_batch(data_len, offsets, lengths, ks, B);
        std::vector<uint64_t> oo = out_offsets ? std::vector<uint64_t>(out_offsets, out_offsets + B)
                                               : packed_out_offsets(ks, B);
        uint64_t out_total = 0;
        for (uint64_t t = 0; t < B; ++t) out_total = std::max(out_total, oo[t] + ks[t]);
        Engine& e = h->engine;
        rtk_b200::DeviceGuard dg(e.device());
        e.io_in.ensure(esize(dtype) * std::max<uint64_t>(data_len, 1));
        e.io_vals.ensure(esize(dtype) * out_total);
        e.io_idx.ensure(8 * out_total);
        e.io_piv.ensure(esize(dtype) * B);
        cudaStream_t s = nullptr;
        cuda_check(cudaMemcpyAsync(e.io_in.p, data, esize(dtype) * data_len, cudaMemcpyHostToDevice, s), "h2d");
        int st = rtk_topk_batched(h, e.io_in.p, data_len, offsets, lengths, ks, B, dtype, order, e.io_vals.p,
                                  e.io_idx.as<uint64_t>(), oo.data(), e.io_piv.p, cfg, opts, s);
        if (st != RTK_OK) throw Error{st, g_last_error};
        // outputs may be ragged: copy each row's slots
        bool packed = true;
        for (uint64_t t = 0, acc = 0; t < B; acc += ks[t], ++t) packed &= oo[t] == acc;
        if (packed) {
            cuda_check(cudaMemcpyAsync(out_vals, e.io_vals.p, esize(dtype) * out_total, cudaMemcpyDeviceToHost, s), "d2h");
            cuda_check(cudaMemcpyAsync(out_idx, e.io_idx.p, 8 * out_total, cudaMemcpyDeviceToHost, s), "d2h");
        } else {
            for (uint64_t t = 0; t < B; ++t) {
                cuda_check(cudaMemcpyAsync(static_cast<char*>(out_vals) + esize(dtype) * oo[t],
                                           e.io_vals.as<char>() + esize(dtype) * oo[t], esize(dtype) * ks[t],
                                           cudaMemcpyDeviceToHost, s), "d2h");
                cuda_check(cudaMemcpyAsync(out_idx + oo[t], e.io_idx.as<uint64_t>() + oo[t], 8 * ks[t],
                                           cudaMemcpyDeviceToHost, s), "d2h");
            }
        }
        if (out_pivots)
            cuda_check(cudaMemcpyAsync(out_pivots, e.io_piv.p, esize(dtype) * B, cudaMemcpyDeviceToHost, s), "d2h");
        cuda_check(cudaStreamSynchronize(s), "sync");
    });
}

int rtk_topk_scaled_host(rtk_handle h, const float* in, uint64_t n, uint64_t k, int order, int mode,
                         double trigger_fraction, uint64_t seed, float* out_vals, uint64_t* out_idx,
                         float* out_pivot, rtk_scale_info* info, const rtk_cfg* cfg) {
    return on_handle(h, [&] {
        const rtk_cfg c = cfg ? *cfg : default_cfg();
        if (n == 0) throw Error{RTK_EMPTY_INPUT, "scaled_topk: empty input"};
        if (k == 0 || k > n) throw Error{RTK_RANK_OUT_OF_RANGE, "scaled_topk: k outside [1, n]"};
        check_common(in, n, k, RTK_F32, order, c, "scaled_topk");
        Engine& e = h->engine;
        rtk_b200::DeviceGuard dg(e.device());
        e.io_in.ensure(4 * n);
        e.io_vals.ensure(4 * k);
        e.io_idx.ensure(8 * k);
        e.io_piv.ensure(4);
        cudaStream_t s = nullptr;
        cuda_check(cudaMemcpyAsync(e.io_in.p, in, 4 * n, cudaMemcpyHostToDevice, s), "h2d");
        run_scaled(e, e.io_in.as<float>(), n, k, order, mode, trigger_fraction, seed, e.io_vals.as<float>(),
                   e.io_idx.as<uint64_t>(), e.io_piv.as<float>(), info, c, s);
        cuda_check(cudaMemcpyAsync(out_vals, e.io_vals.p, 4 * k, cudaMemcpyDeviceToHost, s), "d2h");
        cuda_check(cudaMemcpyAsync(out_idx, e.io_idx.p, 8 * k, cudaMemcpyDeviceToHost, s), "d2h");
        if (out_pivot) cuda_check(cudaMemcpyAsync(out_pivot, e.io_piv.p, 4, cudaMemcpyDeviceToHost, s), "d2h");
        cuda_check(cudaStreamSynchronize(s), "sync");
    });
}

int rtk_nccl_get_unique_id(void* id_out) {
    return guarded([&] {
        if (!id_out) throw Error{RTK_INVALID_ARGUMENT, "null id"};
        rtk_b200::nccl_unique_id(id_out);
    });
}

int rtk_nccl_comm_init_rank(void** comm_out, int nranks, const void* id, int rank, int device) {
    return guarded([&] {
        if (!comm_out || !id || nranks < 1 || rank < 0 || rank >= nranks)
            throw Error{RTK_INVALID_ARGUMENT, "nccl comm init: bad arguments"};
        *comm_out = rtk_b200::nccl_comm_init(nranks, id, rank, device);
    });
}

int rtk_nccl_comm_destroy(void* comm) {
    return guarded([&] { rtk_b200::nccl_comm_destroy(comm); });
}

int rtk_topk_sharded(const rtk_handle* handles, void* const* comms, int L, const void* const* d_shards,
                     const uint64_t* shard_n, int world, uint64_t k, int dtype, int order,
                     void* const* d_out_vals, uint64_t* const* d_out_idx, void* const* d_out_pivots,
                     void* const* streams) {
    return guarded([&] {
        if (!handles || !comms || !d_shards || !shard_n || !d_out_vals || !d_out_idx || L < 1 || world < 1 || L > world)
            throw Error{RTK_INVALID_ARGUMENT, "topk_sharded: bad arguments"};
        if (!dtype_ok(dtype)) throw Error{RTK_INVALID_ARGUMENT, "dtype must be F32, U32, F16 or BF16"};
        if (order != RTK_LARGEST && order != RTK_SMALLEST) throw Error{RTK_INVALID_ARGUMENT, "bad order"};
        std::vector<Engine*> eng(L);
        std::vector<rtk_b200::ShardWork*> work(L);
        std::vector<std::unique_lock<std::recursive_mutex>> locks;
        for (int i = 0; i < L; ++i) {
            if (!handles[i] || !comms[i] || !d_shards[i] || !d_out_vals[i] || !d_out_idx[i])
                throw Error{RTK_INVALID_ARGUMENT, "topk_sharded: null entry"};
            locks.emplace_back(handles[i]->mu);
            eng[i] = &handles[i]->engine;
            work[i] = &handles[i]->shard;
        }
        for (int g = 0; g < world; ++g)
            if (shard_n[g] > (uint64_t(1) << 32)) throw Error{RTK_INVALID_ARGUMENT, "shard longer than 2^32"};
        rtk_b200::topk_sharded(eng.data(), work.data(), comms, L, d_shards, shard_n, world, k, eng_dtype(dtype),
                               static_cast<int>(esize(dtype)), order, d_out_vals, d_out_idx, d_out_pivots, streams);
    });
}

int rtk_merge_shards(rtk_handle h, const void* d_cand_vals, const uint64_t* d_cand_idx,
                     const uint64_t* block_len, const uint64_t* shard_base, uint32_t G, uint64_t k,
                     int dtype, int order, void* d_out_vals, uint64_t* d_out_idx, void* d_out_pivot,
                     void* stream) {
    return on_handle(h, [&] {
        if (!block_len || !shard_base || G == 0) throw Error{RTK_INVALID_ARGUMENT, "bad shard descriptor"};
        std::vector<uint64_t> start(G), base(shard_base, shard_base + G);
        uint64_t total = 0;
        for (uint32_t g = 0; g < G; ++g) {
            start[g] = total;
            total += block_len[g];
            if (g && base[g] < base[g - 1]) throw Error{RTK_INVALID_ARGUMENT, "shards must be in index order"};
        }
        const rtk_cfg c = default_cfg();
        check_common(d_cand_vals, total, k, dtype, order, c, "merge_shards");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        // Tie-break surrogate = position in the concatenation: each block is in (key desc,
        // index asc) order and blocks are in ascending index order, so among equal keys
        // position order == global index order.
        h->engine.run(static_cast<const uint32_t*>(d_cand_vals), eng_dtype(dtype), order, false, 0.0f, false,
                      {RowReq{0, total, k, 0}}, static_cast<uint32_t*>(d_out_vals), d_out_idx,
                      static_cast<uint32_t*>(d_out_pivot), s);
        h->engine.remap(k, d_cand_idx, start, base, d_out_idx, s);
    });
}

}  // extern "C"
