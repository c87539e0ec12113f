// rtk/topk.hpp — drop-in C++ front end of the B200 radix top-k.
//
// Same namespace, type and function names as the reference headers
// (/root/reference/proj/include/rtk/{keycodec,engine,batch,scaling}.hpp), so a caller of
// rtk::topk / rtk::batch_topk / rtk::scaled_topk recompiles against this header and links
// librtk_b200.so instead. Every call goes through the C-ABI in include/rtk_c.h with HOST
// spans (the library does the host<->device copies). Results are bit-identical to the
// reference's: sorted by (key desc, index asc), ties at the pivot by ascending index.
//
//   reference                          here
//   SelectionOrder keycodec.hpp:19     SelectionOrder
//   EngineConfig  engine.hpp:48-68     EngineConfig (GPU tuning hints; validate() identical)
//   exceptions    engine.hpp:31-41     rank_out_of_range / invariant_violation / empty_input_error
//   TopKResult    engine.hpp:103-108   TopKResult
//   topk          engine.hpp:422-443   topk -> rtk_topk_host
//   BatchInput    batch.hpp:27-67      BatchInput
//   batch_topk    batch.hpp:261-367    batch_topk -> rtk_topk_batched_host
//   ScalePolicy   scaling.hpp:20-33    ScaleMode / ScalePolicy / ScaleInfo
//   scaled_topk   scaling.hpp:42-86    scaled_topk -> rtk_topk_scaled_host
#ifndef RTK_TOPK_HPP
#define RTK_TOPK_HPP

#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../rtk_c.h"

namespace rtk {

enum class SelectionOrder { Largest, Smallest };

struct rank_out_of_range : std::out_of_range {
    using std::out_of_range::out_of_range;
};
struct invariant_violation : std::logic_error {
    using std::logic_error::logic_error;
};
struct empty_input_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct device_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

enum class BufferPolicy { Naive, FlushEfficient };

struct EngineConfig {
    unsigned d = 12;
    std::size_t block_size = 1024;
    unsigned grid_size = 4;
    BufferPolicy buffer_policy = BufferPolicy::FlushEfficient;
    std::size_t pack_size = 16;
    bool hierarchical_atomics = true;
    std::size_t filter_fixed_ceiling = 4096;

    std::size_t radix() const { return std::size_t{1} << d; }
    void validate() const {
        if (d < 1 || d > 16) throw std::invalid_argument("digit width must be in [1, 16]");
        if (block_size < 1) throw std::invalid_argument("block_size must be >= 1");
        if (grid_size < 1) throw std::invalid_argument("grid_size must be >= 1");
        if (pack_size < 4 || (pack_size & (pack_size - 1)) != 0)
            throw std::invalid_argument("pack_size must be a power of two >= element width");
    }
};

// Work counters of the last call (the subset of engine.hpp:74-101 with GPU meaning).
struct Instrumentation {
    std::uint64_t passes = 0;
    std::uint64_t elements_scanned = 0;
    std::uint64_t candidates = 0;
    std::uint64_t fallback_rows = 0;
    std::uint64_t deep_levels = 0;
    void reset(unsigned = 0) { *this = {}; }
};

template <typename T>
struct TopKResult {
    std::vector<T> values;
    std::vector<std::uint64_t> indices;
    T pivot{};
};

namespace detail {

inline rtk_handle handle() {
    static rtk_handle h = [] {
        rtk_handle out = nullptr;
        if (rtk_handle_create(&out, 0) != RTK_OK) throw device_error(rtk_last_error());
        return out;
    }();
    return h;
}

inline void raise(int status, const std::string& prefix = {}) {
    if (status == RTK_OK) return;
    const std::string msg = prefix + rtk_last_error();
    switch (status) {
        case RTK_EMPTY_INPUT: throw empty_input_error(msg);
        case RTK_RANK_OUT_OF_RANGE: throw rank_out_of_range(msg);
        case RTK_INVARIANT_VIOLATION: throw invariant_violation(msg);
        case RTK_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        default: throw device_error(msg);
    }
}

inline rtk_cfg to_c(const EngineConfig& c) {
    rtk_cfg r;
    r.d = c.d;
    r.block_size = c.block_size;
    r.grid_size = c.grid_size;
    r.buffer_policy = c.buffer_policy == BufferPolicy::Naive ? 0 : 1;
    r.pack_size = c.pack_size;
    r.hierarchical_atomics = c.hierarchical_atomics ? 1 : 0;
    r.filter_fixed_ceiling = c.filter_fixed_ceiling;
    return r;
}

template <typename T>
constexpr int dtype_code() {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, std::uint32_t>,
                  "rtk top-k is defined for float and std::uint32_t keys");
    return std::is_same_v<T, float> ? RTK_F32 : RTK_U32;
}

inline int order_code(SelectionOrder o) { return o == SelectionOrder::Largest ? RTK_LARGEST : RTK_SMALLEST; }

inline void fill(Instrumentation& instr) {
    rtk_stats st{};
    if (rtk_get_stats(handle(), &st) == RTK_OK) {
        instr.passes = st.passes;
        instr.elements_scanned = st.elements_scanned;
        instr.candidates = st.candidates;
        instr.fallback_rows = st.fallback_rows;
        instr.deep_levels = st.deep_levels;
    }
}

}  // namespace detail

template <typename T>
TopKResult<T> topk(std::span<const T> input, std::uint64_t k, SelectionOrder order, const EngineConfig& cfg,
                   Instrumentation& instr) {
    if (input.empty()) throw empty_input_error("topk: empty input");
    if (k == 0 || k > input.size()) throw rank_out_of_range("topk: k outside [1, n]");
    cfg.validate();
    TopKResult<T> r;
    r.values.resize(k);
    r.indices.resize(k);
    const rtk_cfg c = detail::to_c(cfg);
    detail::raise(rtk_topk_host(detail::handle(), input.data(), input.size(), k, detail::dtype_code<T>(),
                                detail::order_code(order), r.values.data(), r.indices.data(), &r.pivot, &c));
    detail::fill(instr);
    return r;
}

template <typename T>
TopKResult<T> topk(std::span<const T> input, std::uint64_t k, SelectionOrder order, const EngineConfig& cfg) {
    Instrumentation instr;
    return topk(input, k, order, cfg, instr);
}

// ---- batch (batch.hpp) ----------------------------------------------------------------------
template <typename T>
struct BatchInput {
    std::vector<T> data;
    std::vector<std::uint64_t> offsets;
    std::vector<std::uint64_t> lengths;
    std::vector<std::uint64_t> ks;

    std::size_t task_count() const { return lengths.size(); }
    std::span<const T> task_view(std::size_t i) const {
        return std::span<const T>(data).subspan(offsets[i], lengths[i]);
    }
    void validate() const {
        if (lengths.empty()) throw std::invalid_argument("batch: no tasks");
        if (offsets.size() != lengths.size() || ks.size() != lengths.size())
            throw std::invalid_argument("batch: descriptor arrays disagree");
        for (std::size_t i = 0; i < lengths.size(); ++i) {
            std::uint64_t next = i + 1 < offsets.size() ? offsets[i + 1] : data.size();
            if (offsets[i] + lengths[i] > next)
                throw std::invalid_argument("batch: task " + std::to_string(i) + " overlaps its successor");
            if (ks[i] == 0 || ks[i] > lengths[i])
                throw std::invalid_argument("batch: task " + std::to_string(i) + " has k outside [1, n]");
        }
    }
    static BatchInput concatenate(std::vector<std::vector<T>> tasks, std::vector<std::uint64_t> ks) {
        BatchInput b;
        b.ks = std::move(ks);
        for (auto& t : tasks) {
            b.offsets.push_back(b.data.size());
            b.lengths.push_back(t.size());
            b.data.insert(b.data.end(), t.begin(), t.end());
        }
        b.validate();
        return b;
    }
};

struct BatchOptions {
    bool rescheduling = true;
    bool padding = true;
};

struct BatchRunInfo {
    std::vector<std::uint64_t> task_passes;
    std::uint64_t phase_b_rounds = 0;
};

template <typename T>
std::vector<TopKResult<T>> batch_topk(const BatchInput<T>& batch, SelectionOrder order, const EngineConfig& cfg,
                                      const BatchOptions& opts, Instrumentation& instr,
                                      BatchRunInfo* info = nullptr) {
    batch.validate();
    cfg.validate();
    const std::size_t B = batch.task_count();
    std::vector<std::uint64_t> out_off(B);
    std::uint64_t total = 0;
    for (std::size_t t = 0; t < B; ++t) {
        out_off[t] = total;
        total += batch.ks[t];
    }
    std::vector<T> vals(total), pivots(B);
    std::vector<std::uint64_t> idx(total);
    const rtk_cfg c = detail::to_c(cfg);
    const rtk_batch_opts o{opts.rescheduling ? 1 : 0, opts.padding ? 1 : 0};
    detail::raise(rtk_topk_batched_host(detail::handle(), batch.data.data(), batch.data.size(), batch.offsets.data(),
                                        batch.lengths.data(), batch.ks.data(), B, detail::dtype_code<T>(),
                                        detail::order_code(order), vals.data(), idx.data(), out_off.data(),
                                        pivots.data(), &c, &o));
    std::vector<TopKResult<T>> res(B);
    for (std::size_t t = 0; t < B; ++t) {
        res[t].values.assign(vals.begin() + out_off[t], vals.begin() + out_off[t] + batch.ks[t]);
        res[t].indices.assign(idx.begin() + out_off[t], idx.begin() + out_off[t] + batch.ks[t]);
        res[t].pivot = pivots[t];
    }
    detail::fill(instr);
    if (info) {  // batch.hpp:138-141 as measured by the engine (rtk_get_batch_info)
        info->task_passes.assign(B, 0);
        detail::raise(rtk_get_batch_info(detail::handle(), info->task_passes.data(), B, &info->phase_b_rounds));
    }
    return res;
}

template <typename T>
std::vector<TopKResult<T>> batch_topk(const BatchInput<T>& batch, SelectionOrder order, const EngineConfig& cfg,
                                      const BatchOptions& opts = {}) {
    Instrumentation instr;
    return batch_topk(batch, order, cfg, opts, instr);
}

// ---- scaling (scaling.hpp) --------------------------------------------------------------------
enum class ScaleMode { Off, Always, Adaptive };

struct ScalePolicy {
    ScaleMode mode = ScaleMode::Off;
    double trigger_fraction = 0.5;
    std::uint64_t seed = 0;
};

struct ScaleInfo {
    bool scaled = false;
    float a_s = 0.0f;
    std::uint64_t a_index = 0;
};

inline TopKResult<float> scaled_topk(std::span<const float> input, std::uint64_t k, SelectionOrder order,
                                     const EngineConfig& cfg, const ScalePolicy& policy, Instrumentation& instr,
                                     ScaleInfo* info = nullptr) {
    if (input.empty()) throw empty_input_error("scaled_topk: empty input");
    if (k == 0 || k > input.size()) throw rank_out_of_range("scaled_topk: k outside [1, n]");
    TopKResult<float> r;
    r.values.resize(k);
    r.indices.resize(k);
    const rtk_cfg c = detail::to_c(cfg);
    rtk_scale_info si{};
    const int mode = policy.mode == ScaleMode::Off ? RTK_SCALE_OFF
                                                   : (policy.mode == ScaleMode::Always ? RTK_SCALE_ALWAYS
                                                                                       : RTK_SCALE_ADAPTIVE);
    detail::raise(rtk_topk_scaled_host(detail::handle(), input.data(), input.size(), k, detail::order_code(order),
                                       mode, policy.trigger_fraction, policy.seed, r.values.data(), r.indices.data(),
                                       &r.pivot, &si, &c));
    if (info) *info = ScaleInfo{si.scaled != 0, si.a_s, si.a_index};
    detail::fill(instr);
    return r;
}

inline TopKResult<float> scaled_topk(std::span<const float> input, std::uint64_t k, SelectionOrder order,
                                     const EngineConfig& cfg, const ScalePolicy& policy) {
    Instrumentation instr;
    return scaled_topk(input, k, order, cfg, policy, instr);
}

}  // namespace rtk

#endif  // RTK_TOPK_HPP
