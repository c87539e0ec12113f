// ref_shim.cpp — C entry points over the UNMODIFIED reference headers (TEST INFRASTRUCTURE).
//
// Compiled by oracle/Makefile against /root/reference/proj/include (never copied into this
// repo) into oracle/_ref/librtk_ref.so. Used only by tests/ (golden vectors, parity of the
// C restatement in oracle/rtk_oracle.c) and by bench.py's cpu_baseline / --impl reference
// legs, which time the reference's own CPU engine (rtk::topk, rtk::batch_topk,
// rtk::scaled_topk) on the host cores. The product library never links this.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <span>
#include <stdexcept>
#include <vector>

#include "rtk/batch.hpp"
#include "rtk/datagen.hpp"
#include "rtk/engine.hpp"
#include "rtk/io.hpp"
#include "rtk/oracle.hpp"
#include "rtk/scaling.hpp"

namespace {

// Status codes shared with include/rtk_c.h.
enum { OK = 0, EMPTY = 1, RANK = 2, INVARIANT = 3, INVALID = 4, OTHER = 7 };

int code_of(const std::exception_ptr& p) {
    try {
        std::rethrow_exception(p);
    } catch (const rtk::empty_input_error&) {
        return EMPTY;
    } catch (const rtk::rank_out_of_range&) {
        return RANK;
    } catch (const rtk::invariant_violation&) {
        return INVARIANT;
    } catch (const std::invalid_argument&) {
        return INVALID;
    } catch (...) {
        return OTHER;
    }
}

rtk::EngineConfig make_cfg(unsigned d, unsigned grid) {
    rtk::EngineConfig cfg;
    cfg.d = d;
    cfg.block_size = 1024;
    cfg.grid_size = grid;
    return cfg;
}

rtk::SelectionOrder ord(int order) {
    return order == 0 ? rtk::SelectionOrder::Largest : rtk::SelectionOrder::Smallest;
}

template <typename T>
void emit(const rtk::TopKResult<T>& r, void* out_vals, std::uint64_t* out_idx, void* out_pivot) {
    std::memcpy(out_vals, r.values.data(), r.values.size() * sizeof(T));
    std::memcpy(out_idx, r.indices.data(), r.indices.size() * sizeof(std::uint64_t));
    std::memcpy(out_pivot, &r.pivot, sizeof(T));
}

}  // namespace

extern "C" {

int ref_topk(const void* in, std::uint64_t n, std::uint64_t k, int dtype, int order, unsigned d,
             unsigned grid, void* out_vals, std::uint64_t* out_idx, void* out_pivot,
             std::uint64_t* passes) {
    try {
        auto cfg = make_cfg(d, grid);
        rtk::Instrumentation instr;
        instr.reset(grid);
        if (dtype == 0) {
            auto r = rtk::topk(std::span<const float>(static_cast<const float*>(in), n), k,
                               ord(order), cfg, instr);
            emit(r, out_vals, out_idx, out_pivot);
        } else {
            auto r = rtk::topk(
                std::span<const std::uint32_t>(static_cast<const std::uint32_t*>(in), n), k,
                ord(order), cfg, instr);
            emit(r, out_vals, out_idx, out_pivot);
        }
        if (passes) *passes = instr.passes;
        return OK;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

int ref_oracle_topk(const void* in, std::uint64_t n, std::uint64_t k, int dtype, int order,
                    void* out_vals, std::uint64_t* out_idx, void* out_pivot) {
    try {
        if (dtype == 0) {
            auto r = rtk::oracle_topk(std::span<const float>(static_cast<const float*>(in), n),
                                      k, ord(order));
            emit(r, out_vals, out_idx, out_pivot);
        } else {
            auto r = rtk::oracle_topk(
                std::span<const std::uint32_t>(static_cast<const std::uint32_t*>(in), n), k,
                ord(order));
            emit(r, out_vals, out_idx, out_pivot);
        }
        return OK;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// Dense or ragged batch. Outputs for task t start at out_offsets[t].
int ref_batch_topk(const void* data, std::uint64_t data_len, const std::uint64_t* offsets,
                   const std::uint64_t* lengths, const std::uint64_t* ks, std::uint64_t B,
                   int dtype, int order, unsigned d, unsigned grid, int rescheduling,
                   int padding, void* out_vals, std::uint64_t* out_idx,
                   const std::uint64_t* out_offsets, void* out_pivots) {
    try {
        auto cfg = make_cfg(d, grid);
        rtk::BatchOptions opts{rescheduling != 0, padding != 0};
        auto run = [&](auto tag) {
            using T = decltype(tag);
            rtk::BatchInput<T> batch;
            batch.data.assign(static_cast<const T*>(data), static_cast<const T*>(data) + data_len);
            batch.offsets.assign(offsets, offsets + B);
            batch.lengths.assign(lengths, lengths + B);
            batch.ks.assign(ks, ks + B);
            auto res = rtk::batch_topk(batch, ord(order), cfg, opts);
            for (std::uint64_t t = 0; t < B; ++t)
                emit(res[t], static_cast<T*>(out_vals) + out_offsets[t], out_idx + out_offsets[t],
                     static_cast<T*>(out_pivots) + t);
        };
        if (dtype == 0)
            run(float{});
        else
            run(std::uint32_t{});
        return OK;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// mode 0 Off / 1 Always / 2 Adaptive. info = {scaled, a_s bits, a_index}.
int ref_scaled_topk(const float* in, std::uint64_t n, std::uint64_t k, int order, unsigned d,
                    unsigned grid, int mode, double tau, std::uint64_t seed, float* out_vals,
                    std::uint64_t* out_idx, float* out_pivot, std::uint64_t* info) {
    try {
        auto cfg = make_cfg(d, grid);
        rtk::ScalePolicy policy{static_cast<rtk::ScaleMode>(mode), tau, seed};
        rtk::ScaleInfo si;
        rtk::Instrumentation instr;
        instr.reset(grid);
        auto r = rtk::scaled_topk(std::span<const float>(in, n), k, ord(order), cfg, policy,
                                  instr, &si);
        emit(r, out_vals, out_idx, out_pivot);
        std::uint32_t bits;
        std::memcpy(&bits, &si.a_s, 4);
        info[0] = si.scaled;
        info[1] = bits;
        info[2] = si.a_index;
        return OK;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// rtk::generate<T> (datagen.hpp:71-141). kind: 0 Uniform 1 Normal 2 Zipf 3 Peaked.
int ref_generate(int kind, double a, double b, double s, double mass, unsigned modes,
                 std::uint64_t seed, std::uint64_t n, int dtype, void* out) {
    try {
        rtk::DistributionSpec spec;
        spec.kind = static_cast<rtk::DistKind>(kind);
        spec.a = a;
        spec.b = b;
        spec.s = s;
        spec.mass = mass;
        spec.modes = modes;
        spec.seed = seed;
        spec.n = n;
        if (dtype == 0) {
            auto v = rtk::generate<float>(spec);
            std::memcpy(out, v.data(), n * 4);
        } else {
            auto v = rtk::generate<std::uint32_t>(spec);
            std::memcpy(out, v.data(), n * 4);
        }
        return OK;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

int ref_count_bins(const std::uint32_t* keys, std::uint64_t m, unsigned low, unsigned high,
                   unsigned grid, std::uint64_t* hist) {
    try {
        auto cfg = make_cfg(high - low, grid);
        std::vector<rtk::RadixKey> k(m);
        for (std::uint64_t i = 0; i < m; ++i) k[i].bits = keys[i];
        rtk::Instrumentation instr;
        instr.reset(grid);
        auto h = rtk::count_bins(k, rtk::DigitWindow{low, high}, cfg, instr);
        std::memcpy(hist, h.data(), h.size() * 8);
        return OK;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

int ref_select_bin(const std::uint64_t* hist, std::uint64_t nbins, std::uint64_t k,
                   std::uint32_t* bin, std::uint64_t* k_new) {
    try {
        auto sel = rtk::select_bin(rtk::Histogram(hist, hist + nbins), k);
        *bin = sel.bin;
        *k_new = sel.k_new;
        return OK;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

std::uint32_t ref_encode_f32(float v, int order) { return rtk::encode_key(v, ord(order)).bits; }

// ---- rtk/io.hpp (io.cpp compiled in place): RTK1 / RTKB containers ------------------------
static thread_local std::string g_io_msg;
const char* ref_io_error(void) { return g_io_msg.c_str(); }

int ref_write_dataset(const char* path, int dtype, const void* data, std::uint64_t n) {
    try {
        if (dtype == 0) rtk::write_dataset(path, std::span<const float>(static_cast<const float*>(data), n));
        else rtk::write_dataset(path, std::span<const std::uint32_t>(static_cast<const std::uint32_t*>(data), n));
        return OK;
    } catch (const std::exception& e) {
        g_io_msg = e.what();
        return OTHER;
    }
}

// two-call: out == nullptr returns dtype / count only
int ref_read_dataset(const char* path, int* dtype, std::uint64_t* n, void* out) {
    try {
        rtk::Dataset ds = rtk::read_dataset(path);
        *dtype = static_cast<int>(ds.dtype);
        *n = ds.size();
        if (out) std::memcpy(out, ds.dtype == rtk::DType::F32 ? static_cast<const void*>(ds.f32.data())
                                                              : static_cast<const void*>(ds.u32.data()),
                             ds.size() * 4);
        return OK;
    } catch (const std::exception& e) {
        g_io_msg = e.what();
        return OTHER;
    }
}

int ref_write_batch(const char* path, const std::uint64_t* lengths, std::uint32_t tasks, const void* payload,
                    std::uint64_t bytes) {
    try {
        rtk::write_batch(path, std::vector<std::uint64_t>(lengths, lengths + tasks),
                         std::span<const std::uint8_t>(static_cast<const std::uint8_t*>(payload), bytes));
        return OK;
    } catch (const std::exception& e) {
        g_io_msg = e.what();
        return OTHER;
    }
}

int ref_read_batch(const char* path, std::uint32_t* tasks, std::uint64_t* bytes, std::uint64_t* lengths,
                   void* payload) {
    try {
        rtk::BatchFile b = rtk::read_batch(path);
        *tasks = static_cast<std::uint32_t>(b.lengths.size());
        *bytes = b.payload.size();
        if (lengths) std::memcpy(lengths, b.lengths.data(), b.lengths.size() * 8);
        if (payload) std::memcpy(payload, b.payload.data(), b.payload.size());
        return OK;
    } catch (const std::exception& e) {
        g_io_msg = e.what();
        return OTHER;
    }
}

}  // extern "C"
