// rtk_engine.h — host orchestration of the B200 radix top-k (C++; no torch types).
//
// One Engine per rtk_handle. It plans a launch sequence for a set of rows (one query = one
// row; a batch = B rows over one base pointer), owns the device workspace, and replaces the
// reference's std::thread worker pool (engine.hpp:112-122) with grid launches on a stream.
#pragma once
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rtk_c.h"
#include "rtk_device.cuh"
#include "rtk_kernels.h"

namespace rtk_b200 {

struct Error {
    int code;
    std::string msg;
};

struct RowReq {
    uint64_t in_off;   // element offset of the row in the input base
    uint64_t n;        // elements
    uint64_t k;        // rank
    uint64_t out_off;  // element offset of the row's outputs
};

// Makes `dev` current for the scope and restores the caller's device afterwards (the caller's
// framework, e.g. torch.cuda.current_device(), must not see a different device after a call).
class DeviceGuard {
public:
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev_) != cudaSuccess) prev_ = -1;
        if (prev_ != dev) {
            const cudaError_t e = cudaSetDevice(dev);
            if (e != cudaSuccess) throw Error{RTK_CUDA_ERROR, std::string("cudaSetDevice: ") + cudaGetErrorString(e)};
            set_ = true;
        }
    }
    ~DeviceGuard() {
        if (set_ && prev_ >= 0) cudaSetDevice(prev_);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;

private:
    int prev_ = -1;
    bool set_ = false;
};

// Growable device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void ensure(size_t bytes, bool keep = false, cudaStream_t s = nullptr);
    void release();
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

class Engine {
public:
    explicit Engine(int device);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    // Top-k of every row. Values are written as raw 32-bit words (f32 bits or u32).
    // scaled: keys are encode(x - a_s) (f32); gather: values re-read from the input by index.
    void run(const uint32_t* d_base, int dtype, int smallest, bool scaled, float a_s, bool gather,
             const std::vector<RowReq>& rows, uint32_t* d_vals, uint64_t* d_idx,
             uint32_t* d_pivots, cudaStream_t s);

    // Exact histogram of the first d-bit window of the unscaled keys (adaptive trigger).
    std::vector<uint64_t> first_digit_hist(const uint32_t* d_in, uint64_t n, unsigned d,
                                           int smallest, cudaStream_t s);

    // Remap shard-merge positions to global indices.
    void remap(uint64_t k, const uint64_t* d_cand_idx, const std::vector<uint64_t>& block_start,
               const std::vector<uint64_t>& shard_base, uint64_t* d_idx, cudaStream_t s);

    uint32_t read_word(const uint32_t* d, uint64_t i, cudaStream_t s);

    // scaled_topk decided on the device (scaling.hpp:47-67): first-window histogram + one-CTA
    // select_bin / trigger / a_s fetch, stream-ordered, no host round trip. The next run() with
    // use_device_scale() reads the decision in every kernel. mode: 1 Always, 2 Adaptive.
    void enqueue_scale_decide(const uint32_t* d_in, uint64_t n, uint64_t k, unsigned d, int smallest,
                              int mode, double tau, uint64_t a_index, cudaStream_t s);
    const uint32_t* device_scale() const { return adapt_buf_.as<uint32_t>(); }
    // Adaptive without the counting pass: k_scale_guess decides from a sample; the next run()
    // with set_trigger_count(true) counts the exact #{digit > b} / #{digit == b} of the unscaled
    // first window over all n (k_compact), readable afterwards through trigger_counts()
    void enqueue_scale_guess(const uint32_t* d_in, uint64_t n, uint64_t k, unsigned d, int smallest, double tau,
                             uint64_t a_index, cudaStream_t s);
    void set_trigger_count(bool on) { trig_count_ = on; }
    void trigger_counts(uint64_t* gt, uint64_t* eq) const {
        *gt = trig_words_[0] | (static_cast<uint64_t>(trig_words_[1]) << 32);
        *eq = trig_words_[2] | (static_cast<uint64_t>(trig_words_[3]) << 32);
    }
    // {flag, a_s bits} of the last decision (valid once the following run() returned)
    void scale_result(bool* scaled, float* a_s) const;
    void set_adapt(const uint32_t* p) { adapt_ = p; }

    // stats of the last call; total_ms is resolved lazily (waits for the call's last event)
    const rtk_stats& last_stats();
    void set_timing(bool on) { timing_ = on; }
    // bench: events recorded on the call's stream right before its first and after its last
    // device operation (host planning and the completion wait stay outside); null = off
    void set_call_events(cudaEvent_t start, cudaEvent_t end) { call_start_ = start; call_end_ = end; }

    // test switches (rtk_set_option): "force_exact", "force_deep"; false for unknown names
    bool set_option(const std::string& name, int64_t value);
    // full reads of each row's input in the last call (BatchRunInfo::task_passes)
    const std::vector<uint64_t>& row_passes() const { return row_passes_; }

    int device() const { return device_; }
    rtk_stats stats{};
    DevBuf io_in, io_vals, io_idx, io_piv, io_aux;

private:
    // Plan arena: host bytes are staged then copied into a bump-allocated device region.
    struct Plan {
        std::vector<uint8_t> bytes;
        template <typename T>
        size_t add(const std::vector<T>& v) {
            size_t off = (bytes.size() + 15) & ~size_t(15);
            bytes.resize(off + v.size() * sizeof(T));
            if (!v.empty()) std::memcpy(bytes.data() + off, v.data(), v.size() * sizeof(T));
            return off;
        }
    };
    uint8_t* upload(const Plan& p, cudaStream_t s);
    void sync(cudaStream_t s, const char* what);
    void release_retired();
    void mark(const char* name, cudaStream_t s);
    void report_rows_trace(size_t nrows, cudaStream_t s);
    void report_marks();
    struct Mark {
        const char* name;
        cudaEvent_t ev;
        std::chrono::steady_clock::time_point host;
    };
    bool profile_ = false;
    bool count_stats_ = false;   // read candidate counts back (stats.candidates)
    double sample_r_ = 512.0;    // huge rows: target sample rank k*s/n (RTK_SAMPLE_R)
    std::vector<Mark> marks_;
    // State of one run() call shared by the finish / fallback stages.
    struct Call {
        InputSrc src;
        bool gather;
        const uint64_t* d_row_k;
        const uint64_t* d_row_out;
        const uint64_t* d_row_in;
        uint32_t* d_vals;
        uint64_t* d_idx;
        cudaStream_t s;
        std::vector<uint64_t> cap;       // candidate capacity per row
        std::vector<uint64_t> cand_off;  // candidate region per row (buffer A/B)
        uint64_t cand_total;
        std::vector<uint64_t> scratch;
        int R;
        const uint64_t* d_cap;   // device copies of cap / cand_off (plan arena)
        const uint64_t* d_coff;
        uint32_t* d_pivots;
    };
    struct FinishPrep {
        int NR = 0;
        uint64_t big_rows = 0, max_groups = 0, ntiles = 0;
        uint8_t* D = nullptr;
        size_t o_rid = 0, o_tiles = 0;
        uint64_t max_wgroups = 0;
        int cs = 2;
        uint64_t max_cap = 0;
        const SegSlot* slots = nullptr;  // level-0 slots (null: written by k_compact's plan)
        GroupList gl{}, wgl{};
        SlotList nextA{};
    };
    FinishPrep prepare_finish(Call& c, const std::vector<uint32_t>& rids);
    PlanArgs plan_args(const Call& c, const FinishPrep& f);
    void launch_finish(Call& c, const FinishPrep& f);
    void fallback(const uint32_t* d_base, const InputSrc& src, const std::vector<RowReq>& rows,
                  const std::vector<uint32_t>& fb, Call& c, cudaStream_t s);
    void drain(Call& c, uint32_t (&ctl)[8]);
    SortArgs sort_args(const Call& c, const GroupList& gl);
    void launch_sort(uint32_t max_groups, const SortArgs& a, cudaStream_t s);
    CallTail tail_args();
    void set_clean(CallTail& t, int R);
    void wait_signal(cudaStream_t s);
    void record(int i, cudaStream_t s);
    void enqueue(const uint32_t* d_base, int dtype, int smallest, bool scaled, float a_s, bool gather,
                 const std::vector<RowReq>& rows, uint32_t* d_vals, uint64_t* d_idx, uint32_t* d_pivots,
                 cudaStream_t s, Call& c);
    void complete(const uint32_t* d_base, const std::vector<RowReq>& rows, Call& c, cudaStream_t s);

    // CUDA-graph replay of the common path (plan upload .. sort) for repeated identical calls
    struct CallKey {
        const uint32_t* base = nullptr;
        int dtype = 0, smallest = 0, scaled = 0, gather = 0;
        uint32_t a_s_bits = 0;
        const uint32_t* adapt = nullptr;
        void *vals = nullptr, *idx = nullptr, *piv = nullptr;
        cudaStream_t s = nullptr;
        std::vector<RowReq> rows;
        bool operator==(const CallKey& o) const;
    };
    struct Upload {
        uint8_t* d;
        const uint8_t* h;
        size_t bytes;
    };
    std::vector<Upload> cap_uploads_;
    cudaStream_t user_s_ = nullptr;
    uint64_t arena_tag_ = 0;      // bumped by every plan upload (arena content changed)
    struct GraphCache {
        bool valid = false;
        CallKey key;
        uint64_t gen = 0;
        cudaGraphExec_t exec = nullptr;
        std::vector<uint8_t> pinned;  // plan bytes the captured memcpy reads from pin_
        Call call;
        rtk_stats stats{};
        uint32_t seq_incr = 0;
        bool has_init = false;
        int clean_rows = 0;
        size_t arena_used = 0, pin_used = 0;
        std::vector<Upload> uploads;  // plan uploads done outside the graph at capture time
        uint64_t arena_tag = 0;
        uint64_t group_base = 0, wgroup_base = 0;
    };
    GraphCache graph_;
    CallKey last_key_;
    uint64_t last_gen_ = 0;
    bool have_last_ = false;
    bool graphs_ = true;          // RTK_GRAPHS=0 disables
    bool stats_pending_ = false;
    bool capturing_ = false;
    bool needs_init_ = true;      // per-call counters not known to be clean
    bool self_clean_ = false;     // the next main sort launch resets the counters
    bool self_clean_ok_ = true;   // RTK_SELFCLEAN=0 disables
    bool force_init_ = false;
    bool no_graph_events_ = true;   // no stats events inside graphs (RTK_GRAPH_EVENTS=1 keeps them)
    cudaEvent_t call_start_ = nullptr, call_end_ = nullptr;
    bool timing_ = false;           // rtk_set_timing: no graph replay, events around k_compact
    bool trig_count_ = false;       // count the speculative Adaptive trigger in the main compaction
    uint32_t trig_words_[4] = {0, 0, 0, 0};  // ctl[10..13] as the main path left them
    uint32_t drain_trig_[4] = {0, 0, 0, 0};
    bool force_exact_ = false;      // RTK_FORCE_EXACT / "force_exact"
    bool force_deep_ = false;       // RTK_FORCE_DEEP / "force_deep"
    bool in_fallback_ = false;      // the exact path's own compaction (no forced failure there)
    std::vector<uint64_t> row_passes_;
    uint32_t level0_bits() const { return force_deep_ ? 6u : static_cast<uint32_t>(msd_max_bits_); }
    bool no_fused_ = false;
    bool no_rcluster_ = false;  // RTK_NO_RCLUSTER=1: single long rows take the general path
    bool no_dense_ = false;
    int sparse_max_ = 96;            // RTK_SPARSE_MAX (k_compact sparse-hit path threshold)
    int lsd_mode_ = 2;               // RTK_LSD: dense rows' LSD sort: 0 off (MSD + bucket sorts), 1 16-bit keys, 2 all
    size_t lsd_hist_cap_ = 0;
    DevBuf lsd_a_, lsd_b_, lsd_status_, lsd_meta_;
    int sparse_sel_ = 1;
    int dyn_per_cta_ = 12;            // RTK_DYN: k_compact dynamic-tail tiles per CTA (0: static split)             // RTK_SPARSE_SEL (sparse hits from registers, no L2 re-read)
    uint32_t dense_bits_ = 0;       // RTK_DENSE_BITS: level-0 digit of dense rows (0: fine_bits)         // RTK_NO_DENSE=1: dense rows are compacted too         // RTK_NO_FUSED=1: short rows take the general path too
    int tile_contig_ = -1;          // RTK_TILE_CONTIG: force k_compact's tile order (-1: by row count)
    int msd_cs_ = 0;                // RTK_MSD_CS: force the level-0 MSD cluster size
    int rows_pf0_ = 0;              // one-shot L2 prefetch at the row's start, chunks (RTK_ROWS_PF0)
    int rows_pf_ = 0;               // L2 prefetch distance of the per-row ring (RTK_ROWS_PF)
    bool lsd_rr_ = true;            // RTK_LSD_RR=0: LSD tiles claimed row by row (no round-robin order)
    bool lsd_trace_ = false;        // RTK_LSD_TRACE: per-tile phase timestamps of k_lsd_pass
    DevBuf lsd_trace_buf_;
    bool rows_trace_ = false;       // per-CTA phase timestamps of k_rows_fused (RTK_ROWS_TRACE)
    DevBuf trace_;
    int prefetch_mb_ = 24;          // L2 prefetch budget of k_compact (RTK_PREFETCH_MB)
    int clean_rows_ = 0;
    int clean_upto_ = 0;          // rows whose counters the last call left clean
    bool did_init_ = false;
    uint32_t first_flags_ = 0;    // flag word of the last drain's first readback
    bool sig_pending_ = false;    // a signalling sort launch is in flight
    uint32_t expected_seq_ = 0;
    cudaStream_t cap_s_ = nullptr; // private capture stream
    uint32_t* hmap_ = nullptr;    // mapped pinned signal words (host view)
    uint32_t* d_hmap_ = nullptr;  // device view

    int device_;
    DevBuf arena_;
    size_t arena_used_ = 0;
    std::vector<DevBuf> retired_;
    cudaEvent_t pin_ev_ = nullptr;  // recorded after a stream-ordered remap's plan upload
    bool pin_ev_pending_ = false;
    uint8_t* pin_ = nullptr;       // pinned staging for plan uploads
    size_t pin_cap_ = 0, pin_used_ = 0;
    std::vector<uint8_t*> retired_pinned_;
    uint32_t* hctl_ = nullptr;     // pinned readback of the control words
    uint64_t* hcount_ = nullptr;   // pinned readback of candidate counts
    size_t hcount_cap_ = 0;
    cudaEvent_t ev_[4] = {nullptr, nullptr, nullptr, nullptr};
    DevBuf sel_, T_, count_, kmin_, kmax_, kor_, ghist_, samples_, cand_a_, cand_b_, seg_hist_,
        gcursor_, bstart_, dcap_, dcoff_, ctl_, row_fail_, groups_, slots0_, slotsA_, slotsB_, done_,
        seg_ticket_, dbg_, wgroups_, ctot_, sig_;
    uint64_t group_base_ = 0, wgroup_base_ = 0;
    uint32_t next_cap_ = 0;
    uint32_t wgroup_cap_ = 0;
    uint32_t bar_gen_ = 0;        // grid-barrier target of the level-0 MSD (ctl[7], reset per call)
    int msd_q_max_ = 32;          // clusters per huge slot (RTK_MSD_Q)
    int msd_max_bits_ = kMsdMaxBits;  // RTK_MSD_BITS
    const uint32_t* adapt_ = nullptr;  // device scale decision read by the next run() (set_adapt)
    DevBuf adapt_buf_, scale_hist_, scale_plan_;
    uint32_t* hscale_ = nullptr;       // mapped {flag, a_s bits} written by k_scale_decide
    uint32_t* d_hscale_ = nullptr;
    const uint32_t* scale_plan_in_ = nullptr;  // input the cached first-window plan describes
    uint64_t scale_plan_n_ = 0;
};

}  // namespace rtk_b200
