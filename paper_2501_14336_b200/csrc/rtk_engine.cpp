// rtk_engine.cpp — host orchestration (see rtk_engine.h and DESIGN.md §3).
//
// Pipeline per call (all rows of a batch share each launch):
//   1. sample:   k_sample_gather -> 3 x k_radix_pass(samples)   (no host sync)
//                -> key threshold T per row, chosen so #{K >= T} >= k with high probability
//   2. compact:  k_compact over the input — the ONE full read of the data
//   3. verify:   read back candidate counts; rows where count < k or the buffer overflowed
//                take the exact path: k_radix_pass over the input until #{K >= T} is small
//                (early stop at count == k), then k_compact again. Correctness never
//                depends on the sample.
//   4. finish:   candidates (all K >= T, count m >= k) are ordered descending and the first
//                k are gathered: one CTA smem sort for m <= 16384, else MSD partitioning
//                (k_seg_hist / k_seg_scatter) into CTA-sized groups.
#include "rtk_engine.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "rtk_kernels.h"

namespace rtk_b200 {

namespace {

// bumped whenever a device / pinned buffer is (re)allocated or freed: captured graphs embed
// raw pointers and are only replayed while the generation is unchanged
std::atomic<uint64_t> g_buf_gen{1};

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error{e == cudaErrorMemoryAllocation ? RTK_OUT_OF_MEMORY : RTK_CUDA_ERROR,
                    std::string(what) + ": " + cudaGetErrorString(e)};
}

uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

template <typename T>
const T* at(uint8_t* base, size_t off) {
    return reinterpret_cast<const T*>(base + off);
}

}  // namespace

void DevBuf::ensure(size_t bytes, bool keep, cudaStream_t s) {
    if (bytes <= cap) return;
    size_t ncap = std::max(bytes, cap + cap / 2);
    ncap = (ncap + 255) & ~size_t(255);
    void* np = nullptr;
    check(cudaMalloc(&np, ncap), "cudaMalloc");
    g_buf_gen.fetch_add(1);
    if (keep && p && cap) {
        check(cudaMemcpyAsync(np, p, cap, cudaMemcpyDeviceToDevice, s), "grow copy");
        check(cudaStreamSynchronize(s), "grow sync");
    }
    if (p) cudaFree(p);
    p = np;
    cap = ncap;
}

void DevBuf::release() {
    if (p) g_buf_gen.fetch_add(1);
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
}

Engine::Engine(int device) : device_(device) {
    const char* p = std::getenv("RTK_PROFILE");
    profile_ = p && *p && *p != '0';
    if (const char* sr = std::getenv("RTK_SAMPLE_R")) sample_r_ = std::max(1.0, std::atof(sr));
    if (const char* mq = std::getenv("RTK_MSD_Q")) msd_q_max_ = std::max(1, std::atoi(mq));
    if (const char* mb = std::getenv("RTK_MSD_BITS")) msd_max_bits_ = std::min(kMsdMaxBits, std::max(11, std::atoi(mb)));
    if (const char* g = std::getenv("RTK_GRAPHS")) graphs_ = *g && *g != '0';
    if (const char* g = std::getenv("RTK_SELFCLEAN")) self_clean_ok_ = *g && *g != '0';
    if (const char* g = std::getenv("RTK_FORCE_INIT")) force_init_ = *g && *g != '0';
    if (const char* g = std::getenv("RTK_GRAPH_EVENTS")) no_graph_events_ = *g == '0';
    if (const char* g = std::getenv("RTK_PREFETCH_MB")) prefetch_mb_ = std::max(0, std::atoi(g));
    if (const char* g = std::getenv("RTK_NO_FUSED")) no_fused_ = *g && *g != '0';
    if (const char* g = std::getenv("RTK_NO_RCLUSTER")) no_rcluster_ = *g && *g != '0';
    if (const char* g = std::getenv("RTK_NO_DENSE")) no_dense_ = *g && *g != '0';
    if (const char* g = std::getenv("RTK_SPARSE_MAX")) sparse_max_ = std::atoi(g);
    if (const char* g = std::getenv("RTK_SPARSE_SEL")) sparse_sel_ = std::atoi(g);
    if (const char* g = std::getenv("RTK_DYN")) dyn_per_cta_ = std::max(0, std::atoi(g));
    if (const char* g = std::getenv("RTK_LSD")) lsd_mode_ = std::strcmp(g, "16") == 0 ? 1 : std::strcmp(g, "off") == 0 ? 0 : 2;
    if (const char* g = std::getenv("RTK_ROWS_PF")) rows_pf_ = std::atoi(g);
    if (const char* g = std::getenv("RTK_ROWS_PF0")) rows_pf0_ = std::atoi(g);
    if (const char* g = std::getenv("RTK_ROWS_TRACE")) rows_trace_ = *g && *g != '0';
    if (const char* g = std::getenv("RTK_LSD_TRACE")) lsd_trace_ = *g && *g != '0';
    if (const char* g = std::getenv("RTK_LSD_RR")) lsd_rr_ = *g != '0';
    if (const char* g = std::getenv("RTK_MSD_CS")) msd_cs_ = std::atoi(g);
    if (const char* g = std::getenv("RTK_TILE_CONTIG")) tile_contig_ = std::atoi(g);
    if (const char* g = std::getenv("RTK_DENSE_BITS")) dense_bits_ = static_cast<uint32_t>(std::atoi(g));
    if (const char* g = std::getenv("RTK_FORCE_EXACT")) force_exact_ = *g && *g != '0';
    if (const char* g = std::getenv("RTK_FORCE_DEEP")) force_deep_ = *g && *g != '0';
    const char* cs = std::getenv("RTK_COUNT_STATS");
    count_stats_ = profile_ || (cs && *cs && *cs != '0');
}

bool Engine::set_option(const std::string& name, int64_t value) {
    if (name == "force_exact") force_exact_ = value != 0;
    else if (name == "force_deep") force_deep_ = value != 0;
    else return false;
    graph_.valid = false;  // captured graphs embed the previous plan
    have_last_ = false;
    needs_init_ = true;
    return true;
}

Engine::~Engine() {
    if (graph_.exec) cudaGraphExecDestroy(graph_.exec);
    if (cap_s_) cudaStreamDestroy(cap_s_);
    if (hmap_) cudaFreeHost(hmap_);
    if (hscale_) cudaFreeHost(hscale_);
    if (pin_) cudaFreeHost(pin_);
    if (hctl_) cudaFreeHost(hctl_);
    if (hcount_) cudaFreeHost(hcount_);
    for (auto& e : ev_)
        if (e) cudaEventDestroy(e);
    if (pin_ev_) cudaEventDestroy(pin_ev_);
    for (DevBuf* b : {&arena_, &sel_, &T_, &count_, &kmin_, &kmax_, &kor_, &ghist_, &samples_, &cand_a_,
                      &cand_b_, &seg_hist_, &gcursor_, &bstart_, &dcap_, &dcoff_, &ctl_, &row_fail_, &groups_, &slots0_, &slotsA_, &slotsB_, &done_, &seg_ticket_, &wgroups_, &ctot_, &sig_, &io_in, &io_vals, &io_idx,
                      &io_piv, &io_aux, &adapt_buf_, &scale_hist_, &scale_plan_})
        b->release();
}

uint8_t* Engine::upload(const Plan& p, cudaStream_t s) {
    if (pin_ev_pending_) {  // a stream-ordered remap's plan copy may still read the pinned staging
        check(cudaEventSynchronize(pin_ev_), "remap plan copy");
        pin_ev_pending_ = false;
    }
    const size_t need = (p.bytes.size() + 255) & ~size_t(255);
    if (arena_used_ + need > arena_.cap) {
        // earlier plan regions may still be referenced by queued kernels and by pointers the
        // caller holds: retire the old arena (freed at the end of the call), start a new one
        if (arena_.p) retired_.push_back(arena_);
        arena_ = DevBuf{};
        arena_.ensure(std::max<size_t>(need * 2, size_t(4) << 20));
        arena_used_ = 0;
        g_buf_gen.fetch_add(1);
    }
    uint8_t* d = arena_.as<uint8_t>() + arena_used_;
    arena_used_ += need;
    if (!p.bytes.empty()) {
        // stage through pinned memory so the copy is truly asynchronous
        if (pin_used_ + need > pin_cap_) {
            if (pin_) retired_pinned_.push_back(pin_);
            pin_cap_ = std::max<size_t>(need * 2, size_t(4) << 20);
            check(cudaHostAlloc(reinterpret_cast<void**>(&pin_), pin_cap_, cudaHostAllocDefault), "cudaHostAlloc");
            pin_used_ = 0;
            g_buf_gen.fetch_add(1);
        }
        uint8_t* h = pin_ + pin_used_;
        pin_used_ += need;
        std::memcpy(h, p.bytes.data(), p.bytes.size());
        if (capturing_) {
            // not part of the graph: the plan is uploaded now on the caller's stream, and again
            // before a replay only if another call has overwritten the arena since (arena_tag_)
            check(cudaMemcpyAsync(d, h, p.bytes.size(), cudaMemcpyHostToDevice, user_s_), "plan upload");
            cap_uploads_.push_back({d, h, p.bytes.size()});
        } else {
            check(cudaMemcpyAsync(d, h, p.bytes.size(), cudaMemcpyHostToDevice, s), "plan upload");
        }
        ++arena_tag_;
    }
    return d;
}

void Engine::mark(const char* name, cudaStream_t s) {
    if (!profile_) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    marks_.push_back({name, e, std::chrono::steady_clock::now()});
}

// RTK_ROWS_TRACE: per-phase end times of every k_rows_fused CTA (ns after the earliest CTA
// start): percentiles over CTAs, and the spread of CTA finish times by SM load.
void Engine::report_rows_trace(size_t nrows, cudaStream_t s) {
    std::vector<unsigned long long> t(nrows * 16);
    cudaStreamSynchronize(s);
    cudaMemcpy(t.data(), trace_.p, t.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, tend = 0;
    int nph = 0;
    for (size_t b = 0; b < nrows; ++b) {
        t0 = std::min(t0, t[b * 16]);
        int n = 0;
        while (n < 15 && t[b * 16 + n]) ++n;
        nph = std::max(nph, n);
        tend = std::max(tend, t[b * 16 + n - 1]);
    }
    std::fprintf(stderr, "[rtk rows trace] rows=%zu span=%.1fus phase end (us after first start) p0/p50/p100:", nrows,
                 (tend - t0) * 1e-3);
    for (int ph = 0; ph < nph; ++ph) {
        std::vector<double> v;
        for (size_t b = 0; b < nrows; ++b)
            if (t[b * 16 + ph]) v.push_back((t[b * 16 + ph] - t0) * 1e-3);
        std::sort(v.begin(), v.end());
        if (v.empty()) continue;
        std::fprintf(stderr, " [%d] %.1f/%.1f/%.1f", ph, v.front(), v[v.size() / 2], v.back());
    }
    std::vector<int> per_sm(1024, 0);
    for (size_t b = 0; b < nrows; ++b) ++per_sm[t[b * 16 + 15] & 1023];
    // phase durations by how many rows share the SM
    for (int load = 1; load <= 4; ++load) {
        double dur[15] = {0};
        int cnt = 0;
        for (size_t b = 0; b < nrows; ++b) {
            if (per_sm[t[b * 16 + 15] & 1023] != load) continue;
            ++cnt;
            for (int ph = 1; ph < nph; ++ph)
                if (t[b * 16 + ph]) dur[ph] += (t[b * 16 + ph] - t[b * 16 + ph - 1]) * 1e-3;
        }
        if (!cnt) continue;
        std::fprintf(stderr, "\n  rows on SMs with %d rows: %d, mean phase us:", load, cnt);
        for (int ph = 1; ph < nph; ++ph) std::fprintf(stderr, " %.1f", dur[ph] / cnt);
        double wait = 0;  // slot 14: thread 0's ring-stage waits inside the stream phase
        for (size_t b = 0; b < nrows; ++b)
            if (per_sm[t[b * 16 + 15] & 1023] == load) wait += t[b * 16 + 14] * 1e-3;
        std::fprintf(stderr, " (stream: thread 0 waited %.1f us for stages)", wait / cnt);
    }
    std::fprintf(stderr, "\n");
}

void Engine::report_marks() {
    if (!profile_ || marks_.empty()) return;
    cudaEventSynchronize(marks_.back().ev);
    if (dbg_.p) {
        unsigned long long d[64];
        cudaMemcpy(d, dbg_.p, sizeof(d), cudaMemcpyDeviceToHost);
        for (int blk = 0; blk < 2; ++blk) {
            const unsigned long long* e = d + 32 * blk;
            std::fprintf(stderr, "[rtk dbg %s phases ns]", blk ? "sample" : "msd/rows");
            for (unsigned long long i = 1; i < e[31] && i < 31; ++i) std::fprintf(stderr, " %llu", e[i] - e[i - 1]);
            if (!blk && e[12]) std::fprintf(stderr, " | plan: %llu %llu %llu", e[10] - e[3], e[11] - e[10], e[12] - e[11]);
            std::fprintf(stderr, "\n");
        }
        cudaMemset(dbg_.p, 0, sizeof(d));
    }
    std::fprintf(stderr, "[rtk profile]");
    for (size_t i = 1; i < marks_.size(); ++i) {
        float ms = 0;
        cudaEventElapsedTime(&ms, marks_[i - 1].ev, marks_[i].ev);
        const double host_us = std::chrono::duration<double, std::micro>(marks_[i].host - marks_[i - 1].host).count();
        std::fprintf(stderr, " %s=%.1fus(h%.1f)", marks_[i].name, ms * 1000.0f, host_us);
    }
    std::fprintf(stderr, "\n");
    for (auto& m : marks_) cudaEventDestroy(m.ev);
    marks_.clear();
}

void Engine::release_retired() {
    for (DevBuf& b : retired_) b.release();
    retired_.clear();
    for (uint8_t* p : retired_pinned_) cudaFreeHost(p);
    retired_pinned_.clear();
}

void Engine::sync(cudaStream_t s, const char* what) {
    check(cudaGetLastError(), what);
    check(cudaStreamSynchronize(s), what);
}

uint32_t Engine::read_word(const uint32_t* d, uint64_t i, cudaStream_t s) {
    uint32_t v = 0;
    check(cudaMemcpyAsync(&v, d + i, 4, cudaMemcpyDeviceToHost, s), "read word");
    sync(s, "read word");
    return v;
}

// ---------------------------------------------------------------------------------------
bool Engine::CallKey::operator==(const CallKey& o) const {
    if (base != o.base || dtype != o.dtype || smallest != o.smallest || scaled != o.scaled || gather != o.gather ||
        adapt != o.adapt ||
        a_s_bits != o.a_s_bits || vals != o.vals || idx != o.idx || piv != o.piv || s != o.s ||
        rows.size() != o.rows.size())
        return false;
    for (size_t i = 0; i < rows.size(); ++i)
        if (rows[i].in_off != o.rows[i].in_off || rows[i].n != o.rows[i].n || rows[i].k != o.rows[i].k ||
            rows[i].out_off != o.rows[i].out_off)
            return false;
    return true;
}

const rtk_stats& Engine::last_stats() {
    if (stats_pending_) {
        cudaEventSynchronize(ev_[3]);
        cudaEventElapsedTime(&stats.total_ms, ev_[0], ev_[3]);
        // events not recorded in this call (graph replay without event nodes) leave compact_ms
        float ms = 0.0f;
        if (cudaEventElapsedTime(&ms, ev_[1], ev_[2]) == cudaSuccess) stats.compact_ms = ms;
        cudaGetLastError();
        stats_pending_ = false;
    }
    return stats;
}

void Engine::run(const uint32_t* d_base, int dtype, int smallest, bool scaled, float a_s,
                 bool gather, const std::vector<RowReq>& rows, uint32_t* d_vals, uint64_t* d_idx,
                 uint32_t* d_pivots, cudaStream_t s) {
    DeviceGuard dg(device_);
    if (rows.empty()) return;
    if (!ev_[0]) {
        for (auto& e : ev_) check(cudaEventCreate(&e), "cudaEventCreate");
    }
    if (!hmap_) {
        check(cudaHostAlloc(reinterpret_cast<void**>(&hmap_), 64, cudaHostAllocMapped), "cudaHostAlloc");
        std::memset(hmap_, 0, 64);
        check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_hmap_), hmap_, 0), "mapped pointer");
        sig_.ensure(64);
        check(cudaMemsetAsync(sig_.p, 0, 64, s), "memset");
        check(cudaStreamSynchronize(s), "sync");
        expected_seq_ = 0;
    }
    CallKey key;
    key.base = d_base;
    key.dtype = dtype;
    key.smallest = smallest;
    key.scaled = scaled ? 1 : 0;
    key.gather = gather ? 1 : 0;
    std::memcpy(&key.a_s_bits, &a_s, 4);
    key.adapt = adapt_;
    key.vals = d_vals;
    key.idx = d_idx;
    key.piv = d_pivots;
    key.s = s;
    key.rows = rows;
    const bool usable = graphs_ && !profile_ && !count_stats_ && !timing_;
    const uint64_t gen0 = g_buf_gen.load();
    if (gen0 != last_gen_) needs_init_ = true;  // buffers reallocated: counters are garbage
    if (usable && graph_.valid && graph_.gen == gen0 && graph_.key == key) {
        // replay: restore the plan bytes the captured upload reads, launch, finish on the host
        if (call_start_) check(cudaEventRecord(call_start_, s), "event");
        if (arena_tag_ != graph_.arena_tag) {  // another call reused the arena: re-upload the plan
            if (!graph_.pinned.empty()) std::memcpy(pin_, graph_.pinned.data(), graph_.pinned.size());
            for (const auto& u : graph_.uploads)
                check(cudaMemcpyAsync(u.d, u.h, u.bytes, cudaMemcpyHostToDevice, s), "plan upload");
            arena_tag_ = graph_.arena_tag;
        }
        arena_used_ = graph_.arena_used;  // later (host-driven) uploads go after the captured plan
        pin_used_ = graph_.pin_used;
        group_base_ = graph_.group_base;
        wgroup_base_ = graph_.wgroup_base;
        stats = graph_.stats;
        const int R = static_cast<int>(rows.size());
        row_passes_.assign(R, 1);
        if (!graph_.has_init && (needs_init_ || R > clean_upto_)) {
            launch_init_call(R, count_.as<unsigned long long>(), kmin_.as<unsigned long long>(),
                             kmax_.as<unsigned long long>(), kor_.as<uint32_t>(), T_.as<uint64_t>(), row_fail_.as<uint32_t>(),
                             ctl_.as<uint32_t>(), seg_hist_.as<uint32_t>(), done_.as<uint32_t>(),
                             seg_ticket_.as<uint32_t>(), s);
        }
        clean_rows_ = graph_.clean_rows;
        check(cudaEventRecord(ev_[0], s), "event");
        check(cudaGraphLaunch(graph_.exec, s), "graph launch");
        if (call_end_) check(cudaEventRecord(call_end_, s), "event");
        check(cudaEventRecord(ev_[3], s), "event");
        expected_seq_ += graph_.seq_incr;
        sig_pending_ = graph_.seq_incr > 0;
        Call c = graph_.call;
        complete(d_base, rows, c, s);
        last_gen_ = g_buf_gen.load();
        return;
    }
    const bool capture = usable && have_last_ && last_gen_ == gen0 && last_key_ == key;
    Call c{};
    // capture on a private stream (the caller's may be the legacy default stream, which cannot
    // be captured); the graph is then launched into the caller's stream
    if (capture && !cap_s_) {
        if (cudaStreamCreateWithFlags(&cap_s_, cudaStreamNonBlocking) != cudaSuccess) {
            cudaGetLastError();
            cap_s_ = nullptr;
        }
    }
    if (capture && cap_s_ && cudaStreamBeginCapture(cap_s_, cudaStreamCaptureModeRelaxed) == cudaSuccess) {
        const uint32_t seq0 = expected_seq_;
        cudaGraph_t graph = nullptr;
        bool ok = true;
        capturing_ = true;
        user_s_ = s;
        cap_uploads_.clear();
        try {
            enqueue(d_base, dtype, smallest, scaled, a_s, gather, rows, d_vals, d_idx, d_pivots, cap_s_, c);
        } catch (const Error&) {
            ok = false;
        }
        capturing_ = false;
        c.s = s;
        ok = cudaStreamEndCapture(cap_s_, &graph) == cudaSuccess && ok;
        cudaGraphExec_t exec = nullptr;
        ok = ok && g_buf_gen.load() == gen0 && cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
        if (graph && std::getenv("RTK_GRAPH_DUMP")) cudaGraphDebugDotPrint(graph, std::getenv("RTK_GRAPH_DUMP"), 0);
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        if (!ok) {
            if (exec) cudaGraphExecDestroy(exec);
            graphs_ = false;  // capture not possible here: plain launches from now on
            expected_seq_ = seq0;
            run(d_base, dtype, smallest, scaled, a_s, gather, rows, d_vals, d_idx, d_pivots, s);
            return;
        }
        if (graph_.exec) cudaGraphExecDestroy(graph_.exec);
        graph_.exec = exec;
        graph_.key = key;
        graph_.gen = gen0;
        graph_.pinned.assign(pin_, pin_ + pin_used_);
        graph_.uploads = cap_uploads_;
        graph_.arena_tag = arena_tag_;
        graph_.call = c;
        graph_.stats = stats;
        graph_.seq_incr = expected_seq_ - seq0;
        graph_.has_init = did_init_;
        graph_.arena_used = arena_used_;
        graph_.pin_used = pin_used_;
        graph_.group_base = group_base_;
        graph_.wgroup_base = wgroup_base_;
        graph_.clean_rows = clean_rows_;
        graph_.valid = true;
        check(cudaEventRecord(ev_[0], s), "event");
        if (call_start_) check(cudaEventRecord(call_start_, s), "event");
        check(cudaGraphLaunch(exec, s), "graph launch");
        if (call_end_) check(cudaEventRecord(call_end_, s), "event");
        check(cudaEventRecord(ev_[3], s), "event");
    } else {
        cudaGetLastError();
        if (call_start_) check(cudaEventRecord(call_start_, s), "event");
        enqueue(d_base, dtype, smallest, scaled, a_s, gather, rows, d_vals, d_idx, d_pivots, s, c);
        if (call_end_) check(cudaEventRecord(call_end_, s), "event");
    }
    last_key_ = std::move(key);
    have_last_ = true;
    complete(d_base, rows, c, s);
    last_gen_ = g_buf_gen.load();
}

// Everything up to the last kernel of the common path, stream-ordered, no host synchronisation
// (capturable into a CUDA graph).
void Engine::enqueue(const uint32_t* d_base, int dtype, int smallest, bool scaled, float a_s, bool gather,
                     const std::vector<RowReq>& rows, uint32_t* d_vals, uint64_t* d_idx, uint32_t* d_pivots,
                     cudaStream_t s, Call& c_out) {
    arena_used_ = 0;
    pin_used_ = 0;
    stats = rtk_stats{};
    const int R = static_cast<int>(rows.size());
    row_passes_.assign(R, 1);  // one streaming read per row (sampled, fused, dense and LSD rows)
    record(0, s);
    mark("start", s);
    group_base_ = 0;
    wgroup_base_ = 0;
    bar_gen_ = 0;
    sig_pending_ = false;
    self_clean_ = !count_stats_ && self_clean_ok_;  // the main finish resets counters; fallback/deeper levels never
    clean_rows_ = 0;
    did_init_ = false;
    InputSrc src{d_base, dtype, smallest, scaled ? 1 : 0, a_s, adapt_};
    const uint64_t base_words = reinterpret_cast<uintptr_t>(d_base) / elem_bytes(dtype);  // base in elements

    // ---- 1. per-row plan: sample size s, sample rank r', candidate capacity -------------
    std::vector<uint32_t> rid(R), lead(R), sampled(R);
    std::vector<uint64_t> off(R), len(R), tile_start(R + 1, 0), cand_off(R), cap(R), row_k(R),
        row_out(R), row_in(R);
    struct SampleGroup {
        std::vector<uint32_t> rid;
        std::vector<uint64_t> off, len, nseg, k, target;
        uint32_t per_cta = 0;
        int cs = 1;  // cluster size
    } sg[2];  // [0]: one CTA per row, [1]: a 16-CTA cluster per row
    uint64_t cand_total = 0;
    // K6 routing: short rows with small k finish in one CTA each (k_rows_fused); the rest take
    // the general multi-CTA pipeline (sampled threshold -> k_compact -> MSD -> sort groups)
    std::vector<uint32_t> grow, frow[2];
    bool row_cluster = false;  // the one row goes to k_row_cluster (frow[1] holds it)
    std::vector<uint64_t> f_off[2], f_len[2], f_k[2];
    // returns -1 (general path), 0 (large-buffer fused variant) or 1 (small-buffer variant)
    auto fused_class = [&](const RowReq& q) {
        if (no_fused_ || force_exact_) return -1;
        if (q.k == 0 || q.k > rows_fused_kmax(false)) return -1;
        if (R == 1 && !no_rcluster_ && !trig_count_ && q.n > (uint64_t(1) << 18) && q.n <= (uint64_t(1) << 21) &&
            q.k <= row_cluster_kmax()) {  // one long query: a 16-CTA cluster (k_row_cluster)
            const double rr = static_cast<double>(q.k) * 4096.0 / static_cast<double>(q.n);
            const double rp = std::ceil(rr + 4.0 * std::sqrt(rr) + 3.0);
            if (static_cast<double>(q.n) / 4096.0 * (rp + 5.0 * std::sqrt(rp)) <= 8192.0) return 2;
        }
        if (q.n > (uint64_t(1) << 18) && R < 64) return -1;  // long rows want many CTAs
        for (int small = 1; small >= 0; --small) {
            if (q.k > rows_fused_kmax(small)) continue;
            const uint64_t cap = rows_fused_cand(small);
            if (q.n <= cap) return small;
            // expected candidates above the rp-th sample and their spread: (n/s) * Gamma(rp)
            const double s = rows_fused_sample(small);
            const double rr = static_cast<double>(q.k) * s / static_cast<double>(q.n);
            const double rp = std::ceil(rr + 4.0 * std::sqrt(rr) + 3.0);
            const double gap = static_cast<double>(q.n) / s;
            if (q.n > s && gap * (rp + 5.0 * std::sqrt(rp)) <= static_cast<double>(cap)) return small;
        }
        return -1;
    };
    std::vector<uint64_t> g_off, g_len, g_tile{0};
    std::vector<uint32_t> g_lead;
    for (int r = 0; r < R; ++r) {
        const RowReq& q = rows[r];
        rid[r] = r;
        off[r] = q.in_off;
        len[r] = q.n;
        lead[r] = static_cast<uint32_t>((base_words + q.in_off) & 7);
        tile_start[r + 1] = tile_start[r] + ceil_div(lead[r] + q.n, kTile);
        row_k[r] = q.k;
        row_out[r] = q.out_off;
        row_in[r] = q.in_off;
        int fc = fused_class(q);
        if (fc == 2) {
            row_cluster = true;
            fc = 1;
        }
        if (fc >= 0) {
            frow[fc].push_back(r);
            f_off[fc].push_back(q.in_off);
            f_len[fc].push_back(q.n);
            f_k[fc].push_back(q.k);
            cap[r] = q.n;  // only used if the row falls back to the exact path
            cand_off[r] = 0;
            stats.elements_scanned += q.n;
            continue;
        }
        grow.push_back(r);
        g_off.push_back(q.in_off);
        g_len.push_back(q.n);
        g_lead.push_back(lead[r]);
        g_tile.push_back(g_tile.back() + ceil_div(lead[r] + q.n, kTile));
        bool samp = q.k < q.n && q.n >= 4 * kSortCap;
        uint64_t ns = 0, rp = 0;
        if (samp) {
            // stratified sample: 2^-7 of huge rows (cluster of 8 CTAs), 2^-6 of the others
            // huge rows: enough samples that ~sample_r_ of them land above the threshold
            // (r = k s / n), 2^14..2^17 and <= n/128; a 16-CTA cluster per row when s > 8192
            if (q.n >= (uint64_t(1) << 22)) {
                const double want = static_cast<double>(sample_r_) * static_cast<double>(q.n) / static_cast<double>(q.k);
                uint64_t p2 = uint64_t(1) << 14;
                while (p2 < want && p2 < (uint64_t(1) << 17)) p2 <<= 1;
                ns = std::min<uint64_t>(p2, q.n / 128);
            } else {
                ns = std::min<uint64_t>(8192, std::max<uint64_t>(2048, q.n / 64));
            }
            ns &= ~uint64_t(31);
            const double rr = static_cast<double>(q.k) * static_cast<double>(ns) / static_cast<double>(q.n);
            rp = static_cast<uint64_t>(std::ceil(rr + 4.0 * std::sqrt(rr) + 3.0));
            if (rp >= ns / 2) samp = false;
        }
        sampled[r] = samp;
        if (samp) {
            const double ratio = static_cast<double>(q.n) / static_cast<double>(ns);
            cap[r] = std::min<uint64_t>(q.n, static_cast<uint64_t>(ratio * (2.0 * rp + 16.0)) + 1024);
            const int grp = ns > 8192 ? 1 : 0;
            SampleGroup& g = sg[grp];
            g.rid.push_back(r);
            g.off.push_back(q.in_off);
            g.len.push_back(q.n);
            g.nseg.push_back(ns / 32);
            g.k.push_back(rp);
            g.target.push_back(rp + rp / 10 + 8);
            if (grp) {  // a power of two: the sample kernel splits its 2048 bins into cs equal slices
                int cs = 1;
                while (cs * 2 <= 16 && static_cast<uint64_t>(cs * 2) * 4096 <= ns) cs *= 2;
                g.cs = std::max<int>(g.cs, cs);
            }
            g.per_cta = std::max<uint32_t>(g.per_cta, static_cast<uint32_t>(ns / g.cs));
        } else {
            cap[r] = q.n;
        }
        cand_off[r] = (cand_total + 3) & ~uint64_t(3);
        cand_total = cand_off[r] + cap[r];
        stats.elements_scanned += q.n + ns;
    }

    sel_.ensure(sizeof(RowSel) * R);
    T_.ensure(8 * R);
    count_.ensure(8 * R);
    kmin_.ensure(8 * R);
    kmax_.ensure(8 * R);
    kor_.ensure(4 * R);
    ghist_.ensure(8ull * kBins * R);
    cand_a_.ensure(8 * std::max<uint64_t>(cand_total, 1));

    // Dense mode: every general row is unsampled with k >= n/2 (e.g. k = vocab): all elements are
    // candidates, so the compaction would only rewrite the rows as composites. The level-0 MSD
    // reads the input instead (slot.src = 1), its digit the top bits of the key.
    bool dense = !grow.empty() && no_dense_ == false && !force_exact_;
    std::vector<SegSlot> dslots;
    for (uint32_t r : grow) {
        const RowReq& q = rows[r];
        if (sampled[r] || 2 * q.k < q.n || q.n <= kSortCap) { dense = false; break; }
        const uint32_t bits = std::min<uint32_t>(dense_bits_ ? dense_bits_ : fine_bits(q.n), level0_bits());
        SegSlot sl{cand_off[r], q.n, 0, r, 64u - bits, bits, 1u, q.in_off};
        dslots.push_back(sl);
    }
    if (!dense) dslots.clear();
    // dense rows of >= 2 tiles each: the segmented one-sweep LSD sort (rtk_lsd.cu)
    // (RTK_LSD=off: the MSD + bucket-sort path; RTK_LSD=16: 16-bit keys only)
    const bool lsd = dense && (lsd_mode_ == 2 || (lsd_mode_ == 1 && dtype == kF16));
    std::vector<uint64_t> l_tile{0}, l_len, l_in, l_buf, l_k, l_out;
    std::vector<uint32_t> l_order;
    uint64_t l_total = 0;
    if (lsd) {
        for (uint32_t r : grow) {
            const RowReq& q = rows[r];
            l_tile.push_back(l_tile.back() + ceil_div(q.n, lsd_tile()));
            l_len.push_back(q.n);
            l_in.push_back(q.in_off);
            l_buf.push_back(l_total);
            l_total += (q.n + 3) & ~uint64_t(3);
            l_k.push_back(q.k);
            l_out.push_back(q.out_off);
        }
        // claim order of the LSD tiles: round-robin over the rows (tile 0 of every row, then tile
        // 1, ...), so a tile's predecessor in its row was claimed ~R claims earlier and has
        // usually published its inclusive prefix by the time the tile looks back
        if (lsd_rr_) {
            const size_t NR = l_len.size();
            uint64_t maxt = 0;
            for (size_t j = 0; j < NR; ++j) maxt = std::max(maxt, l_tile[j + 1] - l_tile[j]);
            l_order.reserve(l_tile.back());
            for (uint64_t t = 0; t < maxt; ++t)
                for (size_t j = 0; j < NR; ++j)
                    if (l_tile[j] + t < l_tile[j + 1]) l_order.push_back(static_cast<uint32_t>(l_tile[j] + t));
        }
    }
    Plan P;
    const size_t o_dslots = P.add(dslots);
    const size_t o_ltile = P.add(l_tile), o_llen = P.add(l_len), o_lin = P.add(l_in), o_lbuf = P.add(l_buf),
                 o_lk = P.add(l_k), o_lout = P.add(l_out), o_lord = P.add(l_order);
    const size_t o_rid = P.add(rid), o_off = P.add(off), o_len = P.add(len), o_lead = P.add(lead),
                 o_tile = P.add(tile_start), o_coff = P.add(cand_off), o_cap = P.add(cap),
                 o_k = P.add(row_k), o_out = P.add(row_out), o_in = P.add(row_in),
                 o_grow = P.add(grow), o_goff = P.add(g_off), o_glen = P.add(g_len), o_glead = P.add(g_lead),
                 o_gtile = P.add(g_tile);
    size_t o_f[2][4];
    for (int v = 0; v < 2; ++v) {
        o_f[v][0] = P.add(frow[v]);
        o_f[v][1] = P.add(f_off[v]);
        o_f[v][2] = P.add(f_len[v]);
        o_f[v][3] = P.add(f_k[v]);
    }
    size_t o_sg[2][6];
    for (int g = 0; g < 2; ++g) {
        o_sg[g][0] = P.add(sg[g].rid);
        o_sg[g][1] = P.add(sg[g].off);
        o_sg[g][2] = P.add(sg[g].len);
        o_sg[g][3] = P.add(sg[g].nseg);
        o_sg[g][4] = P.add(sg[g].k);
        o_sg[g][5] = P.add(sg[g].target);
    }
    uint8_t* D = upload(P, s);
    mark("plan", s);

    ctl_.ensure(64);
    row_fail_.ensure(4 * R);
    done_.ensure(4 * R);
    seg_ticket_.ensure(4 * R);
    seg_hist_.ensure(4ull * kBins * R);
    // one kernel resets every per-call counter (unsampled rows keep T = 0) — unless the previous
    // call's last sort CTA already did (self-cleaning, see SortArgs::R_clean)
    if (needs_init_ || R > clean_upto_ || force_init_) {
    needs_init_ = false;
    did_init_ = true;
    launch_init_call(R, count_.as<unsigned long long>(), kmin_.as<unsigned long long>(),
                     kmax_.as<unsigned long long>(), kor_.as<uint32_t>(), T_.as<uint64_t>(), row_fail_.as<uint32_t>(),
                     ctl_.as<uint32_t>(), seg_hist_.as<uint32_t>(), done_.as<uint32_t>(),
                     seg_ticket_.as<uint32_t>(), s);
    ++stats.kernel_launches;
    }
    mark("init", s);

    for (int g = 0; g < 2; ++g) {
        if (sg[g].rid.empty()) continue;
        if (profile_) dbg_.ensure(4096);
        SampleRows sr{at<uint32_t>(D, o_sg[g][0]), at<uint64_t>(D, o_sg[g][1]), at<uint64_t>(D, o_sg[g][2]),
                      at<uint64_t>(D, o_sg[g][3]), at<uint64_t>(D, o_sg[g][4]), at<uint64_t>(D, o_sg[g][5]),
                      profile_ ? dbg_.as<unsigned long long>() + 32 : nullptr};
        launch_sample_select(static_cast<int>(sg[g].rid.size()), sg[g].cs, sg[g].per_cta, sr, src,
                             T_.as<uint64_t>(), s);
        check(cudaGetLastError(), "sample_select launch");
        ++stats.kernel_launches;
    }
    mark("sample", s);

    // ---- 2-4. compaction (+ fused per-row plan) and the device-planned ordering ----------
    Call c{src, gather, at<uint64_t>(D, o_k), at<uint64_t>(D, o_out), at<uint64_t>(D, o_in), d_vals,
           d_idx, s, cap, cand_off, cand_total, std::vector<uint64_t>(R), R,
           at<uint64_t>(D, o_cap), at<uint64_t>(D, o_coff), d_pivots};
    for (int v = 0; v < 2; ++v) {
        if (frow[v].empty()) continue;
        RowsFusedArgs fa{at<uint32_t>(D, o_f[v][0]), at<uint64_t>(D, o_f[v][1]), at<uint64_t>(D, o_f[v][2]),
                         at<uint64_t>(D, o_f[v][3]), src, c.d_row_out, d_vals, d_idx, d_pivots,
                         row_fail_.as<uint32_t>(), ctl_.as<uint32_t>(), nullptr, CallTail{},
                         static_cast<uint32_t>(rows_pf_) | (static_cast<uint32_t>(rows_pf0_) << 16)};
        if (profile_) {
            dbg_.ensure(4096);
            fa.dbg = dbg_.as<unsigned long long>();
        }
        // the call's last kernel (no general rows, last fused variant): completion signal + clean
        const bool last = grow.empty() && (v == 1 || frow[1].empty());
        if (last && !count_stats_) {
            fa.tail = tail_args();
            if (self_clean_) {
                set_clean(fa.tail, R);
                clean_rows_ = R;
            }
        }
        const size_t nfr = frow[v].size();
        if (rows_trace_) {
            trace_.ensure(nfr * 16 * sizeof(unsigned long long));
            cudaMemsetAsync(trace_.p, 0, nfr * 16 * sizeof(unsigned long long), s);
            fa.trace = trace_.as<unsigned long long>();
        }
        if (v == 1 && row_cluster) launch_row_cluster(fa, s);
        else launch_rows_fused(static_cast<int>(nfr), fa, v == 1, s);
        ++stats.kernel_launches;
        if (rows_trace_) report_rows_trace(nfr, s);
        if (fa.tail.hflags) {
            ++expected_seq_;
            sig_pending_ = true;
        }
        mark("rows_fused", s);
    }
    record(1, s);
    if (!grow.empty() && lsd) {
        record(2, s);
        mark("compact(skipped: dense rows)", s);
        const int NR = static_cast<int>(grow.size());
        const uint64_t tiles = l_tile.back();
        lsd_a_.ensure(8 * std::max<uint64_t>(l_total, 1));
        lsd_b_.ensure(8 * std::max<uint64_t>(l_total, 1));
        // look-back words carry a device epoch (ctr[4]); both are zeroed together whenever either
        // buffer is (re)allocated, so a stale word can never match a later call's epoch
        if (lsd_status_.cap < 8 * 256 * tiles || lsd_hist_cap_ < static_cast<size_t>(NR)) {
            lsd_status_.ensure(std::max<size_t>(lsd_status_.cap, 8 * 256 * tiles));
            lsd_hist_cap_ = std::max<size_t>(lsd_hist_cap_, NR);
            lsd_meta_.ensure(4ull * (1024ull * lsd_hist_cap_ + 8));
            check(cudaMemsetAsync(lsd_status_.p, 0, lsd_status_.cap, s), "memset");
            check(cudaMemsetAsync(lsd_meta_.p, 0, 4ull * (1024ull * lsd_hist_cap_ + 8), s), "memset");
        }
        uint32_t* hist = lsd_meta_.as<uint32_t>();
        uint32_t* ctr = hist + 1024ull * lsd_hist_cap_;
        check(cudaMemsetAsync(hist, 0, 4ull * 1024 * NR, s), "memset");
        check(cudaMemsetAsync(ctr, 0, 16, s), "memset");  // tile counters; ctr[4] (epoch) persists
        LsdArgs la{};
        la.R = NR;
        la.tile_start = at<uint64_t>(D, o_ltile);
        la.order = l_order.empty() ? nullptr : at<uint32_t>(D, o_lord);
        la.len = at<uint64_t>(D, o_llen);
        la.in_off = at<uint64_t>(D, o_lin);
        la.buf_off = at<uint64_t>(D, o_lbuf);
        la.k = at<uint64_t>(D, o_lk);
        la.out_off = at<uint64_t>(D, o_lout);
        la.rid = at<uint32_t>(D, o_grow);
        la.hist = hist;
        la.status = lsd_status_.as<unsigned long long>();
        la.ctr = ctr;
        la.src = lsd_b_.as<unsigned long long>();
        la.dst = lsd_a_.as<unsigned long long>();
        la.in = src;
        la.out_vals = d_vals;
        la.out_idx = d_idx;
        la.pivots = d_pivots;
        la.npass = dtype == kF16 ? 2u : 4u;
        la.shift0 = dtype == kF16 ? 16u : 0u;
        la.tail = tail_args();
        if (self_clean_) {
            set_clean(la.tail, R);
            clean_rows_ = R;
        }
        if (lsd_trace_) {
            lsd_trace_buf_.ensure(8ull * 8 * 4 * tiles);
            check(cudaMemsetAsync(lsd_trace_buf_.p, 0, 8ull * 8 * 4 * tiles, s), "memset");
            la.trace = lsd_trace_buf_.as<unsigned long long>();
        }
        launch_lsd(tiles, la, s);
        check(cudaGetLastError(), "lsd launch");
        if (lsd_trace_) {  // per pass: phase durations (p10/p50/p90 us) and the pass span
            std::vector<unsigned long long> tv(8ull * 4 * tiles);
            check(cudaStreamSynchronize(s), "sync");
            check(cudaMemcpy(tv.data(), lsd_trace_buf_.p, 8 * tv.size(), cudaMemcpyDeviceToHost), "trace");
            for (uint32_t p = 0; p < la.npass; ++p) {
                std::vector<double> ph[6];
                unsigned long long t0 = ~0ull, t1 = 0;
                for (uint64_t t = 0; t < tiles; ++t) {
                    const unsigned long long* e = tv.data() + (p * tiles + t) * 8;
                    if (!e[0] || !e[4]) continue;
                    const int last = e[5] ? 5 : 4;
                    t0 = std::min(t0, e[0]);
                    t1 = std::max(t1, e[last]);
                    for (int i = 1; i <= last; ++i) ph[i - 1].push_back((e[i] - e[i - 1]) * 1e-3);
                    ph[5].push_back((e[last] - e[0]) * 1e-3);
                }
                std::fprintf(stderr, "[rtk lsd trace] pass %u span %.1f us; phase us p10/p50/p90:", p, (t1 - t0) * 1e-3);
                const char* nm[6] = {"rank", "lookback", "scan", "reorder", "store", "tile"};
                for (int i = 0; i < 6; ++i) {
                    auto& v = ph[i];
                    if (v.empty()) continue;
                    std::sort(v.begin(), v.end());
                    std::fprintf(stderr, " %s %.2f/%.2f/%.2f", nm[i], v[v.size() / 10], v[v.size() / 2], v[v.size() * 9 / 10]);
                }
                std::fprintf(stderr, "\n");
            }
        }
        stats.kernel_launches += 1 + la.npass;
        ++expected_seq_;
        sig_pending_ = true;
        mark("lsd sort", s);
    } else if (!grow.empty() && dense) {
        FinishPrep fp = prepare_finish(c, grow);
        fp.slots = at<SegSlot>(D, o_dslots);
        record(2, s);
        mark("compact(skipped: dense rows)", s);
        launch_finish(c, fp);
    } else if (!grow.empty()) {
        FinishPrep fp = prepare_finish(c, grow);
        Rows all{static_cast<int>(grow.size()), at<uint32_t>(D, o_grow), at<uint64_t>(D, o_goff),
                 at<uint64_t>(D, o_glen), at<uint32_t>(D, o_glead), at<uint64_t>(D, o_gtile)};
        launch_compact(g_tile.back(), all, src, T_.as<uint64_t>(), cand_a_.as<uint64_t>(), c.d_coff, c.d_cap,
                       count_.as<unsigned long long>(), kmin_.as<unsigned long long>(),
                       kmax_.as<unsigned long long>(), plan_args(c, fp), s);
        stats.kernel_launches += 1;
        record(2, s);
        mark("compact", s);
        launch_finish(c, fp);
    } else {
        record(2, s);
    }
    record(3, s);
    c_out = std::move(c);
}

// Wait for the common path, then the rare host-driven paths (deeper MSD levels, exact path).
void Engine::complete(const uint32_t* d_base, const std::vector<RowReq>& rows, Call& c, cudaStream_t s) {
    const int R = static_cast<int>(rows.size());
    uint32_t ctl[8];
    self_clean_ = false;
    // the next call may skip the init kernel only if this call's main sort cleaned every row and
    // nothing else (deeper levels, exact path, errors) touches the counters afterwards
    const bool cleaned = clean_rows_ >= R && sig_pending_;
    needs_init_ = true;
    drain(c, ctl);
    std::memcpy(trig_words_, drain_trig_, sizeof(trig_words_));  // the main path's trigger counts
    // host-driven rare paths enqueue more device work: the call's end moves behind it
    const bool extra = (first_flags_ & (kFlagMore | kFlagFail)) != 0;
    // first_flags_: the flag word as the main path left it (drain's deeper levels clear kFlagMore)
    if (cleaned && (first_flags_ & (kFlagFail | kFlagMore | kFlagOverflow)) == 0) {
        needs_init_ = false;
        clean_upto_ = clean_rows_;
    } else {
        clean_upto_ = 0;
    }

    // ---- exact path for rows whose sampled threshold missed (rare) ------------------------
    if (ctl[0] & kFlagFail) {
        std::vector<uint32_t> fail(R), fb;
        check(cudaMemcpyAsync(fail.data(), row_fail_.p, 4 * R, cudaMemcpyDeviceToHost, s), "d2h");
        sync(s, "row_fail");
        for (int r = 0; r < R; ++r)
            if (fail[r]) fb.push_back(r);
        stats.fallback_rows = fb.size();
        fallback(d_base, c.src, rows, fb, c, s);
        drain(c, ctl);
        if (ctl[0] & kFlagFail) throw Error{RTK_INVARIANT_VIOLATION, "filter: pivot inconsistent after exact path"};
        record(3, s);
        if (call_end_) check(cudaEventRecord(call_end_, s), "event");
        sync(s, "finish");
    } else if (extra && call_end_) {
        check(cudaEventRecord(call_end_, s), "event");
    }
    if (count_stats_)
        for (int r = 0; r < R; ++r) stats.candidates += hcount_[r];
    mark("drain", s);
    report_marks();
    release_retired();
    stats_pending_ = true;  // compact_ms / total_ms resolved lazily (the events may still be pending)
    if (profile_) last_stats();
}

// ---------------------------------------------------------------------------------------
// Device-planned ordering of the candidates of rows `rids` (no host round trip):
// [k_compact's last CTA per row plans it] -> MSD level 0: k_seg_hist (+ fused bucket plan)
// -> k_seg_scatter -> k_sort_groups (+ pivots). Level-0 tiles are laid out over the rows'
// candidate CAPACITIES; each tile reads the actual count on the device.
// ---------------------------------------------------------------------------------------
Engine::FinishPrep Engine::prepare_finish(Call& c, const std::vector<uint32_t>& rids) {
    FinishPrep f{};
    f.NR = static_cast<int>(rids.size());
    // level-0 MSD bounds from the capacity (the device picks bits = fine_bits(m) <= fine_bits(cap))
    uint64_t cta_groups = f.NR, warp_groups = 0, max_cap = 0;
    for (int j = 0; j < f.NR; ++j) {
        const uint64_t cp = c.cap[rids[j]];
        if (cp <= kSortCap) continue;
        ++f.big_rows;
        max_cap = std::max(max_cap, cp);
        const uint64_t bins = uint64_t(1) << std::min<uint32_t>(fine_bits(cp), msd_max_bits_);
        cta_groups += std::min<uint64_t>(bins, cp / (kWarpGroupMax + 1) + 1);
        warp_groups += std::min<uint64_t>(bins, cp);
    }
    f.cs = msd_cluster_size(max_cap);
    // many big rows (batched dense rows, k = vocab): smaller clusters run more rows at once; the
    // MSD of one slot is latency-bound (cluster barriers), not bandwidth-bound
    if (msd_cs_) f.cs = msd_cs_;
    else
        while (f.cs > 2 && f.big_rows * static_cast<uint64_t>(f.cs) > 2ull * num_sms()) f.cs >>= 1;
    f.max_cap = max_cap;
    f.max_groups = cta_groups;
    f.max_wgroups = warp_groups;
    groups_.ensure(sizeof(SortGroup) * (group_base_ + f.max_groups), /*keep=*/true, c.s);
    wgroups_.ensure(sizeof(SortGroup) * std::max<uint64_t>(wgroup_base_ + f.max_wgroups, 1), /*keep=*/true, c.s);
    slots0_.ensure(sizeof(SegSlot) * std::max(f.NR, 1));
    const uint64_t max_next = c.cand_total / kSortCap + f.NR + 1;
    slotsA_.ensure(sizeof(SegSlot) * max_next);
    slotsB_.ensure(sizeof(SegSlot) * max_next);
    seg_hist_.ensure(4ull * kBins * std::max<int>(f.NR, 1));
    gcursor_.ensure(4ull * kBins * std::max<int>(f.NR, 1));
    bstart_.ensure(4ull * kBins * std::max<int>(f.NR, 1));
    cand_b_.ensure(8 * std::max<uint64_t>(c.cand_total, 1));
    next_cap_ = static_cast<uint32_t>(max_next);
    uint32_t* ctl = ctl_.as<uint32_t>();
    f.gl = GroupList{groups_.as<SortGroup>(), ctl + 1, static_cast<uint32_t>(group_base_ + f.max_groups)};
    f.wgl = GroupList{wgroups_.as<SortGroup>(), ctl + 5, static_cast<uint32_t>(wgroup_base_ + f.max_wgroups)};
    f.nextA = SlotList{slotsA_.as<SegSlot>(), ctl + 3, next_cap_};
    group_base_ += f.max_groups;
    wgroup_base_ += f.max_wgroups;
    wgroup_cap_ = static_cast<uint32_t>(wgroup_base_);
    return f;
}

PlanArgs Engine::plan_args(const Call& c, const FinishPrep& f) {
    PlanArgs pa{};
    pa.cap = c.d_cap;
    pa.row_k = c.d_row_k;
    pa.cand_off = c.d_coff;
    pa.count = count_.as<unsigned long long>();
    pa.kmin = kmin_.as<unsigned long long>();
    pa.kmax = kmax_.as<unsigned long long>();
    pa.kor = kor_.as<uint32_t>();
    // interleaved tiles stream ~12% faster for one huge row; many rows prefer contiguous runs
    pa.contig = tile_contig_ >= 0 ? static_cast<uint32_t>(tile_contig_) : (f.NR > 8 ? 1u : 0u);
    pa.slots = slots0_.as<SegSlot>();
    pa.groups = f.gl;
    pa.flags = ctl_.as<uint32_t>();
    pa.row_fail = row_fail_.as<uint32_t>();
    pa.done = done_.as<uint32_t>();
    pa.max_bits = level0_bits();
    pa.force_fail = force_exact_ && !in_fallback_ ? 1u : 0u;
    pa.trig = trig_count_ && !in_fallback_ ? 1u : 0u;
    pa.prefetch_mb = static_cast<uint32_t>(prefetch_mb_);
    pa.sparse_max = static_cast<uint32_t>(sparse_max_);
    pa.sparse_sel = static_cast<uint32_t>(sparse_sel_);
    pa.dyn_ctr = dyn_per_cta_ > 0 ? ctl_.as<uint32_t>() + 8 : nullptr;  // ctl[8..9]: zeroed by init / self-clean
    pa.dyn_per_cta = static_cast<uint32_t>(dyn_per_cta_);
    return pa;
}

void Engine::launch_finish(Call& c, const FinishPrep& f) {
    if (f.NR == 0) return;
    if (f.big_rows) {
        FineArgs fa{c.src, c.d_row_k, f.gl, f.wgl, f.nextA, ctl_.as<uint32_t>(), nullptr, 1, nullptr, nullptr, 0};
        const SegSlot* slots = f.slots ? f.slots : slots0_.as<SegSlot>();
        if (profile_) {
            dbg_.ensure(4096);
            fa.dbg = dbg_.as<unsigned long long>();
        }
        // one huge slot: spread it over Q co-resident 8-CTA clusters (>= ~8K composites per CTA)
        int cs = f.cs;
        if (f.NR == 1 && f.cs == 16) {
            const uint64_t want = std::max<uint64_t>(1, f.max_cap / (8 * 8192));
            const uint32_t Q = static_cast<uint32_t>(std::min<uint64_t>(
                std::min<uint64_t>(msd_q_max_, static_cast<uint64_t>(msd_max_clusters(8))), want));
            if (Q > 1) {
                cs = 8;
                fa.Q = Q;
                ctot_.ensure(4ull * fa.Q << kMsdMaxBits);
                fa.ctot = ctot_.as<uint32_t>();
                fa.bar = ctl_.as<uint32_t>() + 7;
                bar_gen_ += fa.Q * cs;
                fa.bar_target = bar_gen_;
            }
        }
        if (!launch_msd_cluster(f.NR, cs, slots, cand_a_.as<uint64_t>(), cand_b_.as<uint64_t>(), fa, c.s)) {
            bar_gen_ -= fa.Q * cs;
            fa.Q = 1;
            launch_msd_cluster(f.NR, f.cs, slots, cand_a_.as<uint64_t>(), cand_b_.as<uint64_t>(), fa, c.s);
        }
        check(cudaGetLastError(), "msd launch");
        stats.kernel_launches += 1;
        mark("msd", c.s);
    }
    SortArgs sa = sort_args(c, f.gl);
    if (self_clean_) {
        set_clean(sa.tail, c.R);
        clean_rows_ = c.R;
    }
    launch_sort(static_cast<uint32_t>(f.max_groups + f.max_wgroups / 8 + 1), sa, c.s);
    mark("sort+pivots", c.s);
}

// stats events: inside a capture they must be external record nodes to be replayed
void Engine::record(int i, cudaStream_t s) {
    if (capturing_ && (i == 0 || i == 3)) return;  // recorded around the graph launch instead
    if (capturing_ && no_graph_events_) return;     // keep kernel->kernel PDL edges unbroken
    check(capturing_ ? cudaEventRecordWithFlags(ev_[i], s, cudaEventRecordExternal) : cudaEventRecord(ev_[i], s),
          "event");
}

void Engine::launch_sort(uint32_t max_groups, const SortArgs& a, cudaStream_t s) {
    launch_sort_groups(max_groups, a, s);
    ++stats.kernel_launches;
    ++expected_seq_;
    sig_pending_ = true;
}

// Spin on the mapped signal word (the last sort CTA's sequence number). The stream is polled
// now and then so a failed kernel surfaces as an error instead of a hang.
void Engine::wait_signal(cudaStream_t s) {
    const volatile uint32_t* f = hmap_;
    for (uint64_t spin = 0;; ++spin) {
        if (((f[15] ^ expected_seq_) & 0x7FFFFFFFu) == 0) return;
        if ((spin & 1023) == 1023) {
            const cudaError_t e = cudaStreamQuery(s);
            if (e == cudaSuccess) {
                if (((f[15] ^ expected_seq_) & 0x7FFFFFFFu) == 0) return;
                throw Error{RTK_INTERNAL, "completion signal missing"};
            }
            if (e != cudaErrorNotReady) check(e, "kernel");
        }
    }
}

CallTail Engine::tail_args() {
    CallTail t{};
    t.ctl = ctl_.as<uint32_t>();
    t.done_ctr = sig_.as<uint32_t>();
    t.seq_ctr = sig_.as<uint32_t>() + 1;
    t.hflags = d_hmap_;
    return t;
}

void Engine::set_clean(CallTail& t, int R) {
    t.R_clean = R;
    t.c_count = count_.as<unsigned long long>();
    t.c_kmin = kmin_.as<unsigned long long>();
    t.c_kmax = kmax_.as<unsigned long long>();
    t.c_kor = kor_.as<uint32_t>();
    t.c_T = T_.as<uint64_t>();
    t.c_done = done_.as<uint32_t>();
    t.c_ticket = seg_ticket_.as<uint32_t>();
}

SortArgs Engine::sort_args(const Call& c, const GroupList& gl) {
    SortArgs a{};
    a.tail = tail_args();
    a.groups = gl;
    a.work = ctl_.as<uint32_t>() + 2;
    a.wgroups = GroupList{wgroups_.as<SortGroup>(), ctl_.as<uint32_t>() + 5, wgroup_cap_};
    a.wwork = ctl_.as<uint32_t>() + 6;
    a.buf0 = cand_a_.as<unsigned long long>();
    a.buf1 = cand_b_.as<unsigned long long>();
    a.row_k = c.d_row_k;
    a.row_out_off = c.d_row_out;
    a.row_in_off = c.d_row_in;
    a.in_base = c.src.base;
    a.out_vals = c.d_vals;
    a.out_idx = c.d_idx;
    a.pivots = c.d_pivots;
    a.gather = c.gather ? 1 : 0;
    a.dtype = c.src.dtype;
    a.smallest = c.src.smallest;
    return a;
}

// Synchronise, then run host-driven deeper MSD levels while some bucket is still larger than
// one CTA's sort (adversarial/clustered candidate sets only). ctl: [flags, groups, work, nA, nB].
void Engine::drain(Call& c, uint32_t (&ctl)[8]) {
    if (!hctl_) check(cudaHostAlloc(reinterpret_cast<void**>(&hctl_), 64, cudaHostAllocDefault), "cudaHostAlloc");
    if (hcount_cap_ < static_cast<size_t>(c.R)) {
        if (hcount_) cudaFreeHost(hcount_);
        hcount_cap_ = std::max<size_t>(c.R, 1024);
        check(cudaHostAlloc(reinterpret_cast<void**>(&hcount_), 8 * hcount_cap_, cudaHostAllocDefault), "cudaHostAlloc");
    }
    if (sig_pending_ && !count_stats_) {
        wait_signal(c.s);  // the last CTA published ctl[0..7] and ctl[10..13]: no copy, no stream sync
        // bit 31 of the sequence word: the words were published; clear: the flags and the
        // trigger counts were zero (the other words matter only under a flag)
        const volatile uint32_t* hw = hmap_;
        const bool words = (hw[15] >> 31) != 0;
        for (int i = 0; i < 8; ++i) ctl[i] = words ? hw[i] : 0u;
        for (int i = 0; i < 4; ++i) drain_trig_[i] = words ? hw[8 + i] : 0u;  // ctl[10..13]
    } else {
        check(cudaMemcpyAsync(hctl_, ctl_.p, 64, cudaMemcpyDeviceToHost, c.s), "d2h");
        if (count_stats_) check(cudaMemcpyAsync(hcount_, count_.p, 8 * c.R, cudaMemcpyDeviceToHost, c.s), "d2h");
        sync(c.s, "finish");
        std::memcpy(ctl, hctl_, 32);
        std::memcpy(drain_trig_, hctl_ + 10, 16);
    }
    sig_pending_ = false;
    first_flags_ = ctl[0];
    if (profile_)
        std::fprintf(stderr, "[rtk ctl] flags=%u cta_groups=%u next_slots=%u warp_groups=%u\n", ctl[0], ctl[1], ctl[3], ctl[5]);
    if (ctl[0] & kFlagOverflow) throw Error{RTK_INTERNAL, "device work list overflow"};
    const uint32_t sticky = ctl[0] & kFlagFail;  // rows for the exact path (kept across levels)
    int src_buf = 1;  // level-0 buckets live in buffer B
    int list = 0;     // next-level slots are in list A (count ctl[3])
    uint32_t nslots = ctl[3];
    while (ctl[0] & kFlagMore) {
        if (nslots > next_cap_) throw Error{RTK_INTERNAL, "MSD slot list overflow"};
        std::vector<SegSlot> sl(nslots);
        DevBuf& cur = list == 0 ? slotsA_ : slotsB_;
        DevBuf& nxt = list == 0 ? slotsB_ : slotsA_;
        check(cudaMemcpyAsync(sl.data(), cur.p, sizeof(SegSlot) * nslots, cudaMemcpyDeviceToHost, c.s), "d2h");
        sync(c.s, "slots");
        std::vector<uint64_t> tiles(nslots + 1, 0);
        for (uint32_t j = 0; j < nslots; ++j) tiles[j + 1] = tiles[j] + ceil_div(sl[j].len + (sl[j].off & 3), kTile64);
        const uint64_t max_groups = uint64_t(nslots) * kBins;
        groups_.ensure(sizeof(SortGroup) * (group_base_ + max_groups), true, c.s);
        seg_hist_.ensure(4ull * kBins * nslots);
        gcursor_.ensure(4ull * kBins * nslots);
        bstart_.ensure(4ull * kBins * nslots);
        seg_ticket_.ensure(4ull * nslots);
        Plan P;
        const size_t o_tiles = P.add(tiles);
        uint8_t* D = upload(P, c.s);
        uint32_t* dctl = ctl_.as<uint32_t>();
        // flags = 0, work = groups so far, next list count = 0
        check(cudaMemsetAsync(dctl, 0, 4, c.s), "memset");
        check(cudaMemcpyAsync(dctl + 2, dctl + 1, 4, cudaMemcpyDeviceToDevice, c.s), "work");
        check(cudaMemcpyAsync(dctl + 6, dctl + 5, 4, cudaMemcpyDeviceToDevice, c.s), "wwork");
        check(cudaMemsetAsync(dctl + (list == 0 ? 4 : 3), 0, 4, c.s), "memset");
        check(cudaMemsetAsync(seg_hist_.p, 0, 4ull * kBins * nslots, c.s), "memset");
        check(cudaMemsetAsync(seg_ticket_.p, 0, 4ull * nslots, c.s), "memset");
        GroupList gl{groups_.as<SortGroup>(), dctl + 1, static_cast<uint32_t>(group_base_ + max_groups)};
        SlotList nl{nxt.as<SegSlot>(), dctl + (list == 0 ? 4 : 3), next_cap_};
        uint64_t* bsrc = src_buf ? cand_b_.as<uint64_t>() : cand_a_.as<uint64_t>();
        uint64_t* bdst = src_buf ? cand_a_.as<uint64_t>() : cand_b_.as<uint64_t>();
        SegPlanArgs pa{seg_hist_.as<uint32_t>(), gcursor_.as<uint32_t>(), c.d_row_k, bstart_.as<uint32_t>(), gl,
                       static_cast<uint32_t>(src_buf ? 0 : 1), nl, dctl, seg_ticket_.as<uint32_t>()};
        launch_seg_hist(tiles.back(), cur.as<SegSlot>(), nslots, at<uint64_t>(D, o_tiles), bsrc, pa, c.s);
        launch_seg_scatter(tiles.back(), cur.as<SegSlot>(), nslots, at<uint64_t>(D, o_tiles), bsrc, bdst,
                           bstart_.as<uint32_t>(), gcursor_.as<uint32_t>(), c.s);
        launch_sort(static_cast<uint32_t>(max_groups), sort_args(c, gl), c.s);
        stats.kernel_launches += 2;
        ++stats.deep_levels;
        group_base_ += max_groups;
        check(cudaMemcpyAsync(hctl_, ctl_.p, 32, cudaMemcpyDeviceToHost, c.s), "d2h");
        sync(c.s, "msd level");
        std::memcpy(ctl, hctl_, 32);
        if (ctl[0] & kFlagOverflow) throw Error{RTK_INTERNAL, "device work list overflow"};
        nslots = list == 0 ? ctl[4] : ctl[3];
        list ^= 1;
        src_buf ^= 1;
    }
    ctl[0] |= sticky;
}

// ---------------------------------------------------------------------------------------
// Exact path (rows whose sampled threshold missed): radix passes over the input with the
// paper's early stop, until #{K >= T} <= target. Mirrors radix_select (engine.hpp:293-312)
// on the composite key, so ties at the pivot are resolved by index inside the same loop.
// ---------------------------------------------------------------------------------------
void Engine::fallback(const uint32_t* d_base, const InputSrc& src, const std::vector<RowReq>& rows,
                      const std::vector<uint32_t>& fb, Call& c, cudaStream_t s) {
    std::vector<uint64_t>& cand_off = c.cand_off;
    uint64_t& cand_total = c.cand_total;
    const uint64_t base_words = reinterpret_cast<uintptr_t>(d_base) / elem_bytes(src.dtype);
    const int R = static_cast<int>(rows.size());
    std::vector<uint32_t> active = fb;
    {
        std::vector<uint64_t> k, target;
        for (uint32_t r : fb) {
            k.push_back(rows[r].k);
            target.push_back(std::min(rows[r].n, rows[r].k + std::max<uint64_t>(8192, rows[r].k / 16)));
        }
        Plan P;
        const size_t o_rid = P.add(fb), o_k = P.add(k), o_t = P.add(target);
        uint8_t* D = upload(P, s);
        launch_init_sel(static_cast<int>(fb.size()), at<uint32_t>(D, o_rid), at<uint64_t>(D, o_k),
                        at<uint64_t>(D, o_t), sel_.as<RowSel>(), s);
        ++stats.kernel_launches;
    }
    check(cudaMemsetAsync(ghist_.p, 0, 8ull * kBins * R, s), "memset");
    // Device-driven passes (radix_select's loop, engine.hpp:293-312): the at most six digit
    // windows of the 64-bit composite are launched back to back with no host round trip; each
    // pass skips rows that already resolved (RowSel::status, set by the pass's last CTA with the
    // early stop count_ge <= target), so only one readback follows all of them.
    {
        std::vector<uint64_t> off, len, tiles{0};
        std::vector<uint32_t> lead;
        for (uint32_t r : active) {
            off.push_back(rows[r].in_off);
            len.push_back(rows[r].n);
            lead.push_back(static_cast<uint32_t>((base_words + rows[r].in_off) & 7));
            tiles.push_back(tiles.back() + ceil_div(lead.back() + rows[r].n, kTile));
        }
        Plan P;
        const size_t o_rid = P.add(active), o_off = P.add(off), o_len = P.add(len),
                     o_lead = P.add(lead), o_tile = P.add(tiles);
        uint8_t* D = upload(P, s);
        Rows rr{static_cast<int>(active.size()), at<uint32_t>(D, o_rid), at<uint64_t>(D, o_off), at<uint64_t>(D, o_len),
                at<uint32_t>(D, o_lead), at<uint64_t>(D, o_tile)};
        for (int pass = 0; pass < 6; ++pass) {
            launch_radix_pass(0, tiles.back(), rr, src, nullptr, sel_.as<RowSel>(), ghist_.as<unsigned long long>(), s);
            ++stats.kernel_launches;
        }
    }
    std::vector<RowSel> st(R);
    std::vector<uint64_t> T(R);
    check(cudaMemcpyAsync(st.data(), sel_.p, sizeof(RowSel) * R, cudaMemcpyDeviceToHost, s), "d2h");
    check(cudaMemcpyAsync(T.data(), T_.p, 8 * R, cudaMemcpyDeviceToHost, s), "d2h");
    sync(s, "exact path passes");
    for (uint32_t r : active) {
        if (st[r].status == 2) throw Error{RTK_INVARIANT_VIOLATION, "select_bin: rank outside histogram total"};
        if (st[r].status != 1) throw Error{RTK_INVARIANT_VIOLATION, "radix select did not resolve"};
        stats.passes += st[r].passes;
        stats.elements_scanned += rows[r].n * st[r].passes;
        row_passes_[r] += st[r].passes;
    }

    // thresholds are full composites now; candidates get fresh regions at the buffer end
    std::vector<uint64_t> expect(R, 0);
    std::vector<uint64_t> off, len, tiles{0};
    std::vector<uint32_t> lead;
    for (uint32_t r : fb) {
        T[r] = st[r].T;
        expect[r] = st[r].count_ge;
        cand_off[r] = (cand_total + 3) & ~uint64_t(3);
        c.cap[r] = expect[r];
        cand_total = cand_off[r] + expect[r];
        off.push_back(rows[r].in_off);
        len.push_back(rows[r].n);
        lead.push_back(static_cast<uint32_t>((base_words + rows[r].in_off) & 7));
        tiles.push_back(tiles.back() + ceil_div(lead.back() + rows[r].n, kTile));
        stats.elements_scanned += rows[r].n;
    }
    cand_a_.ensure(8 * cand_total, /*keep=*/true, s);
    cand_b_.ensure(8 * cand_total, /*keep=*/false, s);
    check(cudaMemcpyAsync(T_.p, T.data(), 8 * R, cudaMemcpyHostToDevice, s), "h2d");
    Plan P;
    const size_t o_rid = P.add(fb), o_off = P.add(off), o_len = P.add(len), o_lead = P.add(lead),
                 o_tile = P.add(tiles), o_coff = P.add(cand_off), o_cap = P.add(c.cap);
    uint8_t* D = upload(P, s);
    c.d_cap = at<uint64_t>(D, o_cap);
    c.d_coff = at<uint64_t>(D, o_coff);
    for (uint32_t r : fb) {
        check(cudaMemsetAsync(count_.as<uint64_t>() + r, 0, 8, s), "memset");
        check(cudaMemsetAsync(kmin_.as<uint64_t>() + r, 0xFF, 8, s), "memset");
        check(cudaMemsetAsync(kmax_.as<uint64_t>() + r, 0, 8, s), "memset");
        check(cudaMemsetAsync(kor_.as<uint32_t>() + r, 0, 4, s), "memset");
        check(cudaMemsetAsync(row_fail_.as<uint32_t>() + r, 0, 4, s), "memset");
        check(cudaMemsetAsync(done_.as<uint32_t>() + r, 0, 4, s), "memset");
    }
    // control words: flags = 0, slot lists empty, work = groups so far; the level-0 MSD's grid
    // barrier restarts from 0 (the main path's MSD may have returned before its barrier — a row
    // whose plan failed has an empty slot — so the device count need not match bar_gen_)
    check(cudaMemsetAsync(ctl_.p, 0, 4, s), "memset");
    check(cudaMemsetAsync(ctl_.as<uint32_t>() + 3, 0, 8, s), "memset");
    check(cudaMemsetAsync(ctl_.as<uint32_t>() + 7, 0, 4, s), "memset");
    bar_gen_ = 0;
    check(cudaMemcpyAsync(ctl_.as<uint32_t>() + 2, ctl_.as<uint32_t>() + 1, 4, cudaMemcpyDeviceToDevice, s), "work");
    check(cudaMemcpyAsync(ctl_.as<uint32_t>() + 6, ctl_.as<uint32_t>() + 5, 4, cudaMemcpyDeviceToDevice, s), "wwork");
    for (uint32_t r : fb) ++row_passes_[r];  // the re-compaction reads the row once more
    FinishPrep fp = prepare_finish(c, fb);
    check(cudaMemsetAsync(seg_hist_.p, 0, 4ull * kBins * fb.size(), s), "memset");
    check(cudaMemsetAsync(seg_ticket_.p, 0, 4ull * fb.size(), s), "memset");
    Rows rr{static_cast<int>(fb.size()), at<uint32_t>(D, o_rid), at<uint64_t>(D, o_off),
            at<uint64_t>(D, o_len), at<uint32_t>(D, o_lead), at<uint64_t>(D, o_tile)};
    in_fallback_ = true;
    const PlanArgs fpa = plan_args(c, fp);
    in_fallback_ = false;
    launch_compact(tiles.back(), rr, src, T_.as<uint64_t>(), cand_a_.as<uint64_t>(),
                   c.d_coff, c.d_cap, count_.as<unsigned long long>(),
                   kmin_.as<unsigned long long>(), kmax_.as<unsigned long long>(), fpa, s);
    ++stats.kernel_launches;
    launch_finish(c, fp);
    std::vector<uint64_t> count(R);
    check(cudaMemcpyAsync(count.data(), count_.p, 8 * R, cudaMemcpyDeviceToHost, s), "d2h");
    sync(s, "fallback compact");
    for (uint32_t r : fb)
        if (count[r] != expect[r] || count[r] < rows[r].k)
            throw Error{RTK_INVARIANT_VIOLATION, "filter: candidate count disagrees with the selected pivot"};
}

// ---------------------------------------------------------------------------------------
std::vector<uint64_t> Engine::first_digit_hist(const uint32_t* d_in, uint64_t n, unsigned d,
                                               int smallest, cudaStream_t s) {
    DeviceGuard dg(device_);
    const uint64_t nb = uint64_t(1) << d;
    DevBuf& h = io_aux;
    h.ensure(8 * nb);
    check(cudaMemsetAsync(h.p, 0, 8 * nb, s), "memset");
    const uint64_t base_words = reinterpret_cast<uintptr_t>(d_in) / 4;
    std::vector<uint32_t> rid{0}, lead{static_cast<uint32_t>(base_words & 7)};
    std::vector<uint64_t> off{0}, len{n}, tiles{0, ceil_div(lead[0] + n, kTile)};
    Plan P;
    const size_t o_rid = P.add(rid), o_off = P.add(off), o_len = P.add(len), o_lead = P.add(lead),
                 o_tile = P.add(tiles);
    uint8_t* D = upload(P, s);
    Rows rr{1, at<uint32_t>(D, o_rid), at<uint64_t>(D, o_off), at<uint64_t>(D, o_len),
            at<uint32_t>(D, o_lead), at<uint64_t>(D, o_tile)};
    InputSrc src{d_in, kF32, smallest, 0, 0.0f, nullptr};
    launch_first_digit_hist(tiles.back(), rr, src, d, h.as<unsigned long long>(), s);
    std::vector<uint64_t> out(nb);
    check(cudaMemcpyAsync(out.data(), h.p, 8 * nb, cudaMemcpyDeviceToHost, s), "d2h");
    sync(s, "first digit hist");
    release_retired();
    return out;
}

void Engine::enqueue_scale_decide(const uint32_t* d_in, uint64_t n, uint64_t k, unsigned d, int smallest,
                                  int mode, double tau, uint64_t a_index, cudaStream_t s) {
    DeviceGuard dg(device_);
    if (!hscale_) {
        check(cudaHostAlloc(reinterpret_cast<void**>(&hscale_), 16, cudaHostAllocMapped), "cudaHostAlloc");
        std::memset(hscale_, 0, 16);
        check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_hscale_), hscale_, 0), "mapped pointer");
    }
    adapt_buf_.ensure(16);
    const uint64_t nb = uint64_t(1) << d;
    unsigned long long* hist = nullptr;
    if (mode == 2) {
        scale_hist_.ensure(8 * nb);
        hist = scale_hist_.as<unsigned long long>();
        check(cudaMemsetAsync(hist, 0, 8 * nb, s), "memset");
        // one-row plan of the trigger pass in its own buffer (not the call arena, whose pinned
        // staging the next run() may rewrite while this copy is pending); re-sent on change only
        const uint64_t base_words = reinterpret_cast<uintptr_t>(d_in) / 4;
        const uint32_t lead = static_cast<uint32_t>(base_words & 7);
        const uint64_t ntiles = ceil_div(lead + n, kTile);
        if (d_in != scale_plan_in_ || n != scale_plan_n_ || !scale_plan_.p) {
            scale_plan_.ensure(64);
            uint64_t plan[8] = {0, 0, n, lead, 0, ntiles, 0, 0};  // rid | off | len | lead | tiles[2]
            // pageable source: the copy is staged before cudaMemcpyAsync returns
            check(cudaMemcpyAsync(scale_plan_.p, plan, sizeof(plan), cudaMemcpyHostToDevice, s), "plan");
            scale_plan_in_ = d_in;
            scale_plan_n_ = n;
        }
        uint8_t* D = scale_plan_.as<uint8_t>();
        Rows rr{1, at<uint32_t>(D, 0), at<uint64_t>(D, 8), at<uint64_t>(D, 16), at<uint32_t>(D, 24),
                at<uint64_t>(D, 32)};
        InputSrc src{d_in, kF32, smallest, 0, 0.0f, nullptr};
        launch_first_digit_hist(ntiles, rr, src, d, hist, s);
    }
    launch_scale_decide(mode, hist, static_cast<uint32_t>(nb), n, k, tau, d_in, a_index,
                        adapt_buf_.as<uint32_t>(), d_hscale_, s);
}

void Engine::enqueue_scale_guess(const uint32_t* d_in, uint64_t n, uint64_t k, unsigned d, int smallest, double tau,
                                 uint64_t a_index, cudaStream_t s) {
    DeviceGuard dg(device_);
    if (!hscale_) {
        check(cudaHostAlloc(reinterpret_cast<void**>(&hscale_), 16, cudaHostAllocMapped), "cudaHostAlloc");
        std::memset(hscale_, 0, 16);
        check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_hscale_), hscale_, 0), "mapped pointer");
    }
    adapt_buf_.ensure(16);
    launch_scale_guess(d_in, n, k, d, smallest, tau, a_index, adapt_buf_.as<uint32_t>(), d_hscale_, s);
    check(cudaGetLastError(), "scale guess launch");
}

void Engine::scale_result(bool* scaled, float* a_s) const {
    const volatile uint32_t* h = hscale_;
    *scaled = h && h[0] != 0;
    const uint32_t bits = h ? h[1] : 0u;
    std::memcpy(a_s, &bits, 4);
}

void Engine::remap(uint64_t k, const uint64_t* d_cand_idx, const std::vector<uint64_t>& block_start,
                   const std::vector<uint64_t>& shard_base, uint64_t* d_idx, cudaStream_t s) {
    Plan P;
    const size_t o_bs = P.add(block_start), o_sb = P.add(shard_base);
    uint8_t* D = upload(P, s);
    launch_remap_idx(k, d_cand_idx, static_cast<uint32_t>(block_start.size()), at<uint64_t>(D, o_bs),
                     at<uint64_t>(D, o_sb), d_idx, s);
    check(cudaGetLastError(), "remap launch");
    // stream-ordered, no host synchronisation: the next plan upload waits for this one's pinned
    // staging to be consumed before it rewrites it (upload())
    if (!pin_ev_) check(cudaEventCreateWithFlags(&pin_ev_, cudaEventDisableTiming), "event");
    check(cudaEventRecord(pin_ev_, s), "event");
    pin_ev_pending_ = true;
}

}  // namespace rtk_b200
