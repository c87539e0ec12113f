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
#include <cmath>
#include <cstring>

#include "rtk_kernels.h"

namespace rtk_b200 {

namespace {

constexpr uint64_t kSmallSort = 4096;   // largest group one CTA sorts in shared memory
constexpr uint64_t kGroupPack = 2048;   // consecutive small buckets are packed up to this

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
    if (keep && p && cap) {
        check(cudaMemcpyAsync(np, p, cap, cudaMemcpyDeviceToDevice, s), "grow copy");
        check(cudaStreamSynchronize(s), "grow sync");
    }
    if (p) cudaFree(p);
    p = np;
    cap = ncap;
}

void DevBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
}

Engine::Engine(int device) : device_(device) {}

Engine::~Engine() {
    for (auto& e : ev_)
        if (e) cudaEventDestroy(e);
    for (DevBuf* b : {&arena_, &sel_, &T_, &count_, &kmin_, &kmax_, &ghist_, &samples_, &cand_a_,
                      &cand_b_, &seg_hist_, &gcursor_, &io_in, &io_vals, &io_idx,
                      &io_piv, &io_aux})
        b->release();
}

uint8_t* Engine::upload(const Plan& p, cudaStream_t s) {
    const size_t need = (p.bytes.size() + 255) & ~size_t(255);
    if (arena_used_ + need > arena_.cap) {
        // earlier plan regions may still be referenced by queued kernels and by pointers the
        // caller holds: retire the old arena (freed at the end of the call), start a new one
        if (arena_.p) retired_.push_back(arena_);
        arena_ = DevBuf{};
        arena_.ensure(std::max<size_t>(need * 2, size_t(4) << 20));
        arena_used_ = 0;
    }
    uint8_t* d = arena_.as<uint8_t>() + arena_used_;
    arena_used_ += need;
    if (!p.bytes.empty())
        check(cudaMemcpyAsync(d, p.bytes.data(), p.bytes.size(), cudaMemcpyHostToDevice, s), "plan upload");
    return d;
}

void Engine::release_retired() {
    for (DevBuf& b : retired_) b.release();
    retired_.clear();
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
void Engine::run(const uint32_t* d_base, int dtype, int smallest, bool scaled, float a_s,
                 bool gather, const std::vector<RowReq>& rows, uint32_t* d_vals, uint64_t* d_idx,
                 uint32_t* d_pivots, cudaStream_t s) {
    check(cudaSetDevice(device_), "cudaSetDevice");
    arena_used_ = 0;
    stats = rtk_stats{};
    const int R = static_cast<int>(rows.size());
    if (R == 0) return;
    if (!ev_[0]) {
        for (auto& e : ev_) check(cudaEventCreate(&e), "cudaEventCreate");
    }
    check(cudaEventRecord(ev_[0], s), "event");
    InputSrc src{d_base, dtype, smallest, scaled ? 1 : 0, a_s};
    const uint64_t base_words = reinterpret_cast<uintptr_t>(d_base) / 4;

    // ---- 1. per-row plan: sample size s, sample rank r', candidate capacity -------------
    std::vector<uint32_t> rid(R), lead(R), sampled(R);
    std::vector<uint64_t> off(R), len(R), tile_start(R + 1, 0), cand_off(R), cap(R), row_k(R),
        row_out(R), row_in(R);
    std::vector<uint32_t> s_rid;
    std::vector<uint64_t> s_inoff, s_n, s_soff, s_len, s_tile{0}, s_nseg{0}, s_k, s_target;
    std::vector<uint32_t> s_lead;
    uint64_t cand_total = 0, sample_total = 0;
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
        bool samp = q.k < q.n && q.n >= 2 * kSmallSort;
        uint64_t ns = 0, rp = 0;
        if (samp) {
            ns = std::min<uint64_t>(uint64_t(1) << 18, std::max<uint64_t>(2048, q.n / 64)) & ~uint64_t(31);
            const double rr = static_cast<double>(q.k) * static_cast<double>(ns) / static_cast<double>(q.n);
            rp = static_cast<uint64_t>(std::ceil(rr + 4.0 * std::sqrt(rr) + 3.0));
            if (rp >= ns / 2) samp = false;
        }
        sampled[r] = samp;
        if (samp) {
            const double ratio = static_cast<double>(q.n) / static_cast<double>(ns);
            cap[r] = std::min<uint64_t>(q.n, static_cast<uint64_t>(ratio * (2.0 * rp + 16.0)) + 1024);
            s_rid.push_back(r);
            s_inoff.push_back(q.in_off);
            s_n.push_back(q.n);
            s_soff.push_back(sample_total);
            s_len.push_back(ns);
            s_lead.push_back(0);  // sample regions are 32-element aligned
            s_tile.push_back(s_tile.back() + ceil_div(ns, kTile64));
            s_nseg.push_back(s_nseg.back() + ns / 32);
            s_k.push_back(rp);
            s_target.push_back(rp + rp / 10 + 8);
            sample_total += ns;
        } else {
            cap[r] = q.n;
        }
        cand_off[r] = cand_total;
        cand_total += cap[r];
        stats.elements_scanned += q.n + ns;
    }
    const int RS = static_cast<int>(s_rid.size());

    sel_.ensure(sizeof(RowSel) * R);
    T_.ensure(8 * R);
    count_.ensure(8 * R);
    kmin_.ensure(8 * R);
    kmax_.ensure(8 * R);
    ghist_.ensure(8ull * kBins * std::max(RS, R));
    samples_.ensure(8 * std::max<uint64_t>(sample_total, 1));
    cand_a_.ensure(8 * std::max<uint64_t>(cand_total, 1));

    Plan P;
    const size_t o_rid = P.add(rid), o_off = P.add(off), o_len = P.add(len), o_lead = P.add(lead),
                 o_tile = P.add(tile_start), o_coff = P.add(cand_off), o_cap = P.add(cap),
                 o_k = P.add(row_k), o_out = P.add(row_out), o_in = P.add(row_in),
                 o_sampled = P.add(sampled), o_srid = P.add(s_rid), o_sin = P.add(s_inoff),
                 o_sn = P.add(s_n), o_soff = P.add(s_soff), o_slen = P.add(s_len),
                 o_stile = P.add(s_tile), o_snseg = P.add(s_nseg), o_sk = P.add(s_k),
                 o_starget = P.add(s_target), o_slead = P.add(s_lead);
    uint8_t* D = upload(P, s);

    check(cudaMemsetAsync(count_.p, 0, 8 * R, s), "memset");
    check(cudaMemsetAsync(kmin_.p, 0xFF, 8 * R, s), "memset");
    check(cudaMemsetAsync(kmax_.p, 0, 8 * R, s), "memset");
    check(cudaMemsetAsync(ghist_.p, 0, 8ull * kBins * std::max(RS, R), s), "memset");

    if (RS > 0) {
        launch_init_sel(RS, at<uint32_t>(D, o_srid), at<uint64_t>(D, o_sk), at<uint64_t>(D, o_starget),
                        sel_.as<RowSel>(), s);
        Rows gather_rows{RS, at<uint32_t>(D, o_srid), at<uint64_t>(D, o_sin), at<uint64_t>(D, o_sn),
                         nullptr, nullptr};
        launch_sample_gather(s_nseg.back(), gather_rows, src, at<uint64_t>(D, o_soff),
                             at<uint64_t>(D, o_snseg), samples_.as<uint64_t>(), s);
        Rows srows{RS, at<uint32_t>(D, o_srid), at<uint64_t>(D, o_soff), at<uint64_t>(D, o_slen),
                   at<uint32_t>(D, o_slead), at<uint64_t>(D, o_stile)};
        for (int pass = 0; pass < 3; ++pass)
            launch_radix_pass(1, s_tile.back(), srows, src, samples_.as<uint64_t>(), sel_.as<RowSel>(),
                              ghist_.as<unsigned long long>(), s);
        stats.kernel_launches += 5;
    }
    launch_set_threshold(R, at<uint32_t>(D, o_rid), at<uint32_t>(D, o_sampled), sel_.as<RowSel>(),
                         T_.as<uint64_t>(), s);
    Rows all{R, at<uint32_t>(D, o_rid), at<uint64_t>(D, o_off), at<uint64_t>(D, o_len),
             at<uint32_t>(D, o_lead), at<uint64_t>(D, o_tile)};
    check(cudaEventRecord(ev_[1], s), "event");
    launch_compact(tile_start.back(), all, src, T_.as<uint64_t>(), cand_a_.as<uint64_t>(),
                   at<uint64_t>(D, o_coff), at<uint64_t>(D, o_cap), count_.as<unsigned long long>(),
                   kmin_.as<unsigned long long>(), kmax_.as<unsigned long long>(), s);
    check(cudaEventRecord(ev_[2], s), "event");
    stats.kernel_launches += 2;

    std::vector<uint64_t> count(R), kmin(R), kmax(R);
    check(cudaMemcpyAsync(count.data(), count_.p, 8 * R, cudaMemcpyDeviceToHost, s), "d2h");
    check(cudaMemcpyAsync(kmin.data(), kmin_.p, 8 * R, cudaMemcpyDeviceToHost, s), "d2h");
    check(cudaMemcpyAsync(kmax.data(), kmax_.p, 8 * R, cudaMemcpyDeviceToHost, s), "d2h");
    sync(s, "compact");

    // ---- 3. verify the sampled thresholds; exact path for the rows that missed -----------
    std::vector<uint32_t> fb;
    for (int r = 0; r < R; ++r)
        if (count[r] < row_k[r] || count[r] > cap[r]) fb.push_back(r);
    if (!fb.empty()) {
        stats.fallback_rows = fb.size();
        fallback(d_base, src, rows, fb, cand_off, count, kmin, kmax, cand_total, s);
    }
    for (int r = 0; r < R; ++r) stats.candidates += count[r];

    // ---- 4. order candidates and gather the first k ------------------------------------
    finish(src, gather, rows, cand_off, count, kmin, kmax, cand_total, at<uint64_t>(D, o_k),
           at<uint64_t>(D, o_out), at<uint64_t>(D, o_in), d_vals, d_idx, s);
    if (d_pivots) {
        launch_pivots(R, at<uint64_t>(D, o_out), at<uint64_t>(D, o_k), d_vals, d_pivots, s);
        ++stats.kernel_launches;
    }
    check(cudaEventRecord(ev_[3], s), "event");
    sync(s, "finish");
    release_retired();
    cudaEventElapsedTime(&stats.compact_ms, ev_[1], ev_[2]);
    cudaEventElapsedTime(&stats.total_ms, ev_[0], ev_[3]);
}

// ---------------------------------------------------------------------------------------
// Exact path (rows whose sampled threshold missed): radix passes over the input with the
// paper's early stop, until #{K >= T} <= target. Mirrors radix_select (engine.hpp:293-312)
// on the composite key, so ties at the pivot are resolved by index inside the same loop.
// ---------------------------------------------------------------------------------------
void Engine::fallback(const uint32_t* d_base, const InputSrc& src, const std::vector<RowReq>& rows,
                      const std::vector<uint32_t>& fb, std::vector<uint64_t>& cand_off,
                      std::vector<uint64_t>& count, std::vector<uint64_t>& kmin,
                      std::vector<uint64_t>& kmax, uint64_t& cand_total, cudaStream_t s) {
    const uint64_t base_words = reinterpret_cast<uintptr_t>(d_base) / 4;
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
    std::vector<RowSel> st(R);
    for (int pass = 0; pass < 6 && !active.empty(); ++pass) {
        const int RA = static_cast<int>(active.size());
        std::vector<uint64_t> off, len, tiles{0};
        std::vector<uint32_t> lead;
        for (uint32_t r : active) {
            off.push_back(rows[r].in_off);
            len.push_back(rows[r].n);
            lead.push_back(static_cast<uint32_t>((base_words + rows[r].in_off) & 7));
            tiles.push_back(tiles.back() + ceil_div(lead.back() + rows[r].n, kTile));
            stats.elements_scanned += rows[r].n;
        }
        Plan P;
        const size_t o_rid = P.add(active), o_off = P.add(off), o_len = P.add(len),
                     o_lead = P.add(lead), o_tile = P.add(tiles);
        uint8_t* D = upload(P, s);
        Rows rr{RA, at<uint32_t>(D, o_rid), at<uint64_t>(D, o_off), at<uint64_t>(D, o_len),
                at<uint32_t>(D, o_lead), at<uint64_t>(D, o_tile)};
        launch_radix_pass(0, tiles.back(), rr, src, nullptr, sel_.as<RowSel>(),
                          ghist_.as<unsigned long long>(), s);
        ++stats.passes;
        ++stats.kernel_launches;
        check(cudaMemcpyAsync(st.data(), sel_.p, sizeof(RowSel) * R, cudaMemcpyDeviceToHost, s), "d2h");
        sync(s, "fallback pass");
        std::vector<uint32_t> still;
        for (uint32_t r : active) {
            if (st[r].status == 2) throw Error{RTK_INVARIANT_VIOLATION, "select_bin: rank outside histogram total"};
            if (st[r].status == 0) still.push_back(r);
        }
        active.swap(still);
    }
    if (!active.empty()) throw Error{RTK_INVARIANT_VIOLATION, "radix select did not resolve"};

    // thresholds are full composites now; candidates get fresh regions at the buffer end
    std::vector<uint64_t> T(R);
    check(cudaMemcpyAsync(T.data(), T_.p, 8 * R, cudaMemcpyDeviceToHost, s), "d2h");
    sync(s, "T");
    std::vector<uint64_t> cap(R, 0), expect(R, 0);
    std::vector<uint64_t> off, len, tiles{0};
    std::vector<uint32_t> lead;
    for (uint32_t r : fb) {
        T[r] = st[r].T;
        expect[r] = st[r].count_ge;
        cand_off[r] = cand_total;
        cap[r] = expect[r];
        cand_total += expect[r];
        off.push_back(rows[r].in_off);
        len.push_back(rows[r].n);
        lead.push_back(static_cast<uint32_t>((base_words + rows[r].in_off) & 7));
        tiles.push_back(tiles.back() + ceil_div(lead.back() + rows[r].n, kTile));
        stats.elements_scanned += rows[r].n;
    }
    cand_a_.ensure(8 * cand_total, /*keep=*/true, s);
    check(cudaMemcpyAsync(T_.p, T.data(), 8 * R, cudaMemcpyHostToDevice, s), "h2d");
    Plan P;
    const size_t o_rid = P.add(fb), o_off = P.add(off), o_len = P.add(len), o_lead = P.add(lead),
                 o_tile = P.add(tiles), o_coff = P.add(cand_off), o_cap = P.add(cap);
    uint8_t* D = upload(P, s);
    for (uint32_t r : fb) {
        check(cudaMemsetAsync(count_.as<uint64_t>() + r, 0, 8, s), "memset");
        check(cudaMemsetAsync(kmin_.as<uint64_t>() + r, 0xFF, 8, s), "memset");
        check(cudaMemsetAsync(kmax_.as<uint64_t>() + r, 0, 8, s), "memset");
    }
    Rows rr{static_cast<int>(fb.size()), at<uint32_t>(D, o_rid), at<uint64_t>(D, o_off),
            at<uint64_t>(D, o_len), at<uint32_t>(D, o_lead), at<uint64_t>(D, o_tile)};
    launch_compact(tiles.back(), rr, src, T_.as<uint64_t>(), cand_a_.as<uint64_t>(),
                   at<uint64_t>(D, o_coff), at<uint64_t>(D, o_cap), count_.as<unsigned long long>(),
                   kmin_.as<unsigned long long>(), kmax_.as<unsigned long long>(), s);
    ++stats.kernel_launches;
    check(cudaMemcpyAsync(count.data(), count_.p, 8 * R, cudaMemcpyDeviceToHost, s), "d2h");
    check(cudaMemcpyAsync(kmin.data(), kmin_.p, 8 * R, cudaMemcpyDeviceToHost, s), "d2h");
    check(cudaMemcpyAsync(kmax.data(), kmax_.p, 8 * R, cudaMemcpyDeviceToHost, s), "d2h");
    sync(s, "fallback compact");
    for (uint32_t r : fb)
        if (count[r] != expect[r] || count[r] < rows[r].k)
            throw Error{RTK_INVARIANT_VIOLATION, "filter: candidate count disagrees with the selected pivot"};
}

// ---------------------------------------------------------------------------------------
// Ordering + gather (normalize_result engine.hpp:402-420 fused with filter's output).
// ---------------------------------------------------------------------------------------
void Engine::finish(const InputSrc& src, bool gather, const std::vector<RowReq>& rows,
                    const std::vector<uint64_t>& cand_off, const std::vector<uint64_t>& count,
                    const std::vector<uint64_t>& kmin, const std::vector<uint64_t>& kmax,
                    uint64_t cand_total, const uint64_t* d_row_k, const uint64_t* d_row_out_off,
                    const uint64_t* d_row_in_off, uint32_t* d_vals, uint64_t* d_idx,
                    cudaStream_t s) {
    struct Seg {
        uint64_t off;
        uint64_t len;
        uint32_t rid;
        uint64_t rank_base;
        uint32_t pos;
    };
    SortGroups g{};
    g.row_k = d_row_k;
    g.row_out_off = d_row_out_off;
    g.row_in_off = d_row_in_off;
    g.in_base = src.base;
    g.out_vals = d_vals;
    g.out_idx = d_idx;
    g.gather = gather ? 1 : 0;
    g.dtype = src.dtype;
    g.smallest = src.smallest;

    auto launch_groups = [&](std::vector<SortGroup>& groups, const uint64_t* buf) {
        if (groups.empty()) return;
        std::sort(groups.begin(), groups.end(),
                  [](const SortGroup& a, const SortGroup& b) { return a.len < b.len; });
        Plan P;
        const size_t o = P.add(groups);
        uint8_t* D = upload(P, s);
        const SortGroup* dg = at<SortGroup>(D, o);
        size_t i = 0;
        for (uint64_t cls : {uint64_t(1024), uint64_t(2048), kSmallSort}) {
            size_t j = i;
            while (j < groups.size() && groups[j].len <= cls) ++j;
            if (j > i) {
                SortGroups gg = g;
                gg.groups = dg + i;
                gg.buf = reinterpret_cast<const unsigned long long*>(buf);
                launch_sort_groups(static_cast<int>(cls), static_cast<int>(j - i), gg, s);
                ++stats.kernel_launches;
            }
            i = j;
        }
    };

    std::vector<SortGroup> groups;
    std::vector<Seg> segs;
    for (size_t r = 0; r < rows.size(); ++r) {
        const uint64_t m = count[r];
        if (m <= kSmallSort) {
            groups.push_back(SortGroup{cand_off[r], static_cast<uint32_t>(m), static_cast<uint32_t>(r), 0});
        } else {
            const uint64_t x = kmin[r] ^ kmax[r];
            const int hb = 63 - __builtin_clzll(x ? x : 1);
            segs.push_back(Seg{cand_off[r], m, static_cast<uint32_t>(r), 0,
                               static_cast<uint32_t>(hb >= 10 ? hb - 10 : 0)});
        }
    }
    launch_groups(groups, cand_a_.as<uint64_t>());
    if (segs.empty()) return;

    cand_b_.ensure(8 * std::max<uint64_t>(cand_total, 1));
    uint64_t* cur = cand_a_.as<uint64_t>();
    uint64_t* nxt = cand_b_.as<uint64_t>();
    while (!segs.empty()) {
        const int NS = static_cast<int>(segs.size());
        std::vector<uint32_t> sid(NS), pos(NS), lead(NS);
        std::vector<uint64_t> off(NS), len(NS), tiles(NS + 1, 0);
        for (int j = 0; j < NS; ++j) {
            sid[j] = j;
            pos[j] = segs[j].pos;
            off[j] = segs[j].off;
            len[j] = segs[j].len;
            lead[j] = static_cast<uint32_t>(segs[j].off & 3);  // both buffers are 256-B aligned
            tiles[j + 1] = tiles[j] + ceil_div(segs[j].len + lead[j], kTile64);
        }
        seg_hist_.ensure(4ull * kBins * NS);
        gcursor_.ensure(4ull * kBins * NS);
        Plan P;
        const size_t o_sid = P.add(sid), o_pos = P.add(pos), o_off = P.add(off), o_len = P.add(len),
                     o_tile = P.add(tiles), o_lead = P.add(lead);
        uint8_t* D = upload(P, s);
        Rows sr{NS, at<uint32_t>(D, o_sid), at<uint64_t>(D, o_off), at<uint64_t>(D, o_len),
                at<uint32_t>(D, o_lead), at<uint64_t>(D, o_tile)};
        check(cudaMemsetAsync(seg_hist_.p, 0, 4ull * kBins * NS, s), "memset");
        check(cudaMemsetAsync(gcursor_.p, 0, 4ull * kBins * NS, s), "memset");
        launch_seg_hist(tiles.back(), sr, at<uint32_t>(D, o_pos), cur, seg_hist_.as<uint32_t>(), s);
        ++stats.kernel_launches;
        std::vector<uint32_t> hist(static_cast<size_t>(kBins) * NS);
        check(cudaMemcpyAsync(hist.data(), seg_hist_.p, 4ull * kBins * NS, cudaMemcpyDeviceToHost, s), "d2h");
        sync(s, "seg hist");

        std::vector<uint32_t> bstart(static_cast<size_t>(kBins) * NS, ~0u);
        std::vector<Seg> next;
        groups.clear();
        for (int j = 0; j < NS; ++j) {
            const Seg& sg = segs[j];
            const uint64_t kr = rows[sg.rid].k;
            const uint32_t* h = hist.data() + static_cast<size_t>(j) * kBins;
            uint32_t* bs = bstart.data() + static_cast<size_t>(j) * kBins;
            uint64_t cum = 0;
            bool open = false;
            SortGroup cg{};
            for (int b = kBins - 1; b >= 0; --b) {
                const uint64_t c = h[b];
                if (!c) continue;
                const uint64_t start_rank = sg.rank_base + cum;
                if (start_rank >= kr) break;
                bs[b] = static_cast<uint32_t>(cum);
                if (c <= kSmallSort) {
                    if (open && cg.len + c <= kGroupPack) {
                        cg.len += static_cast<uint32_t>(c);
                    } else {
                        if (open) groups.push_back(cg);
                        cg = SortGroup{sg.off + cum, static_cast<uint32_t>(c), sg.rid, start_rank};
                        open = true;
                    }
                } else {
                    if (open) groups.push_back(cg);
                    open = false;
                    next.push_back(Seg{sg.off + cum, c, sg.rid, start_rank, sg.pos >= 11 ? sg.pos - 11 : 0});
                }
                cum += c;
            }
            if (open) groups.push_back(cg);
        }
        Plan P2;
        const size_t o_bs = P2.add(bstart);
        uint8_t* D2 = upload(P2, s);
        launch_seg_scatter(tiles.back(), sr, at<uint32_t>(D, o_pos), cur, nxt, at<uint32_t>(D2, o_bs),
                           gcursor_.as<uint32_t>(), s);
        ++stats.kernel_launches;
        launch_groups(groups, nxt);
        segs.swap(next);
        std::swap(cur, nxt);
        if (!segs.empty()) sync(s, "msd level");
    }
}

// ---------------------------------------------------------------------------------------
std::vector<uint64_t> Engine::first_digit_hist(const uint32_t* d_in, uint64_t n, unsigned d,
                                               int smallest, cudaStream_t s) {
    check(cudaSetDevice(device_), "cudaSetDevice");
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
    InputSrc src{d_in, kF32, smallest, 0, 0.0f};
    launch_first_digit_hist(tiles.back(), rr, src, d, h.as<unsigned long long>(), s);
    std::vector<uint64_t> out(nb);
    check(cudaMemcpyAsync(out.data(), h.p, 8 * nb, cudaMemcpyDeviceToHost, s), "d2h");
    sync(s, "first digit hist");
    release_retired();
    return out;
}

void Engine::remap(uint64_t k, const uint64_t* d_cand_idx, const std::vector<uint64_t>& block_start,
                   const std::vector<uint64_t>& shard_base, uint64_t* d_idx, cudaStream_t s) {
    Plan P;
    const size_t o_bs = P.add(block_start), o_sb = P.add(shard_base);
    uint8_t* D = upload(P, s);
    launch_remap_idx(k, d_cand_idx, static_cast<uint32_t>(block_start.size()), at<uint64_t>(D, o_bs),
                     at<uint64_t>(D, o_sb), d_idx, s);
    sync(s, "remap");
    release_retired();
}

}  // namespace rtk_b200
