// rtk_kernels.h — host-visible launchers of the sm_100a kernels (rtk_kernels.cu).
#pragma once
#include <atomic>
#include <cuda_runtime.h>

#include <cstdint>

#include "rtk_device.cuh"

namespace rtk_b200 {

constexpr uint32_t kSortCap = 2048;    // largest group one CTA sorts in shared memory
constexpr uint32_t kGroupPack = 1024;  // small buckets are packed per quantum of this size
constexpr uint32_t kFlagFail = 1;      // some row's sampled threshold missed (exact path)
constexpr uint32_t kFlagMore = 2;      // some bucket needs a deeper MSD level
constexpr uint32_t kFlagOverflow = 4;  // a device work list overflowed its capacity

struct SampleRows {       // rows whose threshold comes from a stratified sample
    const uint32_t* rid;
    const uint64_t* off;     // input element offset
    const uint64_t* len;     // n
    const uint64_t* nseg;    // 32-element segments sampled
    const uint64_t* k;       // sample rank r'
    const uint64_t* target;  // stop once #{sample K >= T} <= target
    unsigned long long* dbg; // optional phase timestamps (RTK_PROFILE)
};

// End-of-call tail of the LAST kernel of a call (k_sort_groups, or k_rows_fused when a batch
// has only short rows): the last CTA to finish copies ctl[0..7] and ctl[10..13] to mapped
// host memory and then writes a per-launch sequence number to hflags[15] (the host spins on it:
// no memcpy, no stream sync); with R_clean > 0 it also resets the per-call counters of R_clean
// state rows and the control words, so the next call needs no init kernel.
struct CallTail {
    const uint32_t* ctl;
    uint32_t* done_ctr;
    uint32_t* seq_ctr;
    volatile uint32_t* hflags;   // null: no tail
    int R_clean;
    unsigned long long* c_count;
    unsigned long long* c_kmin;
    unsigned long long* c_kmax;
    uint32_t* c_kor;
    uint64_t* c_T;
    uint32_t* c_done;
    uint32_t* c_ticket;
};

#ifdef __CUDACC__
// all threads of every CTA call this at the very end; s_flag is one shared word
__device__ __forceinline__ void call_tail(const CallTail& t, uint32_t* s_flag) {
    if (!t.hflags) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        *s_flag = 0;
        if (atomicAdd(t.done_ctr, 1u) == gridDim.x - 1) {
            __threadfence();
            *t.done_ctr = 0;
            const uint32_t seq = atomicAdd(t.seq_ctr, 1u) + 1;
            const volatile uint32_t* c = t.ctl;
            // ctl[0..7] and the trigger counts ctl[10..13] (what the host reads) as words 0..11 in
            // three 16-byte stores (one PCIe write each), then the sequence word with bit 31 set;
            // when the flags ctl[0] and the trigger counts are zero (the common case; the host
            // reads the other words only under a flag) only the sequence word is written, bit 31
            // clear, and no system fence is needed
            uint32_t w[12], any = 0;
#pragma unroll
            for (int i = 0; i < 12; ++i) {
                w[i] = c[i < 8 ? i : i + 2];
                if (i == 0 || i >= 8) any |= w[i];
            }
            if (any) {
                uint32_t* hf = const_cast<uint32_t*>(t.hflags);
#pragma unroll
                for (int q = 0; q < 3; ++q)
                    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(hf + 4 * q),
                                 "r"(w[4 * q]), "r"(w[4 * q + 1]), "r"(w[4 * q + 2]), "r"(w[4 * q + 3]) : "memory");
                __threadfence_system();
                t.hflags[15] = seq | 0x80000000u;
            } else {
                t.hflags[15] = seq & 0x7FFFFFFFu;
            }
            *s_flag = 1;
        }
    }
    __syncthreads();
    if (*s_flag && t.R_clean > 0) {
        for (int r = threadIdx.x; r < t.R_clean; r += blockDim.x) {
            t.c_count[r] = 0;
            t.c_kmin[r] = ~0ull;
            t.c_kmax[r] = 0;
            t.c_kor[r] = 0;
            t.c_T[r] = 0;
            t.c_done[r] = 0;
            t.c_ticket[r] = 0;
        }
        if (threadIdx.x < 16) const_cast<uint32_t*>(t.ctl)[threadIdx.x] = 0;
    }
}
#endif

struct RowsFusedArgs {    // K6 fast path: one CTA per short row (rtk_rows.cu)
    const uint32_t* rid;
    const uint64_t* off;
    const uint64_t* len;
    const uint64_t* k;
    InputSrc in;
    const uint64_t* row_out_off;  // by state row
    uint32_t* out_vals;
    uint64_t* out_idx;
    uint32_t* pivots;             // by state row, nullable
    uint32_t* row_fail;
    uint32_t* flags;
    unsigned long long* dbg;      // optional phase timestamps (RTK_PROFILE)
    CallTail tail;                // set when this is the call's last kernel
    uint32_t pf;                  // L2 prefetch distance of the streaming ring (chunks ahead)
    unsigned long long* trace;    // optional per-CTA phase timestamps [grid][16] (RTK_ROWS_TRACE)
};

struct SortGroup {
    uint64_t off;        // element offset into buffer `buf`
    uint32_t len;        // <= kSortCap
    uint32_t rid;        // state row
    uint32_t buf;        // 0: candidate buffer A, 1: buffer B
    uint32_t pad;
    uint64_t rank_base;  // output rank of the group's first element
};

struct SegSlot {        // one MSD segment; len == 0 means inactive
    uint64_t off;
    uint64_t len;
    uint64_t rank_base;
    uint32_t rid;
    uint32_t pos;        // digit = ((K - base) >> pos) & (2^bits - 1)
    uint32_t bits;       // level 0: 11..14; deeper levels: kDigit
    uint32_t src;        // level 0: 1 = read the INPUT row at in_off (dense row, no compaction)
    uint64_t in_off;     // input element offset of the row (src == 1)
    uint64_t base;       // digit = (rel(K) >> pos) & mask with rel(K) = ((key - key(base)) >> tz) << ib
    uint32_t tz;         //   + (lo(K) - lo(base)): the candidates' RANGE, not their XOR, with the
                         //   key's common trailing zeros squeezed out (order-preserving); tie-heavy
                         //   rows such as C4 split by index bits at level 0. Children inherit all three.
    uint32_t ib;         // index field width: every row index < 2^ib, so |lo(K) - lo(base)| < 2^ib
                         //   and the shifted key difference still dominates (0 = 32)
};

#ifdef __CUDACC__
__device__ __forceinline__ unsigned long long slot_rel(const SegSlot& sl, unsigned long long K) {
    const uint32_t kd = (static_cast<uint32_t>(K >> 32) - static_cast<uint32_t>(sl.base >> 32)) >> sl.tz;
    return (static_cast<unsigned long long>(kd) << (sl.ib ? sl.ib : 32u)) + (K & 0xffffffffull) -
           (sl.base & 0xffffffffull);
}
#endif

struct GroupList {
    SortGroup* groups;
    uint32_t* count;
    uint32_t cap;
};

struct SlotList {
    SegSlot* slots;
    uint32_t* count;
    uint32_t cap;
};

struct SegPlanArgs {      // bucket plan of one MSD level (fused into k_seg_hist)
    uint32_t* ghist;
    uint32_t* gcursor;
    const uint64_t* row_k;
    uint32_t* bstart;
    GroupList groups;
    uint32_t dst_buf;
    SlotList next;
    uint32_t* flags;
    uint32_t* ticket;        // per slot: tiles finished
};

// Level-0 MSD (k_msd_cluster): one thread-block cluster of CS CTAs per slot, chunk c of the
// slot per CTA. Shared-memory histograms of one 2^bits-bin digit; the column scan over the CS
// CTAs runs through distributed shared memory (per-chunk bucket offsets + totals), CTA 0 plans
// the buckets, every CTA scatters its chunk with shared-memory cursors — one kernel, no global
// matrix, no global atomics on the data path. Buckets of <= kWarpGroupMax elements become warp
// groups (tiny/mid ones packed), <= kSortCap CTA groups, larger ones the next (11-bit) level.
constexpr uint32_t kTinyMax = 32;       // packed by 32-quantum  -> warp group <= 63
constexpr uint32_t kMidMax = 128;       // packed by 128-quantum -> warp group <= 255
constexpr uint32_t kWarpGroupMax = 256; // solo warp group up to this size
constexpr int kMsdMaxBits = 14;
struct FineArgs {
    InputSrc in;             // dense rows (slot.src == 1) are read from the input directly
    const uint64_t* row_k;
    GroupList groups;        // CTA groups
    GroupList wgroups;       // warp groups (<= kWarpGroupMax)
    SlotList next;
    uint32_t* flags;
    unsigned long long* dbg; // optional phase timestamps (RTK_PROFILE)
    // multi-cluster mode (Q > 1): ONE slot over Q co-resident clusters (cooperative launch),
    // cluster totals exchanged through ctot (Q x 2^bits) after one grid barrier
    uint32_t Q;
    uint32_t* ctot;
    uint32_t* bar;           // grid barrier counter (monotonic within a call)
    uint32_t bar_target;
};

// digit bits of the level-0 MSD for m candidates (device: m; host: the capacity bound)
__host__ __device__ inline uint32_t fine_bits(uint64_t m) {
    return m <= 16384 ? 11u : (m <= (uint64_t(1) << 18) ? 13u : 14u);
}
// cluster size for the largest slot of a launch
inline int msd_cluster_size(uint64_t max_cap) {
    int cs = 2;
    while (cs < 16 && static_cast<uint64_t>(cs) * 16384 < max_cap) cs <<= 1;
    return cs;
}

struct PlanArgs {         // per-row plan after the compaction (fused into k_compact)
    const uint64_t* cap;
    const uint64_t* row_k;
    const uint64_t* cand_off;
    const unsigned long long* count;
    const unsigned long long* kmin;
    const unsigned long long* kmax;
    uint32_t* kor;           // per state row: OR of (key ^ T.hi) over the candidates (digit stride)
    SegSlot* slots;          // indexed by launch row
    GroupList groups;
    uint32_t* flags;
    uint32_t* row_fail;
    uint32_t* done;          // per state row: tiles finished
    uint32_t max_bits;       // cap on the level-0 MSD digit (RTK_MSD_BITS; default kMsdMaxBits)
    uint32_t prefetch_mb;    // L2 prefetch budget of k_compact's prologue (RTK_PREFETCH_MB)
    uint32_t sparse_max;     // warp-tiles with <= this many hits take the set-bits (L2 re-read) path
    uint32_t sparse_sel;     // set-bits path takes the key from registers (select tree), no re-read
    uint32_t* dyn_ctr;       // [2] dynamic-tail tile counter + CTAs done (self-resetting); null = static
    uint32_t dyn_per_cta;    // dynamic-tail tiles per CTA of the grid
    uint32_t contig;         // 1: contiguous tile runs per CTA (many-row batches), 0: interleaved
    uint32_t force_fail;     // test switch "force_exact": every row takes the exact path
    uint32_t trig;           // count the speculative Adaptive trigger (k_scale_guess) into flags[10..13]
};

struct SortArgs {
    GroupList groups;
    uint32_t* work;
    GroupList wgroups;       // warp-sized groups (<= kWarpGroupMax)
    uint32_t* wwork;
    const unsigned long long* buf0;
    const unsigned long long* buf1;
    const uint64_t* row_k;
    const uint64_t* row_out_off;
    const uint64_t* row_in_off;   // gather mode only
    const uint32_t* in_base;      // gather mode only
    uint32_t* out_vals;
    uint64_t* out_idx;
    uint32_t* pivots;        // per state row, nullable
    int gather;
    int dtype;
    int smallest;
    CallTail tail;           // completion signal + self-cleaning (see CallTail)
};

// One-time setup per DEVICE (kernel attributes such as the dynamic shared-memory limit are
// per device, and handles may live on any device of the process). Idempotent work only: two
// threads racing on the first call may both run it.
struct DeviceOnce {
    std::atomic<uint64_t> done{0};
    template <typename F>
    void operator()(F&& f) {
        int dev = 0;
        cudaGetDevice(&dev);
        const uint64_t bit = uint64_t(1) << (dev & 63);
        if (done.load(std::memory_order_acquire) & bit) return;
        f();
        done.fetch_or(bit, std::memory_order_release);
    }
};

inline int num_sms() {
    static std::atomic<int> sms[64];
    int dev = 0;
    cudaGetDevice(&dev);
    int v = sms[dev & 63].load(std::memory_order_relaxed);
    if (!v) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (v <= 0) v = 148;
        sms[dev & 63].store(v, std::memory_order_relaxed);
    }
    return v;
}

template <typename K>
inline int persistent_grid(K kernel, int threads, size_t smem, uint64_t tiles) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
    if (occ <= 0) occ = 1;
    const uint64_t g = static_cast<uint64_t>(occ) * num_sms();
    return static_cast<int>(tiles < g ? (tiles ? tiles : 1) : g);
}

void launch_init_sel(int R, const uint32_t* rid, const uint64_t* k, const uint64_t* target,
                     RowSel* sel, cudaStream_t s);
void launch_radix_pass(int src, uint64_t tiles, const Rows& rows, const InputSrc& in,
                       const uint64_t* buf, RowSel* sel, unsigned long long* ghist, cudaStream_t s);
void launch_init_call(int R, unsigned long long* count, unsigned long long* kmin, unsigned long long* kmax,
                      uint32_t* kor, uint64_t* T, uint32_t* row_fail, uint32_t* ctl, uint32_t* seg_hist, uint32_t* done,
                      uint32_t* seg_ticket, cudaStream_t s);
void launch_sample_select(int rows, int cs, uint32_t per_cta, const SampleRows& sr, const InputSrc& in,
                          uint64_t* T, cudaStream_t s);
void launch_compact(uint64_t tiles, const Rows& rows, const InputSrc& in, const uint64_t* T,
                    uint64_t* cand, const uint64_t* cand_off, const uint64_t* cap,
                    unsigned long long* count, unsigned long long* kmin, unsigned long long* kmax,
                    const PlanArgs& pa, cudaStream_t s);
void launch_seg_hist(uint64_t tiles, const SegSlot* slots, int nslots, const uint64_t* tile_start,
                     const uint64_t* src, const SegPlanArgs& pa, cudaStream_t s);
void launch_seg_scatter(uint64_t tiles, const SegSlot* slots, int nslots, const uint64_t* tile_start,
                        const uint64_t* src, uint64_t* dst, const uint32_t* bstart, uint32_t* gcursor,
                        cudaStream_t s);
int msd_max_clusters(int cs);  // co-resident clusters of cs CTAs (occupancy API)
// returns false if a multi-cluster (fa.Q > 1) cooperative launch was refused
bool launch_msd_cluster(int nslots, int cs, const SegSlot* slots, const uint64_t* src, uint64_t* dst,
                        const FineArgs& fa, cudaStream_t s);
void launch_sort_groups(uint32_t max_groups, const SortArgs& g, cudaStream_t s);
void launch_pivots(int R, const uint64_t* row_out_off, const uint64_t* row_k, const uint32_t* vals,
                   uint32_t* pivots, cudaStream_t s);
void launch_first_digit_hist(uint64_t tiles, const Rows& rows, const InputSrc& in, unsigned int d,
                             unsigned long long* ghist, cudaStream_t s);
struct LsdArgs {  // dense rows: segmented one-sweep LSD radix sort (rtk_lsd.cu)
    int R;                        // rows of this launch
    const uint64_t* tile_start;   // [R + 1] 4096-element tiles per row, prefix
    const uint64_t* len;          // elements per row
    const uint64_t* in_off;       // row start in the input (elements)
    const uint64_t* buf_off;      // row start in the ping-pong buffers
    const uint64_t* k;
    const uint64_t* out_off;
    const uint32_t* rid;          // state row (pivots)
    uint32_t* hist;               // [R][4][256] digit counts (zeroed per call)
    unsigned long long* status;   // [tiles][256] look-back words (epoch-tagged, never reset)
    uint32_t* ctr;                // [0..3] tile counters (zeroed per call), [4] epoch
    unsigned long long* src;      // pass p > 0 input (swapped per pass by the launcher)
    unsigned long long* dst;
    InputSrc in;
    uint32_t* out_vals;
    uint64_t* out_idx;
    uint32_t* pivots;
    CallTail tail;                // last pass only
    uint32_t npass;               // 4 (32-bit keys) or 2 (16-bit keys: low half constant)
    uint32_t shift0;              // 0 or 16
    unsigned long long* trace;    // RTK_LSD_TRACE: [pass][tile][8] phase timestamps, nullable
    const uint32_t* order;        // claim index -> row-major tile id (round-robin over rows), nullable
};
uint32_t lsd_tile();
void launch_lsd(uint64_t tiles, const LsdArgs& a, cudaStream_t s);
void launch_rows_fused(int R, const RowsFusedArgs& a, bool small, cudaStream_t s);
// one long row (2^18 < n <= 2^21, k <= row_cluster_kmax()) on one 16-CTA cluster (rtk_rows.cu)
void launch_row_cluster(const RowsFusedArgs& a, cudaStream_t s);
uint32_t row_cluster_kmax();
uint32_t rows_fused_kmax(bool small);
uint32_t rows_fused_cand(bool small);
uint32_t rows_fused_sample(bool small);
void launch_philox_uniform(float* out, uint64_t n, uint64_t seed, uint64_t offset, float a, float b,
                           cudaStream_t s);
void launch_sample_rows(uint64_t rows, const void* vals, int fmt, const uint64_t* idx, uint64_t k, float top_p,
                        float temperature, const float* uniform, uint64_t* token, float* probs, cudaStream_t s);
void launch_scale_guess(const uint32_t* x, uint64_t n, uint64_t k, uint32_t d, int smallest, double tau,
                        uint64_t a_index, uint32_t* out, volatile uint32_t* host_out, cudaStream_t s);
void launch_scale_decide(int mode, const unsigned long long* hist, uint32_t nbins, uint64_t n, uint64_t k,
                         double tau, const uint32_t* x, uint64_t a_index, uint32_t* out,
                         volatile uint32_t* host_out, cudaStream_t s);
void launch_remap_idx(uint64_t n, const uint64_t* cand_idx, uint32_t nblocks,
                      const uint64_t* block_start, const uint64_t* shard_base, uint64_t* idx,
                      cudaStream_t s);

}  // namespace rtk_b200
