// rtk_plan.cuh — per-row plan after the compaction (device side, single thread).
#pragma once
#include "rtk_device.cuh"
#include "rtk_kernels.h"

namespace rtk_b200 {

// m = #{K >= T}: m < k or overflow -> exact path; m <= kSortCap -> one sort group;
// larger -> an MSD slot whose first (fine, 11..14-bit) digit is the top of K - kmin over the
// range kmax - kmin.
__device__ __forceinline__ void plan_row(int j, uint32_t r, const PlanArgs& pa, uint64_t n) {
    const uint64_t m = __ldcg(pa.count + r);
    SegSlot sl{pa.cand_off[r], 0, 0, r, 0, 0, 0};
    if (m < pa.row_k[r] || m > pa.cap[r] || pa.force_fail) {
        pa.row_fail[r] = 1;
        atomicOr(pa.flags, kFlagFail);
    } else if (m <= kSortCap) {
        const uint32_t g = atomicAdd(pa.groups.count, 1u);
        pa.groups.groups[g] = SortGroup{pa.cand_off[r], static_cast<uint32_t>(m), r, 0, 0, 0};
    } else {
        const unsigned long long kmin = __ldcg(pa.kmin + r);
        sl.base = kmin;
        // every candidate key is congruent to T.hi modulo 2^tz: squeeze those zeros out
        const uint32_t ko = pa.kor ? __ldcg(pa.kor + r) : 0u;
        sl.tz = ko ? static_cast<uint32_t>(__ffs(ko) - 1) : 0u;
        // row indices need only ib bits: the index part of rel(K) is |lo(K) - lo(kmin)| < 2^ib, so
        // the key difference is shifted by ib instead of 32 and the level-0 digit reaches the
        // index bits that split heavy key ties (C4: 8 keys x 2^26 indices)
        sl.ib = n > 1 ? static_cast<uint32_t>(64 - __clzll(n - 1)) : 1u;
        const unsigned long long x = slot_rel(sl, __ldcg(pa.kmax + r));  // range, not XOR
        const int hb = 63 - __clzll(x ? x : 1ull);
        const int bits = static_cast<int>(min(fine_bits(m), pa.max_bits));  // level 0: fine MSD digit
        sl.len = m;
        sl.bits = static_cast<uint32_t>(bits);
        sl.pos = static_cast<uint32_t>(hb >= bits - 1 ? hb - (bits - 1) : 0);
    }
    pa.slots[j] = sl;
}

}  // namespace rtk_b200
