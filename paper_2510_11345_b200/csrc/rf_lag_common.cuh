// rf_lag_common.cuh — pieces shared by the persistent TMEM-lag kernels
// (rf_ring_lag.cu: loss + dlogits; rf_ring_kl.cu: the same with the exact-KL
// reference row): barrier waits, the softmax-partial rescale factor and the
// tcgen05 tensor-memory helpers.
#pragma once
#include <cuda_runtime.h>

#include "rf_device.cuh"

namespace rf {

namespace {

// Waits.  Consumers and support warps block in mbarrier try_wait with a
// suspend-time hint (measured +2% over nanosleep polling, which costs issue slots
// on the consumers' SMSPs).
__device__ __forceinline__ void cons_wait(uint32_t bar, uint32_t parity) { mbar_wait_sleep(bar, parity); }
__device__ __forceinline__ void support_wait(uint32_t bar, uint32_t parity) { mbar_wait_sleep(bar, parity); }
// Rescale factor 2^(m - mx) (m <= mx, log2 domain) of a partial softmax sum when
// partials are combined: MUFU ex2 of the exact (fp64) difference, relative error
// ~2^-22 — the class of every element's own ex2.approx.  (An fp64 exp2 here sat on
// every warp's per-row critical path: measured 6.3% slower.)
__device__ __forceinline__ double combine_factor(float m, float mx) {
    const double d = static_cast<double>(m) - static_cast<double>(mx);
    return static_cast<double>(ex2_approx(static_cast<float>(d)));
}

__device__ __forceinline__ void tmem_alloc(uint32_t smem_dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_dst), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint4& v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// Two 4-column loads and the wait that makes them usable; the loaded registers are
// threaded through the wait so no consumer can be scheduled above it.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint4& a, uint4& b) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%8];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4, %5, %6, %7}, [%9];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
        : "r"(taddr), "r"(taddr + 4)
        : "memory");
}
// N consecutive 4-column loads (N 16-byte vectors of this thread) and one wait.
template <int N>
__device__ __forceinline__ void tmem_ld_vecs(uint32_t taddr, uint4* e) {
    static_assert(N >= 1 && N <= 5, "1..5 vectors per call");

    if constexpr (N == 1) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n\t"
            "tcgen05.wait::ld.sync.aligned;"
            : "=r"(e[0].x), "=r"(e[0].y), "=r"(e[0].z), "=r"(e[0].w)
            : "r"(taddr)
            : "memory");
    } else if constexpr (N == 2) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%8];\n\t"
            "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4, %5, %6, %7}, [%9];\n\t"
            "tcgen05.wait::ld.sync.aligned;"
            : "=r"(e[0].x), "=r"(e[0].y), "=r"(e[0].z), "=r"(e[0].w), "=r"(e[1].x), "=r"(e[1].y), "=r"(e[1].z),
              "=r"(e[1].w)
            : "r"(taddr), "r"(taddr + 4)
            : "memory");
    } else if constexpr (N == 3) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%12];\n\t"
            "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4, %5, %6, %7}, [%13];\n\t"
            "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%8, %9, %10, %11}, [%14];\n\t"
            "tcgen05.wait::ld.sync.aligned;"
            : "=r"(e[0].x), "=r"(e[0].y), "=r"(e[0].z), "=r"(e[0].w), "=r"(e[1].x), "=r"(e[1].y), "=r"(e[1].z),
              "=r"(e[1].w), "=r"(e[2].x), "=r"(e[2].y), "=r"(e[2].z), "=r"(e[2].w)
            : "r"(taddr), "r"(taddr + 4), "r"(taddr + 8)
            : "memory");
    } else if constexpr (N == 4) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15}, [%16];\n\t"
            "tcgen05.wait::ld.sync.aligned;"
            : "=r"(e[0].x), "=r"(e[0].y), "=r"(e[0].z), "=r"(e[0].w), "=r"(e[1].x), "=r"(e[1].y), "=r"(e[1].z),
              "=r"(e[1].w), "=r"(e[2].x), "=r"(e[2].y), "=r"(e[2].z), "=r"(e[2].w), "=r"(e[3].x), "=r"(e[3].y),
              "=r"(e[3].z), "=r"(e[3].w)
            : "r"(taddr)
            : "memory");
    } else {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15}, [%20];\n\t"
            "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%16, %17, %18, %19}, [%21];\n\t"
            "tcgen05.wait::ld.sync.aligned;"
            : "=r"(e[0].x), "=r"(e[0].y), "=r"(e[0].z), "=r"(e[0].w), "=r"(e[1].x), "=r"(e[1].y), "=r"(e[1].z),
              "=r"(e[1].w), "=r"(e[2].x), "=r"(e[2].y), "=r"(e[2].z), "=r"(e[2].w), "=r"(e[3].x), "=r"(e[3].y),
              "=r"(e[3].z), "=r"(e[3].w), "=r"(e[4].x), "=r"(e[4].y), "=r"(e[4].z), "=r"(e[4].w)
            : "r"(taddr), "r"(taddr + 16)
            : "memory");
    }

}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint4& a) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w)
        : "r"(taddr)
        : "memory");
}

// ---------------------------------------------------------------------------
// Row queue: the rows a CTA processes, in order.  Entry k (k-th row of this CTA) is
// rowq[k % kRowQ] (a token index, or -1 = no more rows), published by completing
// phase k / kRowQ of the count-1 mbarrier bar_rq[k % kRowQ]; the producer, the
// consumer warps and the scalar warps all read it with rq_get.  A cluster's rank-0
// producer publishes into every CTA of the cluster (DSMEM store + remote arrive), so
// all ranks walk the same rows.  Rows are claimed dynamically from a per-launch
// counter (the first row of each cluster is its id, later rows ncl + atomicAdd), so a
// cluster on a faster SM pair takes more rows than one on a slower pair instead of
// every cluster getting T / ncl rows (measured per-cluster row times differ by up to
// 6% in K2 and 18% in the 4-CTA exact-KL groups: profiles/r02_ncu/*_cta_spans.txt).
// Safe as long as no reader trails the publisher by kRowQ rows (the ring of
// TMA slots and the one-row lag bound the distance to ~3).
constexpr uint32_t kRowQ = 8;
constexpr uint32_t kRowLookahead = 2;  // rows published ahead of the row being loaded

__device__ __forceinline__ int64_t rq_get(const int64_t* rowq, uint32_t bar_rq, uint32_t k) {
    const uint32_t bar = bar_rq + 8 * (k % kRowQ), par = (k / kRowQ) & 1;
    uint32_t ok;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(par), "r"(1000000u)
            : "memory");
    } while (!ok);
    return *reinterpret_cast<const volatile int64_t*>(rowq + (k % kRowQ));
}

// Publish entry k = t in CTA `dst` of the cluster (dst == own rank: a local store + arrive).
__device__ __forceinline__ void rq_put(int64_t* rowq, uint32_t bar_rq, uint32_t k, int64_t t, uint32_t dst,
                                       uint32_t own) {
    const uint32_t slot = smem_u32(rowq + (k % kRowQ)), bar = bar_rq + 8 * (k % kRowQ);
    if (dst == own) {
        asm volatile("st.shared.s64 [%0], %1;" ::"r"(slot), "l"(t) : "memory");
        mbar_arrive(bar);
    } else {
        asm volatile("st.shared::cluster.s64 [%0], %1;" ::"r"(mapa(slot, dst)), "l"(t) : "memory");
        mbar_arrive_remote(mapa(bar, dst));
    }
}

// The k-th row of cluster `cid` out of `ncl` (dynamic: k = 0 is cid, later rows are
// claimed from the launch's counter; static: cid + k·ncl), -1 past the end.
__device__ __forceinline__ int64_t rq_claim(const KParams& p, uint32_t k, uint32_t cid, uint32_t ncl) {
    int64_t t;
    if (k == 0)
        t = cid;
    else if (p.row_ctr)
        t = static_cast<int64_t>(ncl) + atomicAdd(p.row_ctr, 1u);
    else
        t = static_cast<int64_t>(cid) + static_cast<int64_t>(k) * ncl;
    return t < p.T ? t : -1;
}

}  // namespace

}  // namespace rf
