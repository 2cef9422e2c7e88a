// rf_lag_common.cuh — pieces shared by the persistent TMEM-lag kernels
// (rf_ring_lag.cu: loss + dlogits; rf_ring_kl.cu: the same with the exact-KL
// reference row): A/B build knobs, barrier waits, the softmax-partial rescale
// factor and the tcgen05 tensor-memory helpers.
#pragma once
#include <cuda_runtime.h>

#include "rf_device.cuh"

namespace rf {

namespace {

// Lanes of each scalar warp taking part in the per-row combine (32: shuffle
// tree; 1: lane 0 alone).  Build-time knob for A/B runs (make variant).
#ifndef RF_SCALAR_LANES
#define RF_SCALAR_LANES 1
#endif
constexpr int kScalarLanes = RF_SCALAR_LANES;
// Producer back-off while the ring is full (ns; 0 = spin) and the consumers' wait
// flavour (1 = try_wait with a suspend-time hint, 0 = spin) — A/B knobs.
#ifndef RF_PROD_SLEEP_NS
#define RF_PROD_SLEEP_NS 256
#endif
#ifndef RF_CONS_SUSPEND
#define RF_CONS_SUSPEND 1
#endif
__device__ __forceinline__ void cons_wait(uint32_t bar, uint32_t parity) {
    if (RF_CONS_SUSPEND)
        mbar_wait_sleep(bar, parity);
    else
        mbar_wait(bar, parity);
}
// Support-warp waits (producer empty slots, scalar partials): 1 = suspend-hint
// try_wait, 0 = nanosleep polling (each poll costs issue slots on a consumer SMSP).
#ifndef RF_SUPPORT_SUSPEND
#define RF_SUPPORT_SUSPEND 1  // A/B on B200: +2% over 128 ns polling
#endif
__device__ __forceinline__ void support_wait(uint32_t bar, uint32_t parity, uint32_t ns) {
    if (RF_SUPPORT_SUSPEND)
        mbar_wait_sleep(bar, parity);
    else
        mbar_wait_backoff(bar, parity, ns);
}
// Parking e_t in TMEM: 0 = all columns then wait::st before streaming row t+1;
// 1 = same stores, wait deferred to just before write_row(t); 2 = stores
// interleaved with row t+1's copy-in (chunk by chunk), wait before write_row(t).
#ifndef RF_PARK_MODE
#define RF_PARK_MODE 2  // A/B on B200: +1.5% over 0, +1% over 1
#endif
// Rescale factor 2^(m - mx) (m <= mx, log2 domain) of a partial softmax sum when
// partials are combined.  RF_FAST_COMBINE (A/B knob): 1 = MUFU ex2 of the exact
// (fp64) difference, relative error ~2^-22 — the class of every element's own
// ex2.approx — instead of a ~200-cycle fp64 exp2 on the per-row critical path.
#ifndef RF_FAST_COMBINE
#define RF_FAST_COMBINE 1  // A/B on B200: +6.3% (the per-lane fp64 exp2 sat on every warp's row path)
#endif
__device__ __forceinline__ double combine_factor(float m, float mx) {
    const double d = static_cast<double>(m) - static_cast<double>(mx);
    if (RF_FAST_COMBINE) return static_cast<double>(ex2_approx(static_cast<float>(d)));
    return exp2(d);
}
// Per-thread softmax sum: 0 = every vector's fp32 sum folded into fp64 (a 25-deep
// F2F + DADD chain), 1 = four fp32 chains folded once (A/B knob).
#ifndef RF_SUM_F32
#define RF_SUM_F32 0
#endif
// Cluster exchange of the CTA partials: 1 = st.async + complete_tx on the peer's
// mbarrier (no fence, no polling); 0 = sequence words with st.release / ld.acquire
// polling (each poll invalidates L1, each release fences) — A/B knob.
#ifndef RF_XCHG_MBAR
#define RF_XCHG_MBAR 0
#endif
#ifndef RF_XCHG_TAG
#define RF_XCHG_TAG 0  // 1: fence-free tagged 64-bit words (see rf_ring_lag.cu)
#endif
#ifndef RF_XCHG_SPIN
#define RF_XCHG_SPIN 0  // exchange wait: 1 = try_wait polling with a 32 ns back-off
#endif
// Scalar lane fences its previous row's global output stores before waiting for the
// next partials, so the exchange's release fence finds nothing outstanding (A/B knob).
#ifndef RF_PREFENCE
#define RF_PREFENCE 0
#endif
// Peer-partial poll: 1 = relaxed loads + one acquire fence after the last (an acquire
// load invalidates L1 on every poll); 0 = ld.acquire per poll (A/B knob).
#ifndef RF_XCHG_RELAXED_POLL
#define RF_XCHG_RELAXED_POLL 0
#endif
// Write phase: straight-line stores for chunks with no padded / missing vectors.
#ifndef RF_WRITE_FAST
#define RF_WRITE_FAST 1  // A/B on B200: +6% (per-vector branches serialised the store math)
#endif

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

}  // namespace

}  // namespace rf
