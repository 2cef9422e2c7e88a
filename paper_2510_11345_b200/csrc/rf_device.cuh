// rf_device.cuh — sm_100a device helpers: mbarrier / bulk-copy (TMA) / cluster
// PTX wrappers, packed bf16/f16 conversion, and the per-token surrogate math
// (reference semantics, fp64).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "rf_offpolicy.h"

namespace rf {

// ---------------------------------------------------------------------------
// Kernel parameter block (passed by value as a __grid_constant__).
// ---------------------------------------------------------------------------
struct KParams {
    // loss config (= LossConfig, losses.hpp:28-41)
    int32_t variant, aggregation;
    double clip_eps, eps_low, eps_high, trunc_cap, kl_weight, w_plus, w_minus, mismatch_cap;
    // batch
    int64_t T;
    int32_t V;
    int32_t logp_f64;  // per-token log-prob arrays are fp64 (else f32)
    const void* logits;
    int64_t row_stride;
    const void* ref_logits;
    int64_t ref_row_stride;
    const int32_t* row_of_token;
    const int32_t* token_ids;
    const int32_t* seq_of_token;
    const int64_t* seq_offsets;
    const double* advantages;
    const void* behavior_logp;
    const void* prox_logp;
    const void* engine_logp;
    int32_t normalization;
    double inv_n;  // 1 / N_global
    double inv_t;  // 1 / T_global
    double grad_sign;
    // outputs
    void* dlogits;
    int64_t dl_stride;
    double* token_logp;
    double* token_ratio;
    double* token_coef;
    double* token_loss;
    uint8_t* token_flags;
    int32_t* status;
    double* partials;  // [num partial slots][RF_NUM_SCALARS]
    // sequence_product / two-pass support (workspace)
    double* tok_lse;   // [T] lse per token (stats pass output / write pass input)
    double* tok_klx;   // [T] KL per token (kl mode)
    double* tok_lseq;  // [T] ref lse per token (kl mode)
    // ring geometry
    int32_t slice_vecs;   // 16-byte vectors per cluster rank
    int32_t row_vecs;     // 16-byte vectors per row (padded)
    int32_t nchunks;      // chunks per slice
    int32_t nslots;       // ring slots
    int32_t mode;         // 0 = fused loss+dlogits, 1 = stats only (lse/lp), 2 = write with known lse/coef
    unsigned long long* dbg;  // optional per-phase cycle counters (RF_DEBUG_COUNTERS), else nullptr
    // exact-KL kernel with CTA groups exchanging through L2 instead of a hardware cluster
    void* xch;                 // [groups][4 row slots][8 ranks] exchange slots (workspace)
    int32_t vcs;               // CTAs per group (0 = hardware cluster)
    // lag kernels: per-launch row counter (zeroed before the launch) for dynamic row
    // claims; nullptr = static rows cid + k·ncl
    unsigned int* row_ctr;
};

// Per-phase cycle counters are compiled in only for the profiling build
// (make PHASE=1 -> librf_offpolicy_phase.so).
#ifndef RF_PHASE_COUNTERS
#define RF_PHASE_COUNTERS 0
#endif
constexpr bool kPhaseCounters = RF_PHASE_COUNTERS != 0;

// Protocol-checked build (make checked -> librf_offpolicy_checked.so, load with
// RF_LIB_VARIANT=checked): every cross-warp handoff of the persistent kernels
// carries the token index it belongs to and the receiver traps on a mismatch
// (a partial or coefficient taken from the wrong row, a stale exchange slot, a
// ring phase slip), plus bounds asserts on the computed dlogits vector indices.
// compute-sanitizer is not available on this GPU pool; this build is its stand-in.
#ifndef RF_CHECKED
#define RF_CHECKED 0
#endif
constexpr bool kChecked = RF_CHECKED != 0;
__device__ __forceinline__ void rf_check(bool ok) {
    if (RF_CHECKED && !ok) __trap();
}

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Profiling build: per-CTA record of consumer warp 0, lane 0 in dbg[kDbgCtaTimes + 8·cta + i]:
// {start ns, end ns (%globaltimer), %smid, rows, full-wait, stream, coef-wait, write cycles}.
constexpr int kDbgCtaTimes = 16;
constexpr int kDbgCtaWords = 8;
constexpr int kDbgWords = kDbgCtaTimes + kDbgCtaWords * 1024;
__device__ __forceinline__ void dbg_cta_begin(unsigned long long* dbg) {
    if (blockIdx.x < 1024) dbg[kDbgCtaTimes + kDbgCtaWords * blockIdx.x] = global_ns();
}
__device__ __forceinline__ void dbg_cta_end(unsigned long long* dbg, uint32_t rows, const unsigned long long* dph) {
    if (blockIdx.x >= 1024) return;
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    unsigned long long* w = dbg + kDbgCtaTimes + kDbgCtaWords * blockIdx.x;
    w[1] = global_ns();
    w[2] = smid;
    w[3] = rows;
    w[4] = dph[0];
    w[5] = dph[1];
    w[6] = dph[3];
    w[7] = dph[4];
}

// Debug phase timer: accumulates clock64 deltas into a per-thread slot array.
struct PhaseClock {
    long long t;
    __device__ __forceinline__ void start() { t = clock64(); }
    __device__ __forceinline__ void lap(unsigned long long& acc) {
        const long long n = clock64();
        acc += static_cast<unsigned long long>(n - t);
        t = n;
    }
};

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// Arrive on a barrier in another CTA of the cluster (32-bit shared::cluster address).
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
// Poll with a nanosleep back-off: for single-lane roles (TMA producer, scalar
// warp) that share an SMSP with compute warps and must not steal issue slots.
__device__ __forceinline__ void mbar_wait_backoff(uint32_t bar, uint32_t parity, uint32_t ns) {
    while (!mbar_try_wait(bar, parity)) __nanosleep(ns);
}
// try_wait with a suspend-time hint: the waiting warp sleeps until the phase
// completes (or the hint expires) instead of re-issuing polls.
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(parity), "r"(1000000u)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
    while (!mbar_try_wait_cluster(bar, parity)) {
    }
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// TMA bulk copy global -> this CTA's shared memory, completing on `bar`.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(policy)
        : "memory");
}
// TMA bulk copy this CTA's shared memory -> global (bulk-group completion), L2 evict-first.
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes, uint64_t policy) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"(src), "r"(bytes), "l"(policy)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most N committed bulk groups still read their shared-memory source
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the async proxy (TMA store source)
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void sts128_raw(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void sts16_raw(uint32_t addr, uint16_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t ncluster_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
// Map a local shared address to the same offset in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_f64(uint32_t addr, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
// Asynchronous store into a peer CTA's shared memory that completes `bytes` of the
// transaction count of the peer's mbarrier (both addresses from mapa): no fence, no
// polling — the receiver waits on its local mbarrier.
__device__ __forceinline__ void st_async_f64(uint32_t cluster_addr, double v, uint32_t cluster_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(cluster_addr),
                 "l"(__double_as_longlong(v)), "r"(cluster_bar)
                 : "memory");
}
__device__ __forceinline__ void st_async_f32(uint32_t cluster_addr, float v, uint32_t cluster_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(cluster_addr),
                 "r"(__float_as_uint(v)), "r"(cluster_bar)
                 : "memory");
}
// Release-store to a peer CTA's shared memory / acquire-load of a local word at
// cluster scope (sequence-number handshakes).
__device__ __forceinline__ void st_release_cluster_u32(uint32_t cluster_addr, uint32_t v) {
    asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_cluster_u32(uint32_t cluster_addr, uint32_t v) {
    asm volatile("st.relaxed.cluster.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_cluster_u64(uint32_t cluster_addr, uint64_t v) {
    asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" ::"r"(cluster_addr), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_cluster_u64(uint32_t addr) {
    uint64_t v;
    asm volatile("ld.relaxed.cluster.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_cluster_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.relaxed.cluster.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }
__device__ __forceinline__ uint32_t ld_acquire_cluster_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.acquire.cluster.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
// gpu-scope exchange through L2 (CTA groups without a hardware cluster)
__device__ __forceinline__ void st_relaxed_gpu_f64(double* a, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu_f32(float* a, float v) {
    asm volatile("st.relaxed.gpu.global.f32 [%0], %1;" ::"l"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu_u64(unsigned long long* a, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu_u64(unsigned long long* a, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu_u64(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ double ld_relaxed_gpu_f64(const double* a) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ float ld_relaxed_gpu_f32(const float* a) {
    float v;
    asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(a) : "memory");
    return v;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
// Streaming stores of dlogits.  RF_STORE_HINT (A/B knob): 0 = .cs (evict-first in
// L1 and L2), 1 = .L1::no_allocate (keeps the small L1 next to the smem ring for
// spills / locals).
#ifndef RF_STORE_HINT
#define RF_STORE_HINT 1  // A/B on B200: +1.9% (L1 hit rate of the consumers' spill reloads)
#endif
__device__ __forceinline__ void stg128_cs(void* p, uint4 v) {
    if (RF_STORE_HINT == 1)
        asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
                     "r"(v.z), "r"(v.w)
                     : "memory");
    else
        asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                     : "memory");
}
__device__ __forceinline__ void stg64_cs(void* p, uint2 v) {
    if (RF_STORE_HINT == 1)
        asm volatile("st.global.L1::no_allocate.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
    else
        asm volatile("st.global.cs.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}

// bf16x2 word -> two floats (exact)
__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
    __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack_f16x2(uint32_t w) {
    __half2 h = *reinterpret_cast<__half2*>(&w);
    return __half22float2(h);
}

__device__ __forceinline__ float load_logit(const void* base, int64_t idx, bool bf16) {
    if (bf16) {
        const uint16_t u = reinterpret_cast<const uint16_t*>(base)[idx];
        return __uint_as_float(static_cast<uint32_t>(u) << 16);
    }
    return reinterpret_cast<const float*>(base)[idx];
}
__device__ __forceinline__ double load_logp(const void* p, int64_t t, int32_t f64) {
    return f64 ? reinterpret_cast<const double*>(p)[t] : static_cast<double>(reinterpret_cast<const float*>(p)[t]);
}

// ---------------------------------------------------------------------------
// Per-token surrogate math, reference semantics in fp64 (losses.cpp:262-320).
// Explicit __dmul_rn/__dadd_rn keep nvcc from contracting into FMA where the
// reference's x86 build rounds each operation separately.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double clipd(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }

struct TokenResult {
    double ratio, k, loss;
    uint32_t flags;
};

// po/tp: decoupled_ppo prox/behaviour and theta/prox ratios; logp: lp (token) or
// logp_sum (sequence).  Flags per include/rf_offpolicy.h.  VARIANT >= 0 fixes the
// variant at compile time (a kernel that serves one variant only, e.g. exact-KL GRPO).
template <int VARIANT = -1>
__device__ __forceinline__ void variant_math(const KParams& p, double r, double A, double po, double tp,
                                             double logp, double& value, double& gw, uint32_t& flags) {
    switch (VARIANT >= 0 ? VARIANT : p.variant) {
        case RF_PPO:
        case RF_GRPO: {
            const double c = clipd(r, 1.0 - p.clip_eps, 1.0 + p.clip_eps);
            const double v1 = __dmul_rn(r, A), v2 = __dmul_rn(c, A);
            value = (v2 < v1) ? v2 : v1;  // std::min(v1, v2)
            gw = v1 <= v2 ? v1 : (r == c ? v1 : 0.0);
            if (!(v1 <= v2) && r != c) flags |= RF_FLAG_CLIPPED;
            break;
        }
        case RF_DECOUPLED_PPO: {
            const double c = clipd(tp, 1.0 - p.clip_eps, 1.0 + p.clip_eps);
            const double v1 = __dmul_rn(r, A), v2 = __dmul_rn(__dmul_rn(po, c), A);
            value = (v2 < v1) ? v2 : v1;
            gw = v1 <= v2 ? v1 : (tp == c ? __dmul_rn(__dmul_rn(po, tp), A) : 0.0);
            if (!(v1 <= v2) && tp != c) flags |= RF_FLAG_CLIPPED;
            break;
        }
        case RF_TIS: {
            const double w = clipd(r, 0.0, p.trunc_cap);
            value = __dmul_rn(__dmul_rn(w, A), logp);
            gw = __dmul_rn(w, A);
            if (r < 0.0 || r > p.trunc_cap) flags |= RF_FLAG_CLIPPED;
            break;
        }
        case RF_NAIVE_IS:
            value = __dmul_rn(__dmul_rn(r, A), logp);
            gw = __dmul_rn(r, A);
            break;
        case RF_CISPO: {
            const double lo = 1.0 - p.eps_low, hi = 1.0 + p.eps_high;
            const double w = clipd(r, lo, hi);
            value = __dmul_rn(__dmul_rn(w, A), logp);
            gw = __dmul_rn(w, A);
            if (r < lo || r > hi) flags |= RF_FLAG_CLIPPED;
            break;
        }
        case RF_TOPR: {
            double w;
            if (A > 0.0) {
                w = p.w_plus;
                flags |= RF_FLAG_TOPR_POS;
            } else {
                w = __dmul_rn(p.w_minus, clipd(r, 0.0, p.trunc_cap));
                if (r < 0.0 || r > p.trunc_cap) flags |= RF_FLAG_CLIPPED;
            }
            value = __dmul_rn(__dmul_rn(w, A), logp);
            gw = __dmul_rn(w, A);
            break;
        }
        default:
            value = 0.0;
            gw = 0.0;
    }
}

__device__ __forceinline__ double token_scale_of(const KParams& p, int64_t seq) {
    if (p.normalization == RF_NORM_GLOBAL_TOKEN) return p.inv_t;
    const double len = static_cast<double>(p.seq_offsets[seq + 1] - p.seq_offsets[seq]);
    return p.inv_n / len;
}

// The lp-independent half of the per-token math (loads + the theta-constant
// factors), computed while the row's softmax is still being reduced.
struct TokenPre {
    double b, lq, A, scale, m, po, eb;  // eb = exp(b)
    uint32_t flags;
};

__device__ __forceinline__ TokenPre token_pre(const KParams& p, int64_t t, int64_t seq) {
    TokenPre q;
    q.flags = 0;
    q.b = load_logp(p.behavior_logp, t, p.logp_f64);
    q.eb = exp(q.b);
    q.A = p.advantages[seq];
    q.scale = token_scale_of(p, seq);
    q.m = 1.0;
    if (p.mismatch_cap > 0.0) {  // losses.cpp:170-176
        const double em = exp(q.b - load_logp(p.engine_logp, t, p.logp_f64));
        q.m = (p.mismatch_cap < em) ? p.mismatch_cap : em;
        if (em > p.mismatch_cap) q.flags |= RF_FLAG_MISMATCH_CAPPED;
    }
    q.lq = 0.0;
    q.po = 0.0;
    if (p.variant == RF_DECOUPLED_PPO) {  // losses.cpp:283-284
        q.lq = load_logp(p.prox_logp, t, p.logp_f64);
        q.po = exp(q.lq - q.b);
    }
    return q;
}

// The lp-dependent half (losses.cpp:264-320).  On the scalar lane's critical path:
// with VARIANT fixed, no other variant's work (e.g. decoupled_ppo's second exp) is
// evaluated and discarded; kNotDecoupled = any variant but decoupled_ppo (runtime).
constexpr int kNotDecoupled = -2;
template <int VARIANT = -1>
__device__ __forceinline__ TokenResult token_post(const KParams& p, const TokenPre& q, double lp) {
    TokenResult o;
    o.flags = q.flags;
    const double r = exp(lp - q.b);
    o.ratio = r;
    if (!isfinite(r)) o.flags |= RF_FLAG_NONFINITE;
    const int variant = VARIANT >= 0 ? VARIANT : p.variant;
    const double tp = (VARIANT != kNotDecoupled && variant == RF_DECOUPLED_PPO) ? exp(lp - q.lq) : 0.0;
    double value, gw;
    variant_math<VARIANT>(p, r, q.A, q.po, tp, lp, value, gw, o.flags);
    const double sm = __dmul_rn(q.scale, q.m);
    o.k = __dmul_rn(p.grad_sign, __dmul_rn(sm, gw));
    o.loss = __dmul_rn(sm, value);
    if (o.k == 0.0) o.flags |= RF_FLAG_ZERO_COEF;
    return o;
}

// token_mean per-token math given lp (losses.cpp:262-320).
__device__ __forceinline__ TokenResult token_math(const KParams& p, int64_t t, double lp, int64_t seq) {
    return token_post(p, token_pre(p, t, seq), lp);
}

// Partial-scalar accumulator kept by the thread that owns a partial slot.
struct Partials {
    double v[RF_NUM_SCALARS];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < RF_NUM_SCALARS; ++i) v[i] = 0.0;
    }
    __device__ __forceinline__ void add_token(const TokenResult& r, double kl_scaled) {
        v[RF_SCALAR_LOSS] += r.loss;
        v[RF_SCALAR_TOKENS] += 1.0;
        v[RF_SCALAR_CLIPPED] += (r.flags & RF_FLAG_CLIPPED) ? 1.0 : 0.0;
        v[RF_SCALAR_NONFINITE] += (r.flags & RF_FLAG_NONFINITE) ? 1.0 : 0.0;
        v[RF_SCALAR_ZERO_COEF] += (r.flags & RF_FLAG_ZERO_COEF) ? 1.0 : 0.0;
        v[RF_SCALAR_MISMATCH] += (r.flags & RF_FLAG_MISMATCH_CAPPED) ? 1.0 : 0.0;
        v[RF_SCALAR_KL] += kl_scaled;
        v[RF_SCALAR_COEF_ABS] += fabs(r.k);
    }
    // One token's row of contributions (the lag kernels write one row per token, so the
    // scalars do not depend on which cluster processed which row).
    __device__ __forceinline__ static void store_token(double* dst, const TokenResult& r, double kl_scaled) {
        Partials q;
        q.zero();
        q.add_token(r, kl_scaled);
        q.store(dst);
    }
    __device__ __forceinline__ void store(double* dst) const {
#pragma unroll
        for (int i = 0; i < RF_NUM_SCALARS; ++i) dst[i] = v[i];
    }
};

}  // namespace rf
