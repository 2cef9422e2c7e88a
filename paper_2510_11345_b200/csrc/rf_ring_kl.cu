// rf_ring_kl.cu — K2kl: the fused loss + dlogits kernel for exact-KL GRPO
// (grpo with kl_weight > 0: losses.cpp:118-133 kl_and_grad, used per trajectory at
// :321-326; per token row here, scaled by the token's normalisation like the
// generic path).  The policy row x and the reference row y of every token are
// co-resident: each CTA of a 4-CTA group (Qwen3 vocabulary) holds a quarter of
// both rows in registers, so one HBM read of x and y and one HBM write of the
// dlogits row suffice — 6·V bytes per token.
//
// Same lag structure as rf_ring_lag.cu (TMA ring -> registers, previous row parked
// in TMEM, two scalar warps), extended with the reference row.  The group is a
// cooperative launch's consecutive CTAs exchanging through L2 (GX, default: all
// 148 SMs) or a hardware cluster exchanging through DSMEM (RF_KL_GX=0):
//
//   sweep:  e_v = 2^(x_v·log2e - C), ey_v = 2^(y_v·log2e - Cy), d_v = x_v - y_v
//           S = Σ e, Sy = Σ ey, T = Σ e·d         (per thread, then warp, CTA, cluster)
//   scalar: lse = M + ln S, lseq = My + ln Sy, D = T/S, KL = D - lse + lseq
//           k from the GRPO clip (token_post), kc = -grad_sign·scale·β
//   write:  dlogit_v = p_v·(kc·(d_v - D) - k) (+ k at the sampled token)
//                    = e_v·(A + B·d_v),  A = -f·(k + kc·D),  B = f·kc,  f = 2^(C - lse·log2e)
//
// e and d are parked in TMEM as f16 (2·NVT·4 columns per thread).  Rows are claimed
// at run time (the group's rank 0 posts them to the group's claim ring in L2, or, in a
// hardware cluster, into every rank's shared-memory row queue: rf_lag_common.cuh).
#include <cuda_runtime.h>
#include <math_constants.h>

#include "rf_device.cuh"
#include "rf_kernels.h"
#include "rf_lag_common.cuh"
#include "rf_ring_common.cuh"

namespace rf {

using namespace ring;

namespace {

// vectors per packed fp32 partial before the fp64 fold (measured on B200: 2 is +1.2% over 1; 4 gains nothing)
constexpr int kKlFold = 2;

// Padding of the two rows: a finite bf16 (-1.0e30) instead of -inf, so padded lanes give e = 0 and
// d = 0 (never 0·inf) without a per-element guard in the sweep.
constexpr uint32_t kKlPad2 = 0xF14AF14Au;
constexpr float kKlPadMax = -1.0e29f;  // a slice max at or below this is all padding
__device__ __forceinline__ uint4 pad_vec_here() {  // volatile: not hoisted out of its branch
    uint4 v;
    asm volatile("mov.b32 %0, %4;\n\tmov.b32 %1, %4;\n\tmov.b32 %2, %4;\n\tmov.b32 %3, %4;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "n"(kKlPad2));
    return v;
}
__device__ __forceinline__ void mask_tail_pad(uint4& v, int valid) {
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        if (e >= valid) {
            const int wi = e >> 1;
            w[wi] = (e & 1) ? ((w[wi] & 0x0000ffffu) | (kKlPad2 & 0xffff0000u)) : ((w[wi] & 0xffff0000u) | (kKlPad2 & 0xffffu));
        }
    }
    v = make_uint4(w[0], w[1], w[2], w[3]);
}

// One 8-element vector of x and of y: e (f16x2) replaces x, d = x - y (f16x2)
// replaces y; packed f32x2 partial sums of e, ey and e·d are accumulated.
__device__ __forceinline__ void kl_vec(uint4& vx, uint4& vy, uint64_t L2, uint64_t negC2, uint64_t negCy2,
                                       uint64_t& se, uint64_t& sy, uint64_t& sd) {
    uint32_t wx[4] = {vx.x, vx.y, vx.z, vx.w};
    uint32_t wy[4] = {vy.x, vy.y, vy.z, vy.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint64_t x2 = bf16x2_to_f32x2(wx[q]);
        const uint64_t y2 = bf16x2_to_f32x2(wy[q]);
        const uint64_t a = ffma2(x2, L2, negC2);
        const uint64_t ay = ffma2(y2, L2, negCy2);
        const float e0 = ex2_approx(lo2(a)), e1 = ex2_approx(hi2(a));
        const float f0 = ex2_approx(lo2(ay)), f1 = ex2_approx(hi2(ay));
        // x - y.  Padding is the finite kKlPad in both rows (d = 0, e = 0); a genuine -inf logit
        // makes e·d = 0·inf = NaN, as p·(lp − lq) does in the reference (losses.cpp:127-130).
        const uint64_t dd = fsub2(x2, y2);
        const float d0 = lo2(dd), d1 = hi2(dd);
        const uint64_t e2 = pk2(e0, e1);
        se = q == 0 ? e2 : fadd2(se, e2);
        sy = q == 0 ? pk2(f0, f1) : fadd2(sy, pk2(f0, f1));
        sd = q == 0 ? fmul2(e2, pk2(d0, d1)) : ffma2(e2, pk2(d0, d1), sd);
        wx[q] = pack_f16x2(e0, e1);
        wy[q] = pack_f16x2(d0, d1);
    }
    vx = make_uint4(wx[0], wx[1], wx[2], wx[3]);
    vy = make_uint4(wy[0], wy[1], wy[2], wy[3]);
}

// dlogits of one vector: e·(A + B·d)
template <bool OUT_BF16>
__device__ __forceinline__ void kl_store_vec(uint8_t* dst, const uint4& e, const uint4& d, uint64_t A2, uint64_t B2) {
    const uint32_t we[4] = {e.x, e.y, e.z, e.w};
    const uint32_t wd[4] = {d.x, d.y, d.z, d.w};
    uint64_t o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float2 he = unpack_f16x2(we[q]);
        const float2 hd = unpack_f16x2(wd[q]);
        o[q] = fmul2(pk2(he.x, he.y), ffma2(pk2(hd.x, hd.y), B2, A2));
    }
    if (OUT_BF16) {
        stg128_cs(dst, make_uint4(pack_bf16x2(lo2(o[0]), hi2(o[0])), pack_bf16x2(lo2(o[1]), hi2(o[1])),
                                  pack_bf16x2(lo2(o[2]), hi2(o[2])), pack_bf16x2(lo2(o[3]), hi2(o[3]))));
    } else {
        stg128_cs(dst, make_uint4(static_cast<uint32_t>(o[0]), static_cast<uint32_t>(o[0] >> 32),
                                  static_cast<uint32_t>(o[1]), static_cast<uint32_t>(o[1] >> 32)));
        stg128_cs(dst + 16, make_uint4(static_cast<uint32_t>(o[2]), static_cast<uint32_t>(o[2] >> 32),
                                       static_cast<uint32_t>(o[3]), static_cast<uint32_t>(o[3] >> 32)));
    }
}

template <bool OUT_BF16>
__device__ __forceinline__ void kl_store_partial(uint8_t* dst, const uint4& e, const uint4& d, float A, float B,
                                                 int valid) {
    const uint32_t we[4] = {e.x, e.y, e.z, e.w};
    const uint32_t wd[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float2 he = unpack_f16x2(we[q]);
        const float2 hd = unpack_f16x2(wd[q]);
        const float o0 = he.x * fmaf(hd.x, B, A), o1 = he.y * fmaf(hd.y, B, A);
        if (2 * q < valid) {
            if (OUT_BF16)
                reinterpret_cast<__nv_bfloat16*>(dst)[2 * q] = __float2bfloat16_rn(o0);
            else
                reinterpret_cast<float*>(dst)[2 * q] = o0;
        }
        if (2 * q + 1 < valid) {
            if (OUT_BF16)
                reinterpret_cast<__nv_bfloat16*>(dst)[2 * q + 1] = __float2bfloat16_rn(o1);
            else
                reinterpret_cast<float*>(dst)[2 * q + 1] = o1;
        }
    }
}

__device__ __forceinline__ uint32_t bf16_max_vec(const uint4& v) { return vec_max2<true>(v); }

__device__ __forceinline__ float vmax_row(const uint4* r, int n) {
    uint32_t m2 = bf16_max_vec(r[0]);
    for (int j = 1; j < n; ++j) {
        const uint32_t v2 = bf16_max_vec(r[j]);
        __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&m2);
        __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&v2);
        a = __hmax2(a, b);
        m2 = *reinterpret_cast<uint32_t*>(&a);
    }
    return fmaxf(bf16lo(m2), bf16hi(m2));
}

}  // namespace

// GX: the row's CTAs form a GROUP of p.vcs consecutive blocks of a cooperative
// (all-resident) launch instead of a hardware cluster, and exchange their partials
// through L2.  4-CTA clusters of one-SM CTAs place only 33 clusters (132 of 148
// SMs); 37 groups of 4 use every SM.
struct XSlotG {  // [group][row % 4][sender rank]
    double S, T, Sy;
    float M, My;
    unsigned long long seq;  // row_iter + 1 (the slots are zeroed before every launch)
};

template <bool OUT_BF16, int NCW, int NVT, bool GX>
__global__ void __launch_bounds__((NCW + 4) * 32, 1) ring_kl_kernel(const __grid_constant__ KParams p) {
    constexpr int NCT = NCW * 32;
    constexpr int EPV = 8;  // bf16 logits
    constexpr int VPC = lag_vpc(NVT);
    constexpr int NCH = (NVT + VPC - 1) / VPC;
    constexpr int CHUNK_VECS = NCT * VPC;
    constexpr uint32_t CHUNK_BYTES = CHUNK_VECS * 16;
    constexpr uint32_t SLOT_BYTES = 2 * CHUNK_BYTES;  // x chunk, then y chunk
    constexpr size_t OES = OUT_BF16 ? 2 : 4;
    static_assert(NCW % 4 == 0 && NCW >= 4 && NCW <= 16, "whole consumer warpgroups");
    constexpr uint32_t TCOLS = lag_tmem_cols(NCW);
    static_assert(NVT * 8 <= static_cast<int>(TCOLS), "a thread's e and d values must fit its TMEM columns");
    constexpr int REGS_C = lag_regs_consumer(NCW);

    extern __shared__ __align__(1024) uint8_t smem[];
    const int nslots = p.nslots;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar_full = sbase + nslots * SLOT_BYTES;
    const uint32_t bar_empty = bar_full + nslots * 8;
    const uint32_t bar_red = bar_empty + nslots * 8 + 16;  // [2] consumers -> scalar (row parity)
    const uint32_t bar_bc = bar_red + 16;                   // [2] scalar -> consumers (row parity)
    uint8_t* tail = smem + nslots * SLOT_BYTES + nslots * 16 + 48;
    struct XSlot {  // cluster exchange [row % 4][sender rank], sequence-word guarded
        double S, T, Sy;
        float M, My;
        uint32_t seq, pad;
    };
    static_assert(sizeof(XSlot) == 40, "exchange slot layout");
    XSlot* xslot = reinterpret_cast<XSlot*>(tail);                    // [4][8]: 1280 B
    double* redS = reinterpret_cast<double*>(tail + 1280);            // [2][NCW]
    double* redT = redS + 2 * NCW;                                    // [2][NCW]
    double* redSy = redT + 2 * NCW;                                   // [2][NCW]
    float* redM = reinterpret_cast<float*>(redSy + 2 * NCW);          // [2][NCW]
    float* redMy = redM + 2 * NCW;                                    // [2][NCW]
    struct Bcast {
        double k, tok_val;
        float A, B, lseL;
        int32_t tok;
    };
    Bcast* bcs = reinterpret_cast<Bcast*>(tail + 1280 + 64 * NCW);  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bcs + 2);
    static_assert(1280 + 64 * NCW + 2 * sizeof(Bcast) + 4 <= 2176, "tail layout");
    int64_t* rowq = reinterpret_cast<int64_t*>(tail + 2176);      // [kRowQ] row queue (rf_lag_common.cuh)
    const uint32_t bar_rq = smem_u32(tail + 2240);                 // [kRowQ] its mbarriers
    int64_t* red_tag = reinterpret_cast<int64_t*>(tail + 2304);  // [2][NCW] checked build: row of each partial
    int64_t* bc_tag = red_tag + 32;                               // [2] checked build: row of each broadcast

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    // CTA groups: when the grid covers every SM exactly once (a cooperative launch of one
    // CTA per SM over contiguous SM ids), a group is 4 neighbouring SM ids (the same GPC)
    // rather than 4 consecutive block ids; otherwise block ids.
    uint32_t gslot = blockIdx.x;
    if (GX) {  // measured +0.5% over block-id groups (profiles/r02_ab/kl_smid_groups_ab.txt)
        uint32_t smid, nsmid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        asm volatile("mov.u32 %0, %%nsmid;" : "=r"(nsmid));
        if (nsmid == gridDim.x) gslot = smid;
    }
    const uint32_t rank = GX ? gslot % static_cast<uint32_t>(p.vcs) : cluster_ctarank();
    const uint32_t csize = GX ? static_cast<uint32_t>(p.vcs) : cluster_nctarank();
    const uint32_t cid = GX ? gslot / static_cast<uint32_t>(p.vcs) : cluster_id_x();
    const uint32_t ncl = GX ? gridDim.x / static_cast<uint32_t>(p.vcs) : ncluster_x();
    static_assert(sizeof(XSlotG) == 40 && kKlGroupXchBytes == 32 * 40 + 8 * kRowQ, "group exchange layout");
    XSlotG* xg = GX ? reinterpret_cast<XSlotG*>(static_cast<uint8_t*>(p.xch) + static_cast<size_t>(cid) * kKlGroupXchBytes)
                    : nullptr;

    if (tid == 0) {
        for (int s = 0; s < nslots; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_empty + 8 * s, NCW);
        }
        for (int q = 0; q < 2; ++q) {
            mbar_init(bar_red + 8 * q, NCW);
            mbar_init(bar_bc + 8 * q, 1);
        }
        for (int q = 0; q < 32; ++q) xslot[q].seq = 0u;
        for (uint32_t q = 0; q < kRowQ; ++q) mbar_init(bar_rq + 8 * q, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(smem_u32(tmem_slot), 512);
    tmem_fence_before();
    if (GX)
        __syncthreads();
    else
        cluster_sync_all();
    tmem_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int slice_begin = static_cast<int>(rank) * p.slice_vecs;
    const int slice_len = max(0, min(p.slice_vecs, p.row_vecs - slice_begin));
    const int nchunks = (slice_len + CHUNK_VECS - 1) / CHUNK_VECS;
    const int tail_vec = p.row_vecs - 1;
    const int tail_valid = p.V - tail_vec * EPV;
    const bool has_tail = tail_valid < EPV;

    if (warp >= NCW) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kLagRegsSupport));
        if (warp == NCW) {
            // ------------------------------ TMA producer ------------------------------
            if (lane == 0) {
                const uint64_t pol = l2_evict_first_policy();
                int s = 0;
                uint32_t phase = 0, uses = 0;
                // rank 0 claims the group's rows; a hardware cluster's ranks get them through
                // DSMEM (rq_put), a CTA group's through the group's claim ring in L2: one 64-bit
                // word per entry, (k + 1) << 32 | (t + 1), single-copy atomic, so no fence
                unsigned long long* claim =
                    GX ? reinterpret_cast<unsigned long long*>(xg + 32) : nullptr;  // [kRowQ] after the slots
                uint32_t pub = 0;
                bool ended = false;
                auto publish_upto = [&](uint32_t upto, bool block) {
                    while (!ended && pub < upto) {
                        int64_t tq;
                        if (rank == 0) {
                            tq = rq_claim(p, pub, cid, ncl);
                            if (GX) {
                                st_relaxed_gpu_u64(claim + pub % kRowQ,
                                                   (static_cast<unsigned long long>(pub + 1) << 32) |
                                                       static_cast<uint32_t>(tq + 1));
                                rq_put(rowq, bar_rq, pub, tq, rank, rank);
                            } else {
                                for (uint32_t q = 0; q < csize; ++q) rq_put(rowq, bar_rq, pub, tq, q, rank);
                            }
                        } else if (GX) {
                            unsigned long long w;
                            while (((w = ld_relaxed_gpu_u64(claim + pub % kRowQ)) >> 32) != pub + 1) {
                                if (!block) return;  // look-ahead: the leader has not claimed it yet
                                __nanosleep(64);
                            }
                            tq = static_cast<int64_t>(static_cast<uint32_t>(w)) - 1;
                            rq_put(rowq, bar_rq, pub, tq, rank, rank);
                        } else {
                            return;  // a cluster's rank 0 publishes into this CTA
                        }
                        ++pub;
                        if (tq < 0) {  // the end, twice: the other scalar warp reads the entry after it
                            if (GX)
                                rq_put(rowq, bar_rq, pub, -1, rank, rank);
                            else
                                for (uint32_t q = 0; q < csize; ++q) rq_put(rowq, bar_rq, pub, -1, q, rank);
                            ++pub;
                            ended = true;
                        }
                    }
                };
                for (uint32_t k = 0;; ++k) {
                    publish_upto(k + 1, true);
                    const int64_t t = rq_get(rowq, bar_rq, k);
                    if (t < 0) break;
                    const int64_t row = p.row_of_token ? static_cast<int64_t>(p.row_of_token[t]) : t;
                    const uint8_t* src = reinterpret_cast<const uint8_t*>(p.logits) + (row * p.row_stride) * 2 +
                                         static_cast<size_t>(slice_begin) * 16;
                    const uint8_t* srf = reinterpret_cast<const uint8_t*>(p.ref_logits) +
                                         (row * p.ref_row_stride) * 2 + static_cast<size_t>(slice_begin) * 16;
                    for (int c = 0; c < nchunks; ++c) {
                        if (uses >= static_cast<uint32_t>(nslots)) support_wait(bar_empty + 8 * s, phase);
                        const int nv = min(CHUNK_VECS, slice_len - c * CHUNK_VECS);
                        const uint32_t bytes = static_cast<uint32_t>(nv) * 16;
                        mbar_arrive_expect_tx(bar_full + 8 * s, 2 * bytes);
                        bulk_g2s(sbase + s * SLOT_BYTES, src + static_cast<size_t>(c) * CHUNK_BYTES, bytes,
                                 bar_full + 8 * s, pol);
                        bulk_g2s(sbase + s * SLOT_BYTES + CHUNK_BYTES, srf + static_cast<size_t>(c) * CHUNK_BYTES,
                                 bytes, bar_full + 8 * s, pol);
                        ++uses;
                        if (++s == nslots) {
                            s = 0;
                            if (uses > static_cast<uint32_t>(nslots)) phase ^= 1;
                        }
                    }
                    publish_upto(k + 1 + kRowLookahead, false);
                }
            }
            __syncwarp();
        } else if (warp == NCW + 1 || warp == NCW + 2) {
            // --------------------------------- scalar ---------------------------------
            // The whole warp combines the consumer warps' partials (one warp per lane, shuffle
            // trees); lane 0 alone runs the exchange, the token math and the broadcast.
            const uint32_t which = static_cast<uint32_t>(warp - NCW - 1);
            unsigned long long d_red = 0, d_x = 0, d_math = 0, d_comb = 0, d_post = 0;  // phase counters (profiling build)
            PhaseClock pc;
            pc.start();
            const long long t_begin = pc.t;
            for (uint32_t row_iter = which;; row_iter += 2) {
                const int64_t t = rq_get(rowq, bar_rq, row_iter);  // all lanes
                if (t < 0) break;
                const int64_t row = p.row_of_token ? static_cast<int64_t>(p.row_of_token[t]) : t;
                const int32_t tok = p.token_ids[t];
                const bool tok_ok = tok >= 0 && tok < p.V;
                const float x_tok = tok_ok ? load_logit(p.logits, row * p.row_stride + tok, true) : 0.0f;
                const float y_tok = tok_ok ? load_logit(p.ref_logits, row * p.ref_row_stride + tok, true) : 0.0f;
                const int64_t seq = p.seq_of_token[t];
                const TokenPre pre = token_pre(p, t, seq);
                const uint32_t par = row_iter & 1, ph = (row_iter >> 1) & 1;
                Bcast* bc = bcs + par;
                if (kPhaseCounters && p.dbg) pc.lap(d_math);
                support_wait(bar_red + 8 * par, ph);
                if (kPhaseCounters && p.dbg) pc.lap(d_red);
                if (kChecked && lane < NCW) rf_check(red_tag[par * NCW + lane] == t);
                // CTA partials: lane w holds consumer warp w's, fixed butterfly trees (lane 0's
                // result is the one used; the same on every launch)
                const bool has = lane < NCW;
                const float m_l = has ? redM[par * NCW + lane] : -CUDART_INF_F;
                const float my_l = has ? redMy[par * NCW + lane] : -CUDART_INF_F;
                const double s_l = has ? redS[par * NCW + lane] : 0.0;
                const double t_l = has ? redT[par * NCW + lane] : 0.0;
                const double sy_l = has ? redSy[par * NCW + lane] : 0.0;
                float Mw = m_l, Myw = my_l;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    Mw = fmaxf(Mw, __shfl_xor_sync(0xffffffffu, Mw, o));
                    Myw = fmaxf(Myw, __shfl_xor_sync(0xffffffffu, Myw, o));
                }
                const double f_l = (s_l != 0.0) ? combine_factor(m_l, Mw) : 0.0;
                double Sw = s_l * f_l, Tw = t_l * f_l;
                double Syw = (sy_l != 0.0) ? sy_l * combine_factor(my_l, Myw) : 0.0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    Sw += __shfl_xor_sync(0xffffffffu, Sw, o);
                    Tw += __shfl_xor_sync(0xffffffffu, Tw, o);
                    Syw += __shfl_xor_sync(0xffffffffu, Syw, o);
                }
                if (lane == 0) {
                double Mc = static_cast<double>(Mw), Myc = static_cast<double>(Myw), Sc = Sw, Tc = Tw, Syc = Syw;
                if (kPhaseCounters && p.dbg) pc.lap(d_comb);
                if (GX && csize > 1) {
                    const uint32_t xs = row_iter & 3;
                    XSlotG* mine = xg + xs * 8 + rank;
                    st_relaxed_gpu_f64(&mine->S, Sw);
                    st_relaxed_gpu_f64(&mine->T, Tw);
                    st_relaxed_gpu_f64(&mine->Sy, Syw);
                    st_relaxed_gpu_f32(&mine->M, Mw);
                    st_relaxed_gpu_f32(&mine->My, Myw);
                    const unsigned long long want = row_iter + 1;
                    st_release_gpu_u64(&mine->seq, want);
                    float Mq[8], Myq[8];
                    double Sq[8], Tq[8], Syq[8];
                    float Mx = -CUDART_INF_F, Myx = -CUDART_INF_F;
                    for (uint32_t q = 0; q < csize; ++q) {
                        if (q == rank) {
                            Mq[q] = Mw, Myq[q] = Myw, Sq[q] = Sw, Tq[q] = Tw, Syq[q] = Syw;
                        } else {
                            XSlotG* o = xg + xs * 8 + q;
                            while (ld_acquire_gpu_u64(&o->seq) != want) __nanosleep(32);
                            Mq[q] = ld_relaxed_gpu_f32(&o->M);
                            Myq[q] = ld_relaxed_gpu_f32(&o->My);
                            Sq[q] = ld_relaxed_gpu_f64(&o->S);
                            Tq[q] = ld_relaxed_gpu_f64(&o->T);
                            Syq[q] = ld_relaxed_gpu_f64(&o->Sy);
                        }
                        Mx = fmaxf(Mx, Mq[q]);
                        Myx = fmaxf(Myx, Myq[q]);
                    }
                    Sc = 0.0;
                    Tc = 0.0;
                    Syc = 0.0;
                    for (uint32_t q = 0; q < csize; ++q) {  // rank order: identical on every CTA
                        if (Sq[q] != 0.0) {
                            const double f = combine_factor(Mq[q], Mx);
                            Sc += Sq[q] * f;
                            Tc += Tq[q] * f;
                        }
                        if (Syq[q] != 0.0) Syc += Syq[q] * combine_factor(Myq[q], Myx);
                    }
                    Mc = static_cast<double>(Mx);
                    Myc = static_cast<double>(Myx);
                } else if (csize > 1) {
                    const uint32_t xs = row_iter & 3;
                    XSlot* mine = &xslot[xs * 8 + rank];
                    // payload to every peer, one cluster fence, then the sequence words
                    // (one fence instead of a release per peer)
                    for (uint32_t q = 0; q < csize; ++q) {
                        if (q == rank) continue;
                        st_cluster_f64(mapa(smem_u32(&mine->S), q), Sw);
                        st_cluster_f64(mapa(smem_u32(&mine->T), q), Tw);
                        st_cluster_f64(mapa(smem_u32(&mine->Sy), q), Syw);
                        st_cluster_f32(mapa(smem_u32(&mine->M), q), Mw);
                        st_cluster_f32(mapa(smem_u32(&mine->My), q), Myw);
                    }
                    fence_acq_rel_cluster();
                    for (uint32_t q = 0; q < csize; ++q)
                        if (q != rank) st_relaxed_cluster_u32(mapa(smem_u32(&mine->seq), q), row_iter + 1);
                    for (uint32_t q = 0; q < csize; ++q) {
                        if (q == rank) continue;
                        const uint32_t a = smem_u32(&xslot[xs * 8 + q].seq);
                        while (ld_acquire_cluster_u32(a) != row_iter + 1) __nanosleep(32);
                    }
                    float Mx = -CUDART_INF_F, Myx = -CUDART_INF_F;
                    for (uint32_t q = 0; q < csize; ++q) {
                        Mx = fmaxf(Mx, (q == rank) ? Mw : xslot[xs * 8 + q].M);
                        Myx = fmaxf(Myx, (q == rank) ? Myw : xslot[xs * 8 + q].My);
                    }
                    Sc = 0.0;
                    Tc = 0.0;
                    Syc = 0.0;
                    for (uint32_t q = 0; q < csize; ++q) {  // rank order: identical on every CTA
                        const XSlot& o = xslot[xs * 8 + q];
                        const float Mq = (q == rank) ? Mw : o.M;
                        const double Sq = (q == rank) ? Sw : o.S;
                        if (Sq != 0.0) {
                            const double f = combine_factor(Mq, Mx);
                            Sc += Sq * f;
                            Tc += ((q == rank) ? Tw : o.T) * f;
                        }
                        const double Syq = (q == rank) ? Syw : o.Sy;
                        if (Syq != 0.0) Syc += Syq * combine_factor((q == rank) ? Myw : o.My, Myx);
                    }
                    Mc = static_cast<double>(Mx);
                    Myc = static_cast<double>(Myx);
                }
                if (kPhaseCounters && p.dbg) pc.lap(d_x);  // the exchange with the group's peers
                // the gradient needs lse, k and D only: publish them first; the reference lse
                // and the KL value (loss and scalars only) follow off the critical path
                const double lse = kLn2 * (Mc + log2(Sc));
                const double D = Tc / Sc;  // Σ p_v (x_v - y_v)
                TokenResult tr;
                double lp = CUDART_NAN;
                if (!tok_ok) {
                    atomicOr(p.status, RF_DEVSTAT_TOKEN_OUT_OF_RANGE);
                    tr.ratio = CUDART_NAN;
                    tr.k = 0.0;
                    tr.loss = 0.0;
                    tr.flags = RF_FLAG_NONFINITE | RF_FLAG_ZERO_COEF;
                } else {
                    lp = static_cast<double>(x_tok) - lse;
                    tr = token_post<RF_GRPO>(p, pre, lp);  // the exact-KL path is GRPO only
                    if (tr.flags & RF_FLAG_NONFINITE) atomicOr(p.status, RF_DEVSTAT_NONFINITE_RATIO);
                }
                const double ks = pre.scale;
                const double kc = -p.grad_sign * ks * p.kl_weight;
                const float lseL = static_cast<float>(lse * 1.4426950408889634);
                bc->k = tr.k;
                bc->A = static_cast<float>(-(tr.k + kc * D));
                bc->B = static_cast<float>(kc);
                bc->lseL = lseL;
                if (tok_ok) {
                    const double pt = tr.ratio * pre.eb;  // exp(lp) = ratio · exp(b)
                    const double dt = static_cast<double>(x_tok) - static_cast<double>(y_tok);
                    bc->tok_val = (tr.k - tr.k * pt) + kc * pt * (dt - D);
                    bc->tok = tok;
                } else {
                    bc->tok_val = 0.0;
                    bc->tok = -1;
                }
                if (kChecked) bc_tag[par] = t;
                mbar_arrive(bar_bc + 8 * par);
                if (kPhaseCounters && p.dbg) pc.lap(d_post);
                const double lseq = kLn2 * (Myc + log2(Syc));
                const double klv = D - lse + lseq;  // Σ p_v (lp_v - lq_v)
                const double kl_scaled = __dmul_rn(ks, klv);
                tr.loss = tr.loss - __dmul_rn(__dmul_rn(ks, p.kl_weight), klv);
                if (rank == 0) {
                    if (p.token_logp) p.token_logp[t] = lp;
                    if (p.token_ratio) p.token_ratio[t] = tr.ratio;
                    if (p.token_coef) p.token_coef[t] = tr.k;
                    if (p.token_loss) p.token_loss[t] = tr.loss;
                    if (p.token_flags) p.token_flags[t] = static_cast<uint8_t>(tr.flags);
                    Partials::store_token(p.partials + static_cast<size_t>(t) * RF_NUM_SCALARS, tr, kl_scaled);
                }
                }  // lane 0
                __syncwarp();
            }
            if (kPhaseCounters && p.dbg && lane == 0) {
                pc.lap(d_math);
                atomicAdd(p.dbg + 6, d_red);
                atomicAdd(p.dbg + 7, d_x);
                atomicAdd(p.dbg + 8, d_math);
                atomicAdd(p.dbg + 12, d_post);
                atomicAdd(p.dbg + 13, d_comb);
                atomicAdd(p.dbg + 9, static_cast<unsigned long long>(clock64() - t_begin));
            }
        }
        __syncwarp();
        tmem_fence_before();
        if (GX)
            __syncthreads();
        else
            cluster_sync_all();
        return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REGS_C));
    {
        // -------------------------------- consumers --------------------------------
        int s = 0;
        uint32_t fphase = 0;
        const uint64_t L2 = pk2(kL2e, kL2e);
        const uint32_t tm = tmem_base + ((32u * (warp & 3)) << 16) + TCOLS * (warp >> 2);  // e: [0, 4·NVT)
        const uint32_t tmd = tm + 4 * NVT;                                                   // d: [4·NVT, 8·NVT)
        uint4 r[NVT], ry[NVT];
        int jmax = 0;
#pragma unroll
        for (int j = 0; j < NVT; ++j) jmax += ((j / VPC) * CHUNK_VECS + (j % VPC) * NCT + tid < slice_len) ? 1 : 0;
        int tail_j = -1;
        if (has_tail) {
            const int svt = tail_vec - slice_begin;
            if (svt >= 0 && svt < slice_len && (svt % CHUNK_VECS) % NCT == tid)
                tail_j = (svt / CHUNK_VECS) * VPC + (svt % CHUNK_VECS) / NCT;
        }
        const int jfull = tail_j >= 0 ? tail_j : jmax;
        const size_t thr_off = static_cast<size_t>(slice_begin + tid) * EPV * OES;
        // phase counters (profiling build): full-wait, stream, park, coef-wait, write, total
        unsigned long long dph[6] = {0, 0, 0, 0, 0, 0};
        PhaseClock pcc;
        pcc.start();
        const long long t_begin = pcc.t;
        const bool dbg = kPhaseCounters && p.dbg != nullptr && lane == 0;
        if (dbg && warp == 0) dbg_cta_begin(p.dbg);

        // copy-in (parking the previous row's e and d chunk by chunk), max, sweep, reduce
        auto stream_row = [&](int64_t t_row, uint32_t row_iter, bool park_prev) -> float {
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                if (park_prev) {
#pragma unroll
                    for (int jj = 0; jj < VPC; ++jj) {
                        const int j = c * VPC + jj;
                        if (j < NVT) {
                            tmem_st4(tm + 4 * j, r[j]);
                            tmem_st4(tmd + 4 * j, ry[j]);
                        }
                    }
                }
                if (c < nchunks) {
                    if (dbg) pcc.lap(dph[1]);
                    cons_wait(bar_full + 8 * s, fphase);
                    if (dbg) pcc.lap(dph[0]);
                    const uint32_t slot = sbase + s * SLOT_BYTES + tid * 16;
                    if (c * VPC + VPC <= jmax) {  // whole chunk inside the slice: plain loads
#pragma unroll
                        for (int jj = 0; jj < VPC; ++jj) {
                            const int j = c * VPC + jj;
                            if (j < NVT) {
                                r[j] = lds128(slot + jj * NCT * 16);
                                ry[j] = lds128(slot + CHUNK_BYTES + jj * NCT * 16);
                            }
                        }
                    } else {  // the slice ends in this chunk: -inf past it
#pragma unroll
                        for (int jj = 0; jj < VPC; ++jj) {
                            const int j = c * VPC + jj;
                            if (j < NVT) {
                                const bool ok = j < jmax;
                                r[j] = ok ? lds128(slot + jj * NCT * 16) : pad_vec_here();
                                ry[j] = ok ? lds128(slot + CHUNK_BYTES + jj * NCT * 16) : pad_vec_here();
                            }
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(bar_empty + 8 * s);
                    if (++s == nslots) {
                        s = 0;
                        fphase ^= 1;
                    }
                } else {
#pragma unroll
                    for (int jj = 0; jj < VPC; ++jj) {
                        const int j = c * VPC + jj;
                        if (j < NVT) r[j] = ry[j] = pad_vec_here();
                    }
                }
            }
            if (tail_j >= 0) {
#pragma unroll
                for (int j = 0; j < NVT; ++j)
                    if (j == tail_j) {
                        mask_tail_pad(r[j], tail_valid);
                        mask_tail_pad(ry[j], tail_valid);
                    }
            }
            const float M = vmax_row(r, NVT), My = vmax_row(ry, NVT);
            const float C = ((M <= kKlPadMax) ? 0.0f : M) * kL2e;
            const float Cy = ((My <= kKlPadMax) ? 0.0f : My) * kL2e;
            const uint64_t negC2 = pk2(-C, -C), negCy2 = pk2(-Cy, -Cy);
            // packed fp32 partial sums over kKlFold vectors, folded into fp64
            double S = 0.0, T = 0.0, Sy = 0.0;
            uint64_t as = 0, ay = 0, ad = 0;
#pragma unroll
            for (int j = 0; j < NVT; ++j) {
                uint64_t se, sy, sd;
                kl_vec(r[j], ry[j], L2, negC2, negCy2, se, sy, sd);
                if (j % kKlFold == 0) {
                    as = se, ay = sy, ad = sd;
                } else {
                    as = fadd2(as, se), ay = fadd2(ay, sy), ad = fadd2(ad, sd);
                }
                if (j % kKlFold == kKlFold - 1 || j == NVT - 1) {
                    S += static_cast<double>(lo2(as) + hi2(as));
                    Sy += static_cast<double>(lo2(ay) + hi2(ay));
                    T += static_cast<double>(lo2(ad) + hi2(ad));
                }
            }
            const float Mr = (S == 0.0) ? -CUDART_INF_F : C;
            const float Myr = (Sy == 0.0) ? -CUDART_INF_F : Cy;
            const uint32_t par = row_iter & 1;
            float Mw = Mr, Myw = Myr;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                Mw = fmaxf(Mw, __shfl_xor_sync(0xffffffffu, Mw, o));
                Myw = fmaxf(Myw, __shfl_xor_sync(0xffffffffu, Myw, o));
            }
            const double f = (S != 0.0) ? combine_factor(Mr, Mw) : 0.0;
            double sw = S * f, tw = T * f;
            double syw = (Sy != 0.0) ? Sy * combine_factor(Myr, Myw) : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                sw += __shfl_xor_sync(0xffffffffu, sw, o);
                tw += __shfl_xor_sync(0xffffffffu, tw, o);
                syw += __shfl_xor_sync(0xffffffffu, syw, o);
            }
            if (lane == 0) {
                redM[par * NCW + warp] = Mw;
                redMy[par * NCW + warp] = Myw;
                redS[par * NCW + warp] = sw;
                redT[par * NCW + warp] = tw;
                redSy[par * NCW + warp] = syw;
                if (kChecked) red_tag[par * NCW + warp] = t_row;
                mbar_arrive(bar_red + 8 * par);
            }
            if (dbg) pcc.lap(dph[1]);
            return C;
        };

        auto write_row = [&](int64_t t, uint32_t row_iter, float C) {
            const uint32_t par = row_iter & 1;
            if (dbg) pcc.lap(dph[4]);
            cons_wait(bar_bc + 8 * par, (row_iter >> 1) & 1);
            if (dbg) pcc.lap(dph[3]);
            if (kChecked) rf_check(bc_tag[par] == t);
            const Bcast* bc = bcs + par;
            const float f = ex2_approx(C - bc->lseL);
            const float A = f * bc->A, B = f * bc->B;
            const uint64_t A2 = pk2(A, A), B2 = pk2(B, B);
            const int tokv = bc->tok;
            const float tv = static_cast<float>(bc->tok_val);
            uint8_t* drow = reinterpret_cast<uint8_t*>(p.dlogits) + static_cast<size_t>(t) * p.dl_stride * OES;
            uint8_t* dthr = drow + thr_off;
#pragma unroll 1
            for (int c = 0; c < NCH; ++c) {
                uint4 e[VPC], d[VPC];
                if (c * VPC + VPC <= NVT) {
                    tmem_ld_vecs<VPC>(tm + 4 * (c * VPC), e);
                    tmem_ld_vecs<VPC>(tmd + 4 * (c * VPC), d);
                } else {
#pragma unroll
                    for (int h = 0; h < VPC; ++h)
                        if (c * VPC + h < NVT) {
                            tmem_ld4(tm + 4 * (c * VPC + h), e[h]);
                            tmem_ld4(tmd + 4 * (c * VPC + h), d[h]);
                        }
                }
                uint8_t* dc = dthr + static_cast<size_t>(c) * CHUNK_VECS * EPV * OES;
                if (c * VPC + VPC <= jfull) {
#pragma unroll
                    for (int h = 0; h < VPC; ++h)
                        kl_store_vec<OUT_BF16>(dc + static_cast<size_t>(h) * NCT * EPV * OES, e[h], d[h], A2, B2);
                    continue;
                }
#pragma unroll
                for (int h = 0; h < VPC; ++h) {
                    const int jj = c * VPC + h;
                    if (jj < jmax) {
                        uint8_t* dst = dc + static_cast<size_t>(h) * NCT * EPV * OES;
                        if (jj != tail_j)
                            kl_store_vec<OUT_BF16>(dst, e[h], d[h], A2, B2);
                        else
                            kl_store_partial<OUT_BF16>(dst, e[h], d[h], A, B, tail_valid);
                    }
                }
            }
            if (tokv >= 0) {  // sampled-token fix-up by the thread that stored its vector
                const int sv = tokv / EPV - slice_begin;
                if (sv >= 0 && sv < slice_len && (sv % CHUNK_VECS) % NCT == tid) {
                    if (OUT_BF16)
                        reinterpret_cast<__nv_bfloat16*>(drow)[tokv] = __float2bfloat16_rn(tv);
                    else
                        reinterpret_cast<float*>(drow)[tokv] = tv;
                }
            }
            if (dbg) pcc.lap(dph[4]);
        };

        uint32_t it = 0;
        int64_t t = rq_get(rowq, bar_rq, 0);
        float C = 0.f;
        if (t >= 0) C = stream_row(t, 0, false);
        while (t >= 0) {
            const int64_t tn = rq_get(rowq, bar_rq, it + 1);
            if (tn < 0) {  // last row: park it whole
#pragma unroll
                for (int j = 0; j < NVT; ++j) {
                    tmem_st4(tm + 4 * j, r[j]);
                    tmem_st4(tmd + 4 * j, ry[j]);
                }
            }
            if (dbg) pcc.lap(dph[2]);
            float Cn = 0.f;
            if (tn >= 0) Cn = stream_row(tn, it + 1, true);
            tmem_wait_st();
            write_row(t, it, C);
            C = Cn;
            t = tn;
            ++it;
        }
        if (dbg) {
            dph[5] = static_cast<unsigned long long>(clock64() - t_begin);
            for (int q = 0; q < 6; ++q) atomicAdd(p.dbg + q, dph[q]);
            if (warp == 0) dbg_cta_end(p.dbg, it, dph);
        }
    }
    tmem_fence_before();
    __syncwarp();
    if (GX)
        __syncthreads();
    else
        cluster_sync_all();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc(tmem_base, 512);
}

namespace {

template <bool OB, int NCW, int NVT>
cudaError_t launch_kl_gx(const KParams& p, int groups, size_t smem, cudaStream_t st) {
    auto kern = ring_kl_kernel<OB, NCW, NVT, true>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(groups * p.vcs));
    cfg.blockDim = dim3((NCW + 4) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // every group's CTAs co-resident
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

template <bool OB, int NCW, int NVT>
cudaError_t launch_kl_t(const KParams& p, int cs, int nclusters, size_t smem, cudaStream_t st, int* maxc) {
    if (p.vcs > 0 && !maxc) return launch_kl_gx<OB, NCW, NVT>(p, nclusters, smem, st);
    auto kern = ring_kl_kernel<OB, NCW, NVT, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>((maxc ? 148 : nclusters) * cs));
    cfg.blockDim = dim3((NCW + 4) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(cs);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (maxc) return cudaOccupancyMaxActiveClusters(maxc, kern, &cfg);
    return cudaLaunchKernelEx(&cfg, kern, p);
}

cudaError_t kl_dispatch(const KParams& p, bool ob, int nvt, int cs, int ncl, size_t smem, cudaStream_t st,
                        int* maxc) {
    if (ob) {
        switch (nvt) {
            case kRingNvtKL[0]: return launch_kl_t<true, kRingWarpsLag, kRingNvtKL[0]>(p, cs, ncl, smem, st, maxc);
            case kRingNvtKL[1]: return launch_kl_t<true, kRingWarpsLag, kRingNvtKL[1]>(p, cs, ncl, smem, st, maxc);
            case kRingNvtKL[2]: return launch_kl_t<true, kRingWarpsLag, kRingNvtKL[2]>(p, cs, ncl, smem, st, maxc);
        }
    } else {
        switch (nvt) {
            case kRingNvtKL[0]: return launch_kl_t<false, kRingWarpsLag, kRingNvtKL[0]>(p, cs, ncl, smem, st, maxc);
            case kRingNvtKL[1]: return launch_kl_t<false, kRingWarpsLag, kRingNvtKL[1]>(p, cs, ncl, smem, st, maxc);
            case kRingNvtKL[2]: return launch_kl_t<false, kRingWarpsLag, kRingNvtKL[2]>(p, cs, ncl, smem, st, maxc);
        }
    }
    return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_ring_kl(const KParams& p, bool out_bf16, int nvt, int cs, int nclusters, size_t smem,
                           cudaStream_t st) {
    return kl_dispatch(p, out_bf16, nvt, cs, nclusters, smem, st, nullptr);
}

cudaError_t ring_kl_max_clusters(bool out_bf16, int nvt, int cs, size_t smem, int* out) {
    KParams p{};
    return kl_dispatch(p, out_bf16, nvt, cs, 0, smem, nullptr, out);
}

}  // namespace rf
