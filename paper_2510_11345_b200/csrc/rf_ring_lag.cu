// rf_ring_lag.cu — K2: the fused off-policy loss + dlogits kernel, with the per-row
// softmax/coefficient round trip taken off the consumers' critical path.
//
// One HBM read of every logits row, one HBM write of its dlogits row: TMA bulk
// loads stream each CTA's slice of the row into a shared-memory ring, the slice is
// held in the register file for the max and exp sweeps, and the consumer warps
// never wait for the coefficient of the row they just reduced:
//
//   row i   : copy-in + max + exp sweep in registers -> warp partials (M,S) -> scalar warp
//   row i+1 : copy-in (parking e_i in TENSOR MEMORY chunk by chunk, tcgen05.st,
//             4·NVT columns per thread) + max + exp sweep -> partials -> scalar warp
//   row i   : wait k_i (computed by a scalar warp while row i+1 streamed in),
//             read e_i back from TMEM (tcgen05.ld) and write its dlogits
//
// TMEM (256 KB per SM, unused by this non-GEMM path) is the second row buffer
// next to the register file; the scalar warps (DSMEM cluster exchange + fp64
// surrogate math, losses.cpp:264-320) have a whole row of streaming to finish.
// One CTA per SM: 12 consumer warps (152 registers via setmaxnreg) + one support
// warpgroup (TMA producer, two scalar warps for even/odd rows, one idle warp).
// Rows are claimed at run time from a per-launch counter by each cluster's rank-0
// producer and handed to every role through a shared-memory row queue
// (rf_lag_common.cuh), so faster SM pairs take more rows.  2-CTA clusters for the
// Qwen3 vocabulary.  The alternatives measured against each design choice are
// logged in profiles/r01_ab/ab_log.txt and profiles/r02_ab/.
#include <cuda_runtime.h>
#include <math_constants.h>

#include "rf_device.cuh"
#include "rf_kernels.h"
#include "rf_ring_common.cuh"
#include "rf_lag_common.cuh"

namespace rf {

using namespace ring;


template <bool IN_BF16, bool OUT_BF16, int NCW, int NVT>
__global__ void __launch_bounds__((NCW + 4) * 32, 1) ring_lag_kernel(const __grid_constant__ KParams p) {
    constexpr int NCT = NCW * 32;
    constexpr int EPV = IN_BF16 ? 8 : 4;
    constexpr int VPC = lag_vpc(NVT);
    constexpr int NCH = (NVT + VPC - 1) / VPC;
    constexpr int CHUNK_VECS = NCT * VPC;
    constexpr uint32_t CHUNK_BYTES = CHUNK_VECS * 16;
    constexpr size_t OES = OUT_BF16 ? 2 : 4;
    constexpr size_t IES = IN_BF16 ? 2 : 4;
    static_assert(NCW % 4 == 0 && NCW >= 4 && NCW <= 16, "whole consumer warpgroups");
    constexpr uint32_t TCOLS = lag_tmem_cols(NCW);  // TMEM columns per consumer warp
    static_assert(NVT * 4 <= static_cast<int>(TCOLS), "a thread's e values must fit its TMEM columns");
    constexpr int REGS_C = lag_regs_consumer(NCW);

    // smem: [nslots chunks][full][empty][x(2)][red(2)][bc(2)] + tail
    extern __shared__ __align__(1024) uint8_t smem[];
    const int nslots = p.nslots;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar_full = sbase + nslots * CHUNK_BYTES;
    const uint32_t bar_empty = bar_full + nslots * 8;
    const uint32_t bar_red = bar_empty + nslots * 8 + 16;  // [2] consumers -> scalar: CTA partial (row parity)
    const uint32_t bar_bc = bar_red + 16;            // [2] scalar -> consumers: coefficient (row parity)
    uint8_t* tail = smem + nslots * CHUNK_BYTES + nslots * 16 + 48;
    // Cluster exchange slots [row % 4][sender rank]: written remotely by the peer's
    // scalar warp, guarded by a sequence word (row + 1) instead of an mbarrier phase,
    // so a peer running ahead can never alias a phase (a peer is at most one row of
    // the same parity ahead, and 4 slots cover it).
    struct XSlot {
        double S;
        float M;
        uint32_t seq;
    };
    XSlot* xslot = reinterpret_cast<XSlot*>(tail);                  // [4][8]
    double* redS = reinterpret_cast<double*>(tail + 512);           // [2][NCW]
    float* redM = reinterpret_cast<float*>(tail + 512 + 16 * NCW);  // [2][NCW]
    struct Bcast {
        double ctaS;
        float ctaM, lseL;
        double k, tok_val;
        float negk;
        int32_t tok;
    };
    Bcast* bcs = reinterpret_cast<Bcast*>(tail + 512 + 24 * NCW + ((24 * NCW) % 8 ? 4 : 0));  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bcs + 2);
    static_assert(512 + 24 * NCW + 4 + 2 * sizeof(Bcast) + 4 <= 896, "tail layout");
    int64_t* rowq = reinterpret_cast<int64_t*>(tail + 896);       // [kRowQ] row queue (rf_lag_common.cuh)
    const uint32_t bar_rq = smem_u32(tail + 960);                  // [kRowQ] its mbarriers
    int64_t* red_tag = reinterpret_cast<int64_t*>(tail + 1088);  // [2][NCW] checked build: row of each partial
    int64_t* bc_tag = red_tag + 32;                               // [2] checked build: row of each broadcast

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_ctarank();
    const uint32_t csize = cluster_nctarank();
    const uint32_t cid = cluster_id_x();
    const uint32_t ncl = ncluster_x();

    if (tid == 0) {
        for (int s = 0; s < nslots; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_empty + 8 * s, NCW);
        }
        for (int q = 0; q < 2; ++q) {
            mbar_init(bar_red + 8 * q, NCW);  // one arrival per consumer warp partial
            mbar_init(bar_bc + 8 * q, 1);
        }
        for (int q = 0; q < 32; ++q) {
            xslot[q].S = 0.0;  // tag 0 in both words: never a live use
            xslot[q].seq = 0u;
        }
        for (uint32_t q = 0; q < kRowQ; ++q) mbar_init(bar_rq + 8 * q, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(smem_u32(tmem_slot), 512);
    tmem_fence_before();
    cluster_sync_all();
    tmem_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int slice_begin = static_cast<int>(rank) * p.slice_vecs;
    const int slice_len = max(0, min(p.slice_vecs, p.row_vecs - slice_begin));
    const int nchunks = (slice_len + CHUNK_VECS - 1) / CHUNK_VECS;
    const int tail_vec = p.row_vecs - 1;
    const int tail_valid = p.V - tail_vec * EPV;  // 1..EPV
    const bool has_tail = tail_valid < EPV;

    // Warpgroup 2 (producer, scalar, 2 idle warps) hands registers to the two
    // consumer warpgroups, whose row slices live in the register file.
    // Each register-budget region runs to its own epilogue (ptxas allocates
    // registers per region after setmaxnreg).
    if (warp >= NCW) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kLagRegsSupport));
        if (warp == NCW) {
        // ------------------------------ TMA producer ------------------------------
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy();
            int s = 0;
            uint32_t phase = 0, uses = 0;
            unsigned long long dw = 0, dt = 0;
            PhaseClock pc;
            pc.start();
            const long long t_begin = pc.t;
            // rank 0 claims the cluster's rows and publishes them to every rank's row queue,
            // kRowLookahead rows ahead of the row it is loading
            uint32_t pub = 0;
            bool ended = false;
            auto publish_upto = [&](uint32_t upto) {
                while (rank == 0 && !ended && pub < upto) {
                    const int64_t tq = rq_claim(p, pub, cid, ncl);
                    for (uint32_t q = 0; q < csize; ++q) rq_put(rowq, bar_rq, pub, tq, q, rank);
                    ++pub;
                    if (tq < 0) {  // the end, twice: the other scalar warp reads the entry after it
                        for (uint32_t q = 0; q < csize; ++q) rq_put(rowq, bar_rq, pub, -1, q, rank);
                        ++pub;
                        ended = true;
                    }
                }
            };
            for (uint32_t k = 0;; ++k) {
                publish_upto(k + 1);
                const int64_t t = rq_get(rowq, bar_rq, k);
                if (t < 0) break;
                const int64_t row = p.row_of_token ? static_cast<int64_t>(p.row_of_token[t]) : t;
                const uint8_t* src = reinterpret_cast<const uint8_t*>(p.logits) + (row * p.row_stride) * IES +
                                     static_cast<size_t>(slice_begin) * 16;
                for (int c = 0; c < nchunks; ++c) {
                    if (uses >= static_cast<uint32_t>(nslots)) {
                        if (kPhaseCounters && p.dbg) pc.start();
                        support_wait(bar_empty + 8 * s, phase);
                        if (kPhaseCounters && p.dbg) pc.lap(dw);
                    }
                    const int nv = min(CHUNK_VECS, slice_len - c * CHUNK_VECS);
                    const uint32_t bytes = static_cast<uint32_t>(nv) * 16;
                    mbar_arrive_expect_tx(bar_full + 8 * s, bytes);
                    bulk_g2s(sbase + s * CHUNK_BYTES, src + static_cast<size_t>(c) * CHUNK_BYTES, bytes,
                             bar_full + 8 * s, pol);
                    ++uses;
                    if (++s == nslots) {
                        s = 0;
                        if (uses > static_cast<uint32_t>(nslots)) phase ^= 1;
                    }
                }
                publish_upto(k + 1 + kRowLookahead);
            }
            if (kPhaseCounters && p.dbg) {
                dt = static_cast<unsigned long long>(clock64() - t_begin);
                atomicAdd(p.dbg + 10, dw);
                atomicAdd(p.dbg + 11, dt);
            }
        }
        __syncwarp();
    } else if (warp == NCW + 1 || warp == NCW + 2) {
        // --------------------------------- scalar ---------------------------------
        // Two scalar warps: warp NCW+1 owns the even rows of this cluster, NCW+2 the
        // odd ones (row parity == buffer parity), so each has two rows of
        // streaming to finish its exchange + fp64 math.  The whole warp combines the
        // consumer warps' partials (one per lane, shuffle trees); lane 0 alone runs the
        // exchange, the token math and the broadcast.
        {
            const uint32_t which = static_cast<uint32_t>(warp - NCW - 1);
            unsigned long long d_red = 0, d_x = 0, d_math = 0, d_post = 0;
            PhaseClock pc;
            pc.start();
            const long long t_begin = pc.t;
            for (uint32_t row_iter = which;; row_iter += 2) {
                const int64_t t = rq_get(rowq, bar_rq, row_iter);
                if (t < 0) break;
                // issue the per-token loads before waiting
                const int64_t row = p.row_of_token ? static_cast<int64_t>(p.row_of_token[t]) : t;
                const int32_t tok = p.token_ids[t];
                const bool tok_ok = tok >= 0 && tok < p.V;
                const float x_tok = tok_ok ? load_logit(p.logits, row * p.row_stride + tok, IN_BF16) : 0.0f;
                const TokenPre pre = token_pre(p, t, p.seq_of_token[t]);
                const uint32_t par = row_iter & 1, ph = (row_iter >> 1) & 1;
                Bcast* bc = bcs + par;
                if (kPhaseCounters && p.dbg) pc.lap(d_math);
                support_wait(bar_red + 8 * par, ph);
                if (kPhaseCounters && p.dbg) pc.lap(d_red);
                if (kChecked && lane < NCW) rf_check(red_tag[par * NCW + lane] == t);
                // combine the consumer warps' partials: lane w holds warp w's, fixed butterfly
                // trees (lane 0's result is the one used; the same on every launch)
                const float m_l = lane < NCW ? redM[par * NCW + lane] : -CUDART_INF_F;
                const double s_l = lane < NCW ? redS[par * NCW + lane] : 0.0;
                float Mw = m_l;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) Mw = fmaxf(Mw, __shfl_xor_sync(0xffffffffu, Mw, o));
                double Sw = (s_l != 0.0) ? s_l * combine_factor(m_l, Mw) : 0.0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) Sw += __shfl_xor_sync(0xffffffffu, Sw, o);
                if (lane == 0) {
                double Mc = static_cast<double>(Mw), Sc = Sw;
                if (csize > 1) {
                    // push (S, M) to every peer's slot [row % 4][my rank], publish it with a
                    // release store of the sequence word row + 1, then poll the peers' words
                    // with acquire loads (an st.async + remote-mbarrier variant measured 4%
                    // slower: longer wake-up on the coefficient's critical path)
                    const uint32_t slot = (row_iter & 3) * 8 + rank;
                    XSlot* mine = &xslot[slot];
                    for (uint32_t q = 0; q < csize; ++q) {
                        if (q == rank) continue;
                        st_cluster_f64(mapa(smem_u32(&mine->S), q), Sw);
                        st_cluster_f32(mapa(smem_u32(&mine->M), q), Mw);
                        st_release_cluster_u32(mapa(smem_u32(&mine->seq), q), row_iter + 1);
                    }
                    if (kPhaseCounters && p.dbg) pc.lap(d_math);
                    for (uint32_t q = 0; q < csize; ++q) {
                        if (q == rank) continue;
                        const uint32_t a = smem_u32(&xslot[(row_iter & 3) * 8 + q].seq);
                        while (ld_acquire_cluster_u32(a) != row_iter + 1) __nanosleep(32);
                    }
                    if (kPhaseCounters && p.dbg) pc.lap(d_x);
                    float Mx = -CUDART_INF_F;
                    for (uint32_t q = 0; q < csize; ++q)
                        Mx = fmaxf(Mx, (q == rank) ? Mw : xslot[(row_iter & 3) * 8 + q].M);
                    Sc = 0.0;
                    for (uint32_t q = 0; q < csize; ++q) {  // rank order: identical on every CTA
                        const float Mq = (q == rank) ? Mw : xslot[(row_iter & 3) * 8 + q].M;
                        const double Sq = (q == rank) ? Sw : xslot[(row_iter & 3) * 8 + q].S;
                        if (Sq != 0.0) Sc += Sq * combine_factor(Mq, Mx);
                    }
                    Mc = static_cast<double>(Mx);
                }
                const double lse = 0.69314718055994530942 * (Mc + log2(Sc));  // natural-log lse
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
                    // uniform branch: the decoupled ratio's exp only where it is used
                    tr = (p.variant == RF_DECOUPLED_PPO) ? token_post<RF_DECOUPLED_PPO>(p, pre, lp)
                                                         : token_post<kNotDecoupled>(p, pre, lp);
                    if (tr.flags & RF_FLAG_NONFINITE) atomicOr(p.status, RF_DEVSTAT_NONFINITE_RATIO);
                }
                bc->k = tr.k;
                // p_tok = exp(lp) = ratio · exp(b) (exp(b) precomputed while waiting)
                bc->tok_val = (tok_ok && tr.k != 0.0) ? tr.k - tr.k * (tr.ratio * pre.eb) : 0.0;
                bc->lseL = static_cast<float>(lse * 1.4426950408889634);
                bc->negk = static_cast<float>(-tr.k);
                bc->tok = tok_ok ? tok : -1;
                if (kChecked) bc_tag[par] = t;
                mbar_arrive(bar_bc + 8 * par);
                if (kPhaseCounters && p.dbg) pc.lap(d_post);  // partials in -> k published (after the peer wait)
                if (rank == 0) {
                    if (p.token_logp) p.token_logp[t] = lp;
                    if (p.token_ratio) p.token_ratio[t] = tr.ratio;
                    if (p.token_coef) p.token_coef[t] = tr.k;
                    if (p.token_loss) p.token_loss[t] = tr.loss;
                    if (p.token_flags) p.token_flags[t] = static_cast<uint8_t>(tr.flags);
                    Partials::store_token(p.partials + static_cast<size_t>(t) * RF_NUM_SCALARS, tr, 0.0);
                }
                if (kPhaseCounters && p.dbg) pc.lap(d_math);
                }  // lane 0
                __syncwarp();
            }
            if (kPhaseCounters && p.dbg && lane == 0) {
                atomicAdd(p.dbg + 6, d_red);
                atomicAdd(p.dbg + 7, d_x);
                atomicAdd(p.dbg + 8, d_math);
                atomicAdd(p.dbg + 12, d_post);
                atomicAdd(p.dbg + 9, static_cast<unsigned long long>(clock64() - t_begin));
            }
        }
        __syncwarp();
        }
        tmem_fence_before();
        __syncwarp();
        cluster_sync_all();
        return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REGS_C));
    {
        // -------------------------------- consumers --------------------------------
        int s = 0;
        uint32_t fphase = 0;
        const uint64_t L2 = pk2(1.4426950408889634f, 1.4426950408889634f);
        const uint32_t tm = tmem_base + ((32u * (warp & 3)) << 16) + TCOLS * (warp >> 2);
        uint4 r[NVT];
        // Thread-constant geometry: vector j of this thread is slice vector
        // sv(j) = (j/VPC)·CHUNK_VECS + (j%VPC)·NCT + tid, increasing in j, so the valid
        // ones are j < jmax; tail_j is the j holding the row's padded tail vector.
        int jmax = 0;
#pragma unroll
        for (int j = 0; j < NVT; ++j) jmax += ((j / VPC) * CHUNK_VECS + (j % VPC) * NCT + tid < slice_len) ? 1 : 0;
        int tail_j = -1;
        if (has_tail) {
            const int svt = tail_vec - slice_begin;
            if (svt >= 0 && svt < slice_len && (svt % CHUNK_VECS) % NCT == tid)
                tail_j = (svt / CHUNK_VECS) * VPC + (svt % CHUNK_VECS) / NCT;
        }
        const int jfull = tail_j >= 0 ? tail_j : jmax;  // j < jfull: complete vectors (tail_j == jmax - 1)
        const size_t thr_off = static_cast<size_t>(slice_begin + tid) * EPV * OES;
        // debug phase counters: full-wait, stream, park, coef-wait, write, total
        unsigned long long dph[6] = {0, 0, 0, 0, 0, 0};
        PhaseClock pcc;
        pcc.start();
        const long long t_begin = pcc.t;
        const bool dbg = kPhaseCounters && p.dbg != nullptr && lane == 0;
        if (dbg && warp == 0) dbg_cta_begin(p.dbg);

        // copy-in + max + exp sweep + CTA reduction of row t into r[]; returns C_t.
        auto stream_row = [&](int64_t t_row, uint32_t row_iter, bool park_prev) -> float {
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                if (park_prev) {  // park the previous row's e in TMEM, chunk by chunk
#pragma unroll
                    for (int jj = 0; jj < VPC; ++jj)
                        if (c * VPC + jj < NVT) tmem_st4(tm + 4 * (c * VPC + jj), r[c * VPC + jj]);
                }
                if (c < nchunks) {
                    if (dbg) pcc.lap(dph[1]);
                    cons_wait(bar_full + 8 * s, fphase);
                    if (dbg) pcc.lap(dph[0]);
                    const uint32_t slot = sbase + s * CHUNK_BYTES + tid * 16;
                    if (c * VPC + VPC <= jmax) {  // whole chunk inside the slice: plain loads
#pragma unroll
                        for (int jj = 0; jj < VPC; ++jj) {
                            const int j = c * VPC + jj;
                            if (j < NVT) r[j] = lds128(slot + jj * NCT * 16);
                        }
                    } else {  // the slice ends in this chunk: -inf past it
#pragma unroll
                        for (int jj = 0; jj < VPC; ++jj) {
                            const int j = c * VPC + jj;
                            if (j < NVT) r[j] = (j < jmax) ? lds128(slot + jj * NCT * 16) : neg_inf_vec_here<IN_BF16>();
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
                        if (j < NVT) r[j] = neg_inf_vec_here<IN_BF16>();
                    }
                }
            }
            if (tail_j >= 0) {
#pragma unroll
                for (int j = 0; j < NVT; ++j)
                    if (j == tail_j) mask_tail<IN_BF16>(r[j], tail_valid);
            }
            float M;
            if (IN_BF16) {
                uint32_t m2 = vec_max2<true>(r[0]);
#pragma unroll
                for (int j = 1; j < NVT; ++j) {
                    const uint32_t v2 = vec_max2<true>(r[j]);
                    __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&m2);
                    __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&v2);
                    a = __hmax2(a, b);
                    m2 = *reinterpret_cast<uint32_t*>(&a);
                }
                M = fmaxf(bf16lo(m2), bf16hi(m2));
            } else {
                M = __uint_as_float(vec_max2<false>(r[0]));
#pragma unroll
                for (int j = 1; j < NVT; ++j) M = fmaxf(M, __uint_as_float(vec_max2<false>(r[j])));
            }
            const float Mt = (M == -CUDART_INF_F) ? 0.0f : M;
            const float C = Mt * 1.4426950408889634f;
            const uint64_t negC2 = pk2(-C, -C);
            // every vector's packed fp32 pair sum folded into fp64
            double S = 0.0;
#pragma unroll
            for (int j = 0; j < NVT; ++j) {
                const uint64_t acc = vec_exp<IN_BF16>(r[j], L2, negC2);
                S += static_cast<double>(lo2(acc) + hi2(acc));
            }
            const float Mr = (S == 0.0) ? -CUDART_INF_F : C;
            // warp reduction of (C, S) pairs in the log2 domain; each warp hands its
            // partial straight to the scalar warp (no CTA-wide barrier on the consumers)
            const uint32_t par = row_iter & 1;
            float Mw = Mr;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) Mw = fmaxf(Mw, __shfl_xor_sync(0xffffffffu, Mw, o));
            double sw = (S != 0.0) ? S * combine_factor(Mr, Mw) : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sw += __shfl_xor_sync(0xffffffffu, sw, o);
            if (lane == 0) {
                redM[par * NCW + warp] = Mw;
                redS[par * NCW + warp] = sw;
                if (kChecked) red_tag[par * NCW + warp] = t_row;
                mbar_arrive(bar_red + 8 * par);  // release: the scalar warp's wait sees the words above
            }
            if (dbg) pcc.lap(dph[1]);
            return C;
        };

        // write the dlogits row t (coefficient of row_iter) from TMEM
        auto write_row = [&](int64_t t, uint32_t row_iter, float C) {
            const uint32_t par = row_iter & 1;
            if (dbg) pcc.lap(dph[4]);
            cons_wait(bar_bc + 8 * par, (row_iter >> 1) & 1);
            if (dbg) pcc.lap(dph[3]);
            if (kChecked) rf_check(bc_tag[par] == t);
            const Bcast* bc = bcs + par;
            const float lseL = bc->lseL;
            const float negk = bc->negk;
            const bool zero = (bc->k == 0.0);
            const int tokv = bc->tok;
            const float tv = static_cast<float>(bc->tok_val);
            const float f = zero ? 0.0f : negk * ex2_approx(C - lseL);
            const uint64_t f2 = pk2(f, f);
            uint8_t* drow = reinterpret_cast<uint8_t*>(p.dlogits) + static_cast<size_t>(t) * p.dl_stride * OES;
            uint8_t* dthr = drow + thr_off;
            // A rolled loop (e comes from TMEM, not from indexed registers): keeps the
            // hot code small enough for the instruction caches.
#pragma unroll 1
            for (int c = 0; c < NCH; ++c) {
                uint4 e[VPC];
                if (c * VPC + VPC <= NVT) {
                    tmem_ld_vecs<VPC>(tm + 4 * (c * VPC), e);  // VPC loads, one wait
                } else {
#pragma unroll
                    for (int h = 0; h < VPC; ++h)
                        if (c * VPC + h < NVT) tmem_ld4(tm + 4 * (c * VPC + h), e[h]);
                }
                uint8_t* dc = dthr + static_cast<size_t>(c) * CHUNK_VECS * EPV * OES;
                if (kChecked)  // every vector this chunk may store lies inside this CTA's slice of the row
                    for (int h = 0; h < VPC; ++h)
                        if (c * VPC + h < jmax)
                            rf_check(c * CHUNK_VECS + h * NCT + tid < slice_len &&
                                     slice_begin + c * CHUNK_VECS + h * NCT + tid < p.row_vecs);
                if (c * VPC + VPC <= jfull) {  // straight-line stores (+6% over per-vector branches)
#pragma unroll
                    for (int h = 0; h < VPC; ++h)
                        store_vec<OUT_BF16, EPV>(dc + static_cast<size_t>(h) * NCT * EPV * OES, e[h], f2, IN_BF16);
                    continue;
                }
#pragma unroll
                for (int h = 0; h < VPC; ++h) {
                    const int jj = c * VPC + h;
                    if (jj < jmax) {
                        uint8_t* dst = dc + static_cast<size_t>(h) * NCT * EPV * OES;
                        if (jj != tail_j)
                            store_vec<OUT_BF16, EPV>(dst, e[h], f2, IN_BF16);
                        else
                            store_vec_partial<OUT_BF16, EPV>(dst, e[h], f, IN_BF16, tail_valid);
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
            // park e_t in TMEM, stream this CTA's next row (if any), then write row t from TMEM
            const int64_t tn = rq_get(rowq, bar_rq, it + 1);
            if (tn < 0) {  // last row: nothing to stream, park it all now
#pragma unroll
                for (int j = 0; j < NVT; ++j) tmem_st4(tm + 4 * j, r[j]);
            }
            if (dbg) pcc.lap(dph[2]);
            float Cn = 0.f;
            if (tn >= 0) Cn = stream_row(tn, it + 1, true);
            tmem_wait_st();  // e_t must be in TMEM before write_row reads it back
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
    cluster_sync_all();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc(tmem_base, 512);
}

namespace {

template <bool IB, bool OB, int NCW, int NVT>
cudaError_t launch_lag_t(const KParams& p, int cs, int nclusters, size_t smem, cudaStream_t st, int* maxc) {
    auto kern = ring_lag_kernel<IB, OB, NCW, NVT>;
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

template <bool IB, bool OB>
cudaError_t lag_cfg(const KParams& p, int ncw, int nvt, int cs, int ncl, size_t smem, cudaStream_t st, int* maxc) {
    if (ncw == kRingWarpsLag) {
        switch (nvt) {
            case kRingNvtLag[0]: return launch_lag_t<IB, OB, kRingWarpsLag, kRingNvtLag[0]>(p, cs, ncl, smem, st, maxc);
            case kRingNvtLag[1]: return launch_lag_t<IB, OB, kRingWarpsLag, kRingNvtLag[1]>(p, cs, ncl, smem, st, maxc);
            case kRingNvtLag[2]: return launch_lag_t<IB, OB, kRingWarpsLag, kRingNvtLag[2]>(p, cs, ncl, smem, st, maxc);
            case kRingNvtLag[3]: return launch_lag_t<IB, OB, kRingWarpsLag, kRingNvtLag[3]>(p, cs, ncl, smem, st, maxc);
        }
    }
    return cudaErrorInvalidValue;
}

cudaError_t lag_dispatch(const KParams& p, bool ib, bool ob, int ncw, int nvt, int cs, int ncl, size_t smem,
                         cudaStream_t st, int* maxc) {
    if (ib && ob) return lag_cfg<true, true>(p, ncw, nvt, cs, ncl, smem, st, maxc);
    if (ib && !ob) return lag_cfg<true, false>(p, ncw, nvt, cs, ncl, smem, st, maxc);
    if (!ib && ob) return lag_cfg<false, true>(p, ncw, nvt, cs, ncl, smem, st, maxc);
    return lag_cfg<false, false>(p, ncw, nvt, cs, ncl, smem, st, maxc);
}

}  // namespace

cudaError_t launch_ring_lag(const KParams& p, bool in_bf16, bool out_bf16, int ncw, int nvt, int cs, int nclusters,
                            size_t smem, cudaStream_t st) {
    return lag_dispatch(p, in_bf16, out_bf16, ncw, nvt, cs, nclusters, smem, st, nullptr);
}

cudaError_t ring_lag_max_clusters(bool in_bf16, bool out_bf16, int ncw, int nvt, int cs, size_t smem, int* out) {
    KParams p{};
    return lag_dispatch(p, in_bf16, out_bf16, ncw, nvt, cs, 0, smem, nullptr, out);
}

}  // namespace rf
