// rf_kernels.cu — sm_100a kernels of the off-policy loss + dlogits hot path.
//
//   K1 grpo_group_kernel   GRPO group statistics        (grpo_advantages, losses.cpp:41-60)
//   K2 ring_kernel         fused log-softmax/gather + ratio + surrogate + dlogits, one HBM
//                          read of the logits row and one write of the dlogits row; the row
//                          is staged by TMA bulk copies into a ring of shared-memory chunk
//                          slots spread over a thread-block cluster (DSMEM exchange of the
//                          softmax partials)        (loss_and_grad token_mean, losses.cpp:262-331)
//   K2g generic_kernel     the same math for layouts the ring cannot take (tiny / unaligned
//                          vocab, exact-KL GRPO, the two passes of sequence_product)
//   K2s seq_kernel         per-sequence scalars of sequence_product   (losses.cpp:180-259)
//   K3 finalize_kernel     deterministic reduction of per-CTA fp64 partials into scalars
#include <cuda_runtime.h>
#include <math_constants.h>

#include "rf_device.cuh"
#include "rf_kernels.h"

namespace rf {

constexpr float kLog2e = 1.4426950408889634f;

// ===========================================================================
// K1: one thread per GRPO group; sequential fp64 sums in the reference order,
// no FMA contraction -> bit-identical to grpo_advantages.
// ===========================================================================
__global__ void grpo_group_kernel(const double* __restrict__ rewards, const int64_t* __restrict__ group_offsets,
                                  int64_t num_groups, double* __restrict__ adv, uint8_t* __restrict__ degenerate,
                                  int32_t* __restrict__ status) {
    const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= num_groups) return;
    const int64_t b = group_offsets[g], e = group_offsets[g + 1];
    if (e - b < 2) {  // losses.cpp:42 throws; host validated, flag defensively
        atomicOr(status, RF_DEVSTAT_TOKEN_OUT_OF_RANGE);
        return;
    }
    const double n = static_cast<double>(e - b);
    double mean = 0.0;
    for (int64_t i = b; i < e; ++i) mean = __dadd_rn(mean, rewards[i]);
    mean = __ddiv_rn(mean, n);
    double var = 0.0;
    for (int64_t i = b; i < e; ++i) {
        const double d = __dsub_rn(rewards[i], mean);
        var = __dadd_rn(var, __dmul_rn(d, d));
    }
    var = __ddiv_rn(var, n);
    const double sd = __dsqrt_rn(var);
    if (sd < 1e-8) {
        degenerate[g] = 1;
        for (int64_t i = b; i < e; ++i) adv[i] = 0.0;
    } else {
        degenerate[g] = 0;
        for (int64_t i = b; i < e; ++i) adv[i] = __ddiv_rn(__dsub_rn(rewards[i], mean), sd);
    }
}

// ===========================================================================
// Softmax partial (running max M, sum of exp(x - M) S) combination helpers.
// ===========================================================================
__device__ __forceinline__ void combine_ms(float& M, double& S, float M2, double S2) {
    const float Mn = fmaxf(M, M2);
    if (Mn == -CUDART_INF_F) return;
    double s = 0.0;
    if (S != 0.0) s += S * exp(static_cast<double>(M - Mn));
    if (S2 != 0.0) s += S2 * exp(static_cast<double>(M2 - Mn));
    M = Mn;
    S = s;
}

// Warp-level (M, S) reduction: max first, then one fp64 rescale per lane, then sum.
__device__ __forceinline__ void warp_reduce_ms(float& M, double& S) {
    float Mw = M;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) Mw = fmaxf(Mw, __shfl_xor_sync(0xffffffffu, Mw, o));
    double s = (S != 0.0) ? S * exp(static_cast<double>(M - Mw)) : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    M = Mw;
    S = s;
}

// ===========================================================================
// K2: the cluster ring kernel.
//
// Grid: persistent, one cluster of CS CTAs per row at a time; cluster c handles
// token rows c, c + nclusters, ...  Each CTA owns a contiguous 1/CS slice of the
// row (16-byte vectors [rank*slice_vecs, ...)).  Warp NCW is the producer: one
// elected lane streams the slice in CHUNK-sized TMA bulk copies into a ring of
// NSLOT shared-memory slots (mbarrier full/empty pairs).  The NCW consumer warps
// make two passes over the slots a row occupies:
//   pass 1  per thread: chunk-local max, x -> e = 2^((x - M)·log2e) on the MUFU,
//           sum in fp32 per chunk / fp64 across chunks, e stored back IN PLACE
//           (f16 for bf16 logits, f32 for f32 logits) with its max M in the
//           slot's per-thread scale word;
//   reduce  warp shuffles -> CTA -> cluster (DSMEM stores + remote mbarrier
//           arrive); every CTA combines the CS partials in rank order -> lse;
//           consumer thread 0 does the fp64 per-token surrogate math -> k;
//   pass 2  dlogit = -k · e · 2^((M - lse)·log2e)  (+k on the sampled token),
//           packed to bf16/f32 and written with 128-bit streaming stores; the
//           slot is released to the producer chunk by chunk, so the next row's
//           TMA loads overlap this row's stores.
// Logits are read from HBM once and dlogits written once: 4·V bytes per token
// for bf16 in/out.
// ===========================================================================
template <bool IN_BF16, bool OUT_BF16, int NCW, int VPT>
__global__ void __launch_bounds__((NCW + 1) * 32, 1) ring_kernel(const __grid_constant__ KParams p) {
    constexpr int NCT = NCW * 32;
    constexpr int EPV = IN_BF16 ? 8 : 4;  // elements per 16-byte vector
    constexpr int CHUNK_VECS = NCT * VPT;
    constexpr uint32_t CHUNK_BYTES = CHUNK_VECS * 16;
    constexpr uint32_t SLOT_BYTES = CHUNK_BYTES + NCT * 4;

    extern __shared__ __align__(1024) uint8_t smem[];
    const int nslots = p.nslots;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar_full = sbase + nslots * SLOT_BYTES;        // [nslots] u64
    const uint32_t bar_empty = bar_full + nslots * 8;             // [nslots] u64
    const uint32_t bar_x = bar_empty + nslots * 8;                // [2] u64 exchange barriers
    uint8_t* tail = smem + nslots * SLOT_BYTES + nslots * 16 + 16;
    // exchange buffers [2][8] of {double S; float M; pad}
    double* xS = reinterpret_cast<double*>(tail);                 // [2*8]
    float* xM = reinterpret_cast<float*>(tail + 2 * 8 * 8);       // [2*8]
    double* redS = reinterpret_cast<double*>(tail + 2 * 8 * 8 + 2 * 8 * 4);  // [NCW]
    float* redM = reinterpret_cast<float*>(tail + 2 * 8 * 8 + 2 * 8 * 4 + NCW * 8);
    struct Bcast {
        double lse, lp_tok, k, kq;
        float k_f, lse_f;
        int32_t tok_vec, tok_lane;
    };
    Bcast* bc = reinterpret_cast<Bcast*>(tail + 2 * 8 * 8 + 2 * 8 * 4 + NCW * 12 + 4);
    // keep Bcast 8-aligned
    bc = reinterpret_cast<Bcast*>((reinterpret_cast<uintptr_t>(bc) + 7) & ~uintptr_t(7));

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
        mbar_init(bar_x, csize > 1 ? csize - 1 : 1);
        mbar_init(bar_x + 8, csize > 1 ? csize - 1 : 1);
        fence_mbar_init();
    }
    cluster_sync_all();

    const int slice_begin = static_cast<int>(rank) * p.slice_vecs;
    const int slice_end = min(slice_begin + p.slice_vecs, p.row_vecs);
    const int slice_len = max(0, slice_end - slice_begin);
    const int nchunks = (slice_len + CHUNK_VECS - 1) / CHUNK_VECS;
    const int tail_vec = p.row_vecs - 1;
    const int tail_valid = p.V - tail_vec * EPV;  // 1..EPV
    const size_t in_es = IN_BF16 ? 2 : 4;

    if (warp == NCW) {
        // ------------------------- producer -------------------------
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy();
            uint32_t g = 0;  // global chunk counter
            for (int64_t t = cid; t < p.T; t += ncl) {
                const int64_t row = p.row_of_token ? static_cast<int64_t>(p.row_of_token[t]) : t;
                const uint8_t* src = reinterpret_cast<const uint8_t*>(p.logits) +
                                     (row * p.row_stride) * in_es + static_cast<size_t>(slice_begin) * 16;
                for (int c = 0; c < nchunks; ++c, ++g) {
                    const uint32_t s = g % nslots;
                    const uint32_t use = g / nslots;
                    if (use > 0) mbar_wait(bar_empty + 8 * s, (use - 1) & 1);
                    const int nv = min(CHUNK_VECS, slice_len - c * CHUNK_VECS);
                    const uint32_t bytes = static_cast<uint32_t>(nv) * 16;
                    mbar_arrive_expect_tx(bar_full + 8 * s, bytes);
                    bulk_g2s(sbase + s * SLOT_BYTES, src + static_cast<size_t>(c) * CHUNK_BYTES, bytes,
                             bar_full + 8 * s, pol);
                }
            }
        }
        __syncwarp();
    } else {
        // ------------------------- consumers -------------------------
        Partials part;
        part.zero();
        uint32_t g = 0;
        uint32_t row_iter = 0;
        const size_t out_es = OUT_BF16 ? 2 : 4;
        for (int64_t t = cid; t < p.T; t += ncl, ++row_iter) {
            // Scalar-thread prefetch of the per-token inputs (latency hidden by pass 1).
            int32_t tok = 0;
            float x_tok = 0.f;
            int64_t seq = 0;
            double A = 0.0;
            if (tid == 0) {
                const int64_t row = p.row_of_token ? static_cast<int64_t>(p.row_of_token[t]) : t;
                tok = p.token_ids[t];
                seq = p.seq_of_token[t];
                A = p.advantages[seq];
                if (tok >= 0 && tok < p.V) x_tok = load_logit(p.logits, row * p.row_stride + tok, IN_BF16);
            }

            // ---------------- pass 1 ----------------
            float M = -CUDART_INF_F;
            double S = 0.0;
            const uint32_t g0 = g;
            for (int c = 0; c < nchunks; ++c) {
                const uint32_t gc = g0 + c;
                const uint32_t s = gc % nslots;
                mbar_wait(bar_full + 8 * s, (gc / nslots) & 1);
                const uint32_t slot = sbase + s * SLOT_BYTES;
                const int nv = min(CHUNK_VECS, slice_len - c * CHUNK_VECS);
                uint4 v[VPT];
#pragma unroll
                for (int j = 0; j < VPT; ++j) {
                    const int idx = j * NCT + tid;
                    if (idx < nv) v[j] = lds128(slot + idx * 16);
                }
                // mask the padded tail of the row with -inf
#pragma unroll
                for (int j = 0; j < VPT; ++j) {
                    const int idx = j * NCT + tid;
                    const int gvec = slice_begin + c * CHUNK_VECS + idx;
                    if (idx < nv && gvec == tail_vec && tail_valid < EPV) {
                        uint32_t* w = reinterpret_cast<uint32_t*>(&v[j]);
#pragma unroll
                        for (int e = 0; e < EPV; ++e) {
                            if (e >= tail_valid) {
                                if (IN_BF16) {
                                    const int wi = e >> 1;
                                    w[wi] = (e & 1) ? ((w[wi] & 0x0000ffffu) | 0xff800000u)
                                                    : ((w[wi] & 0xffff0000u) | 0x0000ff80u);
                                } else {
                                    w[e] = 0xff800000u;
                                }
                            }
                        }
                    }
                }
                float lm = -CUDART_INF_F;
#pragma unroll
                for (int j = 0; j < VPT; ++j) {
                    const int idx = j * NCT + tid;
                    if (idx < nv) {
                        if (IN_BF16) {
                            __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&v[j].x);
                            __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&v[j].y);
                            __nv_bfloat162 cc = *reinterpret_cast<__nv_bfloat162*>(&v[j].z);
                            __nv_bfloat162 d = *reinterpret_cast<__nv_bfloat162*>(&v[j].w);
                            __nv_bfloat162 m2 = __hmax2(__hmax2(a, b), __hmax2(cc, d));
                            lm = fmaxf(lm, fmaxf(__low2float(m2), __high2float(m2)));
                        } else {
                            lm = fmaxf(lm, fmaxf(fmaxf(__uint_as_float(v[j].x), __uint_as_float(v[j].y)),
                                                 fmaxf(__uint_as_float(v[j].z), __uint_as_float(v[j].w))));
                        }
                    }
                }
                const float Mn = fmaxf(M, lm);
                if (Mn > M && S != 0.0) S *= exp(static_cast<double>(M - Mn));
                M = Mn;
                float sacc[4] = {0.f, 0.f, 0.f, 0.f};
                if (M != -CUDART_INF_F) {
#pragma unroll
                    for (int j = 0; j < VPT; ++j) {
                        const int idx = j * NCT + tid;
                        if (idx < nv) {
                            if (IN_BF16) {
                                uint32_t w[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
                                uint32_t o[4];
#pragma unroll
                                for (int q = 0; q < 4; ++q) {
                                    const float e0 = ex2_approx((bf16lo(w[q]) - M) * kLog2e);
                                    const float e1 = ex2_approx((bf16hi(w[q]) - M) * kLog2e);
                                    sacc[q] += e0 + e1;
                                    o[q] = pack_f16x2(e0, e1);
                                }
                                sts128(slot + idx * 16, make_uint4(o[0], o[1], o[2], o[3]));
                            } else {
                                uint32_t w[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
                                uint32_t o[4];
#pragma unroll
                                for (int q = 0; q < 4; ++q) {
                                    const float e0 = ex2_approx((__uint_as_float(w[q]) - M) * kLog2e);
                                    sacc[q] += e0;
                                    o[q] = __float_as_uint(e0);
                                }
                                sts128(slot + idx * 16, make_uint4(o[0], o[1], o[2], o[3]));
                            }
                        }
                    }
                }
                S += static_cast<double>((sacc[0] + sacc[1]) + (sacc[2] + sacc[3]));
                // per-thread scale word of this chunk
                asm volatile("st.shared.f32 [%0], %1;" ::"r"(slot + CHUNK_BYTES + tid * 4), "f"(M) : "memory");
            }

            // ---------------- reduction ----------------
            warp_reduce_ms(M, S);
            if (lane == 0) {
                redM[warp] = M;
                redS[warp] = S;
            }
            named_bar_sync(1, NCT);
            if (warp == 0) {
                float Mw = lane < NCW ? redM[lane] : -CUDART_INF_F;
                double Sw = lane < NCW ? redS[lane] : 0.0;
                warp_reduce_ms(Mw, Sw);
                if (lane == 0) {
                    const uint32_t par = row_iter & 1;
                    float Mr = Mw;
                    double Sr = Sw;
                    if (csize > 1) {
                        const uint32_t myS = smem_u32(&xS[par * 8 + rank]);
                        const uint32_t myM = smem_u32(&xM[par * 8 + rank]);
                        for (uint32_t r = 0; r < csize; ++r) {
                            if (r == rank) continue;
                            st_cluster_f64(mapa(myS, r), Sw);
                            st_cluster_f32(mapa(myM, r), Mw);
                        }
                        for (uint32_t r = 0; r < csize; ++r) {
                            if (r == rank) continue;
                            mbar_arrive_remote(mapa(bar_x + 8 * par, r));
                        }
                        mbar_wait_cluster(bar_x + 8 * par, (row_iter >> 1) & 1);
                        Mr = -CUDART_INF_F;
                        Sr = 0.0;
                        for (uint32_t r = 0; r < csize; ++r) {
                            const float Mq = (r == rank) ? Mw : xM[par * 8 + r];
                            const double Sq = (r == rank) ? Sw : xS[par * 8 + r];
                            combine_ms(Mr, Sr, Mq, Sq);
                        }
                    }
                    const double lse = static_cast<double>(Mr) + log(Sr);
                    // ---------------- per-token scalar math ----------------
                    TokenResult tr;
                    double lp = CUDART_NAN;
                    if (tok < 0 || tok >= p.V) {
                        atomicOr(p.status, RF_DEVSTAT_TOKEN_OUT_OF_RANGE);
                        tr.ratio = CUDART_NAN;
                        tr.k = 0.0;
                        tr.loss = 0.0;
                        tr.flags = RF_FLAG_NONFINITE | RF_FLAG_ZERO_COEF;
                    } else {
                        lp = static_cast<double>(x_tok) - lse;
                        tr = token_math(p, t, lp, A, token_scale_of(p, seq));
                        if (tr.flags & RF_FLAG_NONFINITE) atomicOr(p.status, RF_DEVSTAT_NONFINITE_RATIO);
                    }
                    if (rank == 0) {
                        if (p.token_logp) p.token_logp[t] = lp;
                        if (p.token_ratio) p.token_ratio[t] = tr.ratio;
                        if (p.token_coef) p.token_coef[t] = tr.k;
                        if (p.token_loss) p.token_loss[t] = tr.loss;
                        if (p.token_flags) p.token_flags[t] = static_cast<uint8_t>(tr.flags);
                        part.add_token(tr, 0.0);
                    }
                    bc->lse = lse;
                    bc->lp_tok = lp;
                    bc->k = tr.k;
                    bc->k_f = static_cast<float>(tr.k);
                    bc->lse_f = static_cast<float>(lse);
                    bc->tok_vec = (tok >= 0 && tok < p.V) ? tok / EPV : -1;
                    bc->tok_lane = (tok >= 0 && tok < p.V) ? tok % EPV : 0;
                }
            }
            named_bar_sync(1, NCT);
            const float k_f = bc->k_f;
            const float lse_f = bc->lse_f;
            const int tok_vec = bc->tok_vec;
            const bool zero = (k_f == 0.0f) && (bc->k == 0.0);

            // ---------------- pass 2 ----------------
            uint8_t* drow = reinterpret_cast<uint8_t*>(p.dlogits) + static_cast<size_t>(t) * p.dl_stride * out_es;
            for (int c = 0; c < nchunks; ++c) {
                const uint32_t gc = g0 + c;
                const uint32_t s = gc % nslots;
                const uint32_t slot = sbase + s * SLOT_BYTES;
                const int nv = min(CHUNK_VECS, slice_len - c * CHUNK_VECS);
                float Mc;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(Mc) : "r"(slot + CHUNK_BYTES + tid * 4));
                const float f = zero ? 0.0f : -k_f * ex2_approx((Mc - lse_f) * kLog2e);
                uint4 v[VPT];
#pragma unroll
                for (int j = 0; j < VPT; ++j) {
                    const int idx = j * NCT + tid;
                    if (idx < nv) v[j] = lds128(slot + idx * 16);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_empty + 8 * s);
#pragma unroll
                for (int j = 0; j < VPT; ++j) {
                    const int idx = j * NCT + tid;
                    if (idx >= nv) continue;
                    const int gvec = slice_begin + c * CHUNK_VECS + idx;
                    float out[EPV];
                    if (IN_BF16) {
                        const uint32_t w[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const float2 e2 = unpack_f16x2(w[q]);
                            out[2 * q] = e2.x * f;
                            out[2 * q + 1] = e2.y * f;
                        }
                    } else {
                        out[0] = __uint_as_float(v[j].x) * f;
                        out[1] = __uint_as_float(v[j].y) * f;
                        out[2] = __uint_as_float(v[j].z) * f;
                        out[3] = __uint_as_float(v[j].w) * f;
                    }
                    if (gvec == tok_vec) {
                        // sampled token: k * (1 - p_tok), p_tok = exp(lp) in fp64
                        const double kk = bc->k;
                        const double pt = exp(bc->lp_tok);
                        out[bc->tok_lane] = zero ? 0.0f : static_cast<float>(kk - kk * pt);
                    }
                    uint8_t* dst = drow + static_cast<size_t>(gvec) * EPV * out_es;
                    const bool partial = (gvec == tail_vec) && (tail_valid < EPV);
                    if (!partial) {
                        if (OUT_BF16) {
                            if (IN_BF16) {
                                stg128_cs(dst, make_uint4(pack_bf16x2(out[0], out[1]), pack_bf16x2(out[2], out[3]),
                                                          pack_bf16x2(out[4], out[5]), pack_bf16x2(out[6], out[7])));
                            } else {
                                stg64_cs(dst, make_uint2(pack_bf16x2(out[0], out[1]), pack_bf16x2(out[2], out[3])));
                            }
                        } else {
#pragma unroll
                            for (int q = 0; q < EPV; q += 4)
                                stg128_cs(dst + q * 4, make_uint4(__float_as_uint(out[q]), __float_as_uint(out[q + 1]),
                                                                  __float_as_uint(out[q + 2]),
                                                                  __float_as_uint(out[q + 3])));
                        }
                    } else {
                        for (int e = 0; e < tail_valid; ++e) {
                            if (OUT_BF16) {
                                __nv_bfloat16 h = __float2bfloat16_rn(out[e]);
                                reinterpret_cast<__nv_bfloat16*>(dst)[e] = h;
                            } else {
                                reinterpret_cast<float*>(dst)[e] = out[e];
                            }
                        }
                    }
                }
            }
            g = g0 + nchunks;
        }
        if (tid == 0 && rank == 0) part.store(p.partials + static_cast<size_t>(cid) * RF_NUM_SCALARS);
    }
    __syncwarp();
    cluster_sync_all();
}

// ===========================================================================
// K2g: generic kernel (one CTA per token row, persistent grid-stride).  Reads
// the row from global memory (three sweeps: max, sum, write); handles any
// vocab/stride/alignment, exact-KL GRPO (ref row), and the stats/write halves
// of sequence_product.  mode 0 = fused, 1 = stats (lse/lp/KL), 2 = write from
// precomputed per-token coef + lse.
// ===========================================================================
template <int NT>
__device__ __forceinline__ void block_reduce_max2(float& a, float& b, float* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) {
        sh[w] = a;
        sh[NT / 32 + w] = b;
    }
    __syncthreads();
    a = -CUDART_INF_F;
    b = -CUDART_INF_F;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) {
        a = fmaxf(a, sh[i]);
        b = fmaxf(b, sh[NT / 32 + i]);
    }
}
template <int NT>
__device__ __forceinline__ void block_reduce_sum3(double& a, double& b, double& c, double* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) {
        sh[w] = a;
        sh[NT / 32 + w] = b;
        sh[2 * NT / 32 + w] = c;
    }
    __syncthreads();
    a = b = c = 0.0;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) {
        a += sh[i];
        b += sh[NT / 32 + i];
        c += sh[2 * NT / 32 + i];
    }
}

template <int NT>
__global__ void __launch_bounds__(NT) generic_kernel(const __grid_constant__ KParams p, int in_bf16, int out_bf16) {
    __shared__ float shf[2 * NT / 32];
    __shared__ double shd[3 * NT / 32];
    __shared__ double bc[6];
    const bool kl = (p.variant == RF_GRPO) && (p.kl_weight > 0.0) && p.ref_logits != nullptr;
    Partials part;
    part.zero();
    for (int64_t t = blockIdx.x; t < p.T; t += gridDim.x) {
        const int64_t row = p.row_of_token ? static_cast<int64_t>(p.row_of_token[t]) : t;
        const int64_t xb = row * p.row_stride;
        const int64_t yb = row * p.ref_row_stride;
        const int32_t tok = p.token_ids[t];
        double lse, lseq = 0.0, klv = 0.0;
        if (p.mode != 2) {
            float M = -CUDART_INF_F, My = -CUDART_INF_F;
            for (int v = threadIdx.x; v < p.V; v += NT) {
                M = fmaxf(M, load_logit(p.logits, xb + v, in_bf16));
                if (kl) My = fmaxf(My, load_logit(p.ref_logits, yb + v, in_bf16));
            }
            block_reduce_max2<NT>(M, My, shf);
            double S = 0.0, Sy = 0.0, T1 = 0.0;
            for (int v = threadIdx.x; v < p.V; v += NT) {
                const float x = load_logit(p.logits, xb + v, in_bf16);
                const double e = exp(static_cast<double>(x - M));
                S += e;
                if (kl) {
                    const float y = load_logit(p.ref_logits, yb + v, in_bf16);
                    Sy += exp(static_cast<double>(y - My));
                    T1 += e * (static_cast<double>(x) - static_cast<double>(y));
                }
            }
            block_reduce_sum3<NT>(S, Sy, T1, shd);
            lse = static_cast<double>(M) + log(S);
            if (kl) {
                lseq = static_cast<double>(My) + log(Sy);
                klv = T1 / S - lse + lseq;  // sum_v p_v (lp_v - lq_v)
            }
        } else {
            lse = p.tok_lse[t];
            if (kl) {
                lseq = p.tok_lseq[t];
                klv = p.tok_klx[t];
            }
        }
        if (threadIdx.x == 0) {
            double k = 0.0, lp = CUDART_NAN, ks = 0.0;
            const bool tok_ok = tok >= 0 && tok < p.V;
            if (!tok_ok) atomicOr(p.status, RF_DEVSTAT_TOKEN_OUT_OF_RANGE);
            if (tok_ok) lp = static_cast<double>(load_logit(p.logits, xb + tok, in_bf16)) - lse;
            const int64_t seq = (p.mode != 1) ? static_cast<int64_t>(p.seq_of_token[t]) : 0;
            if (p.mode != 1) ks = token_scale_of(p, seq);
            if (p.mode == 0) {
                TokenResult tr;
                if (tok_ok) {
                    tr = token_math(p, t, lp, p.advantages[seq], ks);
                    if (tr.flags & RF_FLAG_NONFINITE) atomicOr(p.status, RF_DEVSTAT_NONFINITE_RATIO);
                } else {
                    tr.ratio = CUDART_NAN;
                    tr.k = 0.0;
                    tr.loss = 0.0;
                    tr.flags = RF_FLAG_NONFINITE | RF_FLAG_ZERO_COEF;
                }
                double kl_scaled = 0.0;
                if (kl) {
                    kl_scaled = __dmul_rn(ks, klv);
                    tr.loss = tr.loss - __dmul_rn(__dmul_rn(ks, p.kl_weight), klv);
                }
                k = tr.k;
                if (p.token_logp) p.token_logp[t] = lp;
                if (p.token_ratio) p.token_ratio[t] = tr.ratio;
                if (p.token_coef) p.token_coef[t] = tr.k;
                if (p.token_loss) p.token_loss[t] = tr.loss;
                if (p.token_flags) p.token_flags[t] = static_cast<uint8_t>(tr.flags);
                part.add_token(tr, kl_scaled);
            } else if (p.mode == 1) {
                p.tok_lse[t] = lse;
                p.token_logp[t] = lp;
                if (kl) {
                    p.tok_lseq[t] = lseq;
                    p.tok_klx[t] = klv;
                }
            } else {
                k = p.token_coef[t];
            }
            bc[0] = k;
            bc[1] = lp;
            bc[2] = lse;
            bc[3] = ks;
        }
        __syncthreads();
        if (p.mode != 1 && p.dlogits != nullptr) {
            const double k = bc[0];
            const double kc = kl ? -p.grad_sign * bc[3] * p.kl_weight : 0.0;
            const float k_f = static_cast<float>(k);
            const float lse_f = static_cast<float>(lse);
            const int64_t db = t * p.dl_stride;
            for (int v = threadIdx.x; v < p.V; v += NT) {
                const float x = load_logit(p.logits, xb + v, in_bf16);
                float out;
                if (!kl) {
                    const float pv = exp2f((x - lse_f) * kLog2e);
                    out = (k == 0.0) ? 0.0f : -k_f * pv;
                    if (v == tok && k != 0.0) out = static_cast<float>(k - k * exp(bc[1]));
                } else {
                    const double lpv = static_cast<double>(x) - lse;
                    const double pv = exp(lpv);
                    const double lqv = static_cast<double>(load_logit(p.ref_logits, yb + v, in_bf16)) - lseq;
                    double g = 0.0;
                    if (k != 0.0) g = (v == tok) ? (k - k * pv) : -(k * pv);
                    g += kc * pv * ((lpv - lqv) - klv);
                    out = static_cast<float>(g);
                }
                if (out_bf16)
                    reinterpret_cast<__nv_bfloat16*>(p.dlogits)[db + v] = __float2bfloat16_rn(out);
                else
                    reinterpret_cast<float*>(p.dlogits)[db + v] = out;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && p.mode == 0) part.store(p.partials + static_cast<size_t>(blockIdx.x) * RF_NUM_SCALARS);
}

// ===========================================================================
// K2s: sequence_product per-sequence scalars (losses.cpp:180-259).  One thread
// per sequence of this call; token order sums exactly as the reference.
// Writes per-token coef/flags/loss/ratio and a per-sequence partial row.
// ===========================================================================
__global__ void seq_kernel(const __grid_constant__ KParams p, int64_t seq_begin, int64_t nseq,
                           double* __restrict__ coef_out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nseq) return;
    const int64_t s = seq_begin + i;
    const int64_t t_base = p.seq_offsets[0];  // tokens of this call start at seq_offsets[0]
    const int64_t t0 = p.seq_offsets[s] - t_base, t1 = p.seq_offsets[s + 1] - t_base;
    const int64_t len = t1 - t0;
    const bool kl = (p.variant == RF_GRPO) && (p.kl_weight > 0.0);
    double LR = 0.0, logp_sum = 0.0, LPX = 0.0, LM = 0.0;
    for (int64_t t = t0; t < t1; ++t) {
        const double lp = p.token_logp[t];
        const double b = load_logp(p.behavior_logp, t, p.logp_f64);
        LR = __dadd_rn(LR, __dsub_rn(lp, b));
        logp_sum = __dadd_rn(logp_sum, lp);
        if (p.variant == RF_DECOUPLED_PPO) LPX = __dadd_rn(LPX, __dsub_rn(lp, load_logp(p.prox_logp, t, p.logp_f64)));
        if (p.mismatch_cap > 0.0) LM = __dadd_rn(LM, __dsub_rn(b, load_logp(p.engine_logp, t, p.logp_f64)));
    }
    uint32_t flags = 0;
    const double em = exp(LM);
    const double m = p.mismatch_cap > 0.0 ? ((p.mismatch_cap < em) ? p.mismatch_cap : em) : 1.0;
    if (p.mismatch_cap > 0.0 && em > p.mismatch_cap) flags |= RF_FLAG_MISMATCH_CAPPED;
    const double r = exp(LR);
    if (!isfinite(r)) {
        flags |= RF_FLAG_NONFINITE;
        atomicOr(p.status, RF_DEVSTAT_NONFINITE_RATIO);
    }
    const double A = p.advantages[s];
    double po = 0.0, tp = 0.0;
    if (p.variant == RF_DECOUPLED_PPO) {
        po = exp(__dsub_rn(LR, LPX));
        tp = exp(LPX);
    }
    double value, gw;
    variant_math(p, r, A, po, tp, logp_sum, value, gw, flags);
    const double seq_scale = p.normalization == RF_NORM_GLOBAL_TOKEN ? p.inv_t * static_cast<double>(len) : p.inv_n;
    const double sm = __dmul_rn(seq_scale, m);
    const double k = __dmul_rn(p.grad_sign, __dmul_rn(sm, gw));
    if (k == 0.0) flags |= RF_FLAG_ZERO_COEF;
    const double contrib = __dmul_rn(sm, value);
    const double ks = p.normalization == RF_NORM_GLOBAL_TOKEN ? p.inv_t : p.inv_n / static_cast<double>(len);
    Partials part;
    part.zero();
    for (int64_t t = t0; t < t1; ++t) {
        TokenResult tr;
        tr.k = k;
        tr.flags = flags;
        tr.ratio = exp(p.token_logp[t] - load_logp(p.behavior_logp, t, p.logp_f64));
        tr.loss = (t == t0) ? contrib : 0.0;
        double kl_scaled = 0.0;
        if (kl) {
            const double klv = p.tok_klx[t];
            kl_scaled = __dmul_rn(ks, klv);
            tr.loss -= __dmul_rn(__dmul_rn(ks, p.kl_weight), klv);
        }
        coef_out[t] = k;
        if (p.token_ratio) p.token_ratio[t] = tr.ratio;
        if (p.token_loss) p.token_loss[t] = tr.loss;
        if (p.token_flags) p.token_flags[t] = static_cast<uint8_t>(flags);
        part.add_token(tr, kl_scaled);
    }
    part.store(p.partials + static_cast<size_t>(i) * RF_NUM_SCALARS);
}

// ===========================================================================
// K3: scalars[j] += sum_i partials[i][j] in a fixed order (deterministic).
// ===========================================================================
__global__ void finalize_kernel(const double* __restrict__ partials, int64_t n, double* __restrict__ scalars) {
    __shared__ double sh[256];
    for (int j = 0; j < RF_NUM_SCALARS; ++j) {
        double a = 0.0;
        for (int64_t i = threadIdx.x; i < n; i += 256) a += partials[i * RF_NUM_SCALARS + j];
        sh[threadIdx.x] = a;
        __syncthreads();
        for (int o = 128; o > 0; o >>= 1) {
            if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x == 0) scalars[j] += sh[0];
        __syncthreads();
    }
}

// ===========================================================================
// Launch helpers (called from rf_api.cpp)
// ===========================================================================
template <bool IB, bool OB>
static cudaError_t launch_ring_t(const KParams& p, int cs, int nclusters, size_t smem, cudaStream_t st) {
    auto kern = ring_kernel<IB, OB, kRingWarps, kRingVPT>;
    static bool attr_set = false;  // guarded by the caller's once-flag per instance
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        attr_set = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(nclusters * cs));
    cfg.blockDim = dim3((kRingWarps + 1) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(cs);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

cudaError_t launch_ring(const KParams& p, bool in_bf16, bool out_bf16, int cs, int nclusters, size_t smem,
                        cudaStream_t st) {
    if (in_bf16 && out_bf16) return launch_ring_t<true, true>(p, cs, nclusters, smem, st);
    if (in_bf16 && !out_bf16) return launch_ring_t<true, false>(p, cs, nclusters, smem, st);
    if (!in_bf16 && out_bf16) return launch_ring_t<false, true>(p, cs, nclusters, smem, st);
    return launch_ring_t<false, false>(p, cs, nclusters, smem, st);
}

template <bool IB, bool OB>
static cudaError_t ring_max_clusters_t(int cs, size_t smem, int* out) {
    auto kern = ring_kernel<IB, OB, kRingWarps, kRingVPT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(cs * 148));
    cfg.blockDim = dim3((kRingWarps + 1) * 32);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(cs);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaOccupancyMaxActiveClusters(out, kern, &cfg);
}

cudaError_t ring_max_clusters(bool in_bf16, bool out_bf16, int cs, size_t smem, int* out) {
    if (in_bf16 && out_bf16) return ring_max_clusters_t<true, true>(cs, smem, out);
    if (in_bf16 && !out_bf16) return ring_max_clusters_t<true, false>(cs, smem, out);
    if (!in_bf16 && out_bf16) return ring_max_clusters_t<false, true>(cs, smem, out);
    return ring_max_clusters_t<false, false>(cs, smem, out);
}

cudaError_t launch_generic(const KParams& p, bool in_bf16, bool out_bf16, int grid, cudaStream_t st) {
    generic_kernel<kGenericThreads><<<grid, kGenericThreads, 0, st>>>(p, in_bf16 ? 1 : 0, out_bf16 ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_seq(const KParams& p, int64_t seq_begin, int64_t nseq, double* coef, cudaStream_t st) {
    const int nt = 128;
    const int grid = static_cast<int>((nseq + nt - 1) / nt);
    seq_kernel<<<grid, nt, 0, st>>>(p, seq_begin, nseq, coef);
    return cudaGetLastError();
}

cudaError_t launch_finalize(const double* partials, int64_t n, double* scalars, cudaStream_t st) {
    finalize_kernel<<<1, 256, 0, st>>>(partials, n, scalars);
    return cudaGetLastError();
}

cudaError_t launch_grpo(const double* rewards, const int64_t* group_offsets, int64_t num_groups, double* adv,
                        uint8_t* degenerate, int32_t* status, cudaStream_t st) {
    const int nt = 128;
    const int grid = static_cast<int>((num_groups + nt - 1) / nt);
    grpo_group_kernel<<<grid, nt, 0, st>>>(rewards, group_offsets, num_groups, adv, degenerate, status);
    return cudaGetLastError();
}

}  // namespace rf
