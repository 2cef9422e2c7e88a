// rf_ring.cu — K2, the fused off-policy loss + dlogits kernel for sm_100a.
//
// One HBM read of every logits row and one HBM write of its dlogits row
// (4·V bytes per token for bf16 in/out), reference semantics of
// rlsim::loss_and_grad token_mean (losses.cpp:262-331) per token.
//
// Layout: a persistent grid of thread-block clusters; cluster c owns token
// rows c, c + nclusters, ...  Each of the CS CTAs of a cluster owns a 1/CS
// slice of the row (16-byte vectors).  Two CTAs share an SM, so one CTA's
// per-row synchronisation is covered by the other's streaming.  Per CTA:
//
//   producer warp: one lane streams the CTA's slice of every row in chunk-sized
//       TMA bulk copies (cp.async.bulk, L2 evict-first) into a ring of shared
//       memory slots guarded by full/empty mbarriers.  The ring only buffers
//       loads; it runs more than a row slice ahead of the consumers.
//   NCW consumer warps, per row:
//     copy-in  every thread copies its NVT vectors from the ring into REGISTERS
//              (the row slice lives in the register file), releasing each slot
//              at once so the next row's TMA loads start immediately, and tracks
//              its max with packed bf16x2 max;
//     sweep    e = 2^(x·log2e - M_t·log2e) with packed FFMA2 + MUFU ex2, sums in
//              packed fp32 per vector folded into fp64; e overwrites x in the
//              registers as f16x2 (f32 for f32 logits);
//     reduce   warp shuffles -> CTA (smem) -> cluster (DSMEM stores + remote
//              mbarrier arrive); every CTA combines the CS partials in rank
//              order -> lse (fp64); consumer thread 0 finishes the fp64
//              per-token surrogate math (its lp-independent half was done while
//              the slice streamed in) -> row coefficient k;
//     write    dlogit = e · (-k·2^((M_t - lse)·log2e)) with packed FMUL2, packed
//              to bf16/f32 and written with 128-bit streaming stores; the owner of
//              the sampled token then overwrites it with k·(1 - p_tok) (fp64).
#include <cuda_runtime.h>
#include <math_constants.h>

#include "rf_device.cuh"
#include "rf_kernels.h"
#include "rf_ring_common.cuh"

namespace rf {

using namespace ring;


template <bool IN_BF16, bool OUT_BF16, int NCW, int NVT>
__global__ void __launch_bounds__((NCW + 1) * 32, ring_min_blocks(NCW))
    ring_kernel(const __grid_constant__ KParams p) {
    constexpr int NCT = NCW * 32;
    constexpr int EPV = IN_BF16 ? 8 : 4;
    constexpr int VPC = ring_vpc(NVT);
    constexpr int NCH = (NVT + VPC - 1) / VPC;
    constexpr int CHUNK_VECS = NCT * VPC;
    constexpr uint32_t CHUNK_BYTES = CHUNK_VECS * 16;
    constexpr size_t OES = OUT_BF16 ? 2 : 4;
    constexpr size_t IES = IN_BF16 ? 2 : 4;

    // shared memory: [nslots chunk slots][full bars][empty bars][x bars(2)][red bar][bc bar] + tail words
    extern __shared__ __align__(1024) uint8_t smem[];
    const int nslots = p.nslots;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar_full = sbase + nslots * CHUNK_BYTES;
    const uint32_t bar_empty = bar_full + nslots * 8;
    const uint32_t bar_x = bar_empty + nslots * 8;   // [2] cluster exchange (by row parity)
    const uint32_t bar_red = bar_x + 16;              // consumers -> scalar lane: CTA partial ready
    const uint32_t bar_bc = bar_red + 8;              // scalar lane -> consumers: row coefficient ready
    uint8_t* tail = smem + nslots * CHUNK_BYTES + nslots * 16 + 32;
    double* xS = reinterpret_cast<double*>(tail);                  // [2][8] peers' partial sums
    float* xM = reinterpret_cast<float*>(tail + 128);              // [2][8] peers' partial maxima
    double* redS = reinterpret_cast<double*>(tail + 192);          // [NCW] per-warp sums
    float* redM = reinterpret_cast<float*>(tail + 192 + 8 * NCW);  // [NCW] per-warp maxima
    struct Bcast {
        double ctaS;        // this CTA's partial (log2 domain)
        float ctaM, lseL;   // ... and lse·log2e for the write factor
        double k, tok_val;  // row coefficient; dlogit of the sampled token k·(1 - p_tok)
        float negk;         // -k (fp32)
        int32_t tok;        // sampled token (-1: none)
    };
    Bcast* bc = reinterpret_cast<Bcast*>(tail + 192 + 12 * NCW + ((12 * NCW) % 8 ? 4 : 0));

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
        mbar_init(bar_red, 1);
        mbar_init(bar_bc, 1);
        fence_mbar_init();
    }
    cluster_sync_all();

    const int slice_begin = static_cast<int>(rank) * p.slice_vecs;
    const int slice_len = max(0, min(p.slice_vecs, p.row_vecs - slice_begin));
    const int nchunks = (slice_len + CHUNK_VECS - 1) / CHUNK_VECS;
    const int tail_vec = p.row_vecs - 1;
    const int tail_valid = p.V - tail_vec * EPV;  // 1..EPV
    const bool has_tail = tail_valid < EPV;

    if (warp == NCW) {
        if (lane == 0) {
            // ----------------------------- producer lane -----------------------------
            const uint64_t pol = l2_evict_first_policy();
            int s = 0;
            uint32_t phase = 0, uses = 0;
            for (int64_t t = cid; t < p.T; t += ncl) {
                const int64_t row = p.row_of_token ? static_cast<int64_t>(p.row_of_token[t]) : t;
                const uint8_t* src = reinterpret_cast<const uint8_t*>(p.logits) + (row * p.row_stride) * IES +
                                     static_cast<size_t>(slice_begin) * 16;
                for (int c = 0; c < nchunks; ++c) {
                    if (uses >= static_cast<uint32_t>(nslots)) mbar_wait(bar_empty + 8 * s, phase);
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
            }
        } else if (lane == 1) {
            // ------------------------------ scalar lane ------------------------------
            // Per row: gather the sampled logit and the lp-independent token math
            // while the consumers stream the slice, then combine the CTA partial
            // with the cluster peers' (DSMEM), finish the fp64 surrogate math
            // (losses.cpp:264-320) and publish the row coefficient.
            Partials part;
            part.zero();
            uint32_t row_iter = 0;
            for (int64_t t = cid; t < p.T; t += ncl, ++row_iter) {
                const int64_t row = p.row_of_token ? static_cast<int64_t>(p.row_of_token[t]) : t;
                const int32_t tok = p.token_ids[t];
                const bool tok_ok = tok >= 0 && tok < p.V;
                const float x_tok = tok_ok ? load_logit(p.logits, row * p.row_stride + tok, IN_BF16) : 0.0f;
                const TokenPre pre = token_pre(p, t, p.seq_of_token[t]);
                const uint32_t par = row_iter & 1;
                mbar_wait(bar_red, par);
                const float Mw = bc->ctaM;
                const double Sw = bc->ctaS;
                double Mc = static_cast<double>(Mw), Sc = Sw;
                if (csize > 1) {
                    const uint32_t myS = smem_u32(&xS[par * 8 + rank]);
                    const uint32_t myM = smem_u32(&xM[par * 8 + rank]);
                    for (uint32_t q = 0; q < csize; ++q) {
                        if (q == rank) continue;
                        st_cluster_f64(mapa(myS, q), Sw);
                        st_cluster_f32(mapa(myM, q), Mw);
                    }
                    for (uint32_t q = 0; q < csize; ++q) {
                        if (q == rank) continue;
                        mbar_arrive_remote(mapa(bar_x + 8 * par, q));
                    }
                    mbar_wait_cluster(bar_x + 8 * par, (row_iter >> 1) & 1);
                    float Mx = -CUDART_INF_F;
                    for (uint32_t q = 0; q < csize; ++q) Mx = fmaxf(Mx, (q == rank) ? Mw : xM[par * 8 + q]);
                    Sc = 0.0;
                    for (uint32_t q = 0; q < csize; ++q) {  // rank order: identical on every CTA
                        const float Mq = (q == rank) ? Mw : xM[par * 8 + q];
                        const double Sq = (q == rank) ? Sw : xS[par * 8 + q];
                        if (Sq != 0.0) Sc += Sq * exp2(static_cast<double>(Mq) - static_cast<double>(Mx));
                    }
                    Mc = static_cast<double>(Mx);
                }
                // log2-domain total -> natural lse:  lse = ln2·(Mc + log2 Sc)
                const double lse = kLn2 * (Mc + log2(Sc));
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
                    tr = token_post(p, pre, lp);
                    if (tr.flags & RF_FLAG_NONFINITE) atomicOr(p.status, RF_DEVSTAT_NONFINITE_RATIO);
                }
                bc->k = tr.k;
                bc->tok_val = (tok_ok && tr.k != 0.0) ? tr.k - tr.k * exp(lp) : 0.0;
                bc->lseL = static_cast<float>(lse * 1.4426950408889634);
                bc->negk = static_cast<float>(-tr.k);
                bc->tok = tok_ok ? tok : -1;
                mbar_arrive(bar_bc);  // release: the consumers' acquire-wait sees the words above
                if (rank == 0) {
                    if (p.token_logp) p.token_logp[t] = lp;
                    if (p.token_ratio) p.token_ratio[t] = tr.ratio;
                    if (p.token_coef) p.token_coef[t] = tr.k;
                    if (p.token_loss) p.token_loss[t] = tr.loss;
                    if (p.token_flags) p.token_flags[t] = static_cast<uint8_t>(tr.flags);
                    part.add_token(tr, 0.0);
                }
            }
            if (rank == 0) part.store(p.partials + static_cast<size_t>(cid) * RF_NUM_SCALARS);
        }
        __syncwarp();
    } else {
        // ------------------------------ consumers ------------------------------
        int s = 0;
        uint32_t fphase = 0;
        uint32_t row_iter = 0;
        const uint64_t L2 = pk2(kL2e, kL2e);
        for (int64_t t = cid; t < p.T; t += ncl, ++row_iter) {
            // ------------------------ copy-in + running max ------------------------
            uint4 r[NVT];
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                if (c < nchunks) {
                    mbar_wait(bar_full + 8 * s, fphase);
                    const uint32_t slot = sbase + s * CHUNK_BYTES;
#pragma unroll
                    for (int jj = 0; jj < VPC; ++jj) {
                        const int j = c * VPC + jj;
                        if (j < NVT) {
                            const int sv = c * CHUNK_VECS + jj * NCT + tid;
                            r[j] = (sv < slice_len) ? lds128(slot + (jj * NCT + tid) * 16) : neg_inf_vec<IN_BF16>();
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
                        if (j < NVT) r[j] = neg_inf_vec<IN_BF16>();
                    }
                }
            }
            if (has_tail) {
#pragma unroll
                for (int j = 0; j < NVT; ++j) {
                    const int sv = (j / VPC) * CHUNK_VECS + (j % VPC) * NCT + tid;
                    if (slice_begin + sv == tail_vec) mask_tail<IN_BF16>(r[j], tail_valid);
                }
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
            const float C = Mt * kL2e;  // exponent offset (log2 domain), exact in the fp64 combine

            // ------------------------------ exp sweep ------------------------------
            const uint64_t negC2 = pk2(-C, -C);
            double S = 0.0;
#pragma unroll
            for (int j = 0; j < NVT; ++j) {
                const uint64_t acc = vec_exp<IN_BF16>(r[j], L2, negC2);
                S += static_cast<double>(lo2(acc) + hi2(acc));
            }
            // thread partial: S = sum 2^(x·L - C), i.e. (C, S) in the log2 domain
            const float Mr = (S == 0.0) ? -CUDART_INF_F : C;

            // ------------------------------ reduction ------------------------------
            {
                float Mw = Mr;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) Mw = fmaxf(Mw, __shfl_xor_sync(0xffffffffu, Mw, o));
                double sw = (S != 0.0) ? S * exp2(static_cast<double>(Mr) - static_cast<double>(Mw)) : 0.0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sw += __shfl_xor_sync(0xffffffffu, sw, o);
                if (lane == 0) {
                    redM[warp] = Mw;
                    redS[warp] = sw;
                }
            }
            named_bar_sync(1, NCT);
            if (warp == 0) {
                const float Mw = lane < NCW ? redM[lane] : -CUDART_INF_F;
                const double Sw = lane < NCW ? redS[lane] : 0.0;
                float Mx = Mw;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) Mx = fmaxf(Mx, __shfl_xor_sync(0xffffffffu, Mx, o));
                double sx = (Sw != 0.0) ? Sw * exp2(static_cast<double>(Mw) - static_cast<double>(Mx)) : 0.0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sx += __shfl_xor_sync(0xffffffffu, sx, o);
                if (lane == 0) {
                    bc->ctaM = Mx;
                    bc->ctaS = sx;
                    mbar_arrive(bar_red);
                }
            }
            mbar_wait(bar_bc, row_iter & 1);
            const float lseL = bc->lseL;
            const float negk = bc->negk;
            const bool zero = (bc->k == 0.0);
            const int tokv = bc->tok;
            const float tv = static_cast<float>(bc->tok_val);
            const float f = zero ? 0.0f : negk * ex2_approx(C - lseL);
            const uint64_t f2 = pk2(f, f);

            // ------------------------------ write ------------------------------
            uint8_t* drow = reinterpret_cast<uint8_t*>(p.dlogits) + static_cast<size_t>(t) * p.dl_stride * OES;
            if (!has_tail) {
#pragma unroll
                for (int j = 0; j < NVT; ++j) {
                    const int sv = (j / VPC) * CHUNK_VECS + (j % VPC) * NCT + tid;
                    if (sv < slice_len)
                        store_vec<OUT_BF16, EPV>(drow + static_cast<size_t>(slice_begin + sv) * EPV * OES, r[j], f2,
                                                 IN_BF16);
                }
            } else {
#pragma unroll
                for (int j = 0; j < NVT; ++j) {
                    const int sv = (j / VPC) * CHUNK_VECS + (j % VPC) * NCT + tid;
                    if (sv < slice_len) {
                        uint8_t* dst = drow + static_cast<size_t>(slice_begin + sv) * EPV * OES;
                        if (slice_begin + sv != tail_vec)
                            store_vec<OUT_BF16, EPV>(dst, r[j], f2, IN_BF16);
                        else
                            store_vec_partial<OUT_BF16, EPV>(dst, r[j], f, IN_BF16, tail_valid);
                    }
                }
            }
            // sampled-token fix-up by the thread that stored its vector (same-thread order)
            if (tokv >= 0) {
                const int sv = tokv / EPV - slice_begin;
                if (sv >= 0 && sv < slice_len && (sv % CHUNK_VECS) % NCT == tid) {
                    if (OUT_BF16)
                        reinterpret_cast<__nv_bfloat16*>(drow)[tokv] = __float2bfloat16_rn(tv);
                    else
                        reinterpret_cast<float*>(drow)[tokv] = tv;
                }
            }
        }
    }
    __syncwarp();
    cluster_sync_all();
}

namespace {

template <bool IB, bool OB, int NCW, int NVT>
cudaError_t launch_ring_t(const KParams& p, int cs, int nclusters, size_t smem, cudaStream_t st, int* maxc) {
    auto kern = ring_kernel<IB, OB, NCW, NVT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>((maxc ? 296 : nclusters) * cs));
    cfg.blockDim = dim3((NCW + 1) * 32);
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
cudaError_t dispatch_cfg(const KParams& p, int ncw, int nvt, int cs, int ncl, size_t smem, cudaStream_t st,
                         int* maxc) {
    if (ncw == kRingWarpsSmall) {
        switch (nvt) {
            case 4: return launch_ring_t<IB, OB, kRingWarpsSmall, 4>(p, cs, ncl, smem, st, maxc);
            case 16: return launch_ring_t<IB, OB, kRingWarpsSmall, 16>(p, cs, ncl, smem, st, maxc);
            case 30: return launch_ring_t<IB, OB, kRingWarpsSmall, 30>(p, cs, ncl, smem, st, maxc);
        }
    } else if (ncw == kRingWarpsLarge && nvt == 27) {
        return launch_ring_t<IB, OB, kRingWarpsLarge, 27>(p, cs, ncl, smem, st, maxc);
    }
    return cudaErrorInvalidValue;
}

cudaError_t dispatch(const KParams& p, bool ib, bool ob, int ncw, int nvt, int cs, int ncl, size_t smem,
                     cudaStream_t st, int* maxc) {
    if (ib && ob) return dispatch_cfg<true, true>(p, ncw, nvt, cs, ncl, smem, st, maxc);
    if (ib && !ob) return dispatch_cfg<true, false>(p, ncw, nvt, cs, ncl, smem, st, maxc);
    if (!ib && ob) return dispatch_cfg<false, true>(p, ncw, nvt, cs, ncl, smem, st, maxc);
    return dispatch_cfg<false, false>(p, ncw, nvt, cs, ncl, smem, st, maxc);
}

}  // namespace

cudaError_t launch_ring(const KParams& p, bool in_bf16, bool out_bf16, int ncw, int nvt, int cs, int nclusters,
                        size_t smem, cudaStream_t st) {
    return dispatch(p, in_bf16, out_bf16, ncw, nvt, cs, nclusters, smem, st, nullptr);
}

cudaError_t ring_max_clusters(bool in_bf16, bool out_bf16, int ncw, int nvt, int cs, size_t smem, int* out) {
    KParams p{};
    return dispatch(p, in_bf16, out_bf16, ncw, nvt, cs, 0, smem, nullptr, out);
}

}  // namespace rf
