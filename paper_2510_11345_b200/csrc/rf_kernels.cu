// rf_kernels.cu — sm_100a kernels of the off-policy loss + dlogits hot path.
//
//   K1 grpo_group_kernel   GRPO group statistics        (grpo_advantages, losses.cpp:41-60)
//   K2 ring_kernel         (rf_ring.cu) fused log-softmax/gather + ratio + surrogate + dlogits,
//                          one HBM read of the logits row and one write of the dlogits row
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
    if (e - b < 2) {  // losses.cpp:42 throws: flag it, and leave defined outputs behind
        atomicOr(status, RF_DEVSTAT_GROUP_TOO_SMALL);
        degenerate[g] = 0;
        for (int64_t i = b; i < e; ++i) adv[i] = 0.0;
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
                    tr = token_math(p, t, lp, seq);
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
// K2s: sequence_product per-sequence scalars (losses.cpp:180-259).  One warp
// per sequence of this call; deterministic warp-tree sums.
// Writes per-token coef/flags/loss/ratio and a per-sequence partial row.
// ===========================================================================
__global__ void seq_kernel(const __grid_constant__ KParams p, int64_t seq_begin, int64_t nseq,
                           double* __restrict__ coef_out) {
    // One warp per sequence: the trajectory sums as a warp reduction, the per-token
    // outputs written by all lanes in parallel.
    const int lane = threadIdx.x & 31;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= nseq) return;  // whole warps
    const int64_t s = seq_begin + i;
    const int64_t t_base = p.seq_offsets[0];  // tokens of this call start at seq_offsets[0]
    const int64_t t0 = p.seq_offsets[s] - t_base, t1 = p.seq_offsets[s + 1] - t_base;
    const int64_t len = t1 - t0;
    const bool kl = (p.variant == RF_GRPO) && (p.kl_weight > 0.0);
    const bool dppo = p.variant == RF_DECOUPLED_PPO;
    const bool cap = p.mismatch_cap > 0.0;
    // Lane-strided partial sums, then a fixed shuffle tree with lane 0's result
    // broadcast: deterministic, identical on every lane.  The per-token lp the sums
    // read already differ from the reference's in the last bits (fp32 softmax sums),
    // so the reference's strictly sequential order (losses.cpp:187-252) would buy no
    // exactness; it cost a 4-deep fp64 dependency chain per token (0.47 ms per
    // 65K-token chunk on 8K-token sequences).
    double LR = 0.0, logp_sum = 0.0, LPX = 0.0, LM = 0.0;
#pragma unroll 4
    for (int64_t t = t0 + lane; t < t1; t += 32) {
        const double lp = p.token_logp[t];
        const double b = load_logp(p.behavior_logp, t, p.logp_f64);
        LR += __dsub_rn(lp, b);
        logp_sum += lp;
        if (dppo) LPX += __dsub_rn(lp, load_logp(p.prox_logp, t, p.logp_f64));
        if (cap) LM += __dsub_rn(b, load_logp(p.engine_logp, t, p.logp_f64));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        LR += __shfl_down_sync(0xffffffffu, LR, o);
        logp_sum += __shfl_down_sync(0xffffffffu, logp_sum, o);
        LPX += __shfl_down_sync(0xffffffffu, LPX, o);
        LM += __shfl_down_sync(0xffffffffu, LM, o);
    }
    LR = __shfl_sync(0xffffffffu, LR, 0);
    logp_sum = __shfl_sync(0xffffffffu, logp_sum, 0);
    LPX = __shfl_sync(0xffffffffu, LPX, 0);
    LM = __shfl_sync(0xffffffffu, LM, 0);
    uint32_t flags = 0;
    const double em = exp(LM);
    const double m = cap ? ((p.mismatch_cap < em) ? p.mismatch_cap : em) : 1.0;
    if (cap && em > p.mismatch_cap) flags |= RF_FLAG_MISMATCH_CAPPED;
    const double r = exp(LR);
    if (!isfinite(r)) {
        flags |= RF_FLAG_NONFINITE;
        if (lane == 0) atomicOr(p.status, RF_DEVSTAT_NONFINITE_RATIO);
    }
    const double A = p.advantages[s];
    double po = 0.0, tp = 0.0;
    if (dppo) {
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
    double loss_sum = 0.0, kl_sum = 0.0;
    for (int64_t t = t0 + lane; t < t1; t += 32) {
        double loss = (t == t0) ? contrib : 0.0;
        if (kl) {
            const double klv = p.tok_klx[t];
            kl_sum += __dmul_rn(ks, klv);
            loss -= __dmul_rn(__dmul_rn(ks, p.kl_weight), klv);
        }
        coef_out[t] = k;
        if (p.token_ratio) p.token_ratio[t] = exp(p.token_logp[t] - load_logp(p.behavior_logp, t, p.logp_f64));
        if (p.token_loss) p.token_loss[t] = loss;
        if (p.token_flags) p.token_flags[t] = static_cast<uint8_t>(flags);
        loss_sum += loss;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {  // fixed tree: deterministic
        loss_sum += __shfl_xor_sync(0xffffffffu, loss_sum, o);
        kl_sum += __shfl_xor_sync(0xffffffffu, kl_sum, o);
    }
    if (lane == 0) {
        const double n = static_cast<double>(len);
        double* dst = p.partials + static_cast<size_t>(i) * RF_NUM_SCALARS;
        dst[RF_SCALAR_LOSS] = loss_sum;
        dst[RF_SCALAR_TOKENS] = n;
        dst[RF_SCALAR_CLIPPED] = (flags & RF_FLAG_CLIPPED) ? n : 0.0;
        dst[RF_SCALAR_NONFINITE] = (flags & RF_FLAG_NONFINITE) ? n : 0.0;
        dst[RF_SCALAR_ZERO_COEF] = (flags & RF_FLAG_ZERO_COEF) ? n : 0.0;
        dst[RF_SCALAR_MISMATCH] = (flags & RF_FLAG_MISMATCH_CAPPED) ? n : 0.0;
        dst[RF_SCALAR_KL] = kl_sum;
        dst[RF_SCALAR_COEF_ABS] = fabs(k) * n;
    }
}

// ===========================================================================
// K2t: per-token loss math from log-probs given as lse and the sampled logit
// (the LM-head path: lp = x_tok − lse, no logits row).  One thread per token,
// reference semantics (token_math, losses.cpp:262-320); per-block partial rows
// in a fixed tree order.
// ===========================================================================
__global__ void __launch_bounds__(256) token_loss_kernel(const __grid_constant__ KParams p,
                                                         const double* __restrict__ lse,
                                                         const float* __restrict__ xtok) {
    __shared__ double sh[RF_NUM_SCALARS][256];
    Partials part;
    part.zero();
    const int64_t t = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
    if (t < p.T) {
        const int32_t tok = p.token_ids[t];
        TokenResult tr;
        double lp = CUDART_NAN;
        if (tok < 0 || tok >= p.V) {
            atomicOr(p.status, RF_DEVSTAT_TOKEN_OUT_OF_RANGE);
            tr.ratio = CUDART_NAN;
            tr.k = 0.0;
            tr.loss = 0.0;
            tr.flags = RF_FLAG_NONFINITE | RF_FLAG_ZERO_COEF;
        } else {
            lp = static_cast<double>(xtok[t]) - lse[t];
            tr = token_math(p, t, lp, p.seq_of_token[t]);
            if (tr.flags & RF_FLAG_NONFINITE) atomicOr(p.status, RF_DEVSTAT_NONFINITE_RATIO);
        }
        if (p.token_logp) p.token_logp[t] = lp;
        if (p.token_ratio) p.token_ratio[t] = tr.ratio;
        if (p.token_coef) p.token_coef[t] = tr.k;
        if (p.token_loss) p.token_loss[t] = tr.loss;
        if (p.token_flags) p.token_flags[t] = static_cast<uint8_t>(tr.flags);
        part.add_token(tr, 0.0);
    }
    for (int j = 0; j < RF_NUM_SCALARS; ++j) sh[j][threadIdx.x] = part.v[j];
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            for (int j = 0; j < RF_NUM_SCALARS; ++j) sh[j][threadIdx.x] += sh[j][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int j = 0; j < RF_NUM_SCALARS; ++j) p.partials[static_cast<size_t>(blockIdx.x) * RF_NUM_SCALARS + j] = sh[j][0];
}

cudaError_t launch_token_loss(const KParams& p, const double* lse, const float* xtok, cudaStream_t st) {
    const int grid = static_cast<int>((p.T + 255) / 256);
    token_loss_kernel<<<grid, 256, 0, st>>>(p, lse, xtok);
    return cudaGetLastError();
}

// ===========================================================================
// K3: scalars[j] += sum_i partials[i][j] in a fixed order (deterministic).
// ===========================================================================
// K3 also carries the device-side empty-trajectory check (losses.cpp:157 throws on
// an empty trajectory; the host API validates it on the host): this call's tokens
// span sequences [lo, hi] = [seq_of_token[0], seq_of_token[T-1]].  Every empty
// sequence i is then seen by some call: strictly inside [lo, hi], as lo - 1 of the
// call whose first token starts the next non-empty sequence, or as hi + 1 of the
// call holding the batch's last token (trailing).  O(hi - lo) loads per call.
__global__ void finalize_kernel(const double* __restrict__ partials, int64_t n, double* __restrict__ scalars,
                                const int32_t* __restrict__ seq_of_token, const int64_t* __restrict__ seq_offsets,
                                int64_t num_tokens, int64_t num_seqs, int32_t* __restrict__ status) {
    __shared__ double sh[256];
    if (seq_of_token != nullptr && num_tokens > 0) {
        const int64_t lo = seq_of_token[0], hi = seq_of_token[num_tokens - 1];
        bool empty = false;
        for (int64_t i = lo + threadIdx.x; i < hi; i += 256) empty |= seq_offsets[i + 1] <= seq_offsets[i];
        if (threadIdx.x == 0) {
            if (lo > 0 && lo <= num_seqs) empty |= seq_offsets[lo] <= seq_offsets[lo - 1];
            if (hi + 1 < num_seqs) empty |= seq_offsets[hi + 2] <= seq_offsets[hi + 1];
        }
        if (empty) atomicOr(status, RF_DEVSTAT_EMPTY_TRAJECTORY);
    }
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
// Segmented row sums (rf_rows_segment_sum): out[s][v] = Σ_{i in segment s}
// rows[seg_rows[i]][v] in fp64, index order (deterministic).  One thread per
// column, coalesced across a warp; grid (column blocks, segments).  The reference
// binding folds per-token dlogits into LossResult.grad with it (LogProbGrad's
// per-context accumulation, losses.cpp:87-115).
// ===========================================================================
template <typename T>
__global__ void rows_segment_sum_kernel(const T* __restrict__ rows, int64_t row_stride,
                                        const int64_t* __restrict__ seg_offsets, const int32_t* __restrict__ seg_rows,
                                        int32_t width, double* __restrict__ out, int64_t out_stride) {
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t s = blockIdx.y;
    if (v >= width) return;
    double acc = 0.0;
    for (int64_t i = seg_offsets[s]; i < seg_offsets[s + 1]; ++i)
        acc += static_cast<double>(static_cast<float>(rows[static_cast<int64_t>(seg_rows[i]) * row_stride + v]));
    out[s * out_stride + v] = acc;
}

// ===========================================================================
// Launch helpers (called from rf_api.cpp)
// ===========================================================================
cudaError_t launch_generic(const KParams& p, bool in_bf16, bool out_bf16, int grid, cudaStream_t st) {
    generic_kernel<kGenericThreads><<<grid, kGenericThreads, 0, st>>>(p, in_bf16 ? 1 : 0, out_bf16 ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_seq(const KParams& p, int64_t seq_begin, int64_t nseq, double* coef, cudaStream_t st) {
    const int nt = 128;  // four sequences (one per warp) per block
    const int grid = static_cast<int>((nseq + 3) / 4);
    seq_kernel<<<grid, nt, 0, st>>>(p, seq_begin, nseq, coef);
    return cudaGetLastError();
}

// Stage 1 of a long partial-row reduction (one row per token from the lag kernels):
// block b sums the contiguous rows [b·R, (b+1)·R) in a fixed order into row b of `out`.
__global__ void reduce_rows_kernel(const double* __restrict__ partials, int64_t n, double* __restrict__ out) {
    __shared__ double sh[256];
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t lo = static_cast<int64_t>(blockIdx.x) * per, hi = min(n, lo + per);
    for (int j = 0; j < RF_NUM_SCALARS; ++j) {
        double a = 0.0;
        for (int64_t i = lo + threadIdx.x; i < hi; i += 256) a += partials[i * RF_NUM_SCALARS + j];
        sh[threadIdx.x] = a;
        __syncthreads();
        for (int o = 128; o > 0; o >>= 1) {
            if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x == 0) out[static_cast<size_t>(blockIdx.x) * RF_NUM_SCALARS + j] = sh[0];
        __syncthreads();
    }
}

int finalize_launches(int64_t n) { return n > kFinalizeDirectRows ? 2 : 1; }

cudaError_t launch_finalize(const double* partials, int64_t n, double* scalars, const int32_t* seq_of_token,
                            const int64_t* seq_offsets, int64_t num_tokens, int64_t num_seqs, int32_t* status,
                            cudaStream_t st) {
    if (n > kFinalizeDirectRows) {  // scratch rows [n, n + kFinalizeBlocks) follow the partials
        double* mid = const_cast<double*>(partials) + static_cast<size_t>(n) * RF_NUM_SCALARS;
        reduce_rows_kernel<<<kFinalizeBlocks, 256, 0, st>>>(partials, n, mid);
        partials = mid;
        n = kFinalizeBlocks;
    }
    finalize_kernel<<<1, 256, 0, st>>>(partials, n, scalars, seq_of_token, seq_offsets, num_tokens, num_seqs, status);
    return cudaGetLastError();
}

cudaError_t launch_rows_segment_sum(const void* rows, bool bf16, int64_t row_stride, const int64_t* seg_offsets,
                                    const int32_t* seg_rows, int64_t num_segments, int32_t width, double* out,
                                    int64_t out_stride, cudaStream_t st) {
    const dim3 grid(static_cast<unsigned>((width + 255) / 256), static_cast<unsigned>(num_segments));
    if (bf16)
        rows_segment_sum_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(rows), row_stride,
                                                                     seg_offsets, seg_rows, width, out, out_stride);
    else
        rows_segment_sum_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(rows), row_stride, seg_offsets,
                                                             seg_rows, width, out, out_stride);
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
