// rf_stream.cu — K2w: dlogits from a KNOWN per-token coefficient and lse
// (second pass of sequence_product, losses.cpp:180-259: every token's weight
// depends on the whole sequence's ratio, so the stats pass (lse, lp per token)
// and the sequence reduction come first).
//
//   dlogit[t, v] = k_t · (1[v = tok_t] - exp(x[t, v] - lse_t))
//
// A pure streaming kernel: one CTA per row at a time (persistent), 128-bit
// non-allocating loads, several loads in flight per thread, packed FFMA2 + one
// MUFU ex2 per element + packed FMUL2 by −k, 128-bit streaming stores.  2·V bytes
// read + 2·V written.
#include <cuda_runtime.h>

#include <algorithm>
#include <math_constants.h>

#include "rf_device.cuh"
#include "rf_kernels.h"
#include "rf_ring_common.cuh"

namespace rf {

using namespace ring;

namespace {

__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

constexpr int kStreamThreads = 256;

// persistent grid: every CTA resident (grid = SMs x occupancy)
template <typename K>
int resident_grid(K kernel, int64_t T) {
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kStreamThreads, 0);
    return static_cast<int>(std::min<int64_t>(T, static_cast<int64_t>(sms) * std::max(occ, 1)));
}

}  // namespace

// The row after t for this CTA: claimed from the launch's counter (first rows are the block
// ids, so the counter starts at gridDim.x), or the static walk t + gridDim.x without one.  A
// CTA on a slower SM takes fewer rows instead of setting the launch's end.
__device__ __forceinline__ int64_t next_row(const KParams& p, int64_t t) {
    if (p.row_ctr == nullptr) return t + gridDim.x;
    return static_cast<int64_t>(gridDim.x) + atomicAdd(p.row_ctr, 1u);
}

// Vectors in flight per thread (4 measured best of {4, 8}); resident CTAs per SM
// the register allocation is bounded for: the read-only stats stream wants every
// slot filled (8 CTAs, 32 registers: 6.1 vs 5.2 TB/s at 4), the write stream its
// unspilled registers (6.1 vs 5.5 TB/s when bounded for 8).
constexpr int kStreamUnroll = 4;
constexpr int kStatsMinBlocks = 8;
constexpr int kWriteMinBlocks = 1;

template <bool IN_BF16, bool OUT_BF16>
__global__ void __launch_bounds__(kStreamThreads, kWriteMinBlocks) stream_write_kernel(const __grid_constant__ KParams p) {
    constexpr int EPV = IN_BF16 ? 8 : 4;
    constexpr size_t IES = IN_BF16 ? 2 : 4;
    constexpr size_t OES = OUT_BF16 ? 2 : 4;
    constexpr float kL2e = 1.4426950408889634f;
    const int tid = threadIdx.x;
    const int row_vecs = p.row_vecs;
    const int tail_vec = row_vecs - 1;
    const int tail_valid = p.V - tail_vec * EPV;
    const uint64_t L2 = pk2(kL2e, kL2e);
    __shared__ int64_t sRow[2];
    int par = 0;
    for (int64_t t = blockIdx.x; t < p.T; par ^= 1) {
        if (tid == 0) sRow[par] = next_row(p, t);  // claimed while this row streams
        const int64_t row = p.row_of_token ? static_cast<int64_t>(p.row_of_token[t]) : t;
        const uint8_t* src = reinterpret_cast<const uint8_t*>(p.logits) + row * p.row_stride * IES;
        uint8_t* dst = reinterpret_cast<uint8_t*>(p.dlogits) + t * p.dl_stride * OES;
        const double k = p.token_coef[t];
        const double lse = p.tok_lse[t];
        const int32_t tok = p.token_ids[t];
        const float lseL = static_cast<float>(lse * 1.4426950408889634);
        const bool zero = (k == 0.0);
        const float f = zero ? 0.0f : static_cast<float>(-k);
        const uint64_t negC2 = pk2(-lseL, -lseL);
        const uint64_t f2 = pk2(f, f);
        for (int v0 = tid; v0 < row_vecs; v0 += kStreamThreads * kStreamUnroll) {
            uint4 x[kStreamUnroll];
#pragma unroll
            for (int u = 0; u < kStreamUnroll; ++u) {
                const int v = v0 + u * kStreamThreads;
                if (v < row_vecs) x[u] = ldg_nc_v4(src + static_cast<size_t>(v) * 16);
            }
#pragma unroll
            for (int u = 0; u < kStreamUnroll; ++u) {
                const int v = v0 + u * kStreamThreads;
                if (v >= row_vecs) break;
                // p = 2^(x·log2e − lse·log2e) kept in f32 and scaled by −k before the one
                // rounding to the output dtype (p itself is ~1/V: as f16 it would be
                // subnormal, ~3% relative error per entry)
                uint8_t* d = dst + static_cast<size_t>(v) * EPV * OES;
                const bool full = (v != tail_vec || tail_valid == EPV);
                if (IN_BF16) {
                    const uint32_t w[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
                    uint64_t o[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint64_t a = ffma2(bf16x2_to_f32x2(w[q]), L2, negC2);
                        o[q] = fmul2(pk2(ex2_approx(lo2(a)), ex2_approx(hi2(a))), f2);
                    }
                    if (full) {
                        if (OUT_BF16) {
                            stg128_cs(d, make_uint4(pack_bf16x2(lo2(o[0]), hi2(o[0])), pack_bf16x2(lo2(o[1]), hi2(o[1])),
                                                    pack_bf16x2(lo2(o[2]), hi2(o[2])), pack_bf16x2(lo2(o[3]), hi2(o[3]))));
                        } else {
                            stg128_cs(d, make_uint4(static_cast<uint32_t>(o[0]), static_cast<uint32_t>(o[0] >> 32),
                                                    static_cast<uint32_t>(o[1]), static_cast<uint32_t>(o[1] >> 32)));
                            stg128_cs(d + 16, make_uint4(static_cast<uint32_t>(o[2]), static_cast<uint32_t>(o[2] >> 32),
                                                         static_cast<uint32_t>(o[3]), static_cast<uint32_t>(o[3] >> 32)));
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            if (q < tail_valid) {
                                const float val = (q & 1) ? hi2(o[q >> 1]) : lo2(o[q >> 1]);
                                if (OUT_BF16)
                                    reinterpret_cast<__nv_bfloat16*>(d)[q] = __float2bfloat16_rn(val);
                                else
                                    reinterpret_cast<float*>(d)[q] = val;
                            }
                        }
                    }
                } else {
                    const uint64_t a01 = ffma2(pk2(__uint_as_float(x[u].x), __uint_as_float(x[u].y)), L2, negC2);
                    const uint64_t a23 = ffma2(pk2(__uint_as_float(x[u].z), __uint_as_float(x[u].w)), L2, negC2);
                    const uint4 e = make_uint4(__float_as_uint(ex2_approx(lo2(a01))), __float_as_uint(ex2_approx(hi2(a01))),
                                               __float_as_uint(ex2_approx(lo2(a23))), __float_as_uint(ex2_approx(hi2(a23))));
                    if (full)
                        store_vec<OUT_BF16, 4>(d, e, f2, false);
                    else
                        store_vec_partial<OUT_BF16, 4>(d, e, f, false, tail_valid);
                }
                if (v == tok / EPV && tok >= 0 && tok < p.V) {  // sampled token, same thread: k(1 - p_tok)
                    const double lp = static_cast<double>(load_logit(p.logits, row * p.row_stride + tok, IN_BF16)) - lse;
                    const float tv = zero ? 0.0f : static_cast<float>(k - k * exp(lp));
                    if (OUT_BF16)
                        reinterpret_cast<__nv_bfloat16*>(dst)[tok] = __float2bfloat16_rn(tv);
                    else
                        reinterpret_cast<float*>(dst)[tok] = tv;
                }
            }
        }
        __syncthreads();  // the next row (double-buffered slot: one barrier per row)
        t = sRow[par];
    }
}

// K2st: the stats pass of sequence_product as a read-only stream — lse and lp per
// token (policy.cpp:21-40 log-softmax at the sampled token) with an online
// softmax, so no row is held on chip.  Each thread keeps (C, S): C = fl(M·log2e) of
// its running max, S = Σ 2^(x·log2e − C) in fp64 (fp32 per batch of kStreamUnroll
// vectors, rescaled by ex2 of the exact float offset difference when the max moves).
// 2·V bytes read per token.
template <bool IN_BF16>
__global__ void __launch_bounds__(kStreamThreads, kStatsMinBlocks) stream_stats_kernel(const __grid_constant__ KParams p) {
    constexpr int EPV = IN_BF16 ? 8 : 4;
    constexpr size_t IES = IN_BF16 ? 2 : 4;
    constexpr float kL2e = 1.4426950408889634f;
    constexpr int kWarps = kStreamThreads / 32;
    __shared__ float sC[2][kWarps];
    __shared__ double sS[2][kWarps];
    __shared__ int64_t sTag[2][kWarps];  // checked build: row of each slot
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int row_vecs = p.row_vecs;
    const int tail_vec = row_vecs - 1;
    const int tail_valid = p.V - tail_vec * EPV;
    const uint64_t L2 = pk2(kL2e, kL2e);
    __shared__ int64_t sRow[2];
    int par = 0;
    for (int64_t t = blockIdx.x; t < p.T; par ^= 1) {
        const int64_t row = p.row_of_token ? static_cast<int64_t>(p.row_of_token[t]) : t;
        const uint8_t* src = reinterpret_cast<const uint8_t*>(p.logits) + row * p.row_stride * IES;
        int32_t tok = 0;
        float x_tok = 0.0f;
        if (tid == 0) {  // the sampled logit, loaded while the row streams; the next row claimed
            sRow[par] = next_row(p, t);
            tok = p.token_ids[t];
            if (tok >= 0 && tok < p.V) x_tok = load_logit(p.logits, row * p.row_stride + tok, IN_BF16);
        }
        float C = -CUDART_INF_F;
        double S = 0.0;
        for (int v0 = tid; v0 < row_vecs; v0 += kStreamThreads * kStreamUnroll) {
            uint4 x[kStreamUnroll];
#pragma unroll
            for (int u = 0; u < kStreamUnroll; ++u) {
                const int v = v0 + u * kStreamThreads;
                x[u] = (v < row_vecs) ? ldg_nc_v4(src + static_cast<size_t>(v) * 16) : neg_inf_vec<IN_BF16>();
                if (v == tail_vec && tail_valid != EPV) mask_tail<IN_BF16>(x[u], tail_valid);
            }
            float bm = -CUDART_INF_F;
#pragma unroll
            for (int u = 0; u < kStreamUnroll; ++u) {
                const uint32_t m = vec_max2<IN_BF16>(x[u]);
                bm = IN_BF16 ? fmaxf(bm, fmaxf(__uint_as_float(m << 16), __uint_as_float(m & 0xffff0000u)))
                             : fmaxf(bm, __uint_as_float(m));
            }
            if (bm == -CUDART_INF_F) continue;  // fully masked batch
            const float Cb = bm * kL2e;
            if (Cb > C) {
                if (S != 0.0) S *= static_cast<double>(ex2_approx(C - Cb));
                C = Cb;
            }
            const uint64_t negC2 = pk2(-C, -C);
            uint64_t acc = 0;
#pragma unroll
            for (int u = 0; u < kStreamUnroll; ++u) {
                const uint32_t w[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
                if (IN_BF16) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint64_t a = ffma2(bf16x2_to_f32x2(w[q]), L2, negC2);
                        const uint64_t e = pk2(ex2_approx(lo2(a)), ex2_approx(hi2(a)));
                        acc = (u == 0 && q == 0) ? e : fadd2(acc, e);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 4; q += 2) {
                        const uint64_t a = ffma2(pk2(__uint_as_float(w[q]), __uint_as_float(w[q + 1])), L2, negC2);
                        const uint64_t e = pk2(ex2_approx(lo2(a)), ex2_approx(hi2(a)));
                        acc = (u == 0 && q == 0) ? e : fadd2(acc, e);
                    }
                }
            }
            S += static_cast<double>(lo2(acc)) + static_cast<double>(hi2(acc));
        }
        // warp, then CTA combine (rank order: deterministic)
        float Cw = C;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) Cw = fmaxf(Cw, __shfl_xor_sync(0xffffffffu, Cw, o));
        double s = (S != 0.0) ? S * static_cast<double>(ex2_approx(C - Cw)) : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
            sC[par][warp] = Cw;
            sS[par][warp] = s;
            if (kChecked) sTag[par][warp] = t;
        }
        __syncthreads();  // double-buffered slots: one barrier per row
        if (tid == 0) {
            if (kChecked)
                for (int w = 0; w < kWarps; ++w) rf_check(sTag[par][w] == t);
            float Cm = -CUDART_INF_F;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) Cm = fmaxf(Cm, sC[par][w]);
            double Sc = 0.0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w)
                if (sS[par][w] != 0.0) Sc += sS[par][w] * static_cast<double>(ex2_approx(sC[par][w] - Cm));
            const double lse = 0.69314718055994530942 * (static_cast<double>(Cm) + log2(Sc));
            const bool tok_ok = tok >= 0 && tok < p.V;
            p.tok_lse[t] = lse;
            p.token_logp[t] = tok_ok ? static_cast<double>(x_tok) - lse : CUDART_NAN;
            if (!tok_ok) atomicOr(p.status, RF_DEVSTAT_TOKEN_OUT_OF_RANGE);
        }
        t = sRow[par];  // written before this row's barrier
    }
}

cudaError_t launch_stream_stats(const KParams& p, bool in_bf16, cudaStream_t st) {
    if (in_bf16) {
        auto k = stream_stats_kernel<true>;
        k<<<resident_grid(k, p.T), kStreamThreads, 0, st>>>(p);
    } else {
        auto k = stream_stats_kernel<false>;
        k<<<resident_grid(k, p.T), kStreamThreads, 0, st>>>(p);
    }
    return cudaGetLastError();
}

template <bool IB, bool OB>
void launch_write_t(const KParams& p, cudaStream_t st) {
    auto k = stream_write_kernel<IB, OB>;
    k<<<resident_grid(k, p.T), kStreamThreads, 0, st>>>(p);
}

cudaError_t launch_stream_write(const KParams& p, bool in_bf16, bool out_bf16, cudaStream_t st) {
    if (in_bf16 && out_bf16)
        launch_write_t<true, true>(p, st);
    else if (in_bf16)
        launch_write_t<true, false>(p, st);
    else if (out_bf16)
        launch_write_t<false, true>(p, st);
    else
        launch_write_t<false, false>(p, st);
    return cudaGetLastError();
}

}  // namespace rf
