// rf_stream.cu — K2w: dlogits from a KNOWN per-token coefficient and lse
// (second pass of sequence_product, losses.cpp:180-259: every token's weight
// depends on the whole sequence's ratio, so the stats pass (lse, lp per token)
// and the sequence reduction come first).
//
//   dlogit[t, v] = k_t · (1[v = tok_t] - exp(x[t, v] - lse_t))
//
// A pure streaming kernel: one CTA per row at a time (persistent), 128-bit
// non-allocating loads, several loads in flight per thread, packed FFMA2 + one
// MUFU ex2 per element, 128-bit streaming stores.  2·V bytes read + 2·V written.
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
constexpr int kStreamUnroll = 4;

}  // namespace

template <bool IN_BF16, bool OUT_BF16>
__global__ void __launch_bounds__(kStreamThreads) stream_write_kernel(const __grid_constant__ KParams p) {
    constexpr int EPV = IN_BF16 ? 8 : 4;
    constexpr size_t IES = IN_BF16 ? 2 : 4;
    constexpr size_t OES = OUT_BF16 ? 2 : 4;
    constexpr float kL2e = 1.4426950408889634f;
    const int tid = threadIdx.x;
    const int row_vecs = p.row_vecs;
    const int tail_vec = row_vecs - 1;
    const int tail_valid = p.V - tail_vec * EPV;
    const uint64_t L2 = pk2(kL2e, kL2e);
    for (int64_t t = blockIdx.x; t < p.T; t += gridDim.x) {
        const int64_t row = p.row_of_token ? static_cast<int64_t>(p.row_of_token[t]) : t;
        const uint8_t* src = reinterpret_cast<const uint8_t*>(p.logits) + row * p.row_stride * IES;
        uint8_t* dst = reinterpret_cast<uint8_t*>(p.dlogits) + t * p.dl_stride * OES;
        const double k = p.token_coef[t];
        const double lse = p.tok_lse[t];
        const int32_t tok = p.token_ids[t];
        const float lseL = static_cast<float>(lse * 1.4426950408889634);
        const float negk = static_cast<float>(-k);
        const bool zero = (k == 0.0);
        const uint64_t negC2 = pk2(-lseL, -lseL);
        const uint64_t f2 = pk2(zero ? 0.0f : negk, zero ? 0.0f : negk);
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
                // e = 2^(x·L - lse·L) = p, then out = -k·p via the shared packed store path
                uint4 e = x[u];
                uint32_t w[4] = {e.x, e.y, e.z, e.w};
                if (IN_BF16) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint64_t a = ffma2(bf16x2_to_f32x2(w[q]), L2, negC2);
                        w[q] = pack_f16x2(ex2_approx(lo2(a)), ex2_approx(hi2(a)));
                    }
                } else {
                    const uint64_t a01 = ffma2(pk2(__uint_as_float(w[0]), __uint_as_float(w[1])), L2, negC2);
                    const uint64_t a23 = ffma2(pk2(__uint_as_float(w[2]), __uint_as_float(w[3])), L2, negC2);
                    w[0] = __float_as_uint(ex2_approx(lo2(a01)));
                    w[1] = __float_as_uint(ex2_approx(hi2(a01)));
                    w[2] = __float_as_uint(ex2_approx(lo2(a23)));
                    w[3] = __float_as_uint(ex2_approx(hi2(a23)));
                }
                e = make_uint4(w[0], w[1], w[2], w[3]);
                uint8_t* d = dst + static_cast<size_t>(v) * EPV * OES;
                if (v != tail_vec || tail_valid == EPV)
                    store_vec<OUT_BF16, EPV>(d, e, f2, IN_BF16);
                else
                    store_vec_partial<OUT_BF16, EPV>(d, e, zero ? 0.0f : negk, IN_BF16, tail_valid);
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
    }
}

cudaError_t launch_stream_write(const KParams& p, bool in_bf16, bool out_bf16, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = static_cast<int>(std::min<int64_t>(p.T, static_cast<int64_t>(sms) * 8));
    if (in_bf16 && out_bf16)
        stream_write_kernel<true, true><<<grid, kStreamThreads, 0, st>>>(p);
    else if (in_bf16)
        stream_write_kernel<true, false><<<grid, kStreamThreads, 0, st>>>(p);
    else if (out_bf16)
        stream_write_kernel<false, true><<<grid, kStreamThreads, 0, st>>>(p);
    else
        stream_write_kernel<false, false><<<grid, kStreamThreads, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace rf
