// rf_lmhead.cu — K0 (experimental): the LM-head GEMM on the
// 5th-generation tensor cores with the softmax statistics fused into its epilogue,
// so the [T, V] logits of the stats pass never reach HBM.
//
//   logits = H · Wᵀ      H [T, K] bf16 (hidden states), W [V, K] bf16 (vocab projection)
//   out:   lse[t] = log Σ_v exp(logits[t, v]),  x_tok[t] = logits[t, tok_t]
//
// A 2-CTA cluster owns 256 token rows (UMMA M = 256, cta_group::2) and sweeps its
// vocabulary split in 256-column tiles (UMMA N = 256), K in 64-element (128-byte,
// SWIZZLE_128B) chunks:
//   warp 0      TMA producer: each CTA's 128 H rows and half of the W tile into a
//               6-stage shared-memory ring (bytes complete on the leader's barrier)
//   warp 1      the leader's elected lane issues tcgen05.mma (kind::f16, fp32
//               accumulate in tensor memory), double-buffered over two 256-column
//               TMEM accumulators; commits multicast to both CTAs
//   warps 2-5   epilogue: tcgen05.ld of a finished tile (thread = token row), then
//               MODE 0 (stats): online max / Σexp in fp32 and the sampled token's logit;
//               MODE 1 (dlogits): k·(1[v = tok] − exp(x − lse)) as bf16 rows.
// lse is combined across the vocabulary splits in fp64 (lmhead_combine_kernel).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <math_constants.h>

#include "rf_device.cuh"
#include "rf_kernels.h"

namespace rf {

namespace {

constexpr int kLmM = 128, kLmN = 256, kLmK = 64;  // per CTA: 128 token rows, 256-column vocab tiles, K chunks

// K-major operand tile in SWIZZLE_128B layout: rows of 128 bytes, 8-row (1024 B) groups.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((addr & 0x3FFFFu) >> 4);  // start address
    d |= static_cast<uint64_t>(1) << 16;                  // leading byte offset (unused for swizzled K-major)
    d |= static_cast<uint64_t>(1024 >> 4) << 32;          // stride byte offset: 8 rows x 128 B
    d |= static_cast<uint64_t>(1) << 46;                  // descriptor version (sm_100)
    d |= static_cast<uint64_t>(2) << 61;                  // layout: SWIZZLE_128B
    return d;
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// dlogits of one 32-column chunk of a token row: k·(1[v = tok] − exp(x − lse)), bf16
__device__ __forceinline__ void dl_store_chunk(__nv_bfloat16* drow, const float* v, int col0, int V, int tk, float negk,
                                               double kd, float lseL, double lse, bool st256) {
    constexpr float L = 1.4426950408889634f;
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        float o0 = negk * ex2_approx(fmaf(v[2 * i], L, -lseL));
        float o1 = negk * ex2_approx(fmaf(v[2 * i + 1], L, -lseL));
        if (kd == 0.0) o0 = o1 = 0.0f;
        if (tk == col0 + 2 * i) o0 = static_cast<float>(kd - kd * exp(static_cast<double>(v[2 * i]) - lse));
        if (tk == col0 + 2 * i + 1) o1 = static_cast<float>(kd - kd * exp(static_cast<double>(v[2 * i + 1]) - lse));
        w[i] = pack_bf16x2(o0, o1);
    }
    if (col0 + 32 <= V) {
        if (st256) {  // two full 32-byte sectors per thread (STG.256)
#pragma unroll
            for (int i = 0; i < 2; ++i)
                asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(drow + col0 + 16 * i),
                             "r"(w[8 * i]), "r"(w[8 * i + 1]), "r"(w[8 * i + 2]), "r"(w[8 * i + 3]), "r"(w[8 * i + 4]),
                             "r"(w[8 * i + 5]), "r"(w[8 * i + 6]), "r"(w[8 * i + 7])
                             : "memory");
        } else {
            uint4* d4 = reinterpret_cast<uint4*>(drow + col0);
#pragma unroll
            for (int i = 0; i < 4; ++i) d4[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
        }
    } else {
        for (int i = 0; i < 32 && col0 + i < V; ++i)
            drow[col0 + i] = __ushort_as_bfloat16(static_cast<uint16_t>((i & 1) ? (w[i >> 1] >> 16) : (w[i >> 1] & 0xffffu)));
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// Grouped raster over (128-token block, vocab split): panels of `group` token blocks; inside a
// panel the token blocks vary fastest, so the CTAs resident together share W tiles (streamed in
// step) and the panel's H blocks (group·128·K·2 bytes) stay L2-resident.  Split x covers vocab
// tiles [x·tps, min(ntiles, (x+1)·tps)).
// Writes the split's partial (max, Σexp) per token into pm/ps [gridDim.y][T]; the split
// owning the sampled token writes x_tok directly.
// MODE 0 (stats): partial (max, Σexp) per split + the sampled logit.
// MODE 1 (dlogits): recompute the logits tile and write dlogit = k·(1[v = tok] − exp(x − lse))
//         as bf16 rows of stride dl_stride (the input of the backward GEMMs); lse/coef per token.
// ---------------------------------------------------------------------------
// 2-CTA sweep: a cluster pair computes a
// 256 x 256 tile with tcgen05.mma.cta_group::2 (M = 256, N = 256); each CTA stages its
// own 128 H rows and half (128 rows) of the W tile, so operand traffic per FLOP halves.
// The leader (rank 0) issues the MMAs; its full barriers collect both CTAs' TMA bytes;
// commits multicast to both CTAs; each CTA's epilogue reads its own 128 accumulator
// rows and releases the buffer on the leader's barrier.
// ---------------------------------------------------------------------------
namespace {
constexpr int kL2Stages = 6;
constexpr uint32_t kL2AStage = 128 * kLmK * 2, kL2BStage = 128 * kLmK * 2;  // 16 KB + 16 KB
constexpr uint32_t kL2StageBytes = kL2AStage + kL2BStage;
constexpr size_t kL2Smem = static_cast<size_t>(kL2Stages) * kL2StageBytes + 1024 + 256;
constexpr uint32_t kL2Idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(256 >> 3) << 17) |
                              (static_cast<uint32_t>(256 >> 4) << 24);

__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar & 0xFEFFFFFFu)
        : "memory");
}
__device__ __forceinline__ void umma_f16_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}
}  // namespace

template <int MODE>
__global__ void __launch_bounds__(192, 1)
    lmhead2_kernel(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmW,
                   const int32_t* __restrict__ tok, int64_t T, int32_t V, int32_t K, int32_t tps,
                   float* __restrict__ pm, float* __restrict__ ps, float* __restrict__ xtok, int32_t nsplit,
                   int32_t group, const double* __restrict__ lse_in, const double* __restrict__ coef,
                   __nv_bfloat16* __restrict__ dl, int64_t dl_stride) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    const uint32_t bars = sbase + kL2Stages * kL2StageBytes;
    const uint32_t full = bars, empty = bars + 8 * kL2Stages;
    const uint32_t acc_full = bars + 16 * kL2Stages, acc_empty = acc_full + 16;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + (acc_empty + 16 - raw));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    // (256-token pair block, vocab split) of this cluster, grouped raster as in lmhead_kernel
    const int64_t nblk = (T + 255) / 256;
    const int64_t cidx = blockIdx.x >> 1;
    const int64_t per_panel = static_cast<int64_t>(group) * nsplit;
    const int64_t panel = cidx / per_panel, in_panel = cidx % per_panel;
    const int64_t g0 = panel * group, gsz = (nblk - g0 < group) ? (nblk - g0) : static_cast<int64_t>(group);
    const int64_t blk = g0 + in_panel % gsz;
    const int split = static_cast<int>(in_panel / gsz);
    const int64_t row0 = blk * 256 + 128 * rank;
    const int ntiles_all = (V + kLmN - 1) / kLmN, nk = K / kLmK;
    const int nbeg = split * tps;
    const int ntiles = max(0, min(ntiles_all, nbeg + tps) - nbeg);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kL2Stages; ++s) {
            mbar_init(full + 8 * s, 1);
            mbar_init(empty + 8 * s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(acc_full + 8 * b, 1);
            mbar_init(acc_empty + 8 * b, 8);  // four epilogue warps in each CTA of the pair
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // TMA producer (both CTAs): own H rows + own half of the W tile
            uint32_t it = 0;
            for (int n = 0; n < ntiles; ++n) {
                for (int kc = 0; kc < nk; ++kc, ++it) {
                    const uint32_t s = it % kL2Stages;
                    if (it >= static_cast<uint32_t>(kL2Stages)) mbar_wait(empty + 8 * s, ((it / kL2Stages) - 1) & 1);
                    const uint32_t a = sbase + s * kL2StageBytes, b = a + kL2AStage;
                    if (rank == 0) mbar_arrive_expect_tx(full + 8 * s, 2 * kL2StageBytes);  // both CTAs' bytes
                    tma_load_2d_pair(a, &tmH, kc * kLmK, static_cast<int>(row0), full + 8 * s);
                    tma_load_2d_pair(b, &tmW, kc * kLmK, (nbeg + n) * kLmN + 128 * static_cast<int>(rank), full + 8 * s);
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0 && lane == 0) {  // MMA issuer (leader CTA only)
            uint32_t it = 0;
            for (int n = 0; n < ntiles; ++n) {
                const uint32_t buf = n & 1;
                if (n >= 2) mbar_wait(acc_empty + 8 * buf, ((n >> 1) - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t d = tmem + buf * kLmN;
                for (int kc = 0; kc < nk; ++kc, ++it) {
                    const uint32_t s = it % kL2Stages;
                    mbar_wait(full + 8 * s, (it / kL2Stages) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t a = sbase + s * kL2StageBytes, b = a + kL2AStage;
#pragma unroll
                    for (int k = 0; k < kLmK / 16; ++k)
                        umma_f16_pair(d, smem_desc_sw128(a + 32 * k), smem_desc_sw128(b + 32 * k), kL2Idesc,
                                      (kc > 0 || k > 0) ? 1u : 0u);
                    umma_commit_pair(empty + 8 * s);
                }
                umma_commit_pair(acc_full + 8 * buf);
            }
        }
    } else {
        const int q = warp & 3;
        const int64_t row = row0 + 32 * q + lane;
        const int32_t tk = row < T ? tok[row] : -1;
        const float L = 1.4426950408889634f;
        float m = -CUDART_INF_F, ssum = 0.0f, xt = 0.0f;
        const uint32_t acc_empty_leader = mapa(acc_empty, 0);
        const float lseL = (MODE == 1 && row < T) ? static_cast<float>(lse_in[row] * 1.4426950408889634) : 0.0f;
        const double kd = (MODE == 1 && row < T) ? coef[row] : 0.0;
        const float negk = static_cast<float>(-kd);
        __nv_bfloat16* drow = (MODE == 1 && row < T) ? dl + row * dl_stride : nullptr;
        const bool st256 = MODE == 1 && (dl_stride * 2) % 32 == 0 && (reinterpret_cast<uintptr_t>(dl) & 31) == 0;
        for (int n = 0; n < ntiles; ++n) {
            const uint32_t buf = n & 1;
            mbar_wait_sleep(acc_full + 8 * buf, (n >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * q) << 16) + buf * kLmN;
#pragma unroll 1
            for (int c = 0; c < kLmN; c += 32) {
                float v[32];
                tmem_ld32(taddr + c, v);
                const int col0 = (nbeg + n) * kLmN + c;
                if constexpr (MODE == 1) {
                    if (drow == nullptr) continue;
                    dl_store_chunk(drow, v, col0, V, tk, negk, kd, lseL, lse_in[row], st256);
                    continue;
                }
                float cm = -CUDART_INF_F;
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (col0 + i < V) cm = fmaxf(cm, v[i]);
                const float mn = fmaxf(m, cm);
                float acc = 0.0f;
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (col0 + i < V) acc += ex2_approx((v[i] - mn) * L);
                ssum = (m == -CUDART_INF_F ? 0.0f : ssum * ex2_approx((m - mn) * L)) + acc;
                m = mn;
                if (tk >= col0 && tk < col0 + 32) {
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (tk == col0 + i) xt = v[i];
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                 acc_empty_leader + 8 * buf)
                             : "memory");
        }
        if (MODE == 0 && row < T) {
            pm[static_cast<int64_t>(split) * T + row] = m;
            ps[static_cast<int64_t>(split) * T + row] = ssum;
            if (tk >= nbeg * kLmN && tk < (nbeg + ntiles) * kLmN) xtok[row] = xt;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}

// token blocks per raster panel: their H blocks (128·K·2 bytes each) within ~64 MB of L2
int lm_group(int64_t nblk, int32_t K) {
    const int64_t per = static_cast<int64_t>(kLmM) * K * 2;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(nblk, (64LL << 20) / per)));
}

bool make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kLmK), box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// lse[t] = M + ln Σ_s ps[s][t]·exp(pm[s][t] - M), M = max_s pm[s][t] (fixed split order)
__global__ void lmhead_combine_kernel(const float* __restrict__ pm, const float* __restrict__ ps, int32_t nsplit,
                                      int64_t T, double* __restrict__ lse) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= T) return;
    float M = -CUDART_INF_F;
    for (int s = 0; s < nsplit; ++s) M = fmaxf(M, pm[s * T + t]);
    double S = 0.0;
    for (int s = 0; s < nsplit; ++s) {
        const float m = pm[s * T + t];
        if (m != -CUDART_INF_F) S += static_cast<double>(ps[s * T + t]) * exp(static_cast<double>(m - M));
    }
    lse[t] = static_cast<double>(M) + log(S);  // fp64: lp = x_tok - lse keeps the 1e-5 relative budget
}

namespace {

// One 2-CTA sweep over the vocabulary: token pairs of 256 rows x vocab splits, split so
// that pairs x splits fill the SMs for ~8 waves; grouped raster for L2 reuse of W.
template <int MODE>
cudaError_t launch_lmhead2(const void* H, const void* W, const int32_t* tok, int64_t T, int32_t V, int32_t K,
                           float* pm, float* ps, float* xtok, const double* lse, const double* coef,
                           __nv_bfloat16* dl, int64_t dl_stride, int* nsplit_out, cudaStream_t st) {
    if (K % kLmK != 0 || T <= 0 || V <= 0) return cudaErrorInvalidValue;
    CUtensorMap mh, mw;
    if (!make_map(&mh, H, static_cast<uint64_t>(T), static_cast<uint64_t>(K), kLmM)) return cudaErrorInvalidValue;
    if (!make_map(&mw, W, static_cast<uint64_t>(V), static_cast<uint64_t>(K), 128)) return cudaErrorInvalidValue;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t nblk = (T + kLmM - 1) / kLmM;
    const int ntiles = (V + kLmN - 1) / kLmN;
    int nsplit = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ntiles, (8LL * sms + nblk - 1) / nblk)));
    const int tps = (ntiles + nsplit - 1) / nsplit;
    nsplit = (ntiles + tps - 1) / tps;
    if (nsplit_out) *nsplit_out = nsplit;
    if (MODE == 0 && !pm) return cudaSuccess;  // sizing query
    cudaError_t e = cudaFuncSetAttribute(lmhead2_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kL2Smem));
    if (e != cudaSuccess) return e;
    const int64_t npair = (T + 255) / 256;
    const int group2 = std::max(1, lm_group(npair, K) / 2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(2 * npair * nsplit));
    cfg.blockDim = dim3(192);
    cfg.dynamicSmemBytes = kL2Smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, lmhead2_kernel<MODE>, mh, mw, tok, T, V, K, tps, pm, ps, xtok, nsplit, group2,
                              lse, coef, dl, dl_stride);
}

}  // namespace

cudaError_t launch_lmhead_lse(const void* H, const void* W, const int32_t* tok, int64_t T, int32_t V, int32_t K,
                              double* lse, float* xtok, cudaStream_t st) {
    int nsplit = 0;
    cudaError_t e = launch_lmhead2<0>(H, W, tok, T, V, K, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0,
                                      &nsplit, st);
    if (e != cudaSuccess) return e;
    float* part = nullptr;
    e = cudaMallocAsync(&part, static_cast<size_t>(2) * nsplit * T * sizeof(float), st);
    if (e != cudaSuccess) return e;
    e = launch_lmhead2<0>(H, W, tok, T, V, K, part, part + static_cast<size_t>(nsplit) * T, xtok, nullptr, nullptr,
                          nullptr, 0, nullptr, st);
    if (e == cudaSuccess) {
        lmhead_combine_kernel<<<static_cast<unsigned>((T + 255) / 256), 256, 0, st>>>(
            part, part + static_cast<size_t>(nsplit) * T, nsplit, T, lse);
        e = cudaGetLastError();
    }
    cudaFreeAsync(part, st);
    return e;
}

cudaError_t launch_lmhead_dlogits(const void* H, const void* W, const int32_t* tok, int64_t T, int32_t V, int32_t K,
                                  const double* lse, const double* coef, void* dlogits, int64_t dl_stride,
                                  cudaStream_t st) {
    if ((dl_stride * 2) % 16 != 0) return cudaErrorInvalidValue;
    return launch_lmhead2<1>(H, W, tok, T, V, K, nullptr, nullptr, nullptr, lse, coef,
                             static_cast<__nv_bfloat16*>(dlogits), dl_stride, nullptr, st);
}

}  // namespace rf
