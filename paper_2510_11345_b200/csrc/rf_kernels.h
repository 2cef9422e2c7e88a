// rf_kernels.h — launch entry points of the kernels (internal to the library).
#pragma once
#include <cuda_runtime.h>

#include "rf_device.cuh"

namespace rf {

// Lag configuration (rf_ring_lag.cu): NCW/4 consumer warpgroups + one support
// warpgroup (TMA producer, two scalar warps, one idle) that hands its registers to
// the consumers via setmaxnreg; one CTA per SM; the previous row's e parked in
// TMEM.  Default NCW = 12 (3 consumer warps per SMSP, 152 registers each).
constexpr int kRingWarpsLag = 12;
constexpr int kRingNvtLag[4] = {4, 11, 12, 25};  // instances for NCW = 12 (11: V = 32,000 bf16, one CTA per row)
// support warpgroup registers (32, giving the consumers 160, measured 10% slower)
constexpr int kLagRegsSupport = 56;
__host__ __device__ constexpr int lag_launch_regs(int ncw) {
    return ((65536 / ((ncw + 4) * 32)) / 8 * 8) > 248 ? 248 : ((65536 / ((ncw + 4) * 32)) / 8 * 8);
}
__host__ __device__ constexpr int lag_regs_consumer(int ncw) {
    return ((lag_launch_regs(ncw) * (ncw + 4) * 32 - 128 * kLagRegsSupport) / (ncw * 32)) / 8 * 8 > 248
               ? 248
               : ((lag_launch_regs(ncw) * (ncw + 4) * 32 - 128 * kLagRegsSupport) / (ncw * 32)) / 8 * 8;
}
__host__ __device__ constexpr unsigned lag_tmem_cols(int ncw) { return (512u / (ncw / 4)) / 8 * 8; }
// vectors per thread per TMA chunk of the lag kernels: 5 (30 KB chunks at 12
// consumer warps, measured best of {2,3,4,5,7,9,13}) for the long rows, 2 for NVT = 4
__host__ __device__ constexpr int lag_vpc(int nvt) { return nvt >= 9 ? 5 : 2; }
// exchange / reduce / broadcast words (+ the checked build's row tags at 1088: [2][16] + [2])
constexpr size_t kRingLagTailBytes = RF_CHECKED ? 1088 + 32 * 8 + 16 : 1088;
constexpr size_t kRingLagBarrierBytes = 48;

// Exact-KL lag kernel (rf_ring_kl.cu): policy and reference rows co-resident,
// 12 consumer warps, bf16 logits; NVT = 13 covers a quarter Qwen3 row (4-CTA cluster).
// 13: 4-CTA groups at V = 151,936 (larger groups lose: 5-CTA groups at NVT 10 -12%, 7-CTA at NVT 8 -40%,
// profiles/r02_ab/kl_group_and_exchange_ab.txt)
constexpr int kRingNvtKL[3] = {4, 10, 13};
// exact-KL CTA groups (GX): per group [4 row slots][8 ranks] x 40-byte exchange slots, then
// the group's row-claim ring (kRowQ 64-bit words); zeroed before every launch
constexpr size_t kKlGroupXchBytes = 32 * 40 + 64;
// [4][8] 40-byte exchange slots + 5 x [2][NCW] partials + broadcast (+ checked-build row tags)
constexpr size_t kRingKLTailBytes = RF_CHECKED ? 2304 + 2 * 16 * 8 + 16 : 2304;
cudaError_t launch_ring_kl(const KParams& p, bool out_bf16, int nvt, int cs, int nclusters, size_t smem,
                           cudaStream_t st);
cudaError_t ring_kl_max_clusters(bool out_bf16, int nvt, int cs, size_t smem, int* out);
// Experimental LM-head GEMM + fused softmax statistics (rf_lmhead.cu)
cudaError_t launch_lmhead_lse(const void* H, const void* W, const int32_t* tok, int64_t T, int32_t V, int32_t K,
                              double* lse, float* xtok, cudaStream_t st);
cudaError_t launch_lmhead_dlogits(const void* H, const void* W, const int32_t* tok, int64_t T, int32_t V, int32_t K,
                                  const double* lse, const double* coef, void* dlogits, int64_t dl_stride,
                                  cudaStream_t st);
cudaError_t launch_ring_lag(const KParams& p, bool in_bf16, bool out_bf16, int ncw, int nvt, int cs, int nclusters,
                            size_t smem, cudaStream_t st);
cudaError_t ring_lag_max_clusters(bool in_bf16, bool out_bf16, int ncw, int nvt, int cs, size_t smem, int* out);
constexpr int kGenericThreads = 256;
constexpr int kGenericMaxGrid = 148 * 8;
// finalize: up to this many partial rows in one block; more (one row per token from the
// lag kernels) first go through kFinalizeBlocks fixed-range block sums, written into the
// kFinalizeBlocks scratch rows that follow the partials
constexpr int64_t kFinalizeDirectRows = 4096;
constexpr int kFinalizeBlocks = 148;

cudaError_t launch_generic(const KParams& p, bool in_bf16, bool out_bf16, int grid, cudaStream_t st);
// K2w (rf_stream.cu): dlogits from per-token coef + lse (needs p.row_vecs, ring-compatible layout)
cudaError_t launch_stream_write(const KParams& p, bool in_bf16, bool out_bf16, cudaStream_t st);
// K2st (rf_stream.cu): stats pass of sequence_product (lse, lp per token), read-only online softmax
cudaError_t launch_stream_stats(const KParams& p, bool in_bf16, cudaStream_t st);
cudaError_t launch_seq(const KParams& p, int64_t seq_begin, int64_t nseq, double* coef, cudaStream_t st);
cudaError_t launch_token_loss(const KParams& p, const double* lse, const float* xtok, cudaStream_t st);
// K3: scalar reduce + the empty-trajectory check over the sequences this call spans
int finalize_launches(int64_t n);
cudaError_t launch_finalize(const double* partials, int64_t n, double* scalars, const int32_t* seq_of_token,
                            const int64_t* seq_offsets, int64_t num_tokens, int64_t num_seqs, int32_t* status,
                            cudaStream_t st);
cudaError_t launch_rows_segment_sum(const void* rows, bool bf16, int64_t row_stride, const int64_t* seg_offsets,
                                    const int32_t* seg_rows, int64_t num_segments, int32_t width, double* out,
                                    int64_t out_stride, cudaStream_t st);
cudaError_t launch_grpo(const double* rewards, const int64_t* group_offsets, int64_t num_groups, double* adv,
                        uint8_t* degenerate, int32_t* status, cudaStream_t st);

}  // namespace rf
