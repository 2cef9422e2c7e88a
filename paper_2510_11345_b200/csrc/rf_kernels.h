// rf_kernels.h — launch entry points of rf_kernels.cu (internal to the library).
#pragma once
#include <cuda_runtime.h>

#include "rf_device.cuh"

namespace rf {

constexpr int kRingWarps = 8;   // consumer warps per CTA (+1 producer warp)
constexpr int kRingVPT = 4;     // 16-byte vectors per consumer thread per chunk
constexpr int kRingChunkVecs = kRingWarps * 32 * kRingVPT;
constexpr size_t kRingSlotBytes = static_cast<size_t>(kRingChunkVecs) * 16 + kRingWarps * 32 * 4;
constexpr size_t kRingTailBytes = 512;  // barriers' tail: exchange/reduce/broadcast words
constexpr int kGenericThreads = 256;
constexpr int kGenericMaxGrid = 148 * 8;

cudaError_t launch_ring(const KParams& p, bool in_bf16, bool out_bf16, int cs, int nclusters, size_t smem,
                        cudaStream_t st);
cudaError_t ring_max_clusters(bool in_bf16, bool out_bf16, int cs, size_t smem, int* out);
cudaError_t launch_generic(const KParams& p, bool in_bf16, bool out_bf16, int grid, cudaStream_t st);
cudaError_t launch_seq(const KParams& p, int64_t seq_begin, int64_t nseq, double* coef, cudaStream_t st);
cudaError_t launch_finalize(const double* partials, int64_t n, double* scalars, cudaStream_t st);
cudaError_t launch_grpo(const double* rewards, const int64_t* group_offsets, int64_t num_groups, double* adv,
                        uint8_t* degenerate, int32_t* status, cudaStream_t st);

}  // namespace rf
