// tmem_bw.cu — TMEM load / store throughput per SM on this GPU (microbenchmark for
// the lag kernel's park / write phases, which move 2 bytes per element through TMEM).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_tmem_bw tools/tmem_bw.cu
// run (GPU box): ./tools/_tmem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int MODE>  // 0 = ld x16 (2 KB/warp-instr), 1 = st x16, 2 = ld x4 (512 B), 3 = st x4
__global__ void __launch_bounds__(512) tmem_bw(int iters, unsigned long long* cycles, uint32_t* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = slot;
    const int nw = blockDim.x >> 5;
    const uint32_t cols_per = 512u / ((nw + 3) / 4) / 16 * 16;
    const uint32_t tm = base + ((32u * (warp & 3)) << 16) + cols_per * (warp >> 2);
    uint32_t acc = 0;
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * i;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        for (uint32_t c = 0; c + 16 <= cols_per; c += 16) {
            if (MODE == 0) {
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                    "[%16];\n\ttcgen05.wait::ld.sync.aligned;"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                      "=r"(v[15])
                    : "r"(tm + c));
                acc += v[0] ^ v[15];
            } else if (MODE == 1) {
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16};" ::"r"(tm + c),
                    "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                    "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
            } else if (MODE == 2) {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(v[4 * q]), "=r"(v[4 * q + 1]), "=r"(v[4 * q + 2]), "=r"(v[4 * q + 3])
                                 : "r"(tm + c + 4 * q));
                asm volatile("tcgen05.wait::ld.sync.aligned;");
                acc += v[0] ^ v[15];
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(tm + c + 4 * q),
                                 "r"(v[4 * q]), "r"(v[4 * q + 1]), "r"(v[4 * q + 2]), "r"(v[4 * q + 3]));
            }
        }
    }
    if (MODE == 1 || MODE == 3) asm volatile("tcgen05.wait::st.sync.aligned;");
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) atomicAdd(cycles, static_cast<unsigned long long>(t1 - t0));
    if (acc == 0x12345678u) sink[0] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(512));
}

template <int MODE>
void run(int nwarps, const char* name) {
    unsigned long long* cyc;
    uint32_t* sink;
    cudaMalloc(&cyc, 8);
    cudaMalloc(&sink, 4);
    cudaMemset(cyc, 0, 8);
    const int iters = 2000;
    tmem_bw<MODE><<<148, nwarps * 32>>>(iters, cyc, sink);
    cudaMemset(cyc, 0, 8);
    tmem_bw<MODE><<<148, nwarps * 32>>>(iters, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double per_sm_cycles = static_cast<double>(c) / 148.0;
    const uint32_t cols_per = 512u / ((nwarps + 3) / 4) / 16 * 16;
    const double bytes = static_cast<double>(nwarps) * iters * (cols_per / 16) * 2048.0;
    printf("%-10s warps=%2d  %7.1f B/clk/SM  (%s)\n", name, nwarps, bytes / per_sm_cycles, cudaGetErrorString(e));
    cudaFree(cyc);
    cudaFree(sink);
}

int main() {
    for (int w : {4, 8, 12, 16}) {
        run<0>(w, "ld.x16");
        run<2>(w, "ld.4x4");
        run<1>(w, "st.x16");
        run<3>(w, "st.4x4");
    }
    return 0;
}
