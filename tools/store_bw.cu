// store_bw.cu — SM -> L2 write bandwidth per SM on B200: 128-bit STG from registers
// (the dlogits write path of K2) against TMA bulk stores from shared memory
// (cp.async.bulk.global.shared::cta), each SM writing its own contiguous region.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_store_bw tools/store_bw.cu && tools/_store_bw
// The writes total 8 GB per launch (HBM-resident region >> L2), and, as a second
// case, 64 MB rewritten 128 times (L2-resident: the SM->L2 path alone).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) stg_kernel(uint4* out, size_t per_sm_vecs, int reps, size_t wrap_vecs) {
    const uint4 v = make_uint4(threadIdx.x, blockIdx.x, 1, 2);
    for (int r = 0; r < reps; ++r) {
        uint4* base = out + (static_cast<size_t>(blockIdx.x) * per_sm_vecs) % wrap_vecs;
        for (size_t i = threadIdx.x; i < per_sm_vecs; i += blockDim.x)
            asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(base + i), "r"(v.x),
                         "r"(v.y), "r"(v.z), "r"(v.w)
                         : "memory");
    }
}

constexpr uint32_t kChunk = 32768;  // bytes per bulk store
__global__ void __launch_bounds__(128, 1) tma_kernel(uint8_t* out, size_t per_sm_bytes, int reps, size_t wrap_bytes) {
    extern __shared__ __align__(128) uint8_t sm[];
    for (uint32_t i = threadIdx.x; i < 4 * kChunk / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(sm)[i] = make_uint4(i, blockIdx.x, 3, 4);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int r = 0; r < reps; ++r) {
            uint8_t* base = out + (static_cast<size_t>(blockIdx.x) * per_sm_bytes) % wrap_bytes;
            for (size_t off = 0; off < per_sm_bytes; off += kChunk) {
                const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(sm + ((off / kChunk) % 4) * kChunk));
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(base + off),
                             "r"(src), "r"(kChunk)
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");  // up to 4 in flight
            }
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const size_t total = 8ull << 30;
    uint8_t* buf = nullptr;
    if (cudaMalloc(&buf, total) != cudaSuccess) return 1;
    cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kChunk);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    struct Case {
        const char* name;
        size_t per_sm, wrap;
        int reps;
    } cases[] = {{"HBM (8 GB region)", (total / sms) / kChunk * kChunk, total, 1},
                 {"L2-resident (64 MB region, 128 passes)", ((64ull << 20) / sms) / kChunk * kChunk, 64ull << 20, 128}};
    for (const Case& c : cases) {
        for (int k = 0; k < 2; ++k) {
            float best = 1e30f;
            for (int it = 0; it < 5; ++it) {
                cudaEventRecord(a);
                if (k == 0)
                    stg_kernel<<<sms, 512>>>(reinterpret_cast<uint4*>(buf), c.per_sm / 16, c.reps, c.wrap / 16);
                else
                    tma_kernel<<<sms, 128, 4 * kChunk>>>(buf, c.per_sm, c.reps, c.wrap);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms = 0.f;
                cudaEventElapsedTime(&ms, a, b);
                best = ms < best ? ms : best;
            }
            const double bytes = static_cast<double>(c.per_sm) * sms * c.reps;
            const double gbs = bytes / (best * 1e-3) / 1e9;
            std::printf("%-40s %-16s %8.3f ms  %8.1f GB/s  %6.1f B/clk/SM (at the %d MHz boost clock)\n", c.name,
                        k == 0 ? "STG.128" : "TMA bulk store", best, gbs, gbs * 1e9 / sms / (clk * 1e3), clk / 1000);
        }
    }
    const cudaError_t e = cudaDeviceSynchronize();
    std::printf("status: %s\n", cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 2;
}
