// fp64_lat.cu — latency of dependent fp64 operations on one lane (the scalar warp's
// situation in the lag kernel), alone and next to warps running an ex2/FFMA2/F2F
// stream like the consumers'.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_fp64_lat tools/fp64_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(int n, int mode, int nbg, double* out, long long* cyc) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        if (lane != 0) return;
        double x = out[0] + 1.0, y = out[1] + 0.5;
        const long long t0 = clock64();
        for (int i = 0; i < n; ++i) {
            if (mode == 0) x = fma(x, 0.999999, 1e-9);        // DFMA chain
            else if (mode == 1) x = x + y * 1e-12;              // DMUL + DADD
            else if (mode == 2) x = 1.0 / (x + 1.0) + 1.0;      // IEEE division
            else if (mode == 3) x = exp(x * 1e-6);              // exp(double)
            else x = log2(x + 2.0);                             // log2(double)
        }
        cyc[0] = clock64() - t0;
        out[2] = x;
    } else if (warp <= nbg) {
        // background: consumer-like sweep (f32 FMA + ex2 + f64 accumulate)
        float a = lane * 1e-3f;
        double s = 0.0;
        for (int i = 0; i < n * 8; ++i) {
            float e;
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(a * -0.01f));
            a = fmaf(a, 0.9999f, e * 1e-6f);
            s += static_cast<double>(e);
        }
        out[3 + threadIdx.x] = s + a;
    }
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 4096 * sizeof(double));
    cudaMalloc(&cyc, 8);
    cudaMemset(out, 0, 4096 * sizeof(double));
    const char* names[] = {"dfma", "dmul+dadd", "div", "exp", "log2"};
    for (int mode = 0; mode < 5; ++mode) {
        for (int nbg : {0, 12}) {
            const int n = 2000;
            lat<<<148, (nbg + 1) * 32>>>(n, mode, nbg, out, cyc);
            lat<<<148, (nbg + 1) * 32>>>(n, mode, nbg, out, cyc);
            cudaDeviceSynchronize();
            long long c = 0;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("%-10s background warps=%2d  %7.1f cycles/op\n", names[mode], nbg, static_cast<double>(c) / n);
        }
    }
    return 0;
}
