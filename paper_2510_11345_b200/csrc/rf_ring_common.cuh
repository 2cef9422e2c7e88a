// rf_ring_common.cuh — device helpers shared by the ring kernels (packed f32x2 math,
// bf16/f16 vector conversions, masked tails, vectorised dlogits stores).
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

#include "rf_device.cuh"

namespace rf {
namespace ring {

constexpr float kL2e = 1.4426950408889634f;
constexpr double kLn2 = 0.69314718055994530942;

__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
    return static_cast<uint64_t>(__float_as_uint(lo)) | (static_cast<uint64_t>(__float_as_uint(hi)) << 32);
}
__device__ __forceinline__ float lo2(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v)); }
__device__ __forceinline__ float hi2(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v >> 32)); }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {  // one FADD2 with a negated operand
    uint64_t d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
// bf16x2 word -> packed f32x2 (exact)
__device__ __forceinline__ uint64_t bf16x2_to_f32x2(uint32_t w) {
    return static_cast<uint64_t>(w << 16) | (static_cast<uint64_t>(w & 0xffff0000u) << 32);
}

// (M, S) = running max and sum of exp(x - M).  Sums are rescaled in fp64.
__device__ __forceinline__ void combine_ms(float& M, double& S, float M2, double S2) {
    const float Mn = fmaxf(M, M2);
    if (Mn == -CUDART_INF_F) return;
    double s = 0.0;
    if (S != 0.0) s += S * exp(static_cast<double>(M - Mn));
    if (S2 != 0.0) s += S2 * exp(static_cast<double>(M2 - Mn));
    M = Mn;
    S = s;
}

__device__ __forceinline__ void warp_ms(float& M, double& S) {
    float Mw = M;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) Mw = fmaxf(Mw, __shfl_xor_sync(0xffffffffu, Mw, o));
    double s = (S != 0.0) ? S * exp(static_cast<double>(M - Mw)) : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    M = Mw;
    S = s;
}

template <bool IN_BF16>
__device__ __forceinline__ uint4 neg_inf_vec() {
    return IN_BF16 ? make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u)
                   : make_uint4(0xff800000u, 0xff800000u, 0xff800000u, 0xff800000u);
}

// The same fill built by volatile moves: the compiler may not hoist it out of the
// rarely taken branch it is written in (a plain constant fill was hoisted above the
// chunk loads and executed for every chunk of every row: 4 moves per vector).
template <bool IN_BF16>
__device__ __forceinline__ uint4 neg_inf_vec_here() {
    uint4 v;
    asm volatile("mov.b32 %0, %4;\n\tmov.b32 %1, %4;\n\tmov.b32 %2, %4;\n\tmov.b32 %3, %4;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "n"(IN_BF16 ? 0xff80ff80u : 0xff800000u));
    return v;
}

template <bool IN_BF16>
__device__ __forceinline__ void mask_tail(uint4& v, int valid) {
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
    if (IN_BF16) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            if (e >= valid) {
                const int wi = e >> 1;
                w[wi] = (e & 1) ? ((w[wi] & 0x0000ffffu) | 0xff800000u) : ((w[wi] & 0xffff0000u) | 0x0000ff80u);
            }
        }
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (e >= valid) w[e] = 0xff800000u;
    }
    v = make_uint4(w[0], w[1], w[2], w[3]);
}

template <bool IN_BF16>
__device__ __forceinline__ uint32_t vec_max2(const uint4& v) {
    // packed max of the vector's elements, result in both halves (bf16x2) / as f32 bits
    if (IN_BF16) {
        __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&v.x);
        __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&v.y);
        __nv_bfloat162 c = *reinterpret_cast<const __nv_bfloat162*>(&v.z);
        __nv_bfloat162 d = *reinterpret_cast<const __nv_bfloat162*>(&v.w);
        __nv_bfloat162 m = __hmax2(__hmax2(a, b), __hmax2(c, d));
        return *reinterpret_cast<uint32_t*>(&m);
    }
    return __float_as_uint(fmaxf(fmaxf(__uint_as_float(v.x), __uint_as_float(v.y)),
                                 fmaxf(__uint_as_float(v.z), __uint_as_float(v.w))));
}

// x -> e = 2^(x·L - C) in place (C = M·L); returns the vector's packed f32x2 partial sums.
template <bool IN_BF16>
__device__ __forceinline__ uint64_t vec_exp(uint4& v, uint64_t L2, uint64_t negC2) {
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
    if (IN_BF16) {
        uint64_t acc = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint64_t a = ffma2(bf16x2_to_f32x2(w[q]), L2, negC2);
            const float e0 = ex2_approx(lo2(a));
            const float e1 = ex2_approx(hi2(a));
            w[q] = pack_f16x2(e0, e1);
            acc = q == 0 ? pk2(e0, e1) : fadd2(acc, pk2(e0, e1));
        }
        v = make_uint4(w[0], w[1], w[2], w[3]);
        return acc;
    } else {
        const uint64_t a01 = ffma2(pk2(__uint_as_float(w[0]), __uint_as_float(w[1])), L2, negC2);
        const uint64_t a23 = ffma2(pk2(__uint_as_float(w[2]), __uint_as_float(w[3])), L2, negC2);
        const float e0 = ex2_approx(lo2(a01)), e1 = ex2_approx(hi2(a01));
        const float e2 = ex2_approx(lo2(a23)), e3 = ex2_approx(hi2(a23));
        v = make_uint4(__float_as_uint(e0), __float_as_uint(e1), __float_as_uint(e2), __float_as_uint(e3));
        return fadd2(pk2(e0, e1), pk2(e2, e3));
    }
}

// f16x2 e vector -> bf16x2 e·f (the staged dlogits vector of the TMA-store path)
__device__ __forceinline__ uint4 vec_out_bf16(const uint4& e, uint64_t f2) {
    const uint32_t w[4] = {e.x, e.y, e.z, e.w};
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float2 h = unpack_f16x2(w[q]);
        const uint64_t m = fmul2(pk2(h.x, h.y), f2);
        o[q] = pack_bf16x2(lo2(m), hi2(m));
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

template <bool OUT_BF16, int EPV>
__device__ __forceinline__ void store_vec(uint8_t* dst, const uint4& e, uint64_t f2, bool in_bf16) {
    if (in_bf16) {
        const uint32_t w[4] = {e.x, e.y, e.z, e.w};
        uint64_t o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float2 h = unpack_f16x2(w[q]);
            o[q] = fmul2(pk2(h.x, h.y), f2);
        }
        if (OUT_BF16) {
            stg128_cs(dst, make_uint4(pack_bf16x2(lo2(o[0]), hi2(o[0])), pack_bf16x2(lo2(o[1]), hi2(o[1])),
                                      pack_bf16x2(lo2(o[2]), hi2(o[2])), pack_bf16x2(lo2(o[3]), hi2(o[3]))));
        } else {
            stg128_cs(dst, make_uint4(static_cast<uint32_t>(o[0]), static_cast<uint32_t>(o[0] >> 32),
                                      static_cast<uint32_t>(o[1]), static_cast<uint32_t>(o[1] >> 32)));
            stg128_cs(dst + 16, make_uint4(static_cast<uint32_t>(o[2]), static_cast<uint32_t>(o[2] >> 32),
                                           static_cast<uint32_t>(o[3]), static_cast<uint32_t>(o[3] >> 32)));
        }
    } else {
        const uint64_t o0 = fmul2(pk2(__uint_as_float(e.x), __uint_as_float(e.y)), f2);
        const uint64_t o1 = fmul2(pk2(__uint_as_float(e.z), __uint_as_float(e.w)), f2);
        if (OUT_BF16)
            stg64_cs(dst, make_uint2(pack_bf16x2(lo2(o0), hi2(o0)), pack_bf16x2(lo2(o1), hi2(o1))));
        else
            stg128_cs(dst, make_uint4(static_cast<uint32_t>(o0), static_cast<uint32_t>(o0 >> 32),
                                      static_cast<uint32_t>(o1), static_cast<uint32_t>(o1 >> 32)));
    }
}

template <bool OUT_BF16, int EPV>
__device__ __forceinline__ void store_vec_partial(uint8_t* dst, const uint4& e, float f, bool in_bf16, int valid) {
    float out[EPV];
    if (in_bf16) {
        const uint32_t w[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float2 h = unpack_f16x2(w[q]);
            out[(2 * q) % EPV] = h.x * f;
            out[(2 * q + 1) % EPV] = h.y * f;
        }
    } else {
        out[0 % EPV] = __uint_as_float(e.x) * f;
        out[1 % EPV] = __uint_as_float(e.y) * f;
        out[2 % EPV] = __uint_as_float(e.z) * f;
        out[3 % EPV] = __uint_as_float(e.w) * f;
    }
#pragma unroll
    for (int q = 0; q < EPV; ++q) {
        if (q < valid) {
            if (OUT_BF16)
                reinterpret_cast<__nv_bfloat16*>(dst)[q] = __float2bfloat16_rn(out[q]);
            else
                reinterpret_cast<float*>(dst)[q] = out[q];
        }
    }
}

}  // namespace ring
}  // namespace rf
