// common.cuh -- small device/host helpers shared by the libgfwa kernels.
// (Part of the CUDA path only; the fp64 oracle under oracle/ shares nothing.)
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>

#include "../../include/gfwa.h"

namespace gfwa {

// ---------------------------------------------------------------- host side

// Counts kernel launches issued through the library (gfwa_launch_count()).
void note_launch(int n = 1);
// measurement hook (gfwa_debug_stage_events): records the calling thread's
// registered event for `stage` on `st`, if one is registered, and clears it
void stage_event(int stage, cudaStream_t st);
// Records a CUDA error for gfwa_last_cuda_error(); returns GFWA_ERR_CUDA if err.
gfwa_status_t check_launch(cudaError_t err);
inline gfwa_status_t check_launch() { return check_launch(cudaGetLastError()); }

// Argument check: returns INVALID_ARGUMENT; with GFWA_DEBUG set, says which.
#define GFWA_REQUIRE(cond)                                                                       \
    do {                                                                                         \
        if (!(cond)) {                                                                           \
            if (getenv("GFWA_DEBUG")) fprintf(stderr, "gfwa: %s:%d: failed %s\n", __FILE__, __LINE__, #cond); \
            return GFWA_ERR_INVALID_ARGUMENT;                                                    \
        }                                                                                        \
    } while (0)

// ---------------------------------------------------------------- device side

template <typename T>
__device__ __forceinline__ float to_f32(T x);
template <>
__device__ __forceinline__ float to_f32<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T>
__device__ __forceinline__ T from_f32(float x);
template <>
__device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float exp2f_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// softplus(z) = max(z,0) + log1p(exp(-|z|))  (Alg. 1 l.6; reading C-6)
// Accurate expf/log1pf: the gate kernels are HBM-bound, so full-precision
// math is free and keeps U within the 1e-6 relative target.
__device__ __forceinline__ float softplus_f(float z) { return fmaxf(z, 0.f) + log1pf(expf(-fabsf(z))); }
__device__ __forceinline__ float sigmoid_f(float z) { return 1.f / (1.f + expf(-z)); }

// softplus(z) = max(z,0) + log1p(u), u = exp(-|z|) in (0, 1], with ~15
// instructions: u by MUFU.EX2 (relative error <= |z| 4e-8 + 2 ulp), and
// log1p(u) = 2 atanh(s), s = u/(2+u) in [0, 1/3], by its odd series in
// t = s^2 <= 1/9 through s^13 (truncation 3e-8 relative).  Relative error
// ~1e-7 over the whole range: the fp32 gate path stays inside the 1e-6
// relative target on U (sums of positive terms keep the relative error).
// u = exp(-|z|) in (0, 1]: -|z| log2(e) split exactly as n + f (n integer,
// |f| <= 1/2) so the argument rounding does not grow with |z|.  n is rounded
// with the 1.5 * 2^23 magic add (FMA pipe) and read back from the mantissa
// bits, so the only XU instruction is the MUFU.EX2.
__device__ __forceinline__ float exp_neg_abs(float z) {
    const float kMagic = 12582912.0f;  // 1.5 * 2^23
    const float x = fmaxf(-fabsf(z), -87.f);
    const float tm = fmaf(x, 1.4426950408889634f, kMagic);  // rint(x log2e) in the low mantissa bits
    const float n = tm - kMagic;
    const float f = fmaf(x, 1.4426950408889634f, -n) + x * 1.925963033500041e-08f;  // log2(e) - fp32(log2(e))
    const int ni = __float_as_int(tm) - __float_as_int(kMagic);                     // n >= -126: normal result
    return __int_as_float(__float_as_int(exp2f_approx(f)) + (ni << 23));
}

// log1p(u) for u in (0, 1]: 2 atanh(s), s = u/(2+u) in [0, 1/3], odd series in t = s^2
__device__ __forceinline__ float log1p_unit(float u) {
    const float s = __fdividef(u, 2.f + u);
    const float t = s * s;
    float p = 1.f / 13.f;
    p = fmaf(p, t, 1.f / 11.f);
    p = fmaf(p, t, 1.f / 9.f);
    p = fmaf(p, t, 1.f / 7.f);
    p = fmaf(p, t, 1.f / 5.f);
    p = fmaf(p, t, 1.f / 3.f);
    p = fmaf(p, t, 1.f);
    return 2.f * s * p;
}

__device__ __forceinline__ float softplus_fast(float z) { return fmaxf(z, 0.f) + log1p_unit(exp_neg_abs(z)); }

// softplus(z) and sigmoid(z) from one u = exp(-|z|) (the gate chain rule needs both)
__device__ __forceinline__ void softplus_sigmoid_fast(float z, float& sp, float& sg) {
    const float u = exp_neg_abs(z);
    sp = fmaxf(z, 0.f) + log1p_unit(u);
    const float r = __fdividef(1.f, 1.f + u);
    sg = z >= 0.f ? r : u * r;
}

// sigmoid(z) from u = exp(-|z|): 1/(1+u) or u/(1+u) (no cancellation)
__device__ __forceinline__ float sigmoid_fast(float z) {
    const float u = exp2f_approx(-fabsf(z) * 1.4426950408889634f);
    const float r = __fdividef(1.f, 1.f + u);
    return z >= 0.f ? r : u * r;
}

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

}  // namespace gfwa
