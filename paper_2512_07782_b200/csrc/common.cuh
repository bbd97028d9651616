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

// softplus(z) = max(z,0) + log1p(exp(-|z|))  (Alg. 1 l.6; reading C-6)
// Accurate expf/log1pf: the gate kernels are HBM-bound, so full-precision
// math is free and keeps U within the 1e-6 relative target.
__device__ __forceinline__ float softplus_f(float z) { return fmaxf(z, 0.f) + log1pf(expf(-fabsf(z))); }
__device__ __forceinline__ float sigmoid_f(float z) { return 1.f / (1.f + expf(-z)); }

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

}  // namespace gfwa
