// tma_host.cuh -- host-side TMA tensor-map encoding for [B, N, H, d] bf16
// tensors (d contiguous, arbitrary (b, n, h) element strides).
#pragma once
#include <cuda.h>
#include <stdint.h>

#include "driver_api.cuh"

namespace gfwa {

// Box = {64 d-elements (128 B, one swizzle row), 1 head, rows, 1 batch},
// 128-byte swizzle, OOB rows zero-filled (ragged tails, halo edges).
inline bool encode_bnhd_map(CUtensorMap* map, const void* base, int64_t B, int64_t N, int64_t H, int d,
                            const int64_t* s /* element strides b, n, h */, int box_rows) {
    cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)H, (cuuint64_t)N, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)(s[2] * 2), (cuuint64_t)(s[1] * 2), (cuuint64_t)(s[0] * 2)};
    // size-1 dims may carry any stride; keep them legal (multiple of 16, non-zero)
    for (int i = 0; i < 3; ++i)
        if (strides[i] == 0) strides[i] = 16;
    cuuint32_t box[4] = {64u, 1u, (cuuint32_t)box_rows, 1u};
    cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
    CUresult r = drv::tensorMapEncodeTiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims,
                                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// fp32 [B, N, H, d] map with box {32 d-elements (128 B), 1, rows, 1}, 128B swizzle
// (the dQ reduce-add).
inline bool encode_bnhd_map_f32(CUtensorMap* map, const void* base, int64_t B, int64_t N, int64_t H, int d,
                                const int64_t* s, int box_rows) {
    cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)H, (cuuint64_t)N, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)(s[2] * 4), (cuuint64_t)(s[1] * 4), (cuuint64_t)(s[0] * 4)};
    for (int i = 0; i < 3; ++i)
        if (strides[i] == 0) strides[i] = 16;
    cuuint32_t box[4] = {32u, 1u, (cuuint32_t)box_rows, 1u};
    cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
    CUresult r = drv::tensorMapEncodeTiled(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims,
                                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// fp32 [B, H, d, Nq] map (queries contiguous, row pitch nq_pitch elements, a
// multiple of 4) with box {32 queries (128 B), d rows, 1, 1}, 128B swizzle: the
// transposed dQ accumulator of the tensor-core backward (a drain thread owns one
// d row of the dQ^T tile, so it stages whole 16-byte query runs).
inline bool encode_bhdn_map_f32(CUtensorMap* map, const void* base, int64_t B, int64_t H, int d, int64_t Nq,
                                int64_t nq_pitch, int box_q = 32, int box_d = 0) {
    cuuint64_t dims[4] = {(cuuint64_t)Nq, (cuuint64_t)d, (cuuint64_t)H, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)(nq_pitch * 4), (cuuint64_t)(nq_pitch * 4 * d),
                             (cuuint64_t)(nq_pitch * 4 * d * H)};
    cuuint32_t box[4] = {(cuuint32_t)box_q, (cuuint32_t)(box_d > 0 ? box_d : d), 1u, 1u};
    cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
    CUresult r = drv::tensorMapEncodeTiled(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims,
                                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        box_q == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace gfwa
