// tc_selftest.cu -- diagnostic entry point that exercises exactly the
// primitives the attention kernels are built from (TMA 128B-swizzle tile
// loads, K-major SS MMA, TMEM ld/st, bf16 P written to TMEM and consumed as
// the A operand of a TS MMA against an MN-major B) on one 128x128x128 tile:
//   S = Q K^T (fp32, TMEM),  P = bf16(S) (TMEM),  O = P V (fp32, TMEM).
// tests/test_gpu_tc_selftest.py compares S and O with torch.matmul.
#include <cuda_fp16.h>

#include "common.cuh"
#include "sm100.cuh"
#include "tma_host.cuh"

namespace gfwa {
namespace {

using namespace sm100;

constexpr uint32_t kTile = 128 * 128 * 2;  // one bf16 128x128 tile (two 64-col boxes)

__global__ void __launch_bounds__(192, 1) selftest_kernel(const __grid_constant__ CUtensorMap mq,
                                                          const __grid_constant__ CUtensorMap mk,
                                                          const __grid_constant__ CUtensorMap mv, float* S_out,
                                                          float* O_out, int flags) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* Qs = smem;
    uint8_t* Ks = smem + kTile;
    uint8_t* Vs = smem + 2 * kTile;
    __shared__ uint64_t bar_load, bar_s, bar_p, bar_o;
    __shared__ uint32_t tmem_base_sh;
    const int warp = threadIdx.x >> 5;

    if (threadIdx.x == 0) {
        mbar_init(&bar_load, 1);
        mbar_init(&bar_s, 1);
        mbar_init(&bar_p, 4);
        mbar_init(&bar_o, 1);
        fence_barrier_init();
    }
    if (warp == 4) {
        tmem_alloc(&tmem_base_sh, 256);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    if (warp == 5) {
        if (elect_one()) {
            mbar_expect_tx(&bar_load, 3 * kTile);
            for (int half = 0; half < 2; ++half) {
                tma_load_4d(Qs + half * (kTile / 2), &mq, &bar_load, half * 64, 0, 0, 0);
                tma_load_4d(Ks + half * (kTile / 2), &mk, &bar_load, half * 64, 0, 0, 0);
                tma_load_4d(Vs + half * (kTile / 2), &mv, &bar_load, half * 64, 0, 0, 0);
            }
        }
    } else if (warp == 4) {
        mbar_wait(&bar_load, 0);
        tc_fence_after();
        if (elect_one()) {
            const uint32_t idesc_qk = idesc_bf16(128, 128, false, false);
            for (int k = 0; k < 8; ++k) {
                const uint32_t off = (k >> 2) * (kTile / 2) + (k & 3) * 32;
                mma_ss(tmem, sdesc_sw128(smem_u32(Qs) + off, 16, 1024), sdesc_sw128(smem_u32(Ks) + off, 16, 1024),
                       idesc_qk, k > 0);
            }
            tc_commit(&bar_s);
        }
        __syncwarp();
        mbar_wait(&bar_p, 0);
        tc_fence_after();
        if (elect_one()) {
            // flags & 1: P is fp16 in TMEM (A format F16) against bf16 V (B format BF16)
            const uint32_t idesc_pv = idesc_bf16(128, 128, false, true) & ~((flags & 1) ? (7u << 7) : 0u);
            for (int k = 0; k < 8; ++k) {
                // A = P columns [8k, 8k+8) (16 bf16 keys); B = V rows [16k, 16k+16)
                mma_ts(tmem + 128, tmem + k * 8, sdesc_sw128(smem_u32(Vs) + k * 2048, kTile / 2, 1024),
                       idesc_pv, k > 0);
            }
            tc_commit(&bar_o);
        }
        __syncwarp();
    } else {
        // warps 0-3: one thread per row (TMEM lane)
        const int row = warp * 32 + (threadIdx.x & 31);
        const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
        mbar_wait(&bar_s, 0);
        tc_fence_after();
        float s[128];
        for (int c = 0; c < 128; c += 32) {
            uint32_t r[32];
            tmem_ld32(lane_addr + c, r);
            tmem_wait_ld();
            for (int i = 0; i < 32; ++i) s[c + i] = __uint_as_float(r[i]);
        }
        for (int c = 0; c < 128; ++c) S_out[row * 128 + c] = s[c];
        for (int c = 0; c < 64; c += 32) {
            uint32_t r[32];
            for (int i = 0; i < 32; ++i) {
                if (flags & 1) {
                    const __half2 hv = __floats2half2_rn(s[2 * (c + i)], s[2 * (c + i) + 1]);
                    r[i] = *reinterpret_cast<const uint32_t*>(&hv);
                } else {
                    r[i] = pack_bf16x2(s[2 * (c + i)], s[2 * (c + i) + 1]);
                }
            }
            tmem_st32(lane_addr + c, r);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&bar_p);
        mbar_wait(&bar_o, 0);
        tc_fence_after();
        for (int c = 0; c < 128; c += 32) {
            uint32_t r[32];
            tmem_ld32(lane_addr + 128 + c, r);
            tmem_wait_ld();
            for (int i = 0; i < 32; ++i) O_out[row * 128 + c + i] = __uint_as_float(r[i]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 4) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

}  // namespace
}  // namespace gfwa

using namespace gfwa;

// Q, K, V: [128, 128] bf16 row-major device arrays; S_out, O_out: [128,128] fp32.
extern "C" gfwa_status_t gfwa_debug_tc_selftest_ex(const void* Q, const void* K, const void* V, float* S_out,
                                                   float* O_out, int flags, gfwa_stream_t stream) {
    if (!Q || !K || !V || !S_out || !O_out) return GFWA_ERR_INVALID_ARGUMENT;
    CUtensorMap mq, mk, mv;
    const int64_t st[3] = {128 * 128, 128, 128};
    if (!encode_bnhd_map(&mq, Q, 1, 128, 1, 128, st, 128) || !encode_bnhd_map(&mk, K, 1, 128, 1, 128, st, 128) ||
        !encode_bnhd_map(&mv, V, 1, 128, 1, 128, st, 128))
        return GFWA_ERR_INVALID_ARGUMENT;
    const size_t smem = 3 * kTile + 1024;
    cudaFuncSetAttribute(selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    selftest_kernel<<<1, 192, smem, (cudaStream_t)stream>>>(mq, mk, mv, S_out, O_out, flags);
    note_launch();
    return check_launch();
}

extern "C" gfwa_status_t gfwa_debug_tc_selftest(const void* Q, const void* K, const void* V, float* S_out,
                                                float* O_out, gfwa_stream_t stream) {
    return gfwa_debug_tc_selftest_ex(Q, K, V, S_out, O_out, 0, stream);
}
