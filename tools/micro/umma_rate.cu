// Microbenchmark: tcgen05.mma (kind::f16, bf16 in, fp32 accum, cta_group::1) issue-to-
// completion time per instruction for the shapes the attention kernels use: SS
// (A and B from shared memory) vs TS (A from TMEM), M = 128, N = 64 / 128 / 256.
// One CTA per SM, one elected thread issues `reps` MMAs, commit + wait, clock64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2512_07782_b200/csrc \
//        -o /tmp/umma tools/micro/umma_rate.cu -lcuda && /tmp/umma
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace gfwa::sm100;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) k(long long* out, int reps) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t tm;
    for (int i = threadIdx.x; i < 65536 / 16; i += 128) sts128(smem_u32(smem) + i * 16, make_uint4(0, 0, 0, 0));
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    fence_proxy_async();
    if (threadIdx.x < 32) { tmem_alloc(&tm, 512); tmem_relinquish(); }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t t = tm;
    long long dt = 0;
    if (threadIdx.x < 32) {
        const uint32_t id = idesc_bf16(128, N, false, TS);
        const uint32_t a = smem_u32(smem), b = a + 32768;
        for (int pass = 0; pass < 2; ++pass) {
            long long t0 = clock64();
            if (elect_one()) {
                for (int r = 0; r < reps; ++r) {
                    const uint32_t kk = r & 7;
                    if (TS) mma_ts(t + (N >= 256 ? 0 : 256), t + 8 * kk, sdesc_sw128(b + kk * 2048, 16384, 1024), id, 1u);
                    else mma_ss(t + (N >= 256 ? 0 : 256), sdesc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                                sdesc_sw128(b + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), id, 1u);
                }
                tc_commit(&bar);
            }
            __syncwarp();
            mbar_wait(&bar, pass & 1);
            dt = clock64() - t0;
        }
        if (threadIdx.x == 0) out[blockIdx.x] = dt;
    }
    tc_fence_before(); __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(t, 512); }
}

template <int N, bool TS>
void run(const char* name, int reps) {
    long long* d; cudaMalloc(&d, 148 * 8);
    auto kern = k<N, TS>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 70656);
    kern<<<148, 128, 70656>>>(d, reps);
    long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0; for (long long v : h) s += v;
    s /= 148;
    const double flop = 2.0 * 128 * N * 16;
    printf("%-22s reps %5d: %8.1f clk total, %6.1f clk/MMA, %6.0f flop/clk/SM (%s)\n", name, reps, s, s / reps,
           flop * reps / s, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    for (int reps : {18, 64, 256}) {
        run<64, false>("SS M128 N64 K16", reps);
        run<128, false>("SS M128 N128 K16", reps);
        run<64, true>("TS M128 N64 K16", reps);
        run<128, true>("TS M128 N128 K16", reps);
    }
    return 0;
}
