// Microbenchmark: tcgen05.ld / tcgen05.st throughput (32x32b.x32: 32 lanes x 32 columns
// of 32 bits = 4 KB per warp instruction) with W warps per CTA, one CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2512_07782_b200/csrc \
//        -o tools/micro/tmem tools/micro/tmem_rate.cu && tools/micro/tmem
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace gfwa::sm100;

template <bool ST>
__global__ void k(long long* out, float* sink, int reps) {
    __shared__ uint32_t tm;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) { tmem_alloc(&tm, 512); tmem_relinquish(); }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t t = tm + ((uint32_t)((warp & 3) * 32) << 16) + 32 * (warp >> 2);
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = i;
    float acc = 0.f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < reps; ++it) {
        if (ST) { tmem_st32(t, r); }
        else {
            tmem_ld32(t, r); tmem_wait_ld();
            float s0 = 0.f;
#pragma unroll
            for (int i = 0; i < 32; ++i) s0 += __uint_as_float(r[i]);
            acc += s0;
        }
    }
    if (ST) tmem_wait_st();
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 1.2345f) sink[threadIdx.x] = acc;
    tc_fence_before(); __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

template <bool ST>
void run(int warps, int reps) {
    long long* d; float* s; cudaMalloc(&d, 148 * 8); cudaMalloc(&s, 4096);
    k<ST><<<148, 32 * warps>>>(d, s, reps);
    long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double c = 0; for (long long v : h) c += v; c /= 148;
    const double bytes = 4096.0 * warps * reps;
    printf("%s warps %2d: %8.0f clk, %6.1f B/clk/SM (%s)\n", ST ? "tcgen05.st" : "tcgen05.ld+wait", warps, c, bytes / c,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d); cudaFree(s);
}
int main() {
    for (int w : {1, 4, 8, 16}) run<false>(w, 512);
    for (int w : {1, 4, 8, 16}) run<true>(w, 512);
    return 0;
}
