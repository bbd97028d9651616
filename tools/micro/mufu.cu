// Microbenchmark: MUFU.EX2 and FFMA2 throughput per SM (cycles via clock64).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-2f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) a[i] = ex2(a[i]) * -0.5f;       // MUFU + FMUL
            else a[i] = fmaf(a[i], 0.999f, 1e-3f);          // FFMA only
        }
    }
    long long t1 = clock64();
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4 * 4); cudaMalloc(&c, 148 * 4 * 8);
    int iters = 4096;
    for (int mode = 0; mode < 2; ++mode) for (int threads : {256, 512, 1024}) {
        if (mode == 0) k<0><<<148, threads>>>(o, c, iters); else k<1><<<148, threads>>>(o, c, iters);
        cudaDeviceSynchronize();
        long long h[148]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
        double ops = (double)threads * iters * 8;
        printf("mode %s threads %4d: %.2f ops/clk/SM\n", mode ? "FFMA" : "EX2+FMUL", threads, ops / h[0]);
    }
    return 0;
}
