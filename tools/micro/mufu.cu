// Microbenchmark: MUFU.EX2, FFMA, FFMA2 (f32x2), F2FP (cvt bf16x2) throughput per SM
// (cycles via clock64, 1024 threads per SM, 8 independent chains per thread).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu tools/micro/mufu.cu && /tmp/mufu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ uint32_t cvt2(float a, float b) {
    uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b)); return r; }
template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
    float a[8]; uint64_t p[8]; uint32_t u = 0;
    for (int i = 0; i < 8; ++i) { a[i] = -(threadIdx.x * 1e-3f + i * 1e-2f); p[i] = (uint64_t)__float_as_uint(a[i]) | ((uint64_t)__float_as_uint(a[i]) << 32); }
    const uint64_t m = (uint64_t)__float_as_uint(0.999f) | ((uint64_t)__float_as_uint(0.999f) << 32);
    const uint64_t c = (uint64_t)__float_as_uint(1e-3f) | ((uint64_t)__float_as_uint(1e-3f) << 32);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) a[i] = ex2(a[i]);
            else if (MODE == 1) a[i] = fmaf(a[i], 0.999f, 1e-3f);
            else if (MODE == 2) p[i] = ffma2(p[i], m, c);
            else u += cvt2(a[i], a[(i + 1) & 7]);
        }
    }
    long long t1 = clock64();
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float((uint32_t)p[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + u;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 148 * 8);
    const int iters = 2048, threads = 1024;
    const char* names[] = {"MUFU.EX2", "FFMA", "FFMA2 (2 flops/lane)", "F2FP bf16x2"};
    for (int mode = 0; mode < 4; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) k<0><<<148, threads>>>(o, c, iters);
            else if (mode == 1) k<1><<<148, threads>>>(o, c, iters);
            else if (mode == 2) k<2><<<148, threads>>>(o, c, iters);
            else k<3><<<148, threads>>>(o, c, iters);
            cudaDeviceSynchronize();
        }
        long long h[148]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
        double ops = (double)threads * iters * 8;  // instructions x lanes
        printf("%-22s %.2f lane-instr/clk/SM\n", names[mode], ops / h[0]);
    }
    return 0;
}
