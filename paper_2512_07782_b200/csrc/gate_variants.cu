// gate_variants.cu -- the two gate-preprocessing designs the paper compares its
// kernel against, built on B200 for the §8(f) f2 benchmark.
// They are NOT the product path (gfwa_gate_prefix is); they exist so the
// paper's one kernel comparison can be re-measured on this hardware.
//
//   variant 1  "1-pass, one program per head": Alg. 1 launched as
//              the paper describes it ("one program per head ... the only
//              serial dependency is the single-scalar carry"): one CTA per
//              (b, head) walks the time axis in chunks of B_t = 1024 tokens and
//              keeps the carry on chip.  Reads h, beta once, writes U once.
//   variant 2  "Scan-Then-Propagate": App. E.1.  Phase 1 sums
//              -alpha per (chunk, head); phase 2 scans the chunk sums along
//              time; phase 3 re-reads h, beta, recomputes alpha and writes
//              U = offset + in-chunk cumsum (inputs read twice).
//
// Numerics match gfwa_gate_prefix (reading C-9): alpha and in-run sums in fp32,
// everything across runs and chunks in fp64, so both agree with the oracle to
// 1e-6 relative.  Carry-in is 0 (U[b,h,t] = -sum_{q<=t} alpha, C-8).
#include <cstdint>

#include "common.cuh"

namespace gfwa {
namespace {

constexpr int kThreads = 256;
constexpr int kV1Chunk = 1024;  // variant 1: tokens per chunk (4 per thread)
constexpr int kV2Chunk = 256;   // variant 2: tokens per chunk (one (chunk, b) CTA covers all heads)
constexpr int kV2MaxH = 32;     // variant 2 keeps a [H][B_t] alpha tile in smem

// alpha = softplus(beta h)/(beta + eps)  (Eq. 9, Alg. 1 l.5-7; softplus form C-6)
template <typename Tin>
__device__ __forceinline__ float alpha_at(const Tin* h, const Tin* beta, int64_t i, float eps) {
    const float hv = to_f32<Tin>(h[i]), bv = to_f32<Tin>(beta[i]);
    return __fdividef(softplus_fast(bv * hv), bv + eps);
}

// fp64 inclusive scan of one value per thread across the CTA; returns the
// exclusive prefix of this thread and the CTA total
__device__ __forceinline__ double cta_scan(double x, double* s_w, double& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    double before = 0.0;
    total = 0.0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
        const double v = s_w[w];
        if (w < warp) before += v;
        total += v;
    }
    __syncthreads();  // s_w is reused by the next call
    return before + inc - x;
}

// alpha of a contiguous [nt tokens x H heads] tile (h, beta in [B,N,H]) into
// the transposed smem tile sA[head][token] (one pad word per 8-token run):
// 16-byte loads, four per thread in flight, when the tile is 16-byte aligned
constexpr int kV2Pitch = kV2Chunk + kV2Chunk / 8 + 1;
template <typename Tin>
__device__ __forceinline__ void load_alpha_tile(const Tin* h, const Tin* beta, int64_t base, int nt, int H,
                                                float eps, float* sA) {
    constexpr int V = 16 / sizeof(Tin);  // elements per 16-byte vector
    const int n = nt * H;
    const bool vec = ((((uintptr_t)(h + base)) | ((uintptr_t)(beta + base))) & 15) == 0;
    int done = 0;
    if (vec) {
        const int nv = n / V;
        for (int i0 = threadIdx.x; i0 < nv; i0 += 4 * kThreads) {
            uint4 hv[4], bv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * kThreads;
                if (i < nv) {
                    hv[u] = __ldcs(reinterpret_cast<const uint4*>(h + base) + i);
                    bv[u] = __ldcs(reinterpret_cast<const uint4*>(beta + base) + i);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * kThreads;
                if (i >= nv) break;
                const Tin* hp = reinterpret_cast<const Tin*>(&hv[u]);
                const Tin* bp = reinterpret_cast<const Tin*>(&bv[u]);
#pragma unroll
                for (int k = 0; k < V; ++k) {
                    const int e = i * V + k, t = e / H, j = e % H;
                    const float hv1 = to_f32<Tin>(hp[k]), bv1 = to_f32<Tin>(bp[k]);
                    sA[j * kV2Pitch + t + (t >> 3)] = __fdividef(softplus_fast(bv1 * hv1), bv1 + eps);
                }
            }
        }
        done = nv * V;
    }
    for (int e = done + threadIdx.x; e < kV2Chunk * H; e += kThreads) {
        const int t = e / H, j = e % H;
        sA[j * kV2Pitch + t + (t >> 3)] = e < n ? alpha_at(h, beta, base + e, eps) : 0.f;
    }
}

// ------------------------------------------------------------------ variant 1
template <typename Tin>
__global__ void __launch_bounds__(kThreads) gate_v1_kernel(const Tin* __restrict__ h, const Tin* __restrict__ beta,
                                                          int64_t N, int64_t H, float eps, float* __restrict__ U) {
    __shared__ double s_w[kThreads / 32];
    const int64_t hh = blockIdx.x, b = blockIdx.y;
    float* urow = U + (b * H + hh) * N;
    double carry = 0.0;  // sum of alpha over the chunks already written (on chip)
    for (int64_t t0 = 0; t0 < N; t0 += kV1Chunk) {
        const int64_t tb = t0 + 4 * threadIdx.x;
        float a[4], run = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t t = tb + k;
            a[k] = t < N ? alpha_at(h, beta, (b * N + t) * H + hh, eps) : 0.f;
            run += a[k];
            a[k] = run;  // in-run inclusive prefix (fp32)
        }
        double total;
        const double excl = carry + cta_scan((double)run, s_w, total);
        if (tb + 3 < N && (((uintptr_t)(urow + tb)) & 15) == 0) {
            *reinterpret_cast<float4*>(urow + tb) = make_float4((float)(-(excl + a[0])), (float)(-(excl + a[1])),
                                                                (float)(-(excl + a[2])), (float)(-(excl + a[3])));
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (tb + k < N) urow[tb + k] = (float)(-(excl + a[k]));
        }
        carry += total;
    }
}

// ------------------------------------------------------------------ variant 2
// phase 1: S[b, h, c] = sum over chunk c of alpha
template <typename Tin>
__global__ void __launch_bounds__(kThreads) gate_v2_reduce_kernel(const Tin* __restrict__ h,
                                                                 const Tin* __restrict__ beta, int64_t N, int64_t H,
                                                                 float eps, double* __restrict__ S, int n_chunks) {
    __shared__ float sA[kV2MaxH * kV2Pitch];
    const int c = blockIdx.x;
    const int64_t b = blockIdx.y, t0 = (int64_t)c * kV2Chunk;
    const int nt = (int)min64(kV2Chunk, N - t0);
    load_alpha_tile(h, beta, (b * N + t0) * H, nt, (int)H, eps, sA);
    __syncthreads();
    // a warp per head: lane l sums its 8-token run, then the warp sums the runs
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j = warp; j < H; j += kThreads / 32) {
        const float* row = sA + j * kV2Pitch + lane * (kV2Chunk / 32 + 1);
        float run = 0.f;
#pragma unroll
        for (int k = 0; k < kV2Chunk / 32; ++k) run += row[k];
        double x = run;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) S[(b * H + j) * n_chunks + c] = x;
    }
}

// phase 2: O[b, h, c] = sum_{c' < c} S[b, h, c']  (exclusive cumsum along time,
// P:1040-1042): one CTA per (b, h) row, a CTA-wide scan per 256 chunk sums
__global__ void __launch_bounds__(kThreads) gate_v2_scan_kernel(const double* __restrict__ S, double* __restrict__ O,
                                                               int n_chunks) {
    __shared__ double s_w[kThreads / 32];
    const double* srow = S + (int64_t)blockIdx.x * n_chunks;
    double* orow = O + (int64_t)blockIdx.x * n_chunks;
    double carry = 0.0;
    for (int c0 = 0; c0 < n_chunks; c0 += kThreads) {
        const int c = c0 + threadIdx.x;
        const double x = c < n_chunks ? srow[c] : 0.0;
        double total;
        const double excl = cta_scan(x, s_w, total);
        if (c < n_chunks) orow[c] = carry + excl;
        carry += total;
    }
}

// phase 3: recompute alpha, U = -(O[c] + in-chunk inclusive cumsum)
template <typename Tin>
__global__ void __launch_bounds__(kThreads) gate_v2_propagate_kernel(const Tin* __restrict__ h,
                                                                    const Tin* __restrict__ beta, int64_t N,
                                                                    int64_t H, float eps,
                                                                    const double* __restrict__ O,
                                                                    float* __restrict__ U, int n_chunks) {
    constexpr int kPitch = kV2Pitch;
    __shared__ float sA[kV2MaxH * kPitch];  // [head][token], transposed from [token][head]
    const int c = blockIdx.x;
    const int64_t b = blockIdx.y, t0 = (int64_t)c * kV2Chunk;
    const int nt = (int)min64(kV2Chunk, N - t0);
    load_alpha_tile(h, beta, (b * N + t0) * H, nt, (int)H, eps, sA);
    __syncthreads();
    // a warp per head; lane l owns tokens [8l, 8l + 8) of the chunk
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int R = kV2Chunk / 32;
    for (int j = warp; j < H; j += kThreads / 32) {
        const float* row = sA + j * kPitch + lane * (R + 1);
        float pre[R], run = 0.f;
#pragma unroll
        for (int k = 0; k < R; ++k) {
            run += row[k];
            pre[k] = run;
        }
        double inc = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const double excl = O[(b * H + j) * n_chunks + c] + inc - run;
        float* urow = U + (b * H + j) * N + t0 + lane * R;
#pragma unroll
        for (int k = 0; k < R; ++k)
            if (lane * R + k < nt) urow[k] = (float)(-(excl + pre[k]));
    }
}

template <typename Tin>
void launch_variant(int variant, const void* h, const void* beta, int64_t B, int64_t N, int64_t H, float eps,
                    float* U, void* ws, cudaStream_t st) {
    const Tin* hp = (const Tin*)h;
    const Tin* bp = (const Tin*)beta;
    if (variant == 1) {
        gate_v1_kernel<Tin><<<dim3((unsigned)H, (unsigned)B), kThreads, 0, st>>>(hp, bp, N, H, eps, U);
        note_launch();
        return;
    }
    const int n_chunks = (int)((N + kV2Chunk - 1) / kV2Chunk);
    double* S = (double*)ws;
    double* O = S + B * H * n_chunks;
    gate_v2_reduce_kernel<Tin><<<dim3((unsigned)n_chunks, (unsigned)B), kThreads, 0, st>>>(hp, bp, N, H, eps, S,
                                                                                            n_chunks);
    note_launch();
    gate_v2_scan_kernel<<<(unsigned)(B * H), kThreads, 0, st>>>(S, O, n_chunks);
    note_launch();
    gate_v2_propagate_kernel<Tin><<<dim3((unsigned)n_chunks, (unsigned)B), kThreads, 0, st>>>(hp, bp, N, H, eps, O,
                                                                                              U, n_chunks);
    note_launch();
}

}  // namespace
}  // namespace gfwa

using namespace gfwa;

extern "C" size_t gfwa_gate_prefix_variant_workspace_size(int variant, int64_t B, int64_t N, int64_t H) {
    if (variant != 2 || B < 1 || N < 1 || H < 1) return 256;
    const int64_t n_chunks = (N + kV2Chunk - 1) / kV2Chunk;
    return (size_t)(2 * B * H * n_chunks) * sizeof(double);
}

extern "C" gfwa_status_t gfwa_gate_prefix_variant(int variant, gfwa_dtype_t in_dtype, const void* h,
                                                  const void* beta, int64_t B, int64_t N, int64_t H, float eps,
                                                  float* U, void* ws, size_t ws_bytes, gfwa_stream_t stream) {
    if (variant != 1 && variant != 2) return GFWA_ERR_INVALID_ARGUMENT;
    if (!h || !beta || !U || B < 1 || N < 1 || H < 1 || !(eps >= 0.f)) return GFWA_ERR_INVALID_ARGUMENT;
    if (B > 65535 || H > 65535 || N >= ((int64_t)1 << 40)) return GFWA_ERR_INVALID_ARGUMENT;
    if (in_dtype != GFWA_BF16 && in_dtype != GFWA_F32) return GFWA_ERR_UNSUPPORTED;
    if (variant == 2) {
        if (H > kV2MaxH) return GFWA_ERR_UNSUPPORTED;
        if (!ws || ws_bytes < gfwa_gate_prefix_variant_workspace_size(variant, B, N, H)) return GFWA_ERR_WORKSPACE;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (in_dtype == GFWA_BF16)
        launch_variant<__nv_bfloat16>(variant, h, beta, B, N, H, eps, U, ws, st);
    else
        launch_variant<float>(variant, h, beta, B, N, H, eps, U, ws, st);
    return check_launch();
}
