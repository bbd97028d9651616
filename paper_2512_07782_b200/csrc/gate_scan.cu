// gate_scan.cu -- gfwa_gate_prefix / gfwa_gate_prefix_bwd.
//
// Alg. 1 "Fused Tiled Scan" re-designed for B200: instead of one
// program per head walking its chunks serially with an on-chip carry
// (P:271), every (b, head-group, chunk) tile is an independent CTA and the
// carry is resolved with a single-pass *decoupled look-back*.  h and beta are
// read once and U written once (the paper's I/O claim), all accesses
// coalesced:
//   load    [T tokens x HG heads] tile of h, beta ([B,N,H], H contiguous),
//           one batch of independent loads per thread (1024 threads)
//   alpha   softplus(beta h)/(beta + eps) in fp32 -> smem [HG][T] (transpose,
//           one pad word per lane run so the run reads are conflict-free)
//   scan    one warp per head; lane l owns a run of R = T/32 tokens: serial
//           fp32 prefix, run totals scanned across the warp in fp64
//   carry   chunk aggregate published as one 64-bit word (fp64 value with the
//           2-bit status in its lowest mantissa bits: a single relaxed load
//           observes value and status together); all 32 heads look back
//           concurrently, 32 predecessors per round
//   store   U [B,H,N] rows (N contiguous), 16-byte vector stores
// The head-group size is a template parameter (power of two), so all tile
// index math is shifts and masks.  The backward runs the same machinery right
// to left on dU and fuses the chain rule into dh, dbeta.
#include <algorithm>

#include "common.cuh"

namespace gfwa {
namespace {

constexpr int kThreads = 1024;  // 32 warps: one per head of the group
constexpr int kWarps = kThreads / 32;

struct ScanGeom {
    int HG;        // heads per CTA (<= 32)
    int log_hgp;   // log2 of the head-group slot count (power of two >= HG)
    int log_t;     // log2 tokens per chunk (T >= 64)
    int n_hgroups; // ceil(H / HG)
    int n_chunks;  // ceil(N / T)
};

ScanGeom scan_geom(int64_t B, int64_t N, int64_t H) {
    ScanGeom g;
    g.HG = H >= 32 ? 32 : (int)H;
    g.log_hgp = 0;
    while ((1 << g.log_hgp) < g.HG) ++g.log_hgp;
    g.log_t = 13 - g.log_hgp;  // T * HGP = 8192 elements per tile
    g.n_hgroups = (int)((H + g.HG - 1) / g.HG);
    // small problems: shorter chunks so every SM streams (the look-back makes
    // the chunk count free)
    while (g.log_t > 6 && (int64_t)g.n_hgroups * ((N + (1 << g.log_t) - 1) >> g.log_t) * B < 2 * 148) --g.log_t;
    g.n_chunks = (int)((N + (1 << g.log_t) - 1) >> g.log_t);
    return g;
}

struct Lookback {
    unsigned long long* desc;  // per (b, hg, chunk, head): fp64 value | 2-bit status (0 empty, 1 agg, 2 incl)
    unsigned* ticket;
};

size_t lookback_bytes(int64_t B, const ScanGeom& g) {
    size_t n = (size_t)B * g.n_hgroups * g.n_chunks * 32;
    return (n * sizeof(unsigned long long) + 256 + 255) & ~(size_t)255;
}

Lookback carve(void* ws, int64_t B, const ScanGeom& g) {
    size_t n = (size_t)B * g.n_hgroups * g.n_chunks * 32;
    Lookback lb;
    lb.desc = (unsigned long long*)ws;
    lb.ticket = (unsigned*)((char*)ws + ((n * sizeof(unsigned long long) + 15) & ~(size_t)15));
    return lb;
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// value and status in one word: the status replaces the 2 lowest mantissa
// bits (relative perturbation <= 2^-51, far below the fp32 U it feeds)
__device__ __forceinline__ void publish(unsigned long long* p, double v, unsigned status) {
    st_relaxed_u64(p, ((unsigned long long)__double_as_longlong(v) & ~3ull) | status);
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Exclusive prefix over chunks 0..c-1 of this (sequence, head): warp-parallel
// decoupled look-back, 32 predecessors per round.  Whole warp calls.
__device__ double lookback(const unsigned long long* d, int c) {
    const int lane = threadIdx.x & 31;
    double excl = 0.0;
    int pc = c - 1;
    while (pc >= 0) {
        const int q = pc - lane;
        unsigned long long w = 0;
        if (q >= 0) {
            do {
                w = ld_relaxed_u64(d + (size_t)q * 32);
            } while ((w & 3ull) == 0);
        }
        const unsigned st = (unsigned)(w & 3ull);
        const double v = q >= 0 ? __longlong_as_double((long long)(w & ~3ull)) : 0.0;
        const unsigned pmask = __ballot_sync(0xffffffffu, q >= 0 && st == 2);
        if (pmask) {
            const int first = __ffs(pmask) - 1;  // closest chunk with an inclusive prefix
            excl += warp_sum_d(lane <= first ? v : 0.0);
            break;
        }
        excl += warp_sum_d(v);
        pc -= 32;
    }
    return excl;
}

template <typename Tin>
__device__ __forceinline__ float load_in(const Tin* p) { return to_f32<Tin>(*p); }

// smem index of token tt in a head row: one pad word per run of R tokens
__device__ __forceinline__ int sk(int tt, int log_r) { return tt + (tt >> log_r); }

// ---------------------------------------------------------------- forward

template <typename Tin, bool kAlphaIn, int LOG_HGP>
__global__ void __launch_bounds__(kThreads) gate_prefix_kernel(
    const Tin* __restrict__ h, const Tin* __restrict__ beta, int64_t N, int64_t H, float eps,
    const double* __restrict__ carry_in, float* __restrict__ U, double* __restrict__ total, Lookback lb,
    ScanGeom g) {
    constexpr int HGP = 1 << LOG_HGP;
    extern __shared__ float sA[];  // [HGP][pitch]
    __shared__ unsigned s_ticket;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_ticket = atomicAdd(lb.ticket, 1u);
    __syncthreads();
    const unsigned tk = s_ticket;
    const int c = (int)(tk % g.n_chunks);
    const int rest = (int)(tk / g.n_chunks);
    const int hg = rest % g.n_hgroups;
    const int b = rest / g.n_hgroups;
    const int T = 1 << g.log_t, log_r = g.log_t - 5, R = T >> 5;
    const int pitch = T + 32 + 1;
    const int64_t t0 = (int64_t)c << g.log_t;
    const int hh0 = hg * g.HG;
    const int nh = min(g.HG, (int)(H - hh0));
    const int nt = (int)min64(T, N - t0);

    // 1. tile load, alpha in fp32 (Alg. 1 l.4-7)
    const int64_t row0 = ((int64_t)b * N + t0) * H + hh0;
    constexpr int kB = 8;
    for (int e0 = tid; e0 < T * HGP; e0 += kThreads * kB) {
        float hv[kB], bv[kB];
#pragma unroll
        for (int k = 0; k < kB; ++k) {
            const int e = e0 + k * kThreads;
            const int tt = e >> LOG_HGP, j = e & (HGP - 1);
            hv[k] = 0.f;
            bv[k] = 1.f;
            if (e < T * HGP && tt < nt && j < nh) {
                const int64_t i = row0 + (int64_t)tt * H + j;
                hv[k] = load_in(h + i);
                if (!kAlphaIn) bv[k] = load_in(beta + i);
            }
        }
#pragma unroll
        for (int k = 0; k < kB; ++k) {
            const int e = e0 + k * kThreads;
            const int tt = e >> LOG_HGP, j = e & (HGP - 1);
            if (e < T * HGP) {
                float a = 0.f;
                if (tt < nt && j < nh) a = kAlphaIn ? hv[k] : __fdividef(softplus_fast(bv[k] * hv[k]), bv[k] + eps);
                sA[j * pitch + sk(tt, log_r)] = a;
            }
        }
    }
    __syncthreads();
    const int j = warp;  // one head per warp
    if (j >= nh) return;

    // 2. lane runs (fp32), their exclusive scan across the warp (fp64), chunk
    //    aggregate published, look-back, inclusive published
    const float* row = sA + j * pitch + lane * (R + 1);
    float run = 0.f;
    for (int k = 0; k < R; ++k) run += row[k];
    double x = (double)run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    const double agg = __shfl_sync(0xffffffffu, x, 31);
    unsigned long long* d = lb.desc + ((size_t)(b * g.n_hgroups + hg) * g.n_chunks) * 32 + j;
    if (lane == 0) publish(d + (size_t)c * 32, agg, c == 0 ? 2u : 1u);
    const double excl = c == 0 ? 0.0 : lookback(d, c);
    if (lane == 0) {
        if (c > 0) publish(d + (size_t)c * 32, excl + agg, 2u);
        if (total && c == g.n_chunks - 1) total[(int64_t)b * H + hh0 + j] = excl + agg;
    }
    // 3. U_t = carry - (prefix before this run) - (in-run fp32 prefix)  (Alg. 1 l.8-9)
    const double carry = carry_in ? carry_in[(int64_t)b * H + hh0 + j] : 0.0;
    const float cbase = (float)(carry - (excl + x - (double)run));
    float* urow = U + ((int64_t)b * H + hh0 + j) * N + t0 + lane * R;
    const int tl = lane * R;
    float acc = 0.f;
    if (tl + R <= nt && (R & 3) == 0 && ((uintptr_t)urow & 15) == 0) {
        for (int k = 0; k < R; k += 4) {
            float4 o;
            acc += row[k];
            o.x = cbase - acc;
            acc += row[k + 1];
            o.y = cbase - acc;
            acc += row[k + 2];
            o.z = cbase - acc;
            acc += row[k + 3];
            o.w = cbase - acc;
            *reinterpret_cast<float4*>(urow + k) = o;
        }
    } else {
        for (int k = 0; k < R; ++k) {
            acc += row[k];
            if (tl + k < nt) urow[k] = cbase - acc;
        }
    }
}

// ---------------------------------------------------------------- backward

template <typename Tin, bool kAlphaIn, int LOG_HGP>
__global__ void __launch_bounds__(kThreads) gate_prefix_bwd_kernel(
    const Tin* __restrict__ h, const Tin* __restrict__ beta, int64_t N, int64_t H, float eps,
    const float* __restrict__ dU, const double* __restrict__ carry, float* __restrict__ dalpha,
    Tin* __restrict__ dh, Tin* __restrict__ dbeta, Lookback lb, ScanGeom g) {
    constexpr int HGP = 1 << LOG_HGP;
    extern __shared__ float sA[];  // [HGP][pitch]
    __shared__ unsigned s_ticket;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_ticket = atomicAdd(lb.ticket, 1u);
    __syncthreads();
    const unsigned tk = s_ticket;
    const int rc = (int)(tk % g.n_chunks);  // order of processing: right to left
    const int c = g.n_chunks - 1 - rc;
    const int rest = (int)(tk / g.n_chunks);
    const int hg = rest % g.n_hgroups;
    const int b = rest / g.n_hgroups;
    const int T = 1 << g.log_t, log_r = g.log_t - 5, R = T >> 5;
    const int pitch = T + 32 + 1;
    const int64_t t0 = (int64_t)c << g.log_t;
    const int hh0 = hg * g.HG;
    const int nh = min(g.HG, (int)(H - hh0));
    const int nt = (int)min64(T, N - t0);

    // 1. dU rows (N contiguous) -> smem, one batch of independent loads
    constexpr int kB = 8;
    for (int e0 = tid; e0 < T * HGP; e0 += kThreads * kB) {
        float v[kB];
#pragma unroll
        for (int k = 0; k < kB; ++k) {
            const int e = e0 + k * kThreads;
            const int j = e >> g.log_t, tt = e & (T - 1);
            v[k] = (e < T * HGP && tt < nt && j < nh) ? dU[((int64_t)b * H + hh0 + j) * N + t0 + tt] : 0.f;
        }
#pragma unroll
        for (int k = 0; k < kB; ++k) {
            const int e = e0 + k * kThreads;
            if (e < T * HGP) sA[(e >> g.log_t) * pitch + sk(e & (T - 1), log_r)] = v[k];
        }
    }
    __syncthreads();
    const int j = warp;
    if (j < nh) {
        // 2. reverse scan: dalpha_t = carry - sum_{t' >= t} dU_t'  (suffix sums)
        float* row = sA + j * pitch + lane * (R + 1);
        float run = 0.f;
        for (int k = 0; k < R; ++k) run += row[k];
        double x = (double)run;  // inclusive suffix scan of the lane runs
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_down_sync(0xffffffffu, x, o);
            if (lane + o < 32) x += y;
        }
        const double agg = __shfl_sync(0xffffffffu, x, 0);
        unsigned long long* d = lb.desc + ((size_t)(b * g.n_hgroups + hg) * g.n_chunks) * 32 + j;
        if (lane == 0) publish(d + (size_t)rc * 32, agg, rc == 0 ? 2u : 1u);
        const double excl = rc == 0 ? 0.0 : lookback(d, rc);
        if (lane == 0 && rc > 0) publish(d + (size_t)rc * 32, excl + agg, 2u);
        const double cr = carry ? carry[(int64_t)b * H + hh0 + j] : 0.0;
        const float cbase = (float)(cr - (excl + x - (double)run));
        float* arow = dalpha ? dalpha + ((int64_t)b * H + hh0 + j) * N + t0 + lane * R : nullptr;
        const int tl = lane * R;
        float acc = 0.f;
        for (int k = R - 1; k >= 0; --k) {
            acc += row[k];
            const float da = cbase - acc;
            row[k] = da;  // kept for the chain rule
            if (arow && tl + k < nt) arow[k] = da;
        }
    }
    if (!dh && !dbeta) return;
    __syncthreads();
    // 3. chain rule through Eq. 9 into dh, dbeta ([B,N,H], coalesced)
    const int64_t row0 = ((int64_t)b * N + t0) * H + hh0;
    for (int e0 = tid; e0 < T * HGP; e0 += kThreads * kB) {
        float hv[kB], bv[kB];
#pragma unroll
        for (int k = 0; k < kB; ++k) {
            const int e = e0 + k * kThreads;
            const int tt = e >> LOG_HGP, jj = e & (HGP - 1);
            hv[k] = 0.f;
            bv[k] = 1.f;
            if (!kAlphaIn && e < T * HGP && tt < nt && jj < nh) {
                const int64_t i = row0 + (int64_t)tt * H + jj;
                hv[k] = load_in(h + i);
                bv[k] = load_in(beta + i);
            }
        }
#pragma unroll
        for (int k = 0; k < kB; ++k) {
            const int e = e0 + k * kThreads;
            const int tt = e >> LOG_HGP, jj = e & (HGP - 1);
            if (e >= T * HGP || tt >= nt || jj >= nh) continue;
            const int64_t i = row0 + (int64_t)tt * H + jj;
            const float da = sA[jj * pitch + sk(tt, log_r)];
            if (kAlphaIn) {
                if (dh) dh[i] = from_f32<Tin>(da);
            } else {
                const float z = bv[k] * hv[k], be = bv[k] + eps, sg = sigmoid_fast(z);
                const float rbe = __fdividef(1.f, be);
                if (dh) dh[i] = from_f32<Tin>(da * sg * bv[k] * rbe);
                if (dbeta) dbeta[i] = from_f32<Tin>(da * (sg * hv[k] * be - softplus_fast(z)) * (rbe * rbe));
            }
        }
    }
}

template <typename Tin, bool kAlpha, int L>
void launch_fwd_t(const void* h, const void* beta, int64_t B, int64_t N, int64_t H, float eps,
                  const double* carry_in, float* U, double* total, const Lookback& lb, const ScanGeom& g,
                  cudaStream_t st) {
    const size_t smem = (size_t)(1 << L) * ((1 << g.log_t) + 33) * sizeof(float);
    auto k = gate_prefix_kernel<Tin, kAlpha, L>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<(unsigned)(B * g.n_hgroups * g.n_chunks), kThreads, smem, st>>>((const Tin*)h, (const Tin*)beta, N, H, eps,
                                                                       carry_in, U, total, lb, g);
}

template <typename Tin, bool kAlpha, int L>
void launch_bwd_t(const void* h, const void* beta, int64_t B, int64_t N, int64_t H, float eps, const float* dU,
                  const double* carry, float* dalpha, void* dh, void* dbeta, const Lookback& lb, const ScanGeom& g,
                  cudaStream_t st) {
    const size_t smem = (size_t)(1 << L) * ((1 << g.log_t) + 33) * sizeof(float);
    auto k = gate_prefix_bwd_kernel<Tin, kAlpha, L>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<(unsigned)(B * g.n_hgroups * g.n_chunks), kThreads, smem, st>>>(
        (const Tin*)h, (const Tin*)beta, N, H, eps, dU, carry, dalpha, (Tin*)dh, (Tin*)dbeta, lb, g);
}

// dispatch over the head-group size (power of two <= 32)
#define GFWA_HGP_SWITCH(L, CALL)      \
    switch (L) {                      \
        case 0: CALL(0); break;       \
        case 1: CALL(1); break;       \
        case 2: CALL(2); break;       \
        case 3: CALL(3); break;       \
        case 4: CALL(4); break;       \
        default: CALL(5); break;      \
    }

template <typename Tin>
gfwa_status_t launch_fwd(gfwa_gate_kind_t kind, const void* h, const void* beta, int64_t B, int64_t N,
                         int64_t H, float eps, const double* carry_in, float* U, double* total,
                         const Lookback& lb, const ScanGeom& g, cudaStream_t st) {
#define GFWA_CALL(L)                                                                                 \
    if (kind == GFWA_GATE_ALPHA)                                                                     \
        launch_fwd_t<Tin, true, L>(h, beta, B, N, H, eps, carry_in, U, total, lb, g, st);            \
    else                                                                                             \
        launch_fwd_t<Tin, false, L>(h, beta, B, N, H, eps, carry_in, U, total, lb, g, st);
    GFWA_HGP_SWITCH(g.log_hgp, GFWA_CALL)
#undef GFWA_CALL
    note_launch();
    return check_launch();
}

template <typename Tin>
gfwa_status_t launch_bwd(gfwa_gate_kind_t kind, const void* h, const void* beta, int64_t B, int64_t N,
                         int64_t H, float eps, const float* dU, const double* carry, float* dalpha, void* dh,
                         void* dbeta, const Lookback& lb, const ScanGeom& g, cudaStream_t st) {
#define GFWA_CALL(L)                                                                                       \
    if (kind == GFWA_GATE_ALPHA)                                                                           \
        launch_bwd_t<Tin, true, L>(h, beta, B, N, H, eps, dU, carry, dalpha, dh, dbeta, lb, g, st);        \
    else                                                                                                   \
        launch_bwd_t<Tin, false, L>(h, beta, B, N, H, eps, dU, carry, dalpha, dh, dbeta, lb, g, st);
    GFWA_HGP_SWITCH(g.log_hgp, GFWA_CALL)
#undef GFWA_CALL
    note_launch();
    return check_launch();
}

}  // namespace
}  // namespace gfwa

using namespace gfwa;

extern "C" size_t gfwa_gate_prefix_workspace_size(int64_t B, int64_t N, int64_t H) {
    if (B < 1 || N < 1 || H < 1) return 256;
    return lookback_bytes(B, scan_geom(B, N, H));
}

extern "C" size_t gfwa_gate_prefix_bwd_workspace_size(int64_t B, int64_t N, int64_t H) {
    return gfwa_gate_prefix_workspace_size(B, N, H);
}

static bool aligned_ptr(const void* p, size_t a) { return ((uintptr_t)p % a) == 0; }

extern "C" gfwa_status_t gfwa_gate_prefix(gfwa_gate_kind_t kind, gfwa_dtype_t in_dtype, const void* h,
                                          const void* beta, int64_t B, int64_t N, int64_t H, float eps,
                                          const double* carry_in, float* U, double* total, void* ws,
                                          size_t ws_bytes, gfwa_stream_t stream) {
    if (!h || !U || !ws || B < 1 || N < 1 || H < 1) return GFWA_ERR_INVALID_ARGUMENT;
    if (kind != GFWA_GATE_ALPHA && kind != GFWA_GATE_HBETA) return GFWA_ERR_INVALID_ARGUMENT;
    if (kind == GFWA_GATE_HBETA && (!beta || !(eps >= 0.f))) return GFWA_ERR_INVALID_ARGUMENT;
    if (in_dtype != GFWA_F32 && in_dtype != GFWA_BF16) return GFWA_ERR_UNSUPPORTED;
    if (B * H * ((N + 31) / 32) > (int64_t)1 << 31) return GFWA_ERR_INVALID_ARGUMENT;
    if (!aligned_ptr(ws, 256)) return GFWA_ERR_INVALID_ARGUMENT;
    const ScanGeom g = scan_geom(B, N, H);
    if (ws_bytes < lookback_bytes(B, g)) return GFWA_ERR_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    if (gfwa_status_t s = check_launch(cudaMemsetAsync(ws, 0, lookback_bytes(B, g), st))) return s;
    const Lookback lb = carve(ws, B, g);
    if (in_dtype == GFWA_BF16)
        return launch_fwd<__nv_bfloat16>(kind, h, beta, B, N, H, eps, carry_in, U, total, lb, g, st);
    return launch_fwd<float>(kind, h, beta, B, N, H, eps, carry_in, U, total, lb, g, st);
}

extern "C" gfwa_status_t gfwa_gate_prefix_bwd(gfwa_gate_kind_t kind, gfwa_dtype_t in_dtype, const void* h,
                                              const void* beta, int64_t B, int64_t N, int64_t H, float eps,
                                              const float* dU, const double* carry, float* dalpha, void* dh,
                                              void* dbeta, void* ws, size_t ws_bytes, gfwa_stream_t stream) {
    if (!dU || !ws || B < 1 || N < 1 || H < 1) return GFWA_ERR_INVALID_ARGUMENT;
    if (kind != GFWA_GATE_ALPHA && kind != GFWA_GATE_HBETA) return GFWA_ERR_INVALID_ARGUMENT;
    if (!dalpha && !dh && !dbeta) return GFWA_ERR_INVALID_ARGUMENT;
    if (kind == GFWA_GATE_HBETA && (dh || dbeta) && (!h || !beta)) return GFWA_ERR_INVALID_ARGUMENT;
    if (kind == GFWA_GATE_ALPHA && dbeta) return GFWA_ERR_INVALID_ARGUMENT;
    if (in_dtype != GFWA_F32 && in_dtype != GFWA_BF16) return GFWA_ERR_UNSUPPORTED;
    if (!aligned_ptr(ws, 256)) return GFWA_ERR_INVALID_ARGUMENT;
    const ScanGeom g = scan_geom(B, N, H);
    if (ws_bytes < lookback_bytes(B, g)) return GFWA_ERR_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    if (gfwa_status_t s = check_launch(cudaMemsetAsync(ws, 0, lookback_bytes(B, g), st))) return s;
    const Lookback lb = carve(ws, B, g);
    if (in_dtype == GFWA_BF16)
        return launch_bwd<__nv_bfloat16>(kind, h, beta, B, N, H, eps, dU, carry, dalpha, dh, dbeta, lb, g, st);
    return launch_bwd<float>(kind, h, beta, B, N, H, eps, dU, carry, dalpha, dh, dbeta, lb, g, st);
}
