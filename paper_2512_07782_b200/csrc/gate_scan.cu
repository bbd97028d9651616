// gate_scan.cu -- gfwa_gate_prefix / gfwa_gate_prefix_bwd.
//
// Alg. 1 "Fused Tiled Scan" re-designed for B200: instead of one
// program per head walking its chunks serially with an on-chip carry
// (P:271), every (b, head-group, chunk) tile is an independent CTA and the
// carry is resolved with a single-pass *decoupled look-back* (fp64
// aggregates published per chunk).  h and beta are read once and U written
// once (the paper's I/O claim), all accesses coalesced:
//   load    [T tokens x HG heads] tile of h, beta ([B,N,H], H contiguous)
//   alpha   softplus(beta h)/(beta + eps) in fp32 -> smem [HG][T] (transpose)
//   publish chunk aggregate sum(alpha) per head (fp64)
//   lookback warp-parallel over 32 predecessors -> exclusive prefix (fp64)
//   scan    warp shuffles along the 32-token rows, fp64 running carry
//   store   U [B,H,N] rows (N contiguous)
// The backward runs the same machinery right-to-left on dU and
// optionally fuses the chain rule into dh, dbeta.
#include <algorithm>

#include "common.cuh"

namespace gfwa {
namespace {

constexpr int kThreads = 256;
constexpr int kTileElems = 8192;  // T * HGp

struct ScanGeom {
    int HG;        // heads per CTA (<= 32)
    int T;         // tokens per chunk (multiple of 32)
    int n_hgroups; // ceil(H / HG)
    int n_chunks;  // ceil(N / T)
};

ScanGeom scan_geom(int64_t N, int64_t H) {
    ScanGeom g;
    g.HG = H >= 32 ? 32 : (int)H;
    int hgp = 1;
    while (hgp < g.HG) hgp <<= 1;
    g.T = kTileElems / hgp;
    g.n_hgroups = (int)((H + g.HG - 1) / g.HG);
    g.n_chunks = (int)((N + g.T - 1) / g.T);
    return g;
}

struct Lookback {
    int* flag;     // 0 = empty, 1 = aggregate ready, 2 = inclusive ready
    double* agg;
    double* incl;
    unsigned* ticket;
};

size_t lookback_bytes(int64_t B, const ScanGeom& g) {
    size_t n = (size_t)B * g.n_hgroups * g.n_chunks * g.HG;
    size_t bytes = n * (sizeof(int) + 2 * sizeof(double)) + 256;
    return (bytes + 255) & ~(size_t)255;
}

Lookback carve(void* ws, int64_t B, const ScanGeom& g) {
    size_t n = (size_t)B * g.n_hgroups * g.n_chunks * g.HG;
    char* p = (char*)ws;
    Lookback lb;
    lb.agg = (double*)p;
    lb.incl = (double*)(p + n * sizeof(double));
    lb.flag = (int*)(p + 2 * n * sizeof(double));
    lb.ticket = (unsigned*)(((uintptr_t)(p + 2 * n * sizeof(double) + n * sizeof(int)) + 15) & ~(uintptr_t)15);
    return lb;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Exclusive prefix (over chunks 0..c-1 of this sequence) by warp-parallel
// decoupled look-back.  `base` indexes chunk 0 of the (b, hg, head) sequence;
// descriptors of consecutive chunks are `stride` apart.  Whole warp calls.
__device__ double lookback(const Lookback& lb, size_t base, size_t stride, int c) {
    const int lane = threadIdx.x & 31;
    double excl = 0.0;
    int pc = c - 1;
    while (pc >= 0) {
        const int q = pc - lane;
        int f = 0;
        double v = 0.0;
        if (q >= 0) {
            const size_t i = base + (size_t)q * stride;
            do {
                f = ld_acquire(lb.flag + i);
            } while (f == 0);
            v = (f == 2) ? lb.incl[i] : lb.agg[i];
        }
        const unsigned pmask = __ballot_sync(0xffffffffu, q >= 0 && f == 2);
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

// ---------------------------------------------------------------- forward

template <typename Tin, bool kAlphaIn>
__global__ void __launch_bounds__(kThreads) gate_prefix_kernel(
    const Tin* __restrict__ h, const Tin* __restrict__ beta, int64_t N, int64_t H, float eps,
    const double* __restrict__ carry_in, float* __restrict__ U, double* __restrict__ total,
    Lookback lb, ScanGeom g) {
    extern __shared__ float sA[];  // [HG][T + 1]
    __shared__ unsigned s_ticket;
    __shared__ double s_excl[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_ticket = atomicAdd(lb.ticket, 1u);
    __syncthreads();
    const unsigned tk = s_ticket;
    const int c = (int)(tk % g.n_chunks);
    const int rest = (int)(tk / g.n_chunks);
    const int hg = rest % g.n_hgroups;
    const int b = rest / g.n_hgroups;
    const int T = g.T, HG = g.HG, pitch = T + 1;
    const int64_t t0 = (int64_t)c * T;
    const int hh0 = hg * HG;
    const int nh = min(HG, (int)(H - hh0));
    const int nt = (int)min64(T, N - t0);

    // 1. coalesced load of the [T x HG] tile, alpha in fp32 (Alg. 1 l.4-7).
    for (int e = tid; e < T * HG; e += kThreads) {
        const int tt = e / HG, j = e - tt * HG;
        float a = 0.f;
        if (tt < nt && j < nh) {
            const int64_t i = ((int64_t)b * N + t0 + tt) * H + hh0 + j;
            if (kAlphaIn) {
                a = load_in(h + i);
            } else {
                const float bt = load_in(beta + i);
                a = softplus_f(bt * load_in(h + i)) / (bt + eps);
            }
        }
        sA[j * pitch + tt] = a;
    }
    __syncthreads();

    // 2. per-head chunk aggregate, published for the successors.
    const size_t seq_stride = (size_t)HG;  // consecutive chunks of one head
    for (int j = warp; j < nh; j += kThreads / 32) {
        float part = 0.f;
        for (int tt = lane; tt < nt; tt += 32) part += sA[j * pitch + tt];
        const double agg = warp_sum_d((double)part);
        const size_t base = ((size_t)(b * g.n_hgroups + hg) * g.n_chunks) * HG + j;
        const size_t i = base + (size_t)c * seq_stride;
        if (lane == 0) {
            if (c == 0) {
                lb.incl[i] = agg;
                st_release(lb.flag + i, 2);
            } else {
                lb.agg[i] = agg;
                st_release(lb.flag + i, 1);
            }
        }
        if (lane == 0) s_excl[j] = agg;  // temporarily the aggregate
    }
    __syncwarp();
    // 3. look-back -> exclusive prefix; publish the inclusive prefix.
    for (int j = warp; j < nh; j += kThreads / 32) {
        const size_t base = ((size_t)(b * g.n_hgroups + hg) * g.n_chunks) * HG + j;
        const double excl = c == 0 ? 0.0 : lookback(lb, base, seq_stride, c);
        if (lane == 0) {
            const double agg = s_excl[j];
            if (c > 0) {
                const size_t i = base + (size_t)c * seq_stride;
                lb.incl[i] = excl + agg;
                st_release(lb.flag + i, 2);
            }
            if (total && c == g.n_chunks - 1) total[(int64_t)b * H + hh0 + j] = excl + agg;
            s_excl[j] = excl;
        }
    }
    __syncthreads();
    // 4. in-chunk inclusive scan along the 32-token rows, fp64 running sum,
    //    U = carry - prefix (Alg. 1 l.8-9), coalesced row stores.
    for (int j = warp; j < nh; j += kThreads / 32) {
        const int hh = hh0 + j;
        const double carry = carry_in ? carry_in[(int64_t)b * H + hh] : 0.0;
        double run = s_excl[j];
        float* urow = U + ((int64_t)b * H + hh) * N + t0;
        for (int r = 0; r < nt; r += 32) {
            float x = sA[j * pitch + r + lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const float y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (r + lane < nt) urow[r + lane] = (float)(carry - (run + (double)x));
            run += (double)__shfl_sync(0xffffffffu, x, 31);
        }
    }
}

// ---------------------------------------------------------------- backward

template <typename Tin, bool kAlphaIn>
__global__ void __launch_bounds__(kThreads) gate_prefix_bwd_kernel(
    const Tin* __restrict__ h, const Tin* __restrict__ beta, int64_t N, int64_t H, float eps,
    const float* __restrict__ dU, const double* __restrict__ carry, float* __restrict__ dalpha,
    Tin* __restrict__ dh, Tin* __restrict__ dbeta, Lookback lb, ScanGeom g) {
    extern __shared__ float sA[];  // [HG][T + 1]
    __shared__ unsigned s_ticket;
    __shared__ double s_excl[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_ticket = atomicAdd(lb.ticket, 1u);
    __syncthreads();
    const unsigned tk = s_ticket;
    const int rc = (int)(tk % g.n_chunks);  // order of processing: right to left
    const int c = g.n_chunks - 1 - rc;
    const int rest = (int)(tk / g.n_chunks);
    const int hg = rest % g.n_hgroups;
    const int b = rest / g.n_hgroups;
    const int T = g.T, HG = g.HG, pitch = T + 1;
    const int64_t t0 = (int64_t)c * T;
    const int hh0 = hg * HG;
    const int nh = min(HG, (int)(H - hh0));
    const int nt = (int)min64(T, N - t0);

    // 1. load dU rows (N contiguous) into smem.
    for (int e = tid; e < T * HG; e += kThreads) {
        const int j = e / T, tt = e - j * T;
        float v = 0.f;
        if (tt < nt && j < nh) v = dU[((int64_t)b * H + hh0 + j) * N + t0 + tt];
        sA[j * pitch + tt] = v;
    }
    __syncthreads();
    const size_t seq_stride = (size_t)HG;
    for (int j = warp; j < nh; j += kThreads / 32) {
        float part = 0.f;
        for (int tt = lane; tt < nt; tt += 32) part += sA[j * pitch + tt];
        const double agg = warp_sum_d((double)part);
        const size_t base = ((size_t)(b * g.n_hgroups + hg) * g.n_chunks) * HG + j;
        const size_t i = base + (size_t)rc * seq_stride;
        if (lane == 0) {
            if (rc == 0) {
                lb.incl[i] = agg;
                st_release(lb.flag + i, 2);
            } else {
                lb.agg[i] = agg;
                st_release(lb.flag + i, 1);
            }
            s_excl[j] = agg;
        }
    }
    __syncwarp();
    for (int j = warp; j < nh; j += kThreads / 32) {
        const size_t base = ((size_t)(b * g.n_hgroups + hg) * g.n_chunks) * HG + j;
        const double excl = rc == 0 ? 0.0 : lookback(lb, base, seq_stride, rc);
        if (lane == 0) {
            if (rc > 0) {
                const size_t i = base + (size_t)rc * seq_stride;
                lb.incl[i] = excl + s_excl[j];
                st_release(lb.flag + i, 2);
            }
            s_excl[j] = excl;
        }
    }
    __syncthreads();
    // 2. reverse inclusive scan: dalpha_t = carry - sum_{t' >= t} dU_t'.
    for (int j = warp; j < nh; j += kThreads / 32) {
        const int hh = hh0 + j;
        const double cr = carry ? carry[(int64_t)b * H + hh] : 0.0;
        double run = s_excl[j];
        float* arow = dalpha ? dalpha + ((int64_t)b * H + hh) * N + t0 : nullptr;
        const int last_row = ((nt - 1) / 32) * 32;
        for (int r = last_row; r >= 0; r -= 32) {
            float x = (r + lane < nt) ? sA[j * pitch + r + lane] : 0.f;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const float y = __shfl_down_sync(0xffffffffu, x, o);
                if (lane + o < 32) x += y;
            }
            const float da = (float)(cr - (run + (double)x));
            if (r + lane < nt) {
                if (arow) arow[r + lane] = da;
                sA[j * pitch + r + lane] = da;
            }
            run += (double)__shfl_sync(0xffffffffu, x, 0);
        }
    }
    if (!dh && !dbeta) return;
    __syncthreads();
    // 3. chain rule through Eq. 9 into dh, dbeta ([B,N,H], coalesced).
    for (int e = tid; e < T * HG; e += kThreads) {
        const int tt = e / HG, j = e - tt * HG;
        if (tt >= nt || j >= nh) continue;
        const int64_t i = ((int64_t)b * N + t0 + tt) * H + hh0 + j;
        const float da = sA[j * pitch + tt];
        if (kAlphaIn) {
            if (dh) dh[i] = from_f32<Tin>(da);
        } else {
            const float hv = load_in(h + i), bv = load_in(beta + i);
            const float z = bv * hv, be = bv + eps, sg = sigmoid_f(z);
            if (dh) dh[i] = from_f32<Tin>(da * sg * bv / be);
            if (dbeta) dbeta[i] = from_f32<Tin>(da * (sg * hv * be - softplus_f(z)) / (be * be));
        }
    }
}

template <typename Tin>
gfwa_status_t launch_fwd(gfwa_gate_kind_t kind, const void* h, const void* beta, int64_t B, int64_t N,
                         int64_t H, float eps, const double* carry_in, float* U, double* total,
                         const Lookback& lb, const ScanGeom& g, cudaStream_t st) {
    const size_t smem = (size_t)g.HG * (g.T + 1) * sizeof(float);
    const unsigned grid = (unsigned)(B * g.n_hgroups * g.n_chunks);
    auto k = kind == GFWA_GATE_ALPHA ? gate_prefix_kernel<Tin, true> : gate_prefix_kernel<Tin, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, kThreads, smem, st>>>((const Tin*)h, (const Tin*)beta, N, H, eps, carry_in, U, total, lb, g);
    note_launch();
    return check_launch();
}

template <typename Tin>
gfwa_status_t launch_bwd(gfwa_gate_kind_t kind, const void* h, const void* beta, int64_t B, int64_t N,
                         int64_t H, float eps, const float* dU, const double* carry, float* dalpha, void* dh,
                         void* dbeta, const Lookback& lb, const ScanGeom& g, cudaStream_t st) {
    const size_t smem = (size_t)g.HG * (g.T + 1) * sizeof(float);
    const unsigned grid = (unsigned)(B * g.n_hgroups * g.n_chunks);
    auto k = kind == GFWA_GATE_ALPHA ? gate_prefix_bwd_kernel<Tin, true> : gate_prefix_bwd_kernel<Tin, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, kThreads, smem, st>>>((const Tin*)h, (const Tin*)beta, N, H, eps, dU, carry, dalpha, (Tin*)dh,
                                    (Tin*)dbeta, lb, g);
    note_launch();
    return check_launch();
}

}  // namespace
}  // namespace gfwa

using namespace gfwa;

extern "C" size_t gfwa_gate_prefix_workspace_size(int64_t B, int64_t N, int64_t H) {
    if (B < 1 || N < 1 || H < 1) return 256;
    return lookback_bytes(B, scan_geom(N, H));
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
    const ScanGeom g = scan_geom(N, H);
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
    const ScanGeom g = scan_geom(N, H);
    if (ws_bytes < lookback_bytes(B, g)) return GFWA_ERR_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    if (gfwa_status_t s = check_launch(cudaMemsetAsync(ws, 0, lookback_bytes(B, g), st))) return s;
    const Lookback lb = carve(ws, B, g);
    if (in_dtype == GFWA_BF16)
        return launch_bwd<__nv_bfloat16>(kind, h, beta, B, N, H, eps, dU, carry, dalpha, dh, dbeta, lb, g, st);
    return launch_bwd<float>(kind, h, beta, B, N, H, eps, dU, carry, dalpha, dh, dbeta, lb, g, st);
}
