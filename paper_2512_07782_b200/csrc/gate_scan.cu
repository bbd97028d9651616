// gate_scan.cu -- gfwa_gate_prefix / gfwa_gate_prefix_bwd.
//
// Alg. 1 "Fused Tiled Scan" re-designed for B200: instead of one
// program per head walking its chunks serially with an on-chip carry
// (P:271), every (b, head-group, chunk) tile is an independent CTA and the
// carry is resolved with a single-pass *decoupled look-back*.  h and beta are
// read once and U written once (the paper's I/O claim), all accesses
// coalesced and vectorised:
//   load    [T tokens x HG heads] tile of h, beta ([B,N,H], H contiguous),
//           4 heads per load, one batch of independent loads per thread
//   alpha   softplus(beta h)/(beta + eps) in fp32 -> smem [HG][T] (transpose,
//           one pad word per lane run so the run reads are conflict-free)
//   scan    a warp owns HG/8 heads; lane l owns a run of R = T/32 tokens:
//           serial fp32 prefix, run totals scanned across the warp in fp64
//   carry   chunk aggregate published as one 64-bit word (fp64 value with the
//           2-bit status in its lowest mantissa bits: a single relaxed load
//           observes value and status together); a warp looks back for all
//           its heads at once, 32/(heads per warp) predecessors per round
//   store   U [B,H,N] rows (N contiguous), 16-byte vector stores
// 256-thread CTAs, 4 resident per SM, so one CTA's load phase overlaps the
// others' scan and store phases (one 1024-thread CTA per SM left the memory
// system idle during the scan: 0.38 TB/s).  The head-group size is a template
// parameter (power of two), so all tile index math is shifts and masks.  The
// backward runs the same machinery right to left on dU and fuses the
// chain rule into dh, dbeta.
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <type_traits>

#include "common.cuh"

namespace gfwa {
namespace {

constexpr int kThreads = 256;  // 8 warps
constexpr int kWarps = kThreads / 32;
constexpr int kMinBlocks = 4;  // resident CTAs per SM (64 registers / thread)
constexpr unsigned kFull = 0xffffffffu;
#ifndef GFWA_GATE_SMALL_LOG
#define GFWA_GATE_SMALL_LOG 22  // below 2^22 (b, t, h) elements: the LM-shape geometry
#endif

struct ScanGeom {
    int HG;        // heads per CTA (<= 32)
    int log_hgp;   // log2 of the head-group slot count (power of two >= HG)
    int log_t;     // log2 tokens per chunk (128 <= T <= 1024, so 4 <= R <= 32)
    int n_hgroups; // ceil(H / HG)
    int n_chunks;  // ceil(N / T)
    int n_seq;     // B * n_hgroups independent scans
};

ScanGeom scan_geom(int64_t B, int64_t N, int64_t H) {
    // The look-back chain, not HBM, sets the time at every measured size, so
    // chunks are long and head groups narrow (measured on B200, ncu):
    // LM shapes (< 2^22 (b, t, h) elements): 4-head groups x 512 tokens;
    // probe G: 8-head groups x 1024 tokens (32 x 256 before: 80 -> 65 us fwd,
    // 127 -> 93 us bwd).  T * HGP <= 8192 (the fp32 alpha tile in smem).
    ScanGeom g;
    const bool small = B * N * H < ((int64_t)1 << GFWA_GATE_SMALL_LOG);
    int lh = small ? 2 : 3, lt = small ? 9 : 10;
    if (const char* ge = getenv("GFWA_GATE_GEOM")) sscanf(ge, "%d,%d", &lh, &lt);  // experiments
    g.HG = (int)std::min<int64_t>(H, (int64_t)1 << std::min(std::max(lh, 0), 5));
    g.log_hgp = 0;
    while ((1 << g.log_hgp) < g.HG) ++g.log_hgp;
    g.log_t = std::max(7, std::min(lt, std::min(10, 13 - g.log_hgp)));
    g.n_hgroups = (int)((H + g.HG - 1) / g.HG);
    g.n_chunks = (int)((N + (1 << g.log_t) - 1) >> g.log_t);
    g.n_seq = (int)(B * g.n_hgroups);
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

// Exclusive prefixes over chunks 0..c-1 (in processing order) for the HPW
// heads j0, j0 + 8, ... a warp owns: the lanes form HPW groups of LPH =
// 32/HPW, group i walks back over head j_i's descriptors LPH predecessors per
// round until it meets an inclusive prefix.  Every lane returns its group's
// prefix.  d points at (this sequence/head-group, chunk 0, head 0).  Whole
// warp calls.
template <int HPW>
__device__ double lookback(const unsigned long long* d, int c, int j0, int nh) {
    constexpr int LPH = 32 / HPW;
    const int lane = threadIdx.x & 31;
    const int gi = lane / LPH, p = lane % LPH;
    const int j = j0 + kWarps * gi;
    const unsigned gmask = LPH == 32 ? kFull : (((1u << (LPH & 31)) - 1u) << (gi * LPH));
    double excl = 0.0;
    int pc = c - 1;
    bool done = j >= nh || c == 0;  // uniform within a group
    while (__any_sync(kFull, !done)) {
        const int q = pc - p;
        const bool act = !done && q >= 0;
        unsigned long long w = 0;
        if (act) {
            do {
                w = ld_relaxed_u64(d + (size_t)q * 32 + j);
            } while ((w & 3ull) == 0);
        }
        const unsigned incl = __ballot_sync(kFull, act && (w & 3ull) == 2) & gmask;
        double v = act ? __longlong_as_double((long long)(w & ~3ull)) : 0.0;
        if (incl && p > __ffs(incl) - 1 - gi * LPH) v = 0.0;  // beyond the closest inclusive prefix
#pragma unroll
        for (int o = LPH / 2; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        if (!done) excl += v;
        done = done || incl != 0 || pc < LPH;
        pc -= LPH;
    }
    return excl;
}

// 4 consecutive elements <-> fp32 (8-byte bf16 / 16-byte fp32 accesses)
template <typename Tin>
using Raw4 = std::conditional_t<sizeof(Tin) == 2, uint2, float4>;
__device__ __forceinline__ void unpack4(uint2 r, float (&v)[4]) {
    v[0] = __uint_as_float(r.x << 16);
    v[1] = __uint_as_float(r.x & 0xffff0000u);
    v[2] = __uint_as_float(r.y << 16);
    v[3] = __uint_as_float(r.y & 0xffff0000u);
}
__device__ __forceinline__ void unpack4(float4 r, float (&v)[4]) {
    v[0] = r.x;
    v[1] = r.y;
    v[2] = r.z;
    v[3] = r.w;
}
__device__ __forceinline__ void store4(__nv_bfloat16* p, const float (&v)[4]) {
    __nv_bfloat162 r[2] = {__floats2bfloat162_rn(v[0], v[1]), __floats2bfloat162_rn(v[2], v[3])};
    *reinterpret_cast<uint2*>(p) = *reinterpret_cast<const uint2*>(r);
}
__device__ __forceinline__ void store4(float* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}

template <typename Tin>
__device__ __forceinline__ float load_in(const Tin* p) { return to_f32<Tin>(*p); }

// alpha_t = softplus(beta_t h_t) / (beta_t + eps)  (Eq. 9, Alg. 1 l.6)
__device__ __forceinline__ float alpha_of(float hv, float bv, float eps) {
    return __fdividef(softplus_fast(bv * hv), bv + eps);
}

// smem index of token tt in a head row: one pad word per run of R tokens
__device__ __forceinline__ int sk(int tt, int log_r) { return tt + (tt >> log_r); }

// vectorised [B,N,H] tile access: all HGP heads present, rows 4-aligned
template <int HGP, typename Tin>
__device__ __forceinline__ bool tile_vec_ok(int nh, int64_t H, const Tin* a, const Tin* b) {
    return HGP >= 4 && nh == HGP && (H & 3) == 0 && ((uintptr_t)a % (4 * sizeof(Tin))) == 0 &&
           (b == nullptr || ((uintptr_t)b % (4 * sizeof(Tin))) == 0);
}

// ---------------------------------------------------------------- forward

template <typename Tin, bool kAlphaIn, int LOG_HGP>
__global__ void __launch_bounds__(kThreads, kMinBlocks) gate_prefix_kernel(
    const Tin* __restrict__ h, const Tin* __restrict__ beta, int64_t N, int64_t H, float eps,
    const double* __restrict__ carry_in, float* __restrict__ U, double* __restrict__ total, Lookback lb,
    ScanGeom g) {
    constexpr int HGP = 1 << LOG_HGP;
    constexpr int HPW = HGP > kWarps ? HGP / kWarps : 1;  // heads per warp
    extern __shared__ float sA[];                         // [HGP][pitch]
    __shared__ unsigned s_ticket;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_ticket = atomicAdd(lb.ticket, 1u);
    __syncthreads();
    const unsigned tk = s_ticket;
    // chunk-outer ticket order: a wave spans every sequence's leading chunks, so
    // look-back chains are as short as the wave allows
    const int c = (int)(tk / (unsigned)g.n_seq);
    const int rest = (int)(tk % (unsigned)g.n_seq);
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
    if (tile_vec_ok<HGP>(nh, H, h, kAlphaIn ? nullptr : beta)) {
        constexpr int LOG_G4 = LOG_HGP >= 2 ? LOG_HGP - 2 : 0;  // 4-head groups per token
        constexpr int kV = 8 / (int)sizeof(Tin);              // groups per thread per batch (64 B in flight)
        const int ngrp = T << LOG_G4;
        for (int e0 = tid; e0 < ngrp; e0 += kThreads * kV) {
            Raw4<Tin> rh[kV], rb[kV];
#pragma unroll
            for (int k = 0; k < kV; ++k) {
                const int e = e0 + k * kThreads;
                const int tt = e >> LOG_G4, j4 = e & ((1 << LOG_G4) - 1);
                if (e < ngrp && tt < nt) {
                    const int64_t i = row0 + (int64_t)tt * H + 4 * j4;
                    rh[k] = *reinterpret_cast<const Raw4<Tin>*>(h + i);
                    if (!kAlphaIn) rb[k] = *reinterpret_cast<const Raw4<Tin>*>(beta + i);
                }
            }
#pragma unroll
            for (int k = 0; k < kV; ++k) {
                const int e = e0 + k * kThreads;
                const int tt = e >> LOG_G4, j4 = e & ((1 << LOG_G4) - 1);
                if (e >= ngrp) continue;
                float hv[4], bv[4], a[4];
                unpack4(rh[k], hv);
                if (!kAlphaIn) unpack4(rb[k], bv);
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    a[i] = tt >= nt ? 0.f : kAlphaIn ? hv[i] : alpha_of(hv[i], bv[i], eps);
#pragma unroll
                for (int i = 0; i < 4; ++i) sA[(4 * j4 + i) * pitch + sk(tt, log_r)] = a[i];
            }
        }
    } else {
        constexpr int kB = 4;
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
                    if (tt < nt && j < nh) a = kAlphaIn ? hv[k] : alpha_of(hv[k], bv[k], eps);
                    sA[j * pitch + sk(tt, log_r)] = a;
                }
            }
        }
    }
    __syncthreads();

    // 2. lane runs (fp32), their inclusive scan across the warp (fp64), chunk
    //    aggregates published, look-back, inclusive prefixes published
    unsigned long long* d = lb.desc + (size_t)(b * g.n_hgroups + hg) * g.n_chunks * 32;
    float run[HPW];
    double xs[HPW];
#pragma unroll
    for (int i = 0; i < HPW; ++i) {
        const int j = warp + kWarps * i;
        run[i] = 0.f;
        if (j < nh) {
            const float* row = sA + j * pitch + lane * (R + 1);
            for (int k = 0; k < R; ++k) run[i] += row[k];
        }
        double x = (double)run[i];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
        }
        xs[i] = x;
        const double agg = __shfl_sync(kFull, x, 31);
        if (lane == 0 && j < nh) publish(d + (size_t)c * 32 + j, agg, c == 0 ? 2u : 1u);
    }
    const double ex = lookback<HPW>(d, c, warp, nh);

    // 3. U_t = carry - (prefix before this run) - (in-run fp32 prefix)  (Alg. 1 l.8-9)
    const int tl = lane * R;
#pragma unroll
    for (int i = 0; i < HPW; ++i) {
        const int j = warp + kWarps * i;
        if (j >= nh) continue;  // warp-uniform
        const double excl = __shfl_sync(kFull, ex, i * (32 / HPW));
        const double agg = __shfl_sync(kFull, xs[i], 31);
        if (lane == 0) {
            if (c > 0) publish(d + (size_t)c * 32 + j, excl + agg, 2u);
            if (total && c == g.n_chunks - 1) total[(int64_t)b * H + hh0 + j] = excl + agg;
        }
        const double carry = carry_in ? carry_in[(int64_t)b * H + hh0 + j] : 0.0;
        // carry-side base in fp64, split once per run into hi + lo fp32 words: each
        // U_t = hi + (lo - acc) then costs two fp32 adds, the first exact up to the
        // small in-run prefix, so U_t is rounded once (as an fp64 subtraction would)
        const double cbase = carry - (excl + xs[i] - (double)run[i]);
        const float chi = (float)cbase, clo = (float)(cbase - (double)chi);
        const float* row = sA + j * pitch + lane * (R + 1);
        float* urow = U + ((int64_t)b * H + hh0 + j) * N + t0 + tl;
        float acc = 0.f;
        if (tl + R <= nt && ((uintptr_t)urow & 15) == 0) {
            for (int k = 0; k < R; k += 4) {
                float4 o;
                acc += row[k];
                o.x = chi + (clo - acc);
                acc += row[k + 1];
                o.y = chi + (clo - acc);
                acc += row[k + 2];
                o.z = chi + (clo - acc);
                acc += row[k + 3];
                o.w = chi + (clo - acc);
                *reinterpret_cast<float4*>(urow + k) = o;
            }
        } else {
            for (int k = 0; k < R; ++k) {
                acc += row[k];
                if (tl + k < nt) urow[k] = chi + (clo - acc);
            }
        }
    }
}

// ---------------------------------------------------------------- backward

template <typename Tin, bool kAlphaIn, int LOG_HGP>
__global__ void __launch_bounds__(kThreads, kMinBlocks) gate_prefix_bwd_kernel(
    const Tin* __restrict__ h, const Tin* __restrict__ beta, int64_t N, int64_t H, float eps,
    const float* __restrict__ dU, const double* __restrict__ carry, float* __restrict__ dalpha,
    Tin* __restrict__ dh, Tin* __restrict__ dbeta, Lookback lb, ScanGeom g) {
    constexpr int HGP = 1 << LOG_HGP;
    constexpr int HPW = HGP > kWarps ? HGP / kWarps : 1;
    extern __shared__ float sA[];  // [HGP][pitch]
    __shared__ unsigned s_ticket;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_ticket = atomicAdd(lb.ticket, 1u);
    __syncthreads();
    const unsigned tk = s_ticket;
    const int rc = (int)(tk / (unsigned)g.n_seq);  // order of processing: right to left, chunk-outer
    const int c = g.n_chunks - 1 - rc;
    const int rest = (int)(tk % (unsigned)g.n_seq);
    const int hg = rest % g.n_hgroups;
    const int b = rest / g.n_hgroups;
    const int T = 1 << g.log_t, log_r = g.log_t - 5, R = T >> 5;
    const int pitch = T + 32 + 1;
    const int64_t t0 = (int64_t)c << g.log_t;
    const int hh0 = hg * g.HG;
    const int nh = min(g.HG, (int)(H - hh0));
    const int nt = (int)min64(T, N - t0);
    const int tl = lane * R;

    // 1. dU rows (N contiguous): lane l's run of R tokens straight into its
    //    smem run (16-byte loads when aligned; conflict-free stores)
#pragma unroll 1
    for (int i = 0; i < HPW; ++i) {
        const int j = warp + kWarps * i;
        if (j >= nh) continue;
        const float* src = dU + ((int64_t)b * H + hh0 + j) * N + t0 + tl;
        float* row = sA + j * pitch + lane * (R + 1);
        if (tl + R <= nt && ((uintptr_t)src & 15) == 0) {
            float4 v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (4 * k < R) v[k] = *reinterpret_cast<const float4*>(src + 4 * k);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (4 * k < R) {
                    row[4 * k] = v[k].x;
                    row[4 * k + 1] = v[k].y;
                    row[4 * k + 2] = v[k].z;
                    row[4 * k + 3] = v[k].w;
                }
        } else {
            for (int k = 0; k < R; ++k) row[k] = tl + k < nt ? src[k] : 0.f;
        }
    }
    __syncwarp();

    // 2. reverse scan: dalpha_t = carry - sum_{t' >= t} dU_t'  (suffix sums)
    unsigned long long* d = lb.desc + (size_t)(b * g.n_hgroups + hg) * g.n_chunks * 32;
    float run[HPW];
    double xs[HPW];
#pragma unroll
    for (int i = 0; i < HPW; ++i) {
        const int j = warp + kWarps * i;
        run[i] = 0.f;
        if (j < nh) {
            const float* row = sA + j * pitch + lane * (R + 1);
            for (int k = 0; k < R; ++k) run[i] += row[k];
        }
        double x = (double)run[i];  // inclusive suffix scan of the lane runs
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_down_sync(kFull, x, o);
            if (lane + o < 32) x += y;
        }
        xs[i] = x;
        const double agg = __shfl_sync(kFull, x, 0);
        if (lane == 0 && j < nh) publish(d + (size_t)rc * 32 + j, agg, rc == 0 ? 2u : 1u);
    }
    const double ex = lookback<HPW>(d, rc, warp, nh);
#pragma unroll
    for (int i = 0; i < HPW; ++i) {
        const int j = warp + kWarps * i;
        if (j >= nh) continue;  // warp-uniform
        const double excl = __shfl_sync(kFull, ex, i * (32 / HPW));
        const double agg = __shfl_sync(kFull, xs[i], 0);
        if (lane == 0 && rc > 0) publish(d + (size_t)rc * 32 + j, excl + agg, 2u);
        const double cr = carry ? carry[(int64_t)b * H + hh0 + j] : 0.0;
        const double cbase = cr - (excl + xs[i] - (double)run[i]);  // fp64, as in the forward
        float* row = sA + j * pitch + lane * (R + 1);
        float* arow = dalpha ? dalpha + ((int64_t)b * H + hh0 + j) * N + t0 + tl : nullptr;
        float acc = 0.f;
        if (arow && tl + R <= nt && ((uintptr_t)arow & 15) == 0) {
            for (int k = R - 4; k >= 0; k -= 4) {
                float4 o;
                acc += row[k + 3];
                o.w = (float)(cbase - (double)acc);
                acc += row[k + 2];
                o.z = (float)(cbase - (double)acc);
                acc += row[k + 1];
                o.y = (float)(cbase - (double)acc);
                acc += row[k];
                o.x = (float)(cbase - (double)acc);
                row[k] = o.x;  // kept for the chain rule
                row[k + 1] = o.y;
                row[k + 2] = o.z;
                row[k + 3] = o.w;
                *reinterpret_cast<float4*>(arow + k) = o;
            }
        } else {
            for (int k = R - 1; k >= 0; --k) {
                acc += row[k];
                const float da = (float)(cbase - (double)acc);
                row[k] = da;
                if (arow && tl + k < nt) arow[k] = da;
            }
        }
    }
    if (!dh && !dbeta) return;
    __syncthreads();

    // 3. chain rule through Eq. 9 into dh, dbeta ([B,N,H], coalesced):
    //    d alpha/dh = beta sigma(beta h)/(beta+eps),
    //    d alpha/dbeta = (h sigma(beta h)(beta+eps) - softplus(beta h))/(beta+eps)^2
    const int64_t row0 = ((int64_t)b * N + t0) * H + hh0;
    if (tile_vec_ok<HGP>(nh, H, kAlphaIn ? dh : h, kAlphaIn ? nullptr : beta) &&
        (!dh || ((uintptr_t)dh % (4 * sizeof(Tin))) == 0) &&
        (!dbeta || ((uintptr_t)dbeta % (4 * sizeof(Tin))) == 0)) {
        constexpr int LOG_G4 = LOG_HGP >= 2 ? LOG_HGP - 2 : 0;
        constexpr int kV = 4 / (int)sizeof(Tin);
        const int ngrp = T << LOG_G4;
        for (int e0 = tid; e0 < ngrp; e0 += kThreads * kV) {
            Raw4<Tin> rh[kV], rb[kV];
            if (!kAlphaIn) {
#pragma unroll
                for (int k = 0; k < kV; ++k) {
                    const int e = e0 + k * kThreads;
                    const int tt = e >> LOG_G4, j4 = e & ((1 << LOG_G4) - 1);
                    if (e < ngrp && tt < nt) {
                        const int64_t i = row0 + (int64_t)tt * H + 4 * j4;
                        rh[k] = *reinterpret_cast<const Raw4<Tin>*>(h + i);
                        rb[k] = *reinterpret_cast<const Raw4<Tin>*>(beta + i);
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < kV; ++k) {
                const int e = e0 + k * kThreads;
                const int tt = e >> LOG_G4, j4 = e & ((1 << LOG_G4) - 1);
                if (e >= ngrp || tt >= nt) continue;
                const int64_t i = row0 + (int64_t)tt * H + 4 * j4;
                float da[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) da[q] = sA[(4 * j4 + q) * pitch + sk(tt, log_r)];
                if (kAlphaIn) {
                    if (dh) store4(dh + i, da);
                } else {
                    float hv[4], bv[4], gh[4], gb[4];
                    unpack4(rh[k], hv);
                    unpack4(rb[k], bv);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float z = bv[q] * hv[q], be = bv[q] + eps;
                        float sp, sg;
                        softplus_sigmoid_fast(z, sp, sg);
                        const float rbe = __fdividef(1.f, be);
                        gh[q] = da[q] * sg * bv[q] * rbe;
                        gb[q] = da[q] * (sg * hv[q] * be - sp) * (rbe * rbe);
                    }
                    if (dh) store4(dh + i, gh);
                    if (dbeta) store4(dbeta + i, gb);
                }
            }
        }
        return;
    }
    constexpr int kB = 4;
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
                const float z = bv[k] * hv[k], be = bv[k] + eps;
                float sp, sg;
                softplus_sigmoid_fast(z, sp, sg);
                const float rbe = __fdividef(1.f, be);
                if (dh) dh[i] = from_f32<Tin>(da * sg * bv[k] * rbe);
                if (dbeta) dbeta[i] = from_f32<Tin>(da * (sg * hv[k] * be - sp) * (rbe * rbe));
            }
        }
    }
}

template <typename Tin, bool kAlpha, int L>
void launch_fwd_t(const void* h, const void* beta, int64_t B, int64_t N, int64_t H, float eps,
                  const double* carry_in, float* U, double* total, const Lookback& lb, const ScanGeom& g,
                  cudaStream_t st) {
    const size_t smem = (size_t)(1 << L) * ((1 << g.log_t) + 33) * sizeof(float);  // <= 37 KB
    auto k = gate_prefix_kernel<Tin, kAlpha, L>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<(unsigned)(B * g.n_hgroups * g.n_chunks), kThreads, smem, st>>>((const Tin*)h, (const Tin*)beta, N, H, eps,
                                                                       carry_in, U, total, lb, g);
}

template <typename Tin, bool kAlpha, int L>
void launch_bwd_t(const void* h, const void* beta, int64_t B, int64_t N, int64_t H, float eps, const float* dU,
                  const double* carry, float* dalpha, void* dh, void* dbeta, const Lookback& lb, const ScanGeom& g,
                  cudaStream_t st) {
    const size_t smem = (size_t)(1 << L) * ((1 << g.log_t) + 33) * sizeof(float);  // <= 37 KB
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
