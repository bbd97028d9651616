// attn_simt.cu -- CUDA-core (SIMT) GatedFWA forward/backward.
//
// This is the exact-arithmetic parity path (fp32 in, fp32 math; also accepts
// bf16 inputs): Alg. 2 and Alg. E.2 tiled 64x64 with
// the paper's three changes -- window tile pruning, the bias as an
// outer difference of u vectors and the in-tile window mask
// -- and the paper's two-kernel backward split:
//   bwd_kv_kernel : dK, dV, dU^k   (KV-major, loops over in-window Q tiles)
//   bwd_q_kernel  : dQ, dU^q       (Q-major,  loops over in-window K tiles)
// Neither uses atomics, so results are deterministic.  The bf16 tensor-core
// kernels (attn_tc_*.cu) replace this path for BF16 when d = 128.
#include "attn_common.cuh"

namespace gfwa {
namespace {

constexpr int BM = 64;       // rows per CTA
constexpr int BN = 64;       // columns per inner tile
constexpr int kThreads = 256;  // 8 warps x 8 rows

template <typename T>
__device__ __forceinline__ void load_tile(float* dst, int pitch, const T* base, const int64_t* s, int64_t b,
                                          int64_t h, int64_t n0, int64_t nmax, int D) {
    // dst[r][c] = base[b, n0 + r, h, c] as fp32, zero outside [0, nmax)
    for (int e = threadIdx.x; e < 64 * D; e += kThreads) {
        const int r = e / D, c = e - r * D;
        const int64_t n = n0 + r;
        float v = 0.f;
        if (n >= 0 && n < nmax) v = to_f32<T>(base[off3(s, b, n, h) + c]);
        dst[r * pitch + c] = v;
    }
}

// ------------------------------------------------------------------ forward
template <typename T, int D>
__global__ void __launch_bounds__(kThreads) fwd_simt_kernel(AttnParams p) {
    extern __shared__ float sm[];
    constexpr int P = D + 1;
    float* Qs = sm;                 // [64][D+1]
    float* Ks = Qs + 64 * P;        // [64][D+1]
    float* Vs = Ks + 64 * P;        // [64][D+1]
    float* Ps = Vs + 64 * P;        // [64][65]
    float* uq = Ps + 64 * 65;       // [64] u of the query rows
    float* uk = uq + 64;            // [64] u of the key columns
    // The bias is formed as (u_q - u_k) in fp32 first (near-Sterbenz exact for
    // nearby tokens) and only then scaled to log2 units (reading C-18).
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t b = blockIdx.z, h = blockIdx.y;
    const int64_t q0 = (int64_t)blockIdx.x * BM;  // first query of the tile
    const float sl2 = p.scale * kLog2e;           // logits kept in log2 units
    const float* Ubh = p.U + (b * p.H + h) * p.Nkv;

    load_tile<T>(Qs, P, (const T*)p.Q, p.qs, b, h, q0, p.Nq, D);
    for (int r = threadIdx.x; r < BM; r += kThreads) {
        const int64_t t = q0 + r;
        uq[r] = t < p.Nq ? Ubh[t + p.h0] : 0.f;
    }
    // Alg. 2 l.7-9: key range of the tile (key positions g = t + h0)
    const int64_t g_first = q0 + p.h0;
    const int64_t g_last = min(q0 + BM, p.Nq) - 1 + p.h0;
    const int64_t k_lo = max64(0, g_first - p.w + 1);
    const int64_t kt_lo = k_lo / BN, kt_hi = g_last / BN;

    float o[8][D / 32];
    float m[8], l[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        m[i] = -INFINITY;
        l[i] = 0.f;
#pragma unroll
        for (int x = 0; x < D / 32; ++x) o[i][x] = 0.f;
    }
    for (int64_t kt = kt_lo; kt <= kt_hi; ++kt) {
        const int64_t j0 = kt * BN;
        __syncthreads();
        load_tile<T>(Ks, P, (const T*)p.K, p.ks, b, h, j0, p.Nkv, D);
        load_tile<T>(Vs, P, (const T*)p.V, p.vs, b, h, j0, p.Nkv, D);
        for (int c = threadIdx.x; c < BN; c += kThreads) uk[c] = j0 + c < p.Nkv ? Ubh[j0 + c] : 0.f;
        __syncthreads();
        float s[8][2];
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = 0.f;
        for (int k = 0; k < D; ++k) {
            const float k0 = Ks[lane * P + k], k1 = Ks[(lane + 32) * P + k];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float qv = Qs[(warp * 8 + i) * P + k];
                s[i][0] = fmaf(qv, k0, s[i][0]);
                s[i][1] = fmaf(qv, k1, s[i][1]);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int r = warp * 8 + i;
            const int64_t g = q0 + r + p.h0;
            float mx = -INFINITY;
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                const int64_t j = j0 + lane + 32 * cc;
                // Alg. 2 l.12-15: bias u_q - u_k, keep iff g-w+1 <= j <= g
                const bool keep = (q0 + r < p.Nq) && j <= g && j > g - p.w && j < p.Nkv;
                s[i][cc] = keep ? fmaf(s[i][cc], sl2, (uq[r] - uk[lane + 32 * cc]) * kLog2e) : -INFINITY;
                mx = fmaxf(mx, s[i][cc]);
            }
            mx = warp_max(mx);
            const float mn = fmaxf(m[i], mx);
            const float corr = (mn == -INFINITY) ? 1.f : exp2f(m[i] - mn);
            const float p0 = (mn == -INFINITY) ? 0.f : exp2f(s[i][0] - mn);
            const float p1 = (mn == -INFINITY) ? 0.f : exp2f(s[i][1] - mn);
            l[i] = l[i] * corr + warp_sum(p0 + p1);
            m[i] = mn;
#pragma unroll
            for (int x = 0; x < D / 32; ++x) o[i][x] *= corr;
            Ps[r * 65 + lane] = p0;
            Ps[r * 65 + lane + 32] = p1;
        }
        __syncwarp();
        for (int c = 0; c < BN; ++c) {
            float v[D / 32];
#pragma unroll
            for (int x = 0; x < D / 32; ++x) v[x] = Vs[c * P + lane + 32 * x];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float pv = Ps[(warp * 8 + i) * 65 + c];
#pragma unroll
                for (int x = 0; x < D / 32; ++x) o[i][x] = fmaf(pv, v[x], o[i][x]);
            }
        }
    }
    // Alg. 2 l.19-20: o / l, L = m + log l (natural log, C-10)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t t = q0 + warp * 8 + i;
        if (t >= p.Nq) continue;
        const float inv = 1.f / l[i];
        T* orow = (T*)p.O + off3(p.os, b, t, h);
        T* lrow = p.O_lo ? (T*)p.O_lo + off3(p.os, b, t, h) : nullptr;
#pragma unroll
        for (int x = 0; x < D / 32; ++x) {
            const float v = o[i][x] * inv;
            const T hi = from_f32<T>(v);
            orow[lane + 32 * x] = hi;
            if (lrow) lrow[lane + 32 * x] = from_f32<T>(v - to_f32<T>(hi));  // residual of the cast (C-12)
        }
        if (lane == 0) p.LSE[(b * p.H + h) * p.Nq + t] = (m[i] + log2f(l[i])) * kLn2;
    }
}

// --------------------------------------------------------- backward: D = rowsum(O dO)
template <typename T>
__global__ void __launch_bounds__(256) bwd_pre_kernel(AttnParams p) {
    // one warp per (b, t, h) row; Alg. E.2 l.7, O + O_lo when given (C-12)
    const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const int64_t total = p.B * p.Nq * p.H;
    if (row >= total) return;
    const int64_t h = row % p.H, t = (row / p.H) % p.Nq, b = row / (p.H * p.Nq);
    const int64_t oo = off3(p.os, b, t, h);
    const T* dO = (const T*)p.dO + oo;
    float acc = 0.f;
    if (p.Olo) {
        const T* o = (const T*)p.O + oo;
        const T* ol = (const T*)p.Olo + oo;
        for (int c = lane; c < p.d; c += 32) acc = fmaf(to_f32<T>(o[c]) + to_f32<T>(ol[c]), to_f32<T>(dO[c]), acc);
    } else {
        const T* o = (const T*)p.O + oo;
        for (int c = lane; c < p.d; c += 32) acc = fmaf(to_f32<T>(o[c]), to_f32<T>(dO[c]), acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) p.Dv[(b * p.H + h) * p.Nq + t] = acc;
}

// ------------------------------------------------- backward: dK, dV, dU^k (KV-major)
template <typename T, int D>
__global__ void __launch_bounds__(kThreads) bwd_kv_kernel(AttnParams p) {
    extern __shared__ float sm[];
    constexpr int P = D + 1;
    float* Ks = sm;              // [64 keys][D+1]
    float* Vs = Ks + 64 * P;     // [64 keys][D+1]
    float* Qs = Vs + 64 * P;     // [64 queries][D+1]
    float* dOs = Qs + 64 * P;    // [64 queries][D+1]
    float* Ps = dOs + 64 * P;    // [64 keys][65]
    float* dSs = Ps + 64 * 65;   // [64 keys][65]
    float* uq = dSs + 64 * 65;   // [64]
    float* lse = uq + 64;        // [64] log2 units
    float* Dq = lse + 64;        // [64]
    float* uk = Dq + 64;         // [64]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t b = blockIdx.z, h = blockIdx.y;
    const int64_t j0 = (int64_t)blockIdx.x * BN;  // first key of this tile
    const float sl2 = p.scale * kLog2e;
    const float* Ubh = p.U + (b * p.H + h) * p.Nkv;

    load_tile<T>(Ks, P, (const T*)p.K, p.ks, b, h, j0, p.Nkv, D);
    load_tile<T>(Vs, P, (const T*)p.V, p.vs, b, h, j0, p.Nkv, D);
    for (int c = threadIdx.x; c < BN; c += kThreads) uk[c] = j0 + c < p.Nkv ? Ubh[j0 + c] : 0.f;

    float dk[8][D / 32], dv[8][D / 32], dsum[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        dsum[i] = 0.f;
#pragma unroll
        for (int x = 0; x < D / 32; ++x) dk[i][x] = dv[i][x] = 0.f;
    }
    // Alg. E.2 l.12-14: queries whose window reaches this key tile
    const int64_t j_last = min(j0 + BN, p.Nkv) - 1;
    const int64_t t_lo = max64(0, j0 - p.h0);
    const int64_t t_hi = min64(p.Nq - 1, j_last + p.w - 1 - p.h0);
    if (t_lo <= t_hi) {
        for (int64_t qt = t_lo / BM; qt <= t_hi / BM; ++qt) {
            const int64_t q0 = qt * BM;
            __syncthreads();
            load_tile<T>(Qs, P, (const T*)p.Q, p.qs, b, h, q0, p.Nq, D);
            load_tile<T>(dOs, P, (const T*)p.dO, p.os, b, h, q0, p.Nq, D);
            for (int r = threadIdx.x; r < BM; r += kThreads) {
                const int64_t t = q0 + r;
                const bool ok = t < p.Nq;
                uq[r] = ok ? Ubh[t + p.h0] : 0.f;
                lse[r] = ok ? p.LSE[(b * p.H + h) * p.Nq + t] * kLog2e : 0.f;
                Dq[r] = ok ? p.Dv[(b * p.H + h) * p.Nq + t] : 0.f;
            }
            __syncthreads();
            float s[8][2], dp[8][2];
#pragma unroll
            for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = dp[i][0] = dp[i][1] = 0.f;
            for (int k = 0; k < D; ++k) {
                const float q0v = Qs[lane * P + k], q1v = Qs[(lane + 32) * P + k];
                const float g0v = dOs[lane * P + k], g1v = dOs[(lane + 32) * P + k];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float kv = Ks[(warp * 8 + i) * P + k];
                    const float vv = Vs[(warp * 8 + i) * P + k];
                    s[i][0] = fmaf(kv, q0v, s[i][0]);
                    s[i][1] = fmaf(kv, q1v, s[i][1]);
                    dp[i][0] = fmaf(vv, g0v, dp[i][0]);
                    dp[i][1] = fmaf(vv, g1v, dp[i][1]);
                }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int kr = warp * 8 + i;
                const int64_t j = j0 + kr;
                float colsum = 0.f;
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                    const int c = lane + 32 * cc;
                    const int64_t t = q0 + c;
                    const int64_t g = t + p.h0;
                    const bool keep = t < p.Nq && j < p.Nkv && j <= g && j > g - p.w;
                    // P = exp(S - L), dS = P (dP - D)
                    const float pr = keep ? exp2f(fmaf(s[i][cc], sl2, (uq[c] - uk[kr]) * kLog2e) - lse[c]) : 0.f;
                    const float ds = pr * (dp[i][cc] - Dq[c]);
                    Ps[kr * 65 + c] = pr;
                    dSs[kr * 65 + c] = ds;
                    colsum += ds;
                }
                dsum[i] += warp_sum(colsum);
            }
            __syncwarp();
            for (int c = 0; c < BM; ++c) {
                float qv[D / 32], gv[D / 32];
#pragma unroll
                for (int x = 0; x < D / 32; ++x) {
                    qv[x] = Qs[c * P + lane + 32 * x];
                    gv[x] = dOs[c * P + lane + 32 * x];
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float pv = Ps[(warp * 8 + i) * 65 + c];
                    const float dsv = dSs[(warp * 8 + i) * 65 + c];
#pragma unroll
                    for (int x = 0; x < D / 32; ++x) {
                        dv[i][x] = fmaf(pv, gv[x], dv[i][x]);  // dV += P^T dO
                        dk[i][x] = fmaf(dsv, qv[x], dk[i][x]); // dK += dS^T Q
                    }
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t j = j0 + warp * 8 + i;
        if (j >= p.Nkv) continue;
        T* dkr = (T*)p.dK + off3(p.ks, b, j, h);
        T* dvr = (T*)p.dV + off3(p.vs, b, j, h);
#pragma unroll
        for (int x = 0; x < D / 32; ++x) {
            dkr[lane + 32 * x] = from_f32<T>(dk[i][x] * p.scale);  // reading C-3
            dvr[lane + 32 * x] = from_f32<T>(dv[i][x]);
        }
        // dU^k_j = -sum_t dS_tj (reading C-4); dU^q is added by bwd_q_kernel
        if (lane == 0) p.dU[(b * p.H + h) * p.Nkv + j] = -dsum[i];
    }
}

// ------------------------------------------------- backward: dQ, dU^q (Q-major)
template <typename T, int D>
__global__ void __launch_bounds__(kThreads) bwd_q_kernel(AttnParams p) {
    extern __shared__ float sm[];
    constexpr int P = D + 1;
    float* Qs = sm;              // [64 queries][D+1]
    float* dOs = Qs + 64 * P;    // [64 queries][D+1]
    float* Ks = dOs + 64 * P;    // [64 keys][D+1]
    float* Vs = Ks + 64 * P;     // [64 keys][D+1]
    float* dSs = Vs + 64 * P;    // [64 queries][65]
    float* uq = dSs + 64 * 65;
    float* lse = uq + 64;
    float* Dq = lse + 64;
    float* uk = Dq + 64;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t b = blockIdx.z, h = blockIdx.y;
    const int64_t q0 = (int64_t)blockIdx.x * BM;
    const float sl2 = p.scale * kLog2e;
    const float* Ubh = p.U + (b * p.H + h) * p.Nkv;
    load_tile<T>(Qs, P, (const T*)p.Q, p.qs, b, h, q0, p.Nq, D);
    load_tile<T>(dOs, P, (const T*)p.dO, p.os, b, h, q0, p.Nq, D);
    for (int r = threadIdx.x; r < BM; r += kThreads) {
        const int64_t t = q0 + r;
        const bool ok = t < p.Nq;
        uq[r] = ok ? Ubh[t + p.h0] : 0.f;
        lse[r] = ok ? p.LSE[(b * p.H + h) * p.Nq + t] * kLog2e : 0.f;
        Dq[r] = ok ? p.Dv[(b * p.H + h) * p.Nq + t] : 0.f;
    }
    const int64_t g_first = q0 + p.h0;
    const int64_t g_last = min(q0 + BM, p.Nq) - 1 + p.h0;
    const int64_t kt_lo = max64(0, g_first - p.w + 1) / BN, kt_hi = g_last / BN;
    float dq[8][D / 32], rsum[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        rsum[i] = 0.f;
#pragma unroll
        for (int x = 0; x < D / 32; ++x) dq[i][x] = 0.f;
    }
    for (int64_t kt = kt_lo; kt <= kt_hi; ++kt) {
        const int64_t j0 = kt * BN;
        __syncthreads();
        load_tile<T>(Ks, P, (const T*)p.K, p.ks, b, h, j0, p.Nkv, D);
        load_tile<T>(Vs, P, (const T*)p.V, p.vs, b, h, j0, p.Nkv, D);
        for (int c = threadIdx.x; c < BN; c += kThreads) uk[c] = j0 + c < p.Nkv ? Ubh[j0 + c] : 0.f;
        __syncthreads();
        float s[8][2], dp[8][2];
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = dp[i][0] = dp[i][1] = 0.f;
        for (int k = 0; k < D; ++k) {
            const float k0 = Ks[lane * P + k], k1 = Ks[(lane + 32) * P + k];
            const float v0 = Vs[lane * P + k], v1 = Vs[(lane + 32) * P + k];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float qv = Qs[(warp * 8 + i) * P + k];
                const float gv = dOs[(warp * 8 + i) * P + k];
                s[i][0] = fmaf(qv, k0, s[i][0]);
                s[i][1] = fmaf(qv, k1, s[i][1]);
                dp[i][0] = fmaf(gv, v0, dp[i][0]);
                dp[i][1] = fmaf(gv, v1, dp[i][1]);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int r = warp * 8 + i;
            const int64_t t = q0 + r, g = t + p.h0;
            float rs = 0.f;
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                const int c = lane + 32 * cc;
                const int64_t j = j0 + c;
                const bool keep = t < p.Nq && j < p.Nkv && j <= g && j > g - p.w;
                const float pr = keep ? exp2f(fmaf(s[i][cc], sl2, (uq[r] - uk[c]) * kLog2e) - lse[r]) : 0.f;
                const float ds = pr * (dp[i][cc] - Dq[r]);
                dSs[r * 65 + c] = ds;
                rs += ds;
            }
            rsum[i] += warp_sum(rs);
        }
        __syncwarp();
        for (int c = 0; c < BN; ++c) {
            float kv[D / 32];
#pragma unroll
            for (int x = 0; x < D / 32; ++x) kv[x] = Ks[c * P + lane + 32 * x];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float dsv = dSs[(warp * 8 + i) * 65 + c];
#pragma unroll
                for (int x = 0; x < D / 32; ++x) dq[i][x] = fmaf(dsv, kv[x], dq[i][x]);  // dQ += dS K
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t t = q0 + warp * 8 + i;
        if (t >= p.Nq) continue;
        T* dqr = (T*)p.dQ + off3(p.qs, b, t, h);
#pragma unroll
        for (int x = 0; x < D / 32; ++x) dqr[lane + 32 * x] = from_f32<T>(dq[i][x] * p.scale);
        // dU^q_t = rowsum(dS) at key position t + h0 (reading C-11)
        if (lane == 0) p.dU[(b * p.H + h) * p.Nkv + t + p.h0] += rsum[i];
    }
}

template <typename T, int D>
gfwa_status_t fwd_launch(const AttnParams& p, cudaStream_t st) {
    const size_t smem = (size_t)(3 * 64 * (D + 1) + 64 * 65 + 128) * sizeof(float);
    auto k = fwd_simt_kernel<T, D>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((unsigned)((p.Nq + BM - 1) / BM), (unsigned)p.H, (unsigned)p.B);
    k<<<grid, kThreads, smem, st>>>(p);
    note_launch();
    return check_launch();
}

template <typename T, int D>
gfwa_status_t bwd_launch(const AttnParams& p, cudaStream_t st) {
    {
        const size_t smem = (size_t)(4 * 64 * (D + 1) + 2 * 64 * 65 + 256) * sizeof(float);
        auto k = bwd_kv_kernel<T, D>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        dim3 grid((unsigned)((p.Nkv + BN - 1) / BN), (unsigned)p.H, (unsigned)p.B);
        k<<<grid, kThreads, smem, st>>>(p);
        note_launch();
        if (gfwa_status_t s = check_launch()) return s;
    }
    {
        const size_t smem = (size_t)(4 * 64 * (D + 1) + 64 * 65 + 256) * sizeof(float);
        auto k = bwd_q_kernel<T, D>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        dim3 grid((unsigned)((p.Nq + BM - 1) / BM), (unsigned)p.H, (unsigned)p.B);
        k<<<grid, kThreads, smem, st>>>(p);
        note_launch();
        return check_launch();
    }
}

}  // namespace

gfwa_status_t simt_fwd(const AttnParams& p, gfwa_dtype_t dt, cudaStream_t st) {
    if (dt == GFWA_F32) return p.d == 64 ? fwd_launch<float, 64>(p, st) : fwd_launch<float, 128>(p, st);
    return p.d == 64 ? fwd_launch<__nv_bfloat16, 64>(p, st) : fwd_launch<__nv_bfloat16, 128>(p, st);
}

gfwa_status_t bwd_preprocess(const AttnParams& p, gfwa_dtype_t dt, cudaStream_t st) {
    const int64_t rows = p.B * p.Nq * p.H;
    const unsigned grid = (unsigned)((rows + 7) / 8);
    if (dt == GFWA_F32)
        bwd_pre_kernel<float><<<grid, 256, 0, st>>>(p);
    else
        bwd_pre_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(p);
    note_launch();
    return check_launch();
}

gfwa_status_t simt_bwd(const AttnParams& p, gfwa_dtype_t dt, cudaStream_t st) {
    if (dt == GFWA_F32) return p.d == 64 ? bwd_launch<float, 64>(p, st) : bwd_launch<float, 128>(p, st);
    return p.d == 64 ? bwd_launch<__nv_bfloat16, 64>(p, st) : bwd_launch<__nv_bfloat16, 128>(p, st);
}

}  // namespace gfwa
