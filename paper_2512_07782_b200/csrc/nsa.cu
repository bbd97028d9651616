// nsa.cu -- the NSA extension with GatedFWA as its local branch (App. B,
// P:633-703; readings C-28, C-29), forward.
//
//   compress   Kc, Vc = block means of K, V (C-28: phi = mean, length = stride = blk)
//   cmp+select one warp per query (b, h, t): the scores scale q.Kc_i of the blocks
//              that end at or before t (staged in shared memory), their softmax
//              attention o_cmp (online, fp32), and the selection (C-29): the
//              query's own block, then the n_sel complete blocks with the largest
//              scores (ties to the lower index) by n_sel warp arg-max rounds
//   slc        one warp per query: online-softmax attention over the tokens <= t
//              of the selected blocks (lane = 2 or 4 head-dim channels, bf16 K/V
//              rows read coalesced)
//   combine    O = sigmoid(g0) o_cmp + sigmoid(g1) o_slc + sigmoid(g2) o_loc
// The local branch o_loc is gfwa_fwd (the tensor-core GatedFWA kernel).
// These are CUDA-core kernels: the compressed branch is ~N/blk keys per query and
// the selected branch (n_sel + 1) blk keys, a small multiple of the local window.
// The per-query / per-block walks take kU keys (queries) per round: their rows are
// loaded together and the kU warp reductions interleaved, so a round pays one
// load latency and one reduction latency instead of kU (the serial per-key walk
// was latency-bound).
#include "common.cuh"

namespace gfwa {
namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int kU = 8;  // keys per round in the selected-branch kernels (loads in flight, interleaved reductions)

__device__ __forceinline__ uint32_t pack_bf16x2_nsa(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
constexpr int kMaxBlocks = 512;  // compressed blocks per sequence held in shared memory per warp

__global__ void nsa_compress_kernel(const __nv_bfloat16* __restrict__ K, const __nv_bfloat16* __restrict__ V,
                                    float* __restrict__ Kc, float* __restrict__ Vc, int64_t B, int64_t N, int64_t H,
                                    int d, int blk) {
    const int64_t nb = N / blk;
    const int64_t total = B * nb * H * d;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(e % d);
        const int64_t r = e / d;  // (b, i, h)
        const int64_t hh = r % H, i = (r / H) % nb, b = r / (H * nb);
        float sk = 0.f, sv = 0.f;
        for (int j = 0; j < blk; ++j) {
            const int64_t x = ((b * N + i * blk + j) * H + hh) * d + c;
            sk += __bfloat162float(K[x]);
            sv += __bfloat162float(V[x]);
        }
        Kc[e] = sk / (float)blk;
        Vc[e] = sv / (float)blk;
    }
}

template <int D>
__device__ __forceinline__ void load_row(const __nv_bfloat16* p, int lane, float (&v)[D / 32]) {
    constexpr int C = D / 32;  // 2 or 4 consecutive channels per lane
    if constexpr (C == 4) {
        const uint2 w = *reinterpret_cast<const uint2*>(p + 4 * lane);
        v[0] = __uint_as_float(w.x << 16);
        v[1] = __uint_as_float(w.x & 0xffff0000u);
        v[2] = __uint_as_float(w.y << 16);
        v[3] = __uint_as_float(w.y & 0xffff0000u);
    } else {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(p + 2 * lane);
        v[0] = __uint_as_float(w << 16);
        v[1] = __uint_as_float(w & 0xffff0000u);
    }
}

// the same row left packed (C / 2 words of bf16 pairs), unpacked at use
template <int D>
__device__ __forceinline__ void load_raw(const __nv_bfloat16* p, int lane, uint32_t (&w)[D / 64]) {
    if constexpr (D / 64 == 2) {
        const uint2 x = *reinterpret_cast<const uint2*>(p + 4 * lane);
        w[0] = x.x;
        w[1] = x.y;
    } else {
        w[0] = *reinterpret_cast<const uint32_t*>(p + 2 * lane);
    }
}
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

template <int D>
__global__ void __launch_bounds__(32 * kWarpsPerBlock) nsa_cmp_select_kernel(
    const __nv_bfloat16* __restrict__ Q, const float* __restrict__ Kc, const float* __restrict__ Vc,
    float* __restrict__ Ocmp, float* __restrict__ Lcmp, int* __restrict__ sel, int64_t B, int64_t N, int64_t H,
    int blk, int nsel, float scale) {
    constexpr int C = D / 32;
    __shared__ float s_sc[kWarpsPerBlock][kMaxBlocks];
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int64_t row = (int64_t)blockIdx.x * kWarpsPerBlock + wp;  // (b, t, h)
    if (row >= B * N * H) return;
    const int64_t hh = row % H, t = (row / H) % N, b = row / (H * N);
    const int64_t nb = N / blk;
    const int nc = (int)((t + 1) / blk);  // complete blocks: (i + 1) blk - 1 <= t
    float q[C];
    load_row<D>(Q + row * D, lane, q);
    float* sc = s_sc[wp];
    // scores and the online softmax of the compressed branch
    float m = -INFINITY, l = 0.f, acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = 0.f;
    for (int i = 0; i < nc; ++i) {
        const float* kr = Kc + ((b * nb + i) * H + hh) * D + C * lane;
        float s = 0.f;
#pragma unroll
        for (int c = 0; c < C; ++c) s = fmaf(q[c], kr[c], s);
        s = warp_sum(s) * scale;
        if (lane == 0) sc[i] = s;
        const float mn = fmaxf(m, s);
        const float corr = __expf(m - mn), p = __expf(s - mn);
        const float* vr = Vc + ((b * nb + i) * H + hh) * D + C * lane;
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] = acc[c] * corr + p * vr[c];
        l = l * corr + p;
        m = mn;
    }
    float* o = Ocmp + row * D + C * lane;
#pragma unroll
    for (int c = 0; c < C; ++c) o[c] = nc > 0 ? acc[c] / l : 0.f;
    if (lane == 0) Lcmp[(b * H + hh) * N + t] = nc > 0 ? m + __logf(l) : -INFINITY;
    __syncwarp();
    // selection (C-29): own block first, then n_sel arg-max rounds over the other complete blocks
    const int own = (int)(t / blk);
    int* out = sel + ((b * H + hh) * N + t) * (nsel + 1);
    if (lane == 0) out[0] = own;
    if (own < nc && lane == 0) sc[own] = -INFINITY;  // the own block is complete: not a candidate twice
    __syncwarp();
    for (int k = 1; k <= nsel; ++k) {
        float bv = -INFINITY;
        int bi = -1;
        for (int i = lane; i < nc; i += 32) {
            const float v = sc[i];
            if (v > bv) {  // strided ascending: the first maximum seen is the lowest index
                bv = v;
                bi = i;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (ov > bv || (ov == bv && oi >= 0 && (bi < 0 || oi < bi))) {
                bv = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            out[k] = bv == -INFINITY ? -1 : bi;
            if (bi >= 0 && bv != -INFINITY) sc[bi] = -INFINITY;
        }
        __syncwarp();
    }
}

template <int D>
__global__ void __launch_bounds__(32 * kWarpsPerBlock) nsa_slc_kernel(
    const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ K, const __nv_bfloat16* __restrict__ V,
    const int* __restrict__ sel, float* __restrict__ Oslc, float* __restrict__ Lslc, int64_t B, int64_t N, int64_t H,
    int blk, int nsel, float scale) {
    constexpr int C = D / 32;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int64_t row = (int64_t)blockIdx.x * kWarpsPerBlock + wp;
    if (row >= B * N * H) return;
    const int64_t hh = row % H, t = (row / H) % N, b = row / (H * N);
    float q[C];
    load_row<D>(Q + row * D, lane, q);
    const int* sl = sel + ((b * H + hh) * N + t) * (nsel + 1);
    float m = -INFINITY, l = 0.f, acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = 0.f;
    for (int k = 0; k <= nsel; ++k) {
        const int ib = sl[k];
        if (ib < 0) continue;
        const int64_t j1 = min64((int64_t)(ib + 1) * blk - 1, t);
        // kU keys per round: their K and V rows loaded together, the kU dot products
        // reduced across the warp interleaved, one online-softmax update per round
        for (int64_t j = (int64_t)ib * blk; j <= j1; j += kU) {
            const int nk = (int)min64(kU, j1 - j + 1);
            float kv[kU][C], sc[kU];
            uint32_t vv[kU][C / 2];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int64_t ju = u < nk ? j + u : j;  // tail: re-read row j, masked below
                load_row<D>(K + ((b * N + ju) * H + hh) * D, lane, kv[u]);
                load_raw<D>(V + ((b * N + ju) * H + hh) * D, lane, vv[u]);
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                float x = 0.f;
#pragma unroll
                for (int c = 0; c < C; ++c) x = fmaf(q[c], kv[u][c], x);
                sc[u] = x;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int u = 0; u < kU; ++u) sc[u] += __shfl_xor_sync(0xffffffffu, sc[u], o);
            float mx = -INFINITY;
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                sc[u] = u < nk ? sc[u] * scale : -INFINITY;
                mx = fmaxf(mx, sc[u]);
            }
            const float mn = fmaxf(m, mx);  // finite: nk >= 1
            const float corr = __expf(m - mn);
            l *= corr;
#pragma unroll
            for (int c = 0; c < C; ++c) acc[c] *= corr;
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const float pu = __expf(sc[u] - mn);
                l += pu;
#pragma unroll
                for (int c = 0; c < C; c += 2) {
                    acc[c] = fmaf(pu, bf_lo(vv[u][c / 2]), acc[c]);
                    acc[c + 1] = fmaf(pu, bf_hi(vv[u][c / 2]), acc[c + 1]);
                }
            }
            m = mn;
        }
    }
    float* o = Oslc + row * D + C * lane;
#pragma unroll
    for (int c = 0; c < C; ++c) o[c] = acc[c] / l;  // the own block always holds token t: l > 0
    if (lane == 0) Lslc[(b * H + hh) * N + t] = m + __logf(l);
}

__global__ void nsa_combine_kernel(const float* __restrict__ Ocmp, const float* __restrict__ Oslc,
                                   const __nv_bfloat16* __restrict__ Oloc, const float* __restrict__ g,
                                   __nv_bfloat16* __restrict__ O, int64_t rows, int d) {
    const int64_t total = rows * d;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / d;
        const float a = 1.f / (1.f + __expf(-g[3 * r])), s = 1.f / (1.f + __expf(-g[3 * r + 1])),
                    lo = 1.f / (1.f + __expf(-g[3 * r + 2]));
        O[e] = __float2bfloat16_rn(a * Ocmp[e] + s * Oslc[e] + lo * __bfloat162float(Oloc[e]));
    }
}


// ------------------------------------------------------------------ backward (fixed selection)

// per row: the branch gradients of the gated sum and the rows' D terms
template <int D>
__global__ void __launch_bounds__(32 * kWarpsPerBlock) nsa_combine_bwd_kernel(
    const __nv_bfloat16* __restrict__ dO, const float* __restrict__ g, const float* __restrict__ Ocmp,
    const float* __restrict__ Oslc, const __nv_bfloat16* __restrict__ Oloc, const __nv_bfloat16* __restrict__ Ololo,
    float* __restrict__ dOc, float* __restrict__ dOs, __nv_bfloat16* __restrict__ dOl, float* __restrict__ dg,
    float* __restrict__ Dc, float* __restrict__ Ds, int64_t B, int64_t N, int64_t H) {
    constexpr int C = D / 32;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int64_t row = (int64_t)blockIdx.x * kWarpsPerBlock + wp;
    if (row >= B * N * H) return;
    const int64_t hh = row % H, t = (row / H) % N, b = row / (H * N);
    float go[C], ol[C], ll[C];
    load_row<D>(dO + row * D, lane, go);
    load_row<D>(Oloc + row * D, lane, ol);
    if (Ololo) {
        load_row<D>(Ololo + row * D, lane, ll);
#pragma unroll
        for (int c = 0; c < C; ++c) ol[c] += ll[c];
    }
    const float* oc = Ocmp + row * D + C * lane;
    const float* os = Oslc + row * D + C * lane;
    float sgm[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) sgm[k] = 1.f / (1.f + __expf(-g[3 * row + k]));
    float dotc = 0.f, dots = 0.f, dotl = 0.f;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        dotc = fmaf(go[c], oc[c], dotc);
        dots = fmaf(go[c], os[c], dots);
        dotl = fmaf(go[c], ol[c], dotl);
        dOc[row * D + C * lane + c] = sgm[0] * go[c];
        dOs[row * D + C * lane + c] = sgm[1] * go[c];
    }
    if constexpr (C == 4) {
        uint2 w;
        w.x = pack_bf16x2_nsa(sgm[2] * go[0], sgm[2] * go[1]);
        w.y = pack_bf16x2_nsa(sgm[2] * go[2], sgm[2] * go[3]);
        *reinterpret_cast<uint2*>(dOl + row * D + 4 * lane) = w;
    } else {
        *reinterpret_cast<uint32_t*>(dOl + row * D + 2 * lane) = pack_bf16x2_nsa(sgm[2] * go[0], sgm[2] * go[1]);
    }
    dotc = warp_sum(dotc);
    dots = warp_sum(dots);
    dotl = warp_sum(dotl);
    if (lane == 0) {
        dg[3 * row] = sgm[0] * (1.f - sgm[0]) * dotc;
        dg[3 * row + 1] = sgm[1] * (1.f - sgm[1]) * dots;
        dg[3 * row + 2] = sgm[2] * (1.f - sgm[2]) * dotl;
        // D = rowsum(o * dO_branch): dO_branch = sigmoid(g) dO
        Dc[(b * H + hh) * N + t] = sgm[0] * dotc;
        Ds[(b * H + hh) * N + t] = sgm[1] * dots;
    }
}

// compressed branch, query side: dq = scale sum_i p_i (dO_cmp . Vc_i - D) Kc_i
template <int D>
__global__ void __launch_bounds__(32 * kWarpsPerBlock) nsa_cmp_dq_kernel(
    const __nv_bfloat16* __restrict__ Q, const float* __restrict__ Kc, const float* __restrict__ Vc,
    const float* __restrict__ dOc, const float* __restrict__ Lc, const float* __restrict__ Dc,
    float* __restrict__ dQacc, int64_t B, int64_t N, int64_t H, int blk, float scale) {
    constexpr int C = D / 32;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int64_t row = (int64_t)blockIdx.x * kWarpsPerBlock + wp;
    if (row >= B * N * H) return;
    const int64_t hh = row % H, t = (row / H) % N, b = row / (H * N);
    const int64_t nb = N / blk;
    const int nc = (int)((t + 1) / blk);
    float q[C], go[C], dq[C];
    load_row<D>(Q + row * D, lane, q);
#pragma unroll
    for (int c = 0; c < C; ++c) {
        go[c] = dOc[row * D + C * lane + c];
        dq[c] = 0.f;
    }
    const float L = Lc[(b * H + hh) * N + t], Dv = Dc[(b * H + hh) * N + t];
    for (int i0 = 0; i0 < nc; i0 += kU) {
        const int ni = min(kU, nc - i0);
        float kr[kU][C], sc[kU], dp[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int i = u < ni ? i0 + u : i0;
            const float* kp = Kc + ((b * nb + i) * H + hh) * D + C * lane;
            const float* vp = Vc + ((b * nb + i) * H + hh) * D + C * lane;
            float x = 0.f, y = 0.f;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                kr[u][c] = kp[c];
                x = fmaf(q[c], kr[u][c], x);
                y = fmaf(go[c], vp[c], y);
            }
            sc[u] = x;
            dp[u] = y;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                sc[u] += __shfl_xor_sync(0xffffffffu, sc[u], o);
                dp[u] += __shfl_xor_sync(0xffffffffu, dp[u], o);
            }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const float ds = u < ni ? __expf(sc[u] * scale - L) * (dp[u] - Dv) : 0.f;
#pragma unroll
            for (int c = 0; c < C; ++c) dq[c] = fmaf(scale * ds, kr[u][c], dq[c]);
        }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) dQacc[row * D + C * lane + c] = dq[c];
}

// compressed branch, block side (one warp per (b, block, h), every query that sees it):
// dKc = scale sum_t dS q_t, dVc = sum_t p dO_cmp,t
template <int D>
__global__ void __launch_bounds__(32 * kWarpsPerBlock) nsa_cmp_dkv_kernel(
    const __nv_bfloat16* __restrict__ Q, const float* __restrict__ Kc, const float* __restrict__ Vc,
    const float* __restrict__ dOc, const float* __restrict__ Lc, const float* __restrict__ Dc,
    float* __restrict__ dKc, float* __restrict__ dVc, int64_t B, int64_t N, int64_t H, int blk, float scale) {
    constexpr int C = D / 32;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int64_t nb = N / blk;
    const int64_t r = (int64_t)blockIdx.x * kWarpsPerBlock + wp;  // (b, i, h)
    if (r >= B * nb * H) return;
    const int64_t hh = r % H, i = (r / H) % nb, b = r / (H * nb);
    float kc[C], vc[C], dk[C], dv[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        kc[c] = Kc[r * D + C * lane + c];
        vc[c] = Vc[r * D + C * lane + c];
        dk[c] = 0.f;
        dv[c] = 0.f;
    }
    // kU queries per round: their rows, L and D loaded together, reductions interleaved
    for (int64_t t0 = (i + 1) * blk - 1; t0 < N; t0 += kU) {
        const int nt = (int)min64(kU, N - t0);
        float q[kU][C], go[kU][C], sc[kU], dp[kU], Lt[kU], Dt[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t t = u < nt ? t0 + u : t0;
            const int64_t row = (b * N + t) * H + hh;
            load_row<D>(Q + row * D, lane, q[u]);
#pragma unroll
            for (int c = 0; c < C; ++c) go[u][c] = dOc[row * D + C * lane + c];
            Lt[u] = Lc[(b * H + hh) * N + t];
            Dt[u] = Dc[(b * H + hh) * N + t];
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            float x = 0.f, y = 0.f;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                x = fmaf(q[u][c], kc[c], x);
                y = fmaf(go[u][c], vc[c], y);
            }
            sc[u] = x;
            dp[u] = y;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                sc[u] += __shfl_xor_sync(0xffffffffu, sc[u], o);
                dp[u] += __shfl_xor_sync(0xffffffffu, dp[u], o);
            }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const float p = u < nt ? __expf(sc[u] * scale - Lt[u]) : 0.f;
            const float ds = p * (dp[u] - Dt[u]);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                dk[c] = fmaf(scale * ds, q[u][c], dk[c]);
                dv[c] = fmaf(p, go[u][c], dv[c]);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
        dKc[r * D + C * lane + c] = dk[c];
        dVc[r * D + C * lane + c] = dv[c];
    }
}

// selected branch, query side: dq into the query's row (added)
template <int D>
__global__ void __launch_bounds__(32 * kWarpsPerBlock) nsa_slc_bwd_kernel(
    const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ K, const __nv_bfloat16* __restrict__ V,
    const int* __restrict__ sel, const float* __restrict__ dOs, const float* __restrict__ Ls,
    const float* __restrict__ Ds, float* __restrict__ dQacc, int64_t B, int64_t N, int64_t H, int blk, int nsel,
    float scale) {
    constexpr int C = D / 32;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int64_t row = (int64_t)blockIdx.x * kWarpsPerBlock + wp;
    if (row >= B * N * H) return;
    const int64_t hh = row % H, t = (row / H) % N, b = row / (H * N);
    float q[C], go[C], dq[C];
    load_row<D>(Q + row * D, lane, q);
#pragma unroll
    for (int c = 0; c < C; ++c) {
        go[c] = dOs[row * D + C * lane + c];
        dq[c] = 0.f;
    }
    const float L = Ls[(b * H + hh) * N + t], Dv = Ds[(b * H + hh) * N + t];
    const int* sl = sel + ((b * H + hh) * N + t) * (nsel + 1);
    for (int k = 0; k <= nsel; ++k) {
        const int ib = sl[k];
        if (ib < 0) continue;
        const int64_t j1 = min64((int64_t)(ib + 1) * blk - 1, t);
        for (int64_t j = (int64_t)ib * blk; j <= j1; j += kU) {
            const int nk = (int)min64(kU, j1 - j + 1);
            float kv[kU][C], sc[kU], dp[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int64_t kr = (b * N + (u < nk ? j + u : j)) * H + hh;
                float vv[C];
                load_row<D>(K + kr * D, lane, kv[u]);
                load_row<D>(V + kr * D, lane, vv);
                float x = 0.f, y = 0.f;
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    x = fmaf(q[c], kv[u][c], x);
                    y = fmaf(go[c], vv[c], y);
                }
                sc[u] = x;
                dp[u] = y;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    sc[u] += __shfl_xor_sync(0xffffffffu, sc[u], o);
                    dp[u] += __shfl_xor_sync(0xffffffffu, dp[u], o);
                }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const float p = u < nk ? __expf(sc[u] * scale - L) : 0.f, ds = p * (dp[u] - Dv);
#pragma unroll
                for (int c = 0; c < C; ++c) dq[c] = fmaf(scale * ds, kv[u][c], dq[c]);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) dQacc[row * D + C * lane + c] += dq[c];
}


// selected branch, block side: the queries that selected each block are listed
// (count, scan, fill), then one CTA per (b, h, block) accumulates the block's dK, dV
// in registers over its queries -- no atomics on the gradients
__global__ void nsa_sel_count_kernel(const int* __restrict__ sel, int* __restrict__ cnt, int64_t BH, int64_t N,
                                     int nsel, int nbp) {
    const int64_t total = BH * N * (nsel + 1);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int ib = sel[e];
        if (ib >= 0) atomicAdd(cnt + (e / ((int64_t)N * (nsel + 1))) * nbp + ib, 1);
    }
}
// exclusive scan of the counts per (b, h): one warp per (b, h); cur = the fill cursors
__global__ void nsa_sel_scan_kernel(const int* __restrict__ cnt, int* __restrict__ off, int* __restrict__ cur,
                                    int64_t BH, int nbp) {
    const int64_t bh = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (bh >= BH) return;
    int run = 0;
    for (int i0 = 0; i0 < nbp; i0 += 32) {
        const int i = i0 + lane;
        const int v = i < nbp ? cnt[bh * nbp + i] : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (i < nbp) {
            off[bh * nbp + i] = run + x - v;
            cur[bh * nbp + i] = run + x - v;
        }
        run += __shfl_sync(0xffffffffu, x, 31);
    }
}
__global__ void nsa_sel_fill_kernel(const int* __restrict__ sel, int* __restrict__ cur, int* __restrict__ list,
                                    int64_t BH, int64_t N, int nsel, int nbp) {
    const int64_t total = BH * N * (nsel + 1);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int ib = sel[e];
        if (ib < 0) continue;
        const int64_t bh = e / ((int64_t)N * (nsel + 1));
        const int t = (int)((e / (nsel + 1)) % N);
        list[bh * N * (nsel + 1) + atomicAdd(cur + bh * nbp + ib, 1)] = t;
    }
}

// 256 threads: thread = (key kk = tid / 4 of the block's <= 64 keys, channels (tid % 4) + 4 m)
template <int D>
__global__ void __launch_bounds__(256) nsa_slc_dkv_kernel(
    const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ K, const __nv_bfloat16* __restrict__ V,
    const float* __restrict__ dOs, const float* __restrict__ Ls, const float* __restrict__ Ds,
    const int* __restrict__ off, const int* __restrict__ cnt, const int* __restrict__ list,
    float* __restrict__ dKacc, float* __restrict__ dVacc, int64_t B, int64_t N, int64_t H, int blk, int nsel,
    int nbp, float scale) {
    constexpr int M = D / 4;  // channels per thread
    constexpr int kQB = 16;
    __shared__ float s_q[kQB][D], s_go[kQB][D], s_L[kQB], s_D[kQB];
    __shared__ int s_t[kQB];
    const int64_t r = blockIdx.x;  // (b, h, block)
    const int ib = (int)(r % nbp);
    const int64_t bh = r / nbp, hh = bh % H, b = bh / H;
    const int kk = threadIdx.x >> 2, sub = threadIdx.x & 3;
    const int64_t j = (int64_t)ib * blk + kk;
    const bool kvalid = kk < blk && j < N;
    float kr[M], vr[M], dk[M], dv[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const int c = sub + 4 * m;
        kr[m] = kvalid ? __bfloat162float(K[((b * N + j) * H + hh) * D + c]) : 0.f;
        vr[m] = kvalid ? __bfloat162float(V[((b * N + j) * H + hh) * D + c]) : 0.f;
        dk[m] = 0.f;
        dv[m] = 0.f;
    }
    const int n = cnt[r], o0 = off[r];
    const int* lst = list + bh * N * (nsel + 1) + o0;
    // kQB listed queries staged per round (their Q / dO rows, L, D loaded together)
    for (int q0 = 0; q0 < n; q0 += kQB) {
        const int nq = min(kQB, n - q0);
        __syncthreads();  // the previous round's rows are consumed
        for (int e = threadIdx.x; e < nq * D; e += blockDim.x) {
            const int qi = e / D, c = e % D;
            const int64_t row = (b * N + lst[q0 + qi]) * H + hh;
            s_q[qi][c] = __bfloat162float(Q[row * D + c]);
            s_go[qi][c] = dOs[row * D + c];
        }
        if (threadIdx.x < nq) {
            const int t = lst[q0 + threadIdx.x];
            s_t[threadIdx.x] = t;
            s_L[threadIdx.x] = Ls[bh * N + t];
            s_D[threadIdx.x] = Ds[bh * N + t];
        }
        __syncthreads();
        for (int qi = 0; qi < nq; ++qi) {
            float s = 0.f, dp = 0.f;
#pragma unroll
            for (int m = 0; m < M; ++m) {
                s = fmaf(s_q[qi][sub + 4 * m], kr[m], s);
                dp = fmaf(s_go[qi][sub + 4 * m], vr[m], dp);
            }
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            s += __shfl_xor_sync(0xffffffffu, s, 2);
            dp += __shfl_xor_sync(0xffffffffu, dp, 1);
            dp += __shfl_xor_sync(0xffffffffu, dp, 2);
            if (!kvalid || j > s_t[qi]) continue;  // causal inside the block
            const float p = __expf(s * scale - s_L[qi]);
            const float ds = p * (dp - s_D[qi]);
#pragma unroll
            for (int m = 0; m < M; ++m) {
                dk[m] = fmaf(scale * ds, s_q[qi][sub + 4 * m], dk[m]);
                dv[m] = fmaf(p, s_go[qi][sub + 4 * m], dv[m]);
            }
        }
    }
    if (!kvalid) return;
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const int c = sub + 4 * m;
        dKacc[((b * N + j) * H + hh) * D + c] = dk[m];
        dVacc[((b * N + j) * H + hh) * D + c] = dv[m];
    }
}

// dQ = dQ_loc + dQacc; dK = dK_loc + dKacc + dKc(block) / blk; dV likewise -> bf16
__global__ void nsa_finalize_kernel(const __nv_bfloat16* __restrict__ dQl, const __nv_bfloat16* __restrict__ dKl,
                                    const __nv_bfloat16* __restrict__ dVl, const float* __restrict__ dQacc,
                                    const float* __restrict__ dKacc, const float* __restrict__ dVacc,
                                    const float* __restrict__ dKc, const float* __restrict__ dVc,
                                    __nv_bfloat16* __restrict__ dQ, __nv_bfloat16* __restrict__ dK,
                                    __nv_bfloat16* __restrict__ dV, int64_t B, int64_t N, int64_t H, int d, int blk) {
    const int64_t nb = N / blk, total = B * N * H * d;
    const float inv = 1.f / (float)blk;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(e % d);
        const int64_t r = e / d, hh = r % H, j = (r / H) % N, b = r / (H * N);
        float kc = 0.f, vc = 0.f;
        if (j / blk < nb) {
            const int64_t x = ((b * nb + j / blk) * H + hh) * d + c;
            kc = dKc[x] * inv;
            vc = dVc[x] * inv;
        }
        dQ[e] = __float2bfloat16_rn(__bfloat162float(dQl[e]) + dQacc[e]);
        dK[e] = __float2bfloat16_rn(__bfloat162float(dKl[e]) + dKacc[e] + kc);
        dV[e] = __float2bfloat16_rn(__bfloat162float(dVl[e]) + dVacc[e] + vc);
    }
}

}  // namespace

size_t nsa_workspace(int64_t B, int64_t N, int64_t H, int d, int blk, int nsel) {
    const int64_t nb = N / blk;
    size_t n = 0;
    auto add = [&](size_t bytes) { n += (bytes + 255) & ~(size_t)255; };
    add((size_t)B * nb * H * d * 4 * 2);    // Kc, Vc
    add((size_t)B * N * H * d * 4 * 2);     // o_cmp, o_slc
    add((size_t)B * H * N * (nsel + 1) * 4);  // selection
    add((size_t)B * N * H * d * 2);         // o_loc
    add((size_t)B * H * N * 4 * 3);         // LSE of the local, compressed and selected branches
    return n;
}

// the branches and the combination; o_loc (bf16) was written by gfwa_fwd
gfwa_status_t nsa_fwd_branches(const void* Q, const void* K, const void* V, const float* g, int64_t B, int64_t N,
                               int64_t H, int d, int blk, int nsel, float scale, float* Kc, float* Vc, float* Ocmp,
                               float* Oslc, float* Lcmp, float* Lslc, int* sel, const void* Oloc, void* O,
                               cudaStream_t st, bool compress_only) {
    int dev = 0, n_sm = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t nb = N / blk;
    if (nb > 0) {
        nsa_compress_kernel<<<(unsigned)min64((B * nb * H * d + 255) / 256, (int64_t)n_sm * 16), 256, 0, st>>>(
            (const __nv_bfloat16*)K, (const __nv_bfloat16*)V, Kc, Vc, B, N, H, d, blk);
        note_launch();
    }
    if (compress_only) return check_launch();
    const int64_t rows = B * N * H;
    const unsigned grid = (unsigned)((rows + kWarpsPerBlock - 1) / kWarpsPerBlock);
    if (d == 64) {
        nsa_cmp_select_kernel<64><<<grid, 32 * kWarpsPerBlock, 0, st>>>((const __nv_bfloat16*)Q, Kc, Vc, Ocmp, Lcmp,
                                                                        sel, B, N, H, blk, nsel, scale);
        nsa_slc_kernel<64><<<grid, 32 * kWarpsPerBlock, 0, st>>>((const __nv_bfloat16*)Q, (const __nv_bfloat16*)K,
                                                                 (const __nv_bfloat16*)V, sel, Oslc, Lslc, B, N, H,
                                                                 blk, nsel, scale);
    } else {
        nsa_cmp_select_kernel<128><<<grid, 32 * kWarpsPerBlock, 0, st>>>((const __nv_bfloat16*)Q, Kc, Vc, Ocmp, Lcmp,
                                                                         sel, B, N, H, blk, nsel, scale);
        nsa_slc_kernel<128><<<grid, 32 * kWarpsPerBlock, 0, st>>>((const __nv_bfloat16*)Q, (const __nv_bfloat16*)K,
                                                                  (const __nv_bfloat16*)V, sel, Oslc, Lslc, B, N, H,
                                                                  blk, nsel, scale);
    }
    note_launch(2);
    nsa_combine_kernel<<<(unsigned)min64((rows * d + 255) / 256, (int64_t)n_sm * 16), 256, 0, st>>>(
        Ocmp, Oslc, (const __nv_bfloat16*)Oloc, g, (__nv_bfloat16*)O, rows, d);
    note_launch();
    return check_launch();
}

bool nsa_blocks_ok(int64_t N, int blk) { return N / blk <= kMaxBlocks; }

// backward, phase 1: per-row gradients of the gated sum (dO_loc for gfwa_bwd, D terms)
gfwa_status_t nsa_bwd_combine(const void* dO, const float* g, const float* Ocmp, const float* Oslc, const void* Oloc,
                              const void* Ololo, float* dOc, float* dOs, void* dOl, float* dg, float* Dc, float* Ds,
                              int64_t B, int64_t N, int64_t H, int d, cudaStream_t st) {
    const unsigned grid = (unsigned)((B * N * H + kWarpsPerBlock - 1) / kWarpsPerBlock);
    if (d == 64)
        nsa_combine_bwd_kernel<64><<<grid, 32 * kWarpsPerBlock, 0, st>>>(
            (const __nv_bfloat16*)dO, g, Ocmp, Oslc, (const __nv_bfloat16*)Oloc, (const __nv_bfloat16*)Ololo, dOc, dOs,
            (__nv_bfloat16*)dOl, dg, Dc, Ds, B, N, H);
    else
        nsa_combine_bwd_kernel<128><<<grid, 32 * kWarpsPerBlock, 0, st>>>(
            (const __nv_bfloat16*)dO, g, Ocmp, Oslc, (const __nv_bfloat16*)Oloc, (const __nv_bfloat16*)Ololo, dOc, dOs,
            (__nv_bfloat16*)dOl, dg, Dc, Ds, B, N, H);
    note_launch();
    return check_launch();
}

// backward, phase 2: compressed and selected branches, then the sums with the local
// branch's dQ, dK, dV (bf16, from gfwa_bwd)
gfwa_status_t nsa_bwd_branches(const void* Q, const void* K, const void* V, const int* sel, const float* Kc,
                               const float* Vc, const float* dOc, const float* dOs, const float* Lc, const float* Ls,
                               const float* Dc, const float* Ds, float* dQacc, float* dKacc, float* dVacc, float* dKc,
                               float* dVc, const void* dQl, const void* dKl, const void* dVl, void* dQ, void* dK,
                               void* dV, int64_t B, int64_t N, int64_t H, int d, int blk, int nsel, float scale,
                               int* scnt, int* soff, int* scur, int* slist, cudaStream_t st) {
    int dev = 0, n_sm = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t n = B * N * H * d, nb = N / blk;
    if (gfwa_status_t s = check_launch(cudaMemsetAsync(dKacc, 0, n * sizeof(float), st))) return s;
    if (gfwa_status_t s = check_launch(cudaMemsetAsync(dVacc, 0, n * sizeof(float), st))) return s;
    const unsigned gq = (unsigned)((B * N * H + kWarpsPerBlock - 1) / kWarpsPerBlock);
    const unsigned gb = (unsigned)((B * nb * H + kWarpsPerBlock - 1) / kWarpsPerBlock);
    // the queries of each selectable block (own blocks include the partial last one)
    const int nbp = (int)((N + blk - 1) / blk);
    const int64_t nsl = B * H * N * (nsel + 1);
    if (gfwa_status_t s = check_launch(cudaMemsetAsync(scnt, 0, (size_t)B * H * nbp * sizeof(int), st))) return s;
    const unsigned gs = (unsigned)min64((nsl + 255) / 256, (int64_t)n_sm * 16);
    nsa_sel_count_kernel<<<gs, 256, 0, st>>>(sel, scnt, B * H, N, nsel, nbp);
    nsa_sel_scan_kernel<<<(unsigned)((B * H + 7) / 8), 256, 0, st>>>(scnt, soff, scur, B * H, nbp);
    nsa_sel_fill_kernel<<<gs, 256, 0, st>>>(sel, scur, slist, B * H, N, nsel, nbp);
    note_launch(3);
    auto Qb = (const __nv_bfloat16*)Q;
    if (d == 64) {
        nsa_cmp_dq_kernel<64><<<gq, 32 * kWarpsPerBlock, 0, st>>>(Qb, Kc, Vc, dOc, Lc, Dc, dQacc, B, N, H, blk, scale);
        if (nb > 0)
            nsa_cmp_dkv_kernel<64><<<gb, 32 * kWarpsPerBlock, 0, st>>>(Qb, Kc, Vc, dOc, Lc, Dc, dKc, dVc, B, N, H, blk,
                                                                       scale);
        nsa_slc_bwd_kernel<64><<<gq, 32 * kWarpsPerBlock, 0, st>>>(Qb, (const __nv_bfloat16*)K,
                                                                   (const __nv_bfloat16*)V, sel, dOs, Ls, Ds, dQacc,
                                                                   B, N, H, blk, nsel, scale);
        nsa_slc_dkv_kernel<64><<<(unsigned)(B * H * nbp), 256, 0, st>>>(
            Qb, (const __nv_bfloat16*)K, (const __nv_bfloat16*)V, dOs, Ls, Ds, soff, scnt, slist, dKacc, dVacc, B, N,
            H, blk, nsel, nbp, scale);
    } else {
        nsa_cmp_dq_kernel<128><<<gq, 32 * kWarpsPerBlock, 0, st>>>(Qb, Kc, Vc, dOc, Lc, Dc, dQacc, B, N, H, blk, scale);
        if (nb > 0)
            nsa_cmp_dkv_kernel<128><<<gb, 32 * kWarpsPerBlock, 0, st>>>(Qb, Kc, Vc, dOc, Lc, Dc, dKc, dVc, B, N, H,
                                                                        blk, scale);
        nsa_slc_bwd_kernel<128><<<gq, 32 * kWarpsPerBlock, 0, st>>>(Qb, (const __nv_bfloat16*)K,
                                                                    (const __nv_bfloat16*)V, sel, dOs, Ls, Ds, dQacc,
                                                                    B, N, H, blk, nsel, scale);
        nsa_slc_dkv_kernel<128><<<(unsigned)(B * H * nbp), 256, 0, st>>>(
            Qb, (const __nv_bfloat16*)K, (const __nv_bfloat16*)V, dOs, Ls, Ds, soff, scnt, slist, dKacc, dVacc, B, N,
            H, blk, nsel, nbp, scale);
    }
    note_launch(nb > 0 ? 4 : 3);
    nsa_finalize_kernel<<<(unsigned)min64((n + 255) / 256, (int64_t)n_sm * 16), 256, 0, st>>>(
        (const __nv_bfloat16*)dQl, (const __nv_bfloat16*)dKl, (const __nv_bfloat16*)dVl, dQacc, dKacc, dVacc, dKc, dVc,
        (__nv_bfloat16*)dQ, (__nv_bfloat16*)dK, (__nv_bfloat16*)dV, B, N, H, d, blk);
    note_launch();
    return check_launch();
}

}  // namespace gfwa
