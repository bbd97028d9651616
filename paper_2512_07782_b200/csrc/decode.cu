// decode.cu -- gfwa_decode: one new token per sequence over a rolling
// w-entry cache.  The paper only claims "O(wd) per decoding step with a KV
// cache"; reading C-16: decode(t) is row t of Eq. 12 over the
// last min(t+1, w) tokens, so the ring order of the cache is irrelevant.
//
// HBM-bound split-KV design (flash-decoding): grid = (splits, H_kv, B); each
// CTA streams its contiguous slot range of K_cache then V_cache once through a
// per-warp cp.async shared-memory ring (16-byte pieces, 8 iterations in flight
// per lane without holding registers), keeps the partial (m, l, o) of every
// query head of its KV group, and the last CTA of each (b, kv head) merges the
// partials by LSE (atomic ticket, self-resetting counter).  The slot being replaced (t mod w)
// is never read from the cache: its owner CTA uses k_new/v_new directly and
// writes them back, so the in-place update cannot race with the readers (no
// other CTA touches that slot).
//
// GQA (heads_per_gqa_group = 4 in the paper's NSA runs,
// P:1209-1211): G = H / H_kv query heads share one K/V head, so each cache row
// is read once for G queries (G x less HBM per query head).  The gate stays
// per query head (U_cache [B,H,w]: u_tau - u_newest of that head's gate).
#include "common.cuh"
#include "sm100.cuh"

namespace gfwa {
namespace {

constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
constexpr int kMaxSlotsPerCta = 512;

struct DecodeParams {
    int64_t B, H, Hkv;
    int d, w, splits, slots_per_cta;
    float scale, eps;
    int gate_kind;
    const void* q;
    const void* k_new;
    const void* v_new;
    const float* gate_a;
    const float* gate_b;
    void* Kc;
    void* Vc;
    float* Uc;
    const int64_t* pos;
    void* o;
    float* part;        // [B*H][splits][d + 2]
    unsigned* counter;  // [B*H_kv]
};

template <typename T>
struct Vec {  // 16 bytes of T
    static constexpr int E = 16 / sizeof(T);
};

template <typename T>
__device__ __forceinline__ void unpack(const uint4& u, float* f) {
    if constexpr (sizeof(T) == 4) {
        f[0] = __uint_as_float(u.x);
        f[1] = __uint_as_float(u.y);
        f[2] = __uint_as_float(u.z);
        f[3] = __uint_as_float(u.w);
    } else {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 x = __bfloat1622float2(h[i]);
            f[2 * i] = x.x;
            f[2 * i + 1] = x.y;
        }
    }
}

// per-lane asynchronous 16-byte global->smem copies (LDGSTS): rows stream into a
// shared-memory ring without holding registers, many iterations ahead
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    const int n = pred ? 16 : 0;  // src-size 0 zero-fills (no global read)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// G query heads per K/V head (G = 1: multi-head attention, one K/V head per query head)
#ifndef GFWA_DEC_RING
#define GFWA_DEC_RING 8
#endif
constexpr int kRing = GFWA_DEC_RING;  // ring depth: iterations in flight per lane
#ifndef GFWA_DEC_MINB
#define GFWA_DEC_MINB 6
#endif
template <typename T, int D, int G>
__global__ void __launch_bounds__(kThreads, GFWA_DEC_MINB) decode_kernel(DecodeParams p) {
    constexpr int E = Vec<T>::E;           // elements per 16-byte vector
    constexpr int LPR = D / E;             // lanes per cache row
    constexpr int RPW = 32 / LPR;          // rows per warp iteration
    __shared__ float s_score[G][kMaxSlotsPerCta];
    __shared__ float s_red[kWarps][G][D];
    __shared__ float s_m[kWarps][G], s_l[kWarps][G];
    __shared__ bool s_last;
    constexpr int R_ = (G >= 8 && D == 128) ? kRing / 2 : kRing;  // static smem stays under 48 KB
    __shared__ uint4 s_ring[kWarps][R_][32];  // per-warp row ring (16 B per lane per iteration)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int split = blockIdx.x;
    const int64_t hk = blockIdx.y, b = blockIdx.z, bk = b * p.Hkv + hk;  // KV head and its row
    const int64_t bh0 = b * p.H + hk * G;                                // first query head of the group
    const int64_t t = p.pos[b];
    const int w = p.w;
    const int n_valid = (int)min64(t + 1, w);
    const int slot_new = (int)(t % w);
    const int s0 = split * p.slots_per_cta;
    const int s1 = min(s0 + p.slots_per_cta, n_valid);

    // alpha_t per query head.  U_cache holds, per slot, r = u_tau - u_{t-1} >= 0 (the
    // gate sum between the slot's token tau and the newest cached token): the bias of
    // this step is u_t - u_tau = -(r + alpha_t), and the slot is rewritten as
    // r + alpha_t (relative to u_t).  Stored values stay bounded by the window's gate
    // sum whatever the position, so fp32 never loses the small alphas (a running
    // absolute u would: its ulp grows with the position)
    float a_t[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const int64_t bh = bh0 + g;
        if (p.gate_kind == GFWA_GATE_ALPHA) {
            a_t[g] = p.gate_a[bh];
        } else {
            const float hv = p.gate_a[bh], bv = p.gate_b[bh];
            a_t[g] = softplus_f(bv * hv) / (bv + p.eps);
        }
    }

    const T* Kc = (const T*)p.Kc + bk * (int64_t)w * D;
    const T* Vc = (const T*)p.Vc + bk * (int64_t)w * D;
    const T* knew = (const T*)p.k_new + bk * D;
    const T* vnew = (const T*)p.v_new + bk * D;
    const int sub = lane / LPR, li = lane % LPR;  // row within the warp iteration, lane in row

    float qf[G][E];
#pragma unroll
    for (int g = 0; g < G; ++g)
        unpack<T>(*reinterpret_cast<const uint4*>((const T*)p.q + (bh0 + g) * D + li * E), qf[g]);
    const float sl2 = p.scale * kLog2e;

    // bias (u_t - u_i) log2e of every (head, slot) of this CTA, loaded coalesced up front
    // (a per-row u load inside pass 1 would stall the in-order warp on every row); each
    // slot is read and rewritten (r + alpha_t) by the one thread that owns it
    const int nsl = max(s1 - s0, 0);
    constexpr int kU = 8;  // independent u loads in flight per thread
    for (int i0 = threadIdx.x; i0 < G * nsl; i0 += kThreads * kU) {
        float uv[kU];
#pragma unroll
        for (int k = 0; k < kU; ++k) {
            const int i = i0 + k * kThreads;
            uv[k] = 0.f;
            if (i < G * nsl) uv[k] = __ldg(p.Uc + (bh0 + i / nsl) * w + s0 + i % nsl);
        }
#pragma unroll
        for (int k = 0; k < kU; ++k) {
            const int i = i0 + k * kThreads;
            if (i >= G * nsl) break;
            const int g = i / nsl, j = i % nsl;
            float at = a_t[0];
#pragma unroll
            for (int gg = 1; gg < G; ++gg)
                if (g == gg) at = a_t[gg];
            const float r = (s0 + j == slot_new) ? 0.f : uv[k] + at;
            s_score[g][j] = -r * kLog2e;
            p.Uc[(bh0 + g) * w + s0 + j] = r;
        }
    }
    __syncthreads();
    // pass 1: scores (log2 units) s_i = scale q.k_i + (u_t - u_i), each K row read once for G queries
    float mloc[G];
#pragma unroll
    for (int g = 0; g < G; ++g) mloc[g] = -INFINITY;
    // K and V rows stream through a per-warp shared-memory ring: lane li of row
    // group sub copies its own 16-byte piece of row s = base + sub, kRing
    // iterations ahead, and later reads back only that piece (no cross-lane hazard)
    constexpr int STEP = kWarps * RPW;
    const int base0 = s0 + warp * RPW;
    const int niter = base0 < s1 ? (s1 - base0 + STEP - 1) / STEP : 0;  // warp-uniform
    uint4* ring = &s_ring[warp][0][0];
    auto issue = [&](const T* cache, const T* newrow, int it) {
        const int s = base0 + it * STEP + sub;
        const bool ok = it < niter && s < s1;
        const T* src = (s == slot_new) ? newrow : cache + (int64_t)(ok ? s : s0) * D;
        cp_async16(&ring[(it % R_) * 32 + lane], src + li * E, ok);
        cp_async_commit();
    };
#pragma unroll
    for (int it = 0; it < R_ - 1; ++it) issue(Kc, knew, it);
    for (int it = 0; it < niter; ++it) {
        issue(Kc, knew, it + R_ - 1);
        cp_async_wait<R_ - 1>();  // this lane's piece of iteration `it` has landed
        const uint4 kq = ring[(it % R_) * 32 + lane];
        const int s = base0 + it * STEP + sub;
        const bool ok = s < s1;
        float acc[G];
#pragma unroll
        for (int g = 0; g < G; ++g) acc[g] = 0.f;
        if (ok) {
            if constexpr (sizeof(T) == 2) {
                // bf16: element pairs as packed fp32x2 (FFMA2), half the FMA issue slots
                const uint32_t kw[4] = {kq.x, kq.y, kq.z, kq.w};
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    uint64_t a2 = 0ull;
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        a2 = sm100::ffma2(sm100::f2pack(qf[g][2 * i], qf[g][2 * i + 1]), sm100::bf2_to_f2(kw[i]), a2);
                    float lo, hi;
                    sm100::f2unpack(a2, lo, hi);
                    acc[g] = lo + hi;
                }
            } else {
                float kf[E];
                unpack<T>(kq, kf);
#pragma unroll
                for (int g = 0; g < G; ++g)
#pragma unroll
                    for (int e = 0; e < E; ++e) acc[g] = fmaf(qf[g][e], kf[e], acc[g]);
            }
        }
        // transpose-reduce the G partial dots over the row's LPR lanes: each halving
        // stage sends half of the values (log2 G stages, then plain butterflies), so
        // lane li ends with head li / (LPR / G)'s dot in 2G - 1 + log2(LPR / G) shuffles
        int n = G, o = LPR / 2;
#pragma unroll
        for (; n > 1; n >>= 1, o >>= 1) {
            const bool up = li & o;
#pragma unroll
            for (int e = 0; e < n / 2; ++e) {
                const float send = up ? acc[e] : acc[e + n / 2];
                const float keep = up ? acc[e + n / 2] : acc[e];
                acc[e] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
#pragma unroll
        for (; o > 0; o >>= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], o);
        if (ok && li % (LPR / G) == 0) {
            const int g = li / (LPR / G);
            s_score[g][s - s0] = fmaf(acc[0], sl2, s_score[g][s - s0]);
        }
    }
    cp_async_wait<0>();
    __syncthreads();
    // per-head max over the CTA's slots
#pragma unroll
    for (int g = 0; g < G; ++g) {
        for (int i = s0 + threadIdx.x; i < s1; i += kThreads) mloc[g] = fmaxf(mloc[g], s_score[g][i - s0]);
        mloc[g] = warp_max(mloc[g]);
        if (lane == 0) s_m[warp][g] = mloc[g];
    }
    __syncthreads();
    float m[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        m[g] = s_m[0][g];
#pragma unroll
        for (int i = 1; i < kWarps; ++i) m[g] = fmaxf(m[g], s_m[i][g]);
    }
    // G > 1: p_i = exp2(s_i - m) once per (head, slot), in place: the 16 lanes of a row
    // then read it as a shared-memory broadcast instead of each evaluating G exponentials
    constexpr bool kPre = G > 1;
    for (int i = threadIdx.x; kPre && i < G * nsl; i += kThreads) {
        const int g = i / nsl, j = i % nsl;
        float mg = m[0];
#pragma unroll
        for (int gg = 1; gg < G; ++gg)
            if (g == gg) mg = m[gg];
        s_score[g][j] = exp2f(s_score[g][j] - mg);
    }
    if (kPre) __syncthreads();

    // pass 2: o_part = sum_i exp2(s_i - m) v_i, l = sum_i exp2(s_i - m), each V row read once
    float of[G][E], lloc[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        lloc[g] = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) of[g][e] = 0.f;
    }
#pragma unroll
    for (int it = 0; it < R_ - 1; ++it) issue(Vc, vnew, it);
    for (int it = 0; it < niter; ++it) {
        issue(Vc, vnew, it + R_ - 1);
        cp_async_wait<R_ - 1>();
        const uint4 vq = ring[(it % R_) * 32 + lane];
        const int s = base0 + it * STEP + sub;
        if (s < s1) {
            if constexpr (sizeof(T) == 2) {
                const uint32_t vw[4] = {vq.x, vq.y, vq.z, vq.w};
                uint64_t v2[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) v2[i] = sm100::bf2_to_f2(vw[i]);
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const float pr = kPre ? s_score[g][s - s0] : exp2f(s_score[g][s - s0] - m[g]);
                    const uint64_t p2 = sm100::f2pack(pr, pr);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        uint64_t o2 = sm100::f2pack(of[g][2 * i], of[g][2 * i + 1]);
                        o2 = sm100::ffma2(p2, v2[i], o2);
                        sm100::f2unpack(o2, of[g][2 * i], of[g][2 * i + 1]);
                    }
                    if (li == 0) lloc[g] += pr;
                }
            } else {
                float vf[E];
                unpack<T>(vq, vf);
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const float pr = kPre ? s_score[g][s - s0] : exp2f(s_score[g][s - s0] - m[g]);
#pragma unroll
                    for (int e = 0; e < E; ++e) of[g][e] = fmaf(pr, vf[e], of[g][e]);
                    if (li == 0) lloc[g] += pr;
                }
            }
        }
    }
    cp_async_wait<0>();
    // reduce over the RPW rows of the warp (lanes with equal li)
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
        for (int o = LPR; o < 32; o <<= 1) {
#pragma unroll
            for (int e = 0; e < E; ++e) of[g][e] += __shfl_xor_sync(0xffffffffu, of[g][e], o);
        }
        lloc[g] = warp_sum(lloc[g]);
        if (sub == 0) {
#pragma unroll
            for (int e = 0; e < E; ++e) s_red[warp][g][li * E + e] = of[g][e];
        }
        if (lane == 0) s_l[warp][g] = lloc[g];
    }
    __syncthreads();

    // partials of this split -> workspace, one per query head
    for (int i = threadIdx.x; i < G * D; i += kThreads) {
        const int g = i / D, c = i % D;
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < kWarps; ++k) acc += s_red[k][g][c];
        p.part[((bh0 + g) * p.splits + split) * (int64_t)(D + 2) + c] = acc;
    }
    if (threadIdx.x < G) {
        const int g = threadIdx.x;
        float l = 0.f, mm = s_m[0][g];
        for (int k = 0; k < kWarps; ++k) {
            l += s_l[k][g];
            mm = fmaxf(mm, s_m[k][g]);
        }
        float* part = p.part + ((bh0 + g) * p.splits + split) * (int64_t)(D + 2);
        part[D] = (s0 < s1) ? mm : -INFINITY;
        part[D + 1] = l;
    }
    // owner of the new slot writes the token into the ring (no reader races)
    if (slot_new >= s0 && slot_new < s0 + p.slots_per_cta) {
        T* kd = (T*)p.Kc + bk * (int64_t)w * D + (int64_t)slot_new * D;
        T* vd = (T*)p.Vc + bk * (int64_t)w * D + (int64_t)slot_new * D;
        for (int c = threadIdx.x; c < D; c += kThreads) {
            kd[c] = knew[c];
            vd[c] = vnew[c];
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(p.counter + bk, 1u);
        s_last = (prev == (unsigned)p.splits - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // LSE merge of the split partials per query head (o = sum o_i 2^(m_i-M) / L)
#pragma unroll 1
    for (int g = 0; g < G; ++g) {
        const int64_t bh = bh0 + g;
        const float* pb = p.part + bh * p.splits * (int64_t)(D + 2);
        float M = -INFINITY;
        for (int i = 0; i < p.splits; ++i) M = fmaxf(M, __ldcg(pb + i * (D + 2) + D));
        float L = 0.f;
        for (int i = 0; i < p.splits; ++i) {
            const float mi = __ldcg(pb + i * (D + 2) + D);
            if (mi != -INFINITY) L += __ldcg(pb + i * (D + 2) + D + 1) * exp2f(mi - M);
        }
        const float invL = 1.f / L;
        T* orow = (T*)p.o + bh * D;
        for (int c = threadIdx.x; c < D; c += kThreads) {
            float acc = 0.f;
            for (int i = 0; i < p.splits; ++i) {
                const float mi = __ldcg(pb + i * (D + 2) + D);
                if (mi != -INFINITY) acc += __ldcg(pb + i * (D + 2) + c) * exp2f(mi - M);
            }
            orow[c] = from_f32<T>(acc * invL);
        }
    }
    if (threadIdx.x == 0) p.counter[bk] = 0u;  // leave the workspace zeroed
}

int choose_splits(int64_t BH, int w) {
    // enough CTAs to cover the 148 SMs several times, <= 512 slots per CTA
    int splits = (w + kMaxSlotsPerCta - 1) / kMaxSlotsPerCta;
    while (splits < 64 && (int64_t)splits * 2 * BH <= 148 * 16 && (w + splits * 2 - 1) / (splits * 2) >= 64)
        splits *= 2;
    return splits;
}

}  // namespace
}  // namespace gfwa

using namespace gfwa;

static int64_t kv_heads(const gfwa_decode_desc_t* d) { return d->H_kv > 0 ? d->H_kv : d->H; }

extern "C" size_t gfwa_decode_workspace_size(const gfwa_decode_desc_t* d) {
    if (!d || d->B < 1 || d->H < 1 || d->w < 1 || (d->d != 64 && d->d != 128)) return 256;
    const int64_t hkv = kv_heads(d);
    if (hkv < 1 || d->H % hkv) return 256;
    const int splits = choose_splits(d->B * hkv, d->w);
    size_t bytes = (size_t)d->B * d->H * splits * (d->d + 2) * sizeof(float);
    bytes = (bytes + 255) & ~(size_t)255;
    bytes += (size_t)d->B * hkv * sizeof(unsigned);
    return (bytes + 255) & ~(size_t)255;
}

template <typename T, int D>
static void launch_decode(dim3 grid, const DecodeParams& p, int G, cudaStream_t st) {
    switch (G) {
        case 1: decode_kernel<T, D, 1><<<grid, kThreads, 0, st>>>(p); break;
        case 2: decode_kernel<T, D, 2><<<grid, kThreads, 0, st>>>(p); break;
        case 4: decode_kernel<T, D, 4><<<grid, kThreads, 0, st>>>(p); break;
        default: decode_kernel<T, D, 8><<<grid, kThreads, 0, st>>>(p); break;
    }
}

extern "C" gfwa_status_t gfwa_decode(const gfwa_decode_desc_t* d, const void* q, const void* k_new,
                                     const void* v_new, const float* gate_a, const float* gate_b, void* K_cache,
                                     void* V_cache, float* U_cache, const int64_t* pos, void* o, void* ws,
                                     size_t ws_bytes, gfwa_stream_t stream) {
    if (!d || !q || !k_new || !v_new || !gate_a || !K_cache || !V_cache || !U_cache || !pos || !o || !ws)
        return GFWA_ERR_INVALID_ARGUMENT;
    if (d->B < 1 || d->H < 1 || d->w < 1 || d->H_kv < 0) return GFWA_ERR_INVALID_ARGUMENT;
    const int64_t hkv = kv_heads(d);
    if (d->H % hkv) return GFWA_ERR_INVALID_ARGUMENT;
    const int G = (int)(d->H / hkv);
    if (G != 1 && G != 2 && G != 4 && G != 8) return GFWA_ERR_UNSUPPORTED;
    if (d->B > 65535 || hkv > 65535) return GFWA_ERR_INVALID_ARGUMENT;
    if (d->gate_kind == GFWA_GATE_HBETA && !gate_b) return GFWA_ERR_INVALID_ARGUMENT;
    if (d->gate_kind != GFWA_GATE_HBETA && d->gate_kind != GFWA_GATE_ALPHA) return GFWA_ERR_INVALID_ARGUMENT;
    if (d->d != 64 && d->d != 128) return GFWA_ERR_UNSUPPORTED;
    if (d->dtype != GFWA_BF16 && d->dtype != GFWA_F32) return GFWA_ERR_UNSUPPORTED;
    const void* ptrs[] = {q, k_new, v_new, K_cache, V_cache};
    for (const void* pp : ptrs)
        if ((uintptr_t)pp % 16) return GFWA_ERR_INVALID_ARGUMENT;
    if ((uintptr_t)ws % 256) return GFWA_ERR_INVALID_ARGUMENT;
    if (ws_bytes < gfwa_decode_workspace_size(d)) return GFWA_ERR_WORKSPACE;
    DecodeParams p;
    p.B = d->B;
    p.H = d->H;
    p.Hkv = hkv;
    p.d = d->d;
    p.w = d->w;
    p.splits = choose_splits(d->B * hkv, d->w);
    p.slots_per_cta = (d->w + p.splits - 1) / p.splits;
    p.scale = d->scale > 0.f ? d->scale : 1.f / sqrtf((float)d->d);
    p.eps = d->eps;
    p.gate_kind = d->gate_kind;
    p.q = q;
    p.k_new = k_new;
    p.v_new = v_new;
    p.gate_a = gate_a;
    p.gate_b = gate_b;
    p.Kc = K_cache;
    p.Vc = V_cache;
    p.Uc = U_cache;
    p.pos = pos;
    p.o = o;
    size_t part_bytes = ((size_t)d->B * d->H * p.splits * (d->d + 2) * sizeof(float) + 255) & ~(size_t)255;
    p.part = (float*)ws;
    p.counter = (unsigned*)((char*)ws + part_bytes);
    dim3 grid((unsigned)p.splits, (unsigned)hkv, (unsigned)d->B);
    cudaStream_t st = (cudaStream_t)stream;
    if (d->dtype == GFWA_BF16) {
        if (d->d == 128)
            launch_decode<__nv_bfloat16, 128>(grid, p, G, st);
        else
            launch_decode<__nv_bfloat16, 64>(grid, p, G, st);
    } else {
        if (d->d == 128)
            launch_decode<float, 128>(grid, p, G, st);
        else
            launch_decode<float, 64>(grid, p, G, st);
    }
    note_launch();
    return check_launch();
}
