// decode.cu -- gfwa_decode: one new token per sequence over a rolling
// w-entry cache.  The paper only claims "O(wd) per decoding step with a KV
// cache"; reading C-16: decode(t) is row t of Eq. 12 over the
// last min(t+1, w) tokens, so the ring order of the cache is irrelevant.
//
// HBM-bound split-KV design (flash-decoding): grid = (splits, H, B); each CTA
// streams its contiguous slot range of K_cache then V_cache once with 16-byte
// vector loads, keeps the partial (m, l, o) and the last CTA of each (b, h)
// merges the partials by LSE (atomic ticket, self-resetting counter).  The
// slot being replaced (t mod w) is never read from the cache: its owner CTA
// uses k_new/v_new directly and writes them back, so the in-place update
// cannot race with the readers (no other CTA touches that slot).
#include "common.cuh"

namespace gfwa {
namespace {

constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
constexpr int kMaxSlotsPerCta = 512;

struct DecodeParams {
    int64_t B, H;
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
    unsigned* counter;  // [B*H]
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

__device__ __forceinline__ uint4 ld_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

template <typename T, int D>
__global__ void __launch_bounds__(kThreads) decode_kernel(DecodeParams p) {
    constexpr int E = Vec<T>::E;           // elements per 16-byte vector
    constexpr int LPR = D / E;             // lanes per cache row
    constexpr int RPW = 32 / LPR;          // rows per warp iteration
    __shared__ float s_score[kMaxSlotsPerCta];
    __shared__ float s_red[kWarps][D];
    __shared__ float s_m[kWarps], s_l[kWarps];
    __shared__ bool s_last;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int split = blockIdx.x;
    const int64_t h = blockIdx.y, b = blockIdx.z, bh = b * p.H + h;
    const int64_t t = p.pos[b];
    const int w = p.w;
    const int n_valid = (int)min64(t + 1, w);
    const int slot_new = (int)(t % w);
    const int s0 = split * p.slots_per_cta;
    const int s1 = min(s0 + p.slots_per_cta, n_valid);

    // u_t = u_{t-1} - alpha_t, u_{t-1} from the ring (0 before the first token)
    const float u_prev = t > 0 ? p.Uc[bh * w + (int)((t - 1) % w)] : 0.f;
    float alpha;
    if (p.gate_kind == GFWA_GATE_ALPHA) {
        alpha = p.gate_a[bh];
    } else {
        const float hv = p.gate_a[bh], bv = p.gate_b[bh];
        alpha = softplus_f(bv * hv) / (bv + p.eps);
    }
    const float u_t = u_prev - alpha;

    const T* qrow = (const T*)p.q + bh * D;
    const T* Kc = (const T*)p.Kc + bh * (int64_t)w * D;
    const T* Vc = (const T*)p.Vc + bh * (int64_t)w * D;
    const T* knew = (const T*)p.k_new + bh * D;
    const T* vnew = (const T*)p.v_new + bh * D;
    const float* Uc = p.Uc + bh * w;
    const int sub = lane / LPR, li = lane % LPR;  // row within the warp iteration, lane in row

    float qf[E];
    unpack<T>(*reinterpret_cast<const uint4*>(qrow + li * E), qf);
    const float sl2 = p.scale * kLog2e;

    // pass 1: scores (log2 units) s_i = scale q.k_i + (u_t - u_i)
    float mloc = -INFINITY;
    for (int s = s0 + warp * RPW + sub; s - sub < s1; s += kWarps * RPW) {
        const bool ok = s < s1;
        float acc = 0.f;
        float ui = u_t;
        if (ok) {
            const T* krow = (s == slot_new) ? knew : Kc + (int64_t)s * D;
            float kf[E];
            unpack<T>(ld_stream(krow + li * E), kf);
#pragma unroll
            for (int e = 0; e < E; ++e) acc = fmaf(qf[e], kf[e], acc);
            if (s != slot_new) ui = Uc[s];
        }
#pragma unroll
        for (int o = LPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (ok && li == 0) {
            const float sc = fmaf(acc, sl2, (u_t - ui) * kLog2e);
            s_score[s - s0] = sc;
            mloc = fmaxf(mloc, sc);
        }
    }
    mloc = warp_max(mloc);
    if (lane == 0) s_m[warp] = mloc;
    __syncthreads();
    float m = s_m[0];
#pragma unroll
    for (int i = 1; i < kWarps; ++i) m = fmaxf(m, s_m[i]);

    // pass 2: o_part = sum_i exp2(s_i - m) v_i, l = sum_i exp2(s_i - m)
    float of[E];
#pragma unroll
    for (int e = 0; e < E; ++e) of[e] = 0.f;
    float lloc = 0.f;
    for (int s = s0 + warp * RPW + sub; s - sub < s1; s += kWarps * RPW) {
        if (s < s1) {
            const float pr = exp2f(s_score[s - s0] - m);
            const T* vrow = (s == slot_new) ? vnew : Vc + (int64_t)s * D;
            float vf[E];
            unpack<T>(ld_stream(vrow + li * E), vf);
#pragma unroll
            for (int e = 0; e < E; ++e) of[e] = fmaf(pr, vf[e], of[e]);
            if (li == 0) lloc += pr;
        }
    }
    // reduce over the RPW rows of the warp (lanes with equal li)
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) {
#pragma unroll
        for (int e = 0; e < E; ++e) of[e] += __shfl_xor_sync(0xffffffffu, of[e], o);
    }
    lloc = warp_sum(lloc);
    if (sub == 0) {
#pragma unroll
        for (int e = 0; e < E; ++e) s_red[warp][li * E + e] = of[e];
    }
    if (lane == 0) s_l[warp] = lloc;
    __syncthreads();

    // partial of this split -> workspace
    float* part = p.part + (bh * p.splits + split) * (int64_t)(D + 2);
    for (int c = threadIdx.x; c < D; c += kThreads) {
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < kWarps; ++i) acc += s_red[i][c];
        part[c] = acc;
    }
    if (threadIdx.x == 0) {
        float l = 0.f;
        for (int i = 0; i < kWarps; ++i) l += s_l[i];
        part[D] = (s0 < s1) ? m : -INFINITY;
        part[D + 1] = l;
    }
    // owner of the new slot writes the token into the ring (no reader races)
    if (slot_new >= s0 && slot_new < s0 + p.slots_per_cta) {
        T* kd = (T*)p.Kc + bh * (int64_t)w * D + (int64_t)slot_new * D;
        T* vd = (T*)p.Vc + bh * (int64_t)w * D + (int64_t)slot_new * D;
        for (int c = threadIdx.x; c < D; c += kThreads) {
            kd[c] = knew[c];
            vd[c] = vnew[c];
        }
        if (threadIdx.x == 0) p.Uc[bh * w + slot_new] = u_t;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(p.counter + bh, 1u);
        s_last = (prev == (unsigned)p.splits - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // LSE merge of the split partials (natural layout: o = sum o_i 2^(m_i-M) / L)
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
    if (threadIdx.x == 0) p.counter[bh] = 0u;  // leave the workspace zeroed
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

extern "C" size_t gfwa_decode_workspace_size(const gfwa_decode_desc_t* d) {
    if (!d || d->B < 1 || d->H < 1 || d->w < 1 || (d->d != 64 && d->d != 128)) return 256;
    const int splits = choose_splits(d->B * d->H, d->w);
    size_t bytes = (size_t)d->B * d->H * splits * (d->d + 2) * sizeof(float);
    bytes = (bytes + 255) & ~(size_t)255;
    bytes += (size_t)d->B * d->H * sizeof(unsigned);
    return (bytes + 255) & ~(size_t)255;
}

extern "C" gfwa_status_t gfwa_decode(const gfwa_decode_desc_t* d, const void* q, const void* k_new,
                                     const void* v_new, const float* gate_a, const float* gate_b, void* K_cache,
                                     void* V_cache, float* U_cache, const int64_t* pos, void* o, void* ws,
                                     size_t ws_bytes, gfwa_stream_t stream) {
    if (!d || !q || !k_new || !v_new || !gate_a || !K_cache || !V_cache || !U_cache || !pos || !o || !ws)
        return GFWA_ERR_INVALID_ARGUMENT;
    if (d->B < 1 || d->H < 1 || d->w < 1) return GFWA_ERR_INVALID_ARGUMENT;
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
    p.d = d->d;
    p.w = d->w;
    p.splits = choose_splits(d->B * d->H, d->w);
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
    dim3 grid((unsigned)p.splits, (unsigned)d->H, (unsigned)d->B);
    cudaStream_t st = (cudaStream_t)stream;
    if (d->dtype == GFWA_BF16) {
        if (d->d == 128)
            decode_kernel<__nv_bfloat16, 128><<<grid, kThreads, 0, st>>>(p);
        else
            decode_kernel<__nv_bfloat16, 64><<<grid, kThreads, 0, st>>>(p);
    } else {
        if (d->d == 128)
            decode_kernel<float, 128><<<grid, kThreads, 0, st>>>(p);
        else
            decode_kernel<float, 64><<<grid, kThreads, 0, st>>>(p);
    }
    note_launch();
    return check_launch();
}
