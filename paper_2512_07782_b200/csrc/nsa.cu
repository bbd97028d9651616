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
#include "common.cuh"

namespace gfwa {
namespace {

constexpr int kWarpsPerBlock = 8;
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

template <int D>
__global__ void __launch_bounds__(32 * kWarpsPerBlock) nsa_cmp_select_kernel(
    const __nv_bfloat16* __restrict__ Q, const float* __restrict__ Kc, const float* __restrict__ Vc,
    float* __restrict__ Ocmp, int* __restrict__ sel, int64_t B, int64_t N, int64_t H, int blk, int nsel,
    float scale) {
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
    const int* __restrict__ sel, float* __restrict__ Oslc, int64_t B, int64_t N, int64_t H, int blk, int nsel,
    float scale) {
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
        for (int64_t j = (int64_t)ib * blk; j <= j1; ++j) {
            float kv[C];
            load_row<D>(K + ((b * N + j) * H + hh) * D, lane, kv);
            float s = 0.f;
#pragma unroll
            for (int c = 0; c < C; ++c) s = fmaf(q[c], kv[c], s);
            s = warp_sum(s) * scale;
            const float mn = fmaxf(m, s);
            const float corr = __expf(m - mn), p = __expf(s - mn);
            float vv[C];
            load_row<D>(V + ((b * N + j) * H + hh) * D, lane, vv);
#pragma unroll
            for (int c = 0; c < C; ++c) acc[c] = acc[c] * corr + p * vv[c];
            l = l * corr + p;
            m = mn;
        }
    }
    float* o = Oslc + row * D + C * lane;
#pragma unroll
    for (int c = 0; c < C; ++c) o[c] = acc[c] / l;  // the own block always holds token t: l > 0
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

}  // namespace

size_t nsa_workspace(int64_t B, int64_t N, int64_t H, int d, int blk, int nsel) {
    const int64_t nb = N / blk;
    size_t n = 0;
    auto add = [&](size_t bytes) { n += (bytes + 255) & ~(size_t)255; };
    add((size_t)B * nb * H * d * 4 * 2);    // Kc, Vc
    add((size_t)B * N * H * d * 4 * 2);     // o_cmp, o_slc
    add((size_t)B * H * N * (nsel + 1) * 4);  // selection
    add((size_t)B * N * H * d * 2);         // o_loc
    add((size_t)B * H * N * 4);             // LSE of the local branch
    return n;
}

// the branches and the combination; o_loc (bf16) was written by gfwa_fwd
gfwa_status_t nsa_fwd_branches(const void* Q, const void* K, const void* V, const float* g, int64_t B, int64_t N,
                               int64_t H, int d, int blk, int nsel, float scale, float* Kc, float* Vc, float* Ocmp,
                               float* Oslc, int* sel, const void* Oloc, void* O, cudaStream_t st) {
    int dev = 0, n_sm = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t nb = N / blk;
    if (nb > 0) {
        nsa_compress_kernel<<<(unsigned)min64((B * nb * H * d + 255) / 256, (int64_t)n_sm * 16), 256, 0, st>>>(
            (const __nv_bfloat16*)K, (const __nv_bfloat16*)V, Kc, Vc, B, N, H, d, blk);
        note_launch();
    }
    const int64_t rows = B * N * H;
    const unsigned grid = (unsigned)((rows + kWarpsPerBlock - 1) / kWarpsPerBlock);
    if (d == 64) {
        nsa_cmp_select_kernel<64><<<grid, 32 * kWarpsPerBlock, 0, st>>>((const __nv_bfloat16*)Q, Kc, Vc, Ocmp, sel, B,
                                                                        N, H, blk, nsel, scale);
        nsa_slc_kernel<64><<<grid, 32 * kWarpsPerBlock, 0, st>>>((const __nv_bfloat16*)Q, (const __nv_bfloat16*)K,
                                                                 (const __nv_bfloat16*)V, sel, Oslc, B, N, H, blk,
                                                                 nsel, scale);
    } else {
        nsa_cmp_select_kernel<128><<<grid, 32 * kWarpsPerBlock, 0, st>>>((const __nv_bfloat16*)Q, Kc, Vc, Ocmp, sel,
                                                                         B, N, H, blk, nsel, scale);
        nsa_slc_kernel<128><<<grid, 32 * kWarpsPerBlock, 0, st>>>((const __nv_bfloat16*)Q, (const __nv_bfloat16*)K,
                                                                  (const __nv_bfloat16*)V, sel, Oslc, B, N, H, blk,
                                                                  nsel, scale);
    }
    note_launch(2);
    nsa_combine_kernel<<<(unsigned)min64((rows * d + 255) / 256, (int64_t)n_sm * 16), 256, 0, st>>>(
        Ocmp, Oslc, (const __nv_bfloat16*)Oloc, g, (__nv_bfloat16*)O, rows, d);
    note_launch();
    return check_launch();
}

bool nsa_blocks_ok(int64_t N, int blk) { return N / blk <= kMaxBlocks; }

}  // namespace gfwa
