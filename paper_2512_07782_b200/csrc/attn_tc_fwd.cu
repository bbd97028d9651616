// attn_tc_fwd.cu -- GatedFWA forward on the 5th-generation tensor cores
// (sm_100a): Alg. 2 re-designed for tcgen05/TMEM/TMA.
//
// One CTA owns two 128-row query tiles of one (b, h) and streams the 128-key
// K/V tiles of their joint window once, diagonal first (descending j):
//   warp 9      TMA producer: Q0/Q1 once, then K_j / V_j into 2-stage rings
//               (128B swizzle, OOB rows zero-filled -> ragged tails for free)
//   warp 8      MMA issuer (one elected lane): S_i = Q_i K_j^T (SS, fp32 in
//               TMEM) and O_i += P_i V_j (TS: P read from TMEM), commits to
//               mbarriers; tcgen05.commit tracks all earlier MMAs, so S_full
//               of step n also certifies that PV of step n-1 has landed.
//   warps 0-3/4-7  softmax for tile 0 / tile 1, one thread per query row:
//               tcgen05.ld the S row, add the gate bias (u_q - u_k) (P:377-380,
//               an outer difference of two u vectors, nothing N x w is ever
//               materialised), window-mask only on diagonal / window-edge
//               tiles, online softmax in fp32 with a lazy
//               rescale (only when the running max grows by > 2^8), bf16 P
//               back into the same TMEM columns, then the epilogue O / l and
//               LSE = m + ln l.
// TMEM: S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512) columns x 128 lanes.
// Key tiles outside every row's window are never loaded.
#include "attn_common.cuh"
#include "sm100.cuh"
#include "tma_host.cuh"

namespace gfwa {
namespace {

using namespace sm100;

constexpr int BM = 128;          // query rows per tile
constexpr int BN = 128;          // keys per tile
constexpr int D = 128;           // head dim
constexpr int NST = 2;           // K and V ring stages
constexpr uint32_t kTileBytes = BM * D * 2;  // 32 KB bf16 tile
constexpr int kThreads = 320;    // 8 softmax warps + MMA warp + TMA warp
constexpr float kRescaleThreshold = 8.0f;  // log2 units

struct TcFwdParams {
    const float* U;
    void* O;
    float* O_f32;
    float* LSE;
    int64_t Nq, Nkv, h0, H;
    int w;
    float sl2;  // scale * log2(e)
    int64_t os0, os1, os2;
};

struct __align__(8) Bars {
    uint64_t q_full[2];
    uint64_t k_full[NST], k_empty[NST];
    uint64_t v_full[NST], v_empty[NST];
    uint64_t s_full[2], p_ready[2], o_full[2];
};

__device__ __forceinline__ int64_t kv_tile_lo(int64_t g_lo, int w) { return max64(0, g_lo - w + 1) / BN; }

__global__ void __launch_bounds__(kThreads, 1)
    fwd_tc_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                  const __grid_constant__ CUtensorMap mv, const TcFwdParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* Qs = smem;                            // 2 tiles
    uint8_t* Ks = smem + 2 * kTileBytes;           // NST tiles
    uint8_t* Vs = Ks + NST * kTileBytes;           // NST tiles
    float* ukbuf = (float*)(Vs + NST * kTileBytes);  // [2][BN]
    Bars* bars = (Bars*)(ukbuf + 2 * BN);
    uint32_t* tmem_sh = (uint32_t*)(bars + 1);

    const int warp = threadIdx.x >> 5;
    const int64_t b = blockIdx.z, h = blockIdx.y;
    const int64_t r0 = (int64_t)blockIdx.x * 2 * BM;
    const bool act1 = r0 + BM < p.Nq;
    // Alg. 2 l.7-9 per query tile: key positions g = t + h0
    int64_t jlo[2], jhi[2], glo[2], ghi[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        glo[i] = r0 + i * BM + p.h0;
        ghi[i] = min64(r0 + i * BM + BM - 1, p.Nq - 1) + p.h0;
        jlo[i] = kv_tile_lo(glo[i], p.w);
        jhi[i] = ghi[i] / BN;
    }
    const int64_t J_hi = act1 ? jhi[1] : jhi[0];
    const int64_t J_lo = jlo[0];

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->q_full[i], 1);
            mbar_init(&bars->s_full[i], 1);
            mbar_init(&bars->p_ready[i], 4);
            mbar_init(&bars->o_full[i], 1);
        }
        for (int s = 0; s < NST; ++s) {
            mbar_init(&bars->k_full[s], 1);
            mbar_init(&bars->k_empty[s], 1);
            mbar_init(&bars->v_full[s], 1);
            mbar_init(&bars->v_empty[s], 1);
        }
        fence_barrier_init();
    }
    if (warp == 8) {
        tmem_alloc(tmem_sh, 512);
        tmem_relinquish();
    }
    if (warp == 9 && elect_one()) {
        tma_prefetch(&mq);
        tma_prefetch(&mk);
        tma_prefetch(&mv);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_sh;

    if (warp == 9) {
        // ------------------------------------------------ TMA producer
        if (elect_one()) {
            const uint64_t pol_kv = policy_evict_last();  // K/V tiles are re-read by ~w/128 neighbours
            for (int i = 0; i < 2; ++i) {
                if (i == 1 && !act1) break;
                mbar_expect_tx(&bars->q_full[i], kTileBytes);
                for (int half = 0; half < 2; ++half)
                    tma_load_4d(Qs + i * kTileBytes + half * (kTileBytes / 2), &mq, &bars->q_full[i], half * 64,
                                (int)h, (int)(r0 + i * BM), (int)b);
            }
            int k = 0;
            for (int64_t j = J_hi; j >= J_lo; --j, ++k) {
                const int s = k % NST;
                const uint32_t ph = ((k / NST) & 1) ^ 1;
                mbar_wait(&bars->k_empty[s], ph);
                mbar_expect_tx(&bars->k_full[s], kTileBytes);
                for (int half = 0; half < 2; ++half)
                    tma_load_4d_hint(Ks + s * kTileBytes + half * (kTileBytes / 2), &mk, &bars->k_full[s],
                                     half * 64, (int)h, (int)(j * BN), (int)b, pol_kv);
                mbar_wait(&bars->v_empty[s], ph);
                mbar_expect_tx(&bars->v_full[s], kTileBytes);
                for (int half = 0; half < 2; ++half)
                    tma_load_4d_hint(Vs + s * kTileBytes + half * (kTileBytes / 2), &mv, &bars->v_full[s],
                                     half * 64, (int)h, (int)(j * BN), (int)b, pol_kv);
            }
        }
    } else if (warp == 8) {
        // ------------------------------------------------ MMA issuer
        const uint32_t idesc_qk = idesc_bf16(BM, BN, false, false);
        const uint32_t idesc_pv = idesc_bf16(BM, D, false, true);
        const bool act[2] = {true, act1};
        uint32_t pph[2] = {0, 0};
        int64_t prev[2] = {-1, -1};
        bool first_pv[2] = {true, true};
        mbar_wait(&bars->q_full[0], 0);
        if (act1) mbar_wait(&bars->q_full[1], 0);
        int k = 0;
        for (int64_t j = J_hi; j >= J_lo; --j, ++k) {
            const int s = k % NST;
            mbar_wait(&bars->k_full[s], (k / NST) & 1);
            tc_fence_after();
            int pv_issued = 0;
            for (int i = 0; i < 2; ++i) {
                if (!act[i] || j < jlo[i] || j > jhi[i]) continue;
                if (prev[i] >= 0) {
                    // O_i += P_i(prev) V_prev  (V of tile j+1 sits in stage (k-1) % NST)
                    mbar_wait(&bars->p_ready[i], pph[i]);
                    pph[i] ^= 1;
                    const int vs = (k - 1) % NST;
                    mbar_wait(&bars->v_full[vs], ((k - 1) / NST) & 1);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t vbase = smem_u32(Vs + vs * kTileBytes);
#pragma unroll
                        for (int kk = 0; kk < BN / 16; ++kk)
                            mma_ts(tmem + 256 + 128 * i, tmem + 128 * i + 8 * kk,
                                   sdesc_sw128(vbase + kk * 2048, kTileBytes / 2, 1024), idesc_pv,
                                   (first_pv[i] && kk == 0) ? 0u : 1u);
                    }
                    __syncwarp();
                    first_pv[i] = false;
                    ++pv_issued;
                }
                // S_i = Q_i K_j^T
                if (elect_one()) {
                    const uint32_t qbase = smem_u32(Qs + i * kTileBytes), kbase = smem_u32(Ks + s * kTileBytes);
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t off = (kk >> 2) * (kTileBytes / 2) + (kk & 3) * 32;
                        mma_ss(tmem + 128 * i, sdesc_sw128(qbase + off, 16, 1024),
                               sdesc_sw128(kbase + off, 16, 1024), idesc_qk, kk > 0 ? 1u : 0u);
                    }
                    tc_commit(&bars->s_full[i]);
                }
                __syncwarp();
                prev[i] = j;
            }
            if (elect_one()) {
                tc_commit(&bars->k_empty[s]);
                // release V_{j+1} once every query tile that uses it has issued its PV
                if (pv_issued > 0) {
                    const int64_t jp = j + 1;
                    const int users = (jp >= jlo[0] && jp <= jhi[0]) + (act1 && jp >= jlo[1] && jp <= jhi[1]);
                    if (pv_issued == users) tc_commit(&bars->v_empty[(k - 1) % NST]);
                }
            }
            __syncwarp();
        }
        // flush: last PV of every tile, then signal the epilogue
        for (int i = 0; i < 2; ++i) {
            if (!act[i]) continue;
            mbar_wait(&bars->p_ready[i], pph[i]);
            const int kj = (int)(J_hi - prev[i]);
            const int vs = kj % NST;
            mbar_wait(&bars->v_full[vs], (kj / NST) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t vbase = smem_u32(Vs + vs * kTileBytes);
#pragma unroll
                for (int kk = 0; kk < BN / 16; ++kk)
                    mma_ts(tmem + 256 + 128 * i, tmem + 128 * i + 8 * kk,
                           sdesc_sw128(vbase + kk * 2048, kTileBytes / 2, 1024), idesc_pv,
                           (first_pv[i] && kk == 0) ? 0u : 1u);
                tc_commit(&bars->o_full[i]);
            }
            __syncwarp();
        }
    } else {
        // ------------------------------------------------ softmax warpgroups
        const int i = warp >> 2;  // query tile
        const int r = threadIdx.x & 127;
        if (i == 0 || act1) {
            const int64_t t = r0 + i * BM + r;
            const bool valid = t < p.Nq;
            const int64_t g = t + p.h0;
            const float* Ubh = p.U + (b * p.H + h) * p.Nkv;
            const float uq = valid ? Ubh[g] : 0.f;
            const uint32_t lane_addr = tmem + ((uint32_t)((warp & 3) * 32) << 16);
            const uint32_t scol = 128 * i;
            float* uk = ukbuf + i * BN;
            float m_used = -INFINITY, l = 0.f;
            uint32_t sph = 0;
            int n = 0;
            for (int64_t j = jhi[i]; j >= jlo[i]; --j, ++n) {
                // u of this key tile -> smem (WG-cooperative)
                named_bar_sync(1 + i, 128);
                const int64_t kj = j * BN + r;
                uk[r] = kj < p.Nkv ? Ubh[kj] : 0.f;
                named_bar_sync(1 + i, 128);
                mbar_wait(&bars->s_full[i], sph);
                sph ^= 1;
                tc_fence_after();
                float x[BN];
                {
                    uint32_t rr[32];
#pragma unroll
                    for (int c = 0; c < BN; c += 32) {
                        tmem_ld32(lane_addr + scol + c, rr);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 32; ++e) x[c + e] = __uint_as_float(rr[e]);
                    }
                }
                // logits in log2 units: scale*q.k + (u_q - u_k)  (difference first, C-18)
                const bool interior = (j * BN + BN - 1 <= glo[i]) && (j * BN >= ghi[i] - p.w + 1);
                float mt = -INFINITY;
                if (interior) {
#pragma unroll
                    for (int c = 0; c < BN; c += 4) {
                        const float4 u4 = *reinterpret_cast<const float4*>(uk + c);
                        x[c + 0] = fmaf(x[c + 0], p.sl2, (uq - u4.x) * kLog2e);
                        x[c + 1] = fmaf(x[c + 1], p.sl2, (uq - u4.y) * kLog2e);
                        x[c + 2] = fmaf(x[c + 2], p.sl2, (uq - u4.z) * kLog2e);
                        x[c + 3] = fmaf(x[c + 3], p.sl2, (uq - u4.w) * kLog2e);
                        mt = fmaxf(mt, fmaxf(fmaxf(x[c], x[c + 1]), fmaxf(x[c + 2], x[c + 3])));
                    }
                } else {
                    const int64_t kb = j * BN;
#pragma unroll
                    for (int c = 0; c < BN; c += 4) {
                        const float4 u4 = *reinterpret_cast<const float4*>(uk + c);
                        const float uu[4] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int64_t key = kb + c + e;
                            const bool keep = key <= g && key > g - p.w && key < p.Nkv;
                            x[c + e] = keep ? fmaf(x[c + e], p.sl2, (uq - uu[e]) * kLog2e) : -INFINITY;
                            mt = fmaxf(mt, x[c + e]);
                        }
                    }
                }
                // lazy online softmax: move the reference max only when it grows by > 2^8
                float corr = 1.f;
                bool need = false;
                if (mt > m_used + kRescaleThreshold) {
                    if (m_used != -INFINITY) {
                        corr = ex2(m_used - mt);
                        need = true;
                    }
                    l *= corr;
                    m_used = mt;
                }
                const float mref = (m_used == -INFINITY) ? 0.f : m_used;
                float lsum = 0.f;
#pragma unroll
                for (int c = 0; c < BN; c += 64) {
                    uint32_t pk[32];
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const float p0 = ex2(x[c + 2 * e] - mref), p1 = ex2(x[c + 2 * e + 1] - mref);
                        lsum += p0 + p1;
                        pk[e] = pack_bf16x2(p0, p1);
                    }
                    tmem_st32(lane_addr + scol + c / 2, pk);
                }
                l += lsum;
                // rescale O_i (PV of the previous step is complete: S_full certified it)
                if (__any_sync(0xffffffffu, need) && n > 0) {
                    uint32_t ob[32];
#pragma unroll
                    for (int c = 0; c < D; c += 32) {
                        tmem_ld32(lane_addr + 256 + scol + c, ob);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 32; ++e) ob[e] = __float_as_uint(__uint_as_float(ob[e]) * corr);
                        tmem_st32(lane_addr + 256 + scol + c, ob);
                    }
                }
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if ((threadIdx.x & 31) == 0) mbar_arrive(&bars->p_ready[i]);
            }
            // epilogue: O / l, LSE (Alg. 2 l.19-20)
            mbar_wait(&bars->o_full[i], 0);
            tc_fence_after();
            const float inv = 1.f / l;
            __nv_bfloat16* orow = (__nv_bfloat16*)p.O + b * p.os0 + t * p.os1 + h * p.os2;
            float* frow = p.O_f32 ? p.O_f32 + b * p.os0 + t * p.os1 + h * p.os2 : nullptr;
#pragma unroll
            for (int c = 0; c < D; c += 32) {
                uint32_t ob[32];
                tmem_ld32(lane_addr + 256 + scol + c, ob);
                tmem_wait_ld();
                if (valid) {
                    float v[32];
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(ob[e]) * inv;
#pragma unroll
                    for (int e = 0; e < 32; e += 8) {
                        uint4 pk;
                        pk.x = pack_bf16x2(v[e + 0], v[e + 1]);
                        pk.y = pack_bf16x2(v[e + 2], v[e + 3]);
                        pk.z = pack_bf16x2(v[e + 4], v[e + 5]);
                        pk.w = pack_bf16x2(v[e + 6], v[e + 7]);
                        *reinterpret_cast<uint4*>(orow + c + e) = pk;
                    }
                    if (frow) {
#pragma unroll
                        for (int e = 0; e < 32; e += 4)
                            *reinterpret_cast<float4*>(frow + c + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
                    }
                }
            }
            if (valid) p.LSE[(b * p.H + h) * p.Nq + t] = (m_used + __log2f(l)) * kLn2;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 8) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

constexpr size_t kSmemBytes = 1024 + 2 * kTileBytes + 2 * NST * kTileBytes + 2 * BN * sizeof(float) + sizeof(Bars) + 16;

}  // namespace

bool tc_fwd_supported(const AttnParams& p, gfwa_dtype_t dt) {
    if (dt != GFWA_BF16 || p.d != D) return false;
    if (p.Nkv >= ((int64_t)1 << 31) || p.H >= 65536 || p.B >= 65536) return false;
    if (const char* e = getenv("GFWA_FORCE_SIMT")) return e[0] == '0';
    return true;
}

gfwa_status_t tc_fwd(const AttnParams& p, cudaStream_t st) {
    CUtensorMap mq, mk, mv;
    if (!encode_bnhd_map(&mq, p.Q, p.B, p.Nq, p.H, D, p.qs, BM) ||
        !encode_bnhd_map(&mk, p.K, p.B, p.Nkv, p.H, D, p.ks, BN) ||
        !encode_bnhd_map(&mv, p.V, p.B, p.Nkv, p.H, D, p.vs, BN))
        return GFWA_ERR_INVALID_ARGUMENT;
    TcFwdParams tp;
    tp.U = p.U;
    tp.O = p.O;
    tp.O_f32 = p.O_f32;
    tp.LSE = p.LSE;
    tp.Nq = p.Nq;
    tp.Nkv = p.Nkv;
    tp.h0 = p.h0;
    tp.H = p.H;
    tp.w = p.w;
    tp.sl2 = p.scale * kLog2e;
    tp.os0 = p.os[0];
    tp.os1 = p.os[1];
    tp.os2 = p.os[2];
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
        attr_set = true;
    }
    dim3 grid((unsigned)((p.Nq + 2 * BM - 1) / (2 * BM)), (unsigned)p.H, (unsigned)p.B);
    fwd_tc_kernel<<<grid, kThreads, kSmemBytes, st>>>(mq, mk, mv, tp);
    note_launch();
    return check_launch();
}

}  // namespace gfwa
