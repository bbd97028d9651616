// attn_tc_bwd.cu -- GatedFWA backward on the 5th-generation tensor cores
// (sm_100a): Alg. E.2 with readings C-3, C-4, C-11, C-12.
//
// KV-major: one CTA owns a 128-key tile of one (b, h) (K and V resident in
// smem) and walks the 128-query tiles whose windows reach it.
// Per query tile, all five contractions run on tcgen05 with TMEM accumulators:
//   S^T  = K Q^T          SS  -> TMEM [0,128)
//   dP^T = V dO^T         SS  -> TMEM [128,256)
//   (softmax-grad warps, one thread per key: P^T = exp(S - L), dS^T =
//    P^T (dP^T - D); P^T, dS^T back to TMEM as bf16, dS^T also to smem)
//   dV  += P^T dO         TS  (A = P^T from TMEM)        -> TMEM [256,384)
//   dK  += dS^T Q         TS  (A = dS^T from TMEM)       -> TMEM [384,512)
//   dQ_i = dS K           SS  (A = dS from smem, MN-major) -> TMEM [0,128)
// The paper writes dQ back per tile; here the drain warps add it
// into an fp32 dQ accumulator with vector reductions in L2.  du^k (the column
// sum, C-4) accumulates in registers of the key thread; du^q (the paper's
// rowsum(dS), kept per reading C-11) is a cross-thread sum over keys,
// done in fp32 with a warp butterfly transpose-reduce plus a 4-warp smem
// combine, so both sums see the same fp32 dS and sum_m dU_m telescopes to 0.
// A separate Q-major kernel (the paper's second kernel) is avoided.
#include "attn_common.cuh"
#include "sm100.cuh"
#include "tma_host.cuh"

namespace gfwa {
namespace {

using namespace sm100;

constexpr int BM = 128;  // queries per step
constexpr int BN = 128;  // keys per CTA
constexpr int D = 128;
constexpr uint32_t kTile = 128 * 128 * 2;  // 32 KB bf16 tile
constexpr int kThreads = 320;              // softmax-grad WG, dQ-drain WG, MMA warp, TMA warp

struct TcBwdParams {
    const float* U;
    const float* LSE;
    const float* Dv;
    float* dQacc;   // [B, Nq, H, d] fp32, zeroed by the preprocess kernel
    float* dU;      // [B, H, Nkv] fp32, zeroed by the preprocess kernel
    void* dK;
    void* dV;
    int64_t Nq, Nkv, h0, H;
    int w;
    float sl2, scale;
    int64_t ks0, ks1, ks2, vs0, vs1, vs2;
};

struct __align__(8) Bars {
    uint64_t kv_full, q_full, q_empty, st_full, ds_ready, dq_full, dq_drained, dkdv_full;
};

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}
__device__ __forceinline__ void red_add(float* addr, float a) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(addr), "f"(a) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    bwd_tc_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                  const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mdo,
                  const TcBwdParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* Ks = smem;
    uint8_t* Vs = Ks + kTile;
    uint8_t* Qs = Vs + kTile;
    uint8_t* dOs = Qs + kTile;
    uint8_t* dSs = dOs + kTile;  // dS^T [keys][queries], MN-major A of the dQ MMA
    float* redq = (float*)(dSs + kTile);  // [4 warps][BM] partial du^q
    float* vlse = redq + 4 * BM;          // per-step query vectors (log2 units)
    float* vD = vlse + BM;
    float* vuq = vD + BM;
    Bars* bars = (Bars*)(vuq + BM);
    uint32_t* tmem_sh = (uint32_t*)(bars + 1);

    const int warp = threadIdx.x >> 5;
    const int64_t b = blockIdx.z, h = blockIdx.y;
    const int64_t j0 = (int64_t)blockIdx.x * BN;  // first key of the tile
    const int64_t j_last = min64(j0 + BN, p.Nkv) - 1;
    // Alg. E.2 l.12-14: queries whose window reaches this key tile
    const int64_t t_lo = max64(0, j0 - p.h0);
    const int64_t t_hi = min64(p.Nq - 1, j_last + p.w - 1 - p.h0);
    const int64_t qt_lo = t_lo / BM, qt_hi = t_hi / BM;
    const int nsteps = t_lo <= t_hi ? (int)(qt_hi - qt_lo + 1) : 0;

    if (threadIdx.x == 0) {
        mbar_init(&bars->kv_full, 1);
        mbar_init(&bars->q_full, 1);
        mbar_init(&bars->q_empty, 1);
        mbar_init(&bars->st_full, 1);
        mbar_init(&bars->ds_ready, 4);
        mbar_init(&bars->dq_full, 1);
        mbar_init(&bars->dq_drained, 4);
        mbar_init(&bars->dkdv_full, 1);
        fence_barrier_init();
    }
    if (warp == 8) {
        tmem_alloc(tmem_sh, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_sh;

    if (warp == 9) {
        // ------------------------------------------------ TMA producer
        if (elect_one() && nsteps > 0) {
            mbar_expect_tx(&bars->kv_full, 2 * kTile);
            for (int half = 0; half < 2; ++half) {
                tma_load_4d(Ks + half * (kTile / 2), &mk, &bars->kv_full, half * 64, (int)h, (int)j0, (int)b);
                tma_load_4d(Vs + half * (kTile / 2), &mv, &bars->kv_full, half * 64, (int)h, (int)j0, (int)b);
            }
            for (int n = 0; n < nsteps; ++n) {
                const int64_t t0 = (qt_lo + n) * BM;
                mbar_wait(&bars->q_empty, (n & 1) ^ 1);
                mbar_expect_tx(&bars->q_full, 2 * kTile);
                for (int half = 0; half < 2; ++half) {
                    tma_load_4d(Qs + half * (kTile / 2), &mq, &bars->q_full, half * 64, (int)h, (int)t0, (int)b);
                    tma_load_4d(dOs + half * (kTile / 2), &mdo, &bars->q_full, half * 64, (int)h, (int)t0,
                                (int)b);
                }
            }
        }
    } else if (warp == 8) {
        // ------------------------------------------------ MMA issuer
        const uint32_t id_kk = idesc_bf16(128, 128, false, false);  // S^T, dP^T
        const uint32_t id_tm = idesc_bf16(128, 128, false, true);   // dV, dK (A in TMEM, B MN-major)
        const uint32_t id_dq = idesc_bf16(128, 128, true, true);    // dQ (A, B MN-major)
        if (nsteps > 0) mbar_wait(&bars->kv_full, 0);
        const uint32_t kb = smem_u32(Ks), vb = smem_u32(Vs), qb = smem_u32(Qs), ob = smem_u32(dOs),
                       sb = smem_u32(dSs);
        for (int n = 0; n < nsteps; ++n) {
            mbar_wait(&bars->q_full, n & 1);
            if (n > 0) mbar_wait(&bars->dq_drained, (n - 1) & 1);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint32_t off = (kk >> 2) * (kTile / 2) + (kk & 3) * 32;
                    mma_ss(tmem + 0, sdesc_sw128(kb + off, 16, 1024), sdesc_sw128(qb + off, 16, 1024), id_kk,
                           kk > 0);
                    mma_ss(tmem + 128, sdesc_sw128(vb + off, 16, 1024), sdesc_sw128(ob + off, 16, 1024), id_kk,
                           kk > 0);
                }
                tc_commit(&bars->st_full);
            }
            __syncwarp();
            mbar_wait(&bars->ds_ready, n & 1);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < BM / 16; ++kk) {
                    // dV += P^T dO ; dK += dS^T Q  (A from TMEM, 16 queries = 8 columns)
                    mma_ts(tmem + 256, tmem + 0 + 8 * kk, sdesc_sw128(ob + kk * 2048, kTile / 2, 1024), id_tm,
                           (n > 0 || kk > 0) ? 1u : 0u);
                    mma_ts(tmem + 384, tmem + 128 + 8 * kk, sdesc_sw128(qb + kk * 2048, kTile / 2, 1024), id_tm,
                           (n > 0 || kk > 0) ? 1u : 0u);
                }
#pragma unroll
                for (int kk = 0; kk < BN / 16; ++kk) {
                    // dQ_i = dS K   (contract over the 128 keys)
                    mma_ss(tmem + 0, sdesc_sw128(sb + kk * 2048, kTile / 2, 1024),
                           sdesc_sw128(kb + kk * 2048, kTile / 2, 1024), id_dq, kk > 0);
                }
                tc_commit(&bars->dq_full);
                tc_commit(&bars->q_empty);
                if (n == nsteps - 1) tc_commit(&bars->dkdv_full);
            }
            __syncwarp();
        }
    } else if (warp < 4) {
        // ------------------------------------------------ softmax-grad WG: thread = key
        const int kr = threadIdx.x;  // 0..127
        const int64_t j = j0 + kr;
        const bool kvalid = j < p.Nkv;
        const float* Ubh = p.U + (b * p.H + h) * p.Nkv;
        const float uk = kvalid ? Ubh[j] : 0.f;
        const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
        float colsum = 0.f;
        for (int n = 0; n < nsteps; ++n) {
            const int64_t t0 = (qt_lo + n) * BM;
            named_bar_sync(1, 128);
            {
                const int64_t t = t0 + kr;
                const bool ok = t < p.Nq;
                const int64_t vi = (b * p.H + h) * p.Nq + t;
                vlse[kr] = ok ? p.LSE[vi] * kLog2e : 0.f;
                vD[kr] = ok ? p.Dv[vi] : 0.f;
                vuq[kr] = ok ? Ubh[t + p.h0] : 0.f;
            }
            named_bar_sync(1, 128);
            mbar_wait(&bars->st_full, n & 1);
            tc_fence_after();
            // interior: every (key, query) pair of the tile lies inside the window
            const bool interior = (j0 + BN - 1 <= t0 + p.h0) && (j0 > t0 + BM - 1 + p.h0 - p.w) &&
                                  (t0 + BM <= p.Nq) && (j0 + BN <= p.Nkv);
#pragma unroll 1
            for (int c = 0; c < BM; c += 32) {
                uint32_t sr[32], dr[32];
                tmem_ld32(lane_addr + c, sr);
                tmem_ld32(lane_addr + 128 + c, dr);
                tmem_wait_ld();
                float ds[32];
                uint32_t pk[16], dk[16];
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const int q = c + e;
                    // P = exp(scale q.k + (u_q - u_k) - L_q), log2 units
                    float x = fmaf(__uint_as_float(sr[e]), p.sl2, (vuq[q] - uk) * kLog2e) - vlse[q];
                    if (!interior) {
                        const int64_t t = t0 + q, g = t + p.h0;
                        const bool keep = t < p.Nq && kvalid && j <= g && j > g - p.w;
                        x = keep ? x : -INFINITY;
                    }
                    const float pr = ex2(x);
                    ds[e] = pr * (__uint_as_float(dr[e]) - vD[q]);  // dS = P (dP - D)
                    colsum += ds[e];                                // du^k, fp32 (C-4)
                    if (e & 1) {
                        pk[e / 2] = pack_bf16x2(__uint_as_float(sr[e - 1]), pr);
                        dk[e / 2] = pack_bf16x2(ds[e - 1], ds[e]);
                    } else {
                        sr[e] = __float_as_uint(pr);  // keep P of the even column for packing
                    }
                }
                tmem_st16(lane_addr + c / 2, pk);        // P^T  -> cols [0, 64)
                tmem_st16(lane_addr + 128 + c / 2, dk);  // dS^T -> cols [128, 192)
                // dS^T row -> smem, 128B-swizzled MN-major layout (query chunk ^ key%8)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const int q = c + v * 8;
                    const int half = q >> 6, chunk = ((q & 63) >> 3) ^ (kr & 7);
                    uint4 val = make_uint4(dk[v * 4 + 0], dk[v * 4 + 1], dk[v * 4 + 2], dk[v * 4 + 3]);
                    *reinterpret_cast<uint4*>(dSs + half * (kTile / 2) + kr * 128 + chunk * 16) = val;
                }
                // du^q partial: sum of this warp's 32 keys for each of the 32 query
                // columns, butterfly transpose-reduce -> lane l holds column c + l
                const int lane = threadIdx.x & 31;
#pragma unroll
                for (int s = 16; s >= 1; s >>= 1) {
                    const bool up = lane & s;
#pragma unroll
                    for (int e = 0; e < s; ++e) {
                        const float send = up ? ds[e] : ds[e + s];
                        const float keep = up ? ds[e + s] : ds[e];
                        ds[e] = keep + __shfl_xor_sync(0xffffffffu, send, s);
                    }
                }
                redq[warp * BM + c + lane] = ds[0];
            }
            tmem_wait_st();
            fence_proxy_async();
            tc_fence_before();
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(&bars->ds_ready);
            // du^q_t += rowsum(dS) at key position t + h0 (C-11), 4-warp combine
            named_bar_sync(1, 128);
            {
                const int64_t t = t0 + kr;
                const float rs = redq[kr] + redq[BM + kr] + redq[2 * BM + kr] + redq[3 * BM + kr];
                if (t < p.Nq) red_add(p.dU + (b * p.H + h) * p.Nkv + t + p.h0, rs);
            }
        }
        // epilogue: dK = scale * acc (C-3), dV, du^k = -colsum (C-4)
        __nv_bfloat16* dkrow = (__nv_bfloat16*)p.dK + b * p.ks0 + j * p.ks1 + h * p.ks2;
        __nv_bfloat16* dvrow = (__nv_bfloat16*)p.dV + b * p.vs0 + j * p.vs1 + h * p.vs2;
        if (nsteps > 0) {
            mbar_wait(&bars->dkdv_full, 0);
            tc_fence_after();
        }
#pragma unroll 1
        for (int c = 0; c < D; c += 32) {
            uint32_t kr32[32], vr32[32];
            if (nsteps > 0) {
                tmem_ld32(lane_addr + 384 + c, kr32);
                tmem_ld32(lane_addr + 256 + c, vr32);
                tmem_wait_ld();
            } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) kr32[e] = vr32[e] = 0u;
            }
            if (kvalid) {
#pragma unroll
                for (int e = 0; e < 32; e += 8) {
                    uint4 a, v;
                    a.x = pack_bf16x2(__uint_as_float(kr32[e + 0]) * p.scale, __uint_as_float(kr32[e + 1]) * p.scale);
                    a.y = pack_bf16x2(__uint_as_float(kr32[e + 2]) * p.scale, __uint_as_float(kr32[e + 3]) * p.scale);
                    a.z = pack_bf16x2(__uint_as_float(kr32[e + 4]) * p.scale, __uint_as_float(kr32[e + 5]) * p.scale);
                    a.w = pack_bf16x2(__uint_as_float(kr32[e + 6]) * p.scale, __uint_as_float(kr32[e + 7]) * p.scale);
                    v.x = pack_bf16x2(__uint_as_float(vr32[e + 0]), __uint_as_float(vr32[e + 1]));
                    v.y = pack_bf16x2(__uint_as_float(vr32[e + 2]), __uint_as_float(vr32[e + 3]));
                    v.z = pack_bf16x2(__uint_as_float(vr32[e + 4]), __uint_as_float(vr32[e + 5]));
                    v.w = pack_bf16x2(__uint_as_float(vr32[e + 6]), __uint_as_float(vr32[e + 7]));
                    *reinterpret_cast<uint4*>(dkrow + c + e) = a;
                    *reinterpret_cast<uint4*>(dvrow + c + e) = v;
                }
            }
        }
        if (kvalid) red_add(p.dU + (b * p.H + h) * p.Nkv + j, -colsum);
    } else if (warp < 8) {
        // ------------------------------------------------ dQ drain WG: thread = query
        const int qr = threadIdx.x - 128;
        const uint32_t lane_addr = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        for (int n = 0; n < nsteps; ++n) {
            const int64_t t = (qt_lo + n) * BM + qr;
            const bool valid = t < p.Nq;
            mbar_wait(&bars->dq_full, n & 1);
            tc_fence_after();
            float* dq = p.dQacc + ((b * p.Nq + t) * p.H + h) * D;
#pragma unroll 1
            for (int c = 0; c < D; c += 32) {
                uint32_t r[32];
                tmem_ld32(lane_addr + c, r);
                tmem_wait_ld();
                if (valid) {
#pragma unroll
                    for (int e = 0; e < 32; e += 4)
                        red_add_v4(dq + c + e, __uint_as_float(r[e]), __uint_as_float(r[e + 1]),
                                   __uint_as_float(r[e + 2]), __uint_as_float(r[e + 3]));
                }
            }
            tc_fence_before();
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(&bars->dq_drained);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 8) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

constexpr size_t kSmemBytes = 1024 + 5 * kTile + 7 * BM * sizeof(float) + sizeof(Bars) + 16;

// dQacc, dU zeroing fused with D = rowsum(O dO); dQ = scale * dQacc -> bf16
__global__ void __launch_bounds__(256) bwd_tc_pre_kernel(AttnParams p) {
    const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const int64_t total = p.B * p.Nq * p.H;
    if (row >= total) return;
    const int64_t h = row % p.H, t = (row / p.H) % p.Nq, b = row / (p.H * p.Nq);
    const int64_t oo = b * p.os[0] + t * p.os[1] + h * p.os[2];
    const __nv_bfloat16* dO = (const __nv_bfloat16*)p.dO + oo;
    float acc = 0.f;
    const int c = lane * 4;  // d = 128: 4 elements per lane
    const uint2 g2 = *reinterpret_cast<const uint2*>(dO + c);
    const float2 g01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&g2.x));
    const float2 g23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&g2.y));
    if (p.Ofp) {
        const float4 o = *reinterpret_cast<const float4*>(p.Ofp + oo + c);
        acc = o.x * g01.x + o.y * g01.y + o.z * g23.x + o.w * g23.y;
    } else {
        const uint2 o2 = *reinterpret_cast<const uint2*>((const __nv_bfloat16*)p.O + oo + c);
        const float2 o01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&o2.x));
        const float2 o23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&o2.y));
        acc = o01.x * g01.x + o01.y * g01.y + o23.x * g23.x + o23.y * g23.y;
    }
    acc = warp_sum(acc);
    if (lane == 0) p.Dv[(b * p.H + h) * p.Nq + t] = acc;
    *reinterpret_cast<float4*>(p.dQacc + ((b * p.Nq + t) * p.H + h) * D + c) = make_float4(0.f, 0.f, 0.f, 0.f);
}

__global__ void __launch_bounds__(256) bwd_tc_post_kernel(AttnParams p) {
    const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const int64_t total = p.B * p.Nq * p.H;
    if (row >= total) return;
    const int64_t h = row % p.H, t = (row / p.H) % p.Nq, b = row / (p.H * p.Nq);
    const int c = lane * 4;
    const float4 a = *reinterpret_cast<const float4*>(p.dQacc + ((b * p.Nq + t) * p.H + h) * D + c);
    uint2 o;
    o.x = pack_bf16x2(a.x * p.scale, a.y * p.scale);  // dQ = scale dS K (C-3)
    o.y = pack_bf16x2(a.z * p.scale, a.w * p.scale);
    *reinterpret_cast<uint2*>((__nv_bfloat16*)p.dQ + b * p.qs[0] + t * p.qs[1] + h * p.qs[2] + c) = o;
}

}  // namespace

bool tc_bwd_supported(const AttnParams& p, gfwa_dtype_t dt) {
    if (dt != GFWA_BF16 || p.d != D) return false;
    if (p.Nkv >= ((int64_t)1 << 31) || p.H >= 65536 || p.B >= 65536) return false;
    if (const char* e = getenv("GFWA_FORCE_SIMT")) return e[0] == '0';
    return true;
}

size_t tc_bwd_workspace(const AttnParams& p) { return (size_t)p.B * p.Nq * p.H * D * sizeof(float); }

gfwa_status_t tc_bwd(const AttnParams& pin, cudaStream_t st, void* ws) {
    AttnParams p = pin;
    p.dQacc = (float*)ws;
    CUtensorMap mq, mk, mv, mdo;
    GFWA_REQUIRE(encode_bnhd_map(&mq, p.Q, p.B, p.Nq, p.H, D, p.qs, BM));
    GFWA_REQUIRE(encode_bnhd_map(&mk, p.K, p.B, p.Nkv, p.H, D, p.ks, BN));
    GFWA_REQUIRE(encode_bnhd_map(&mv, p.V, p.B, p.Nkv, p.H, D, p.vs, BN));
    GFWA_REQUIRE(encode_bnhd_map(&mdo, p.dO, p.B, p.Nq, p.H, D, p.os, BM));
    const int64_t rows = p.B * p.Nq * p.H;
    const unsigned rgrid = (unsigned)((rows + 7) / 8);
    if (gfwa_status_t s = check_launch(cudaMemsetAsync(p.dU, 0, (size_t)p.B * p.H * p.Nkv * sizeof(float), st)))
        return s;
    bwd_tc_pre_kernel<<<rgrid, 256, 0, st>>>(p);
    note_launch();
    if (gfwa_status_t s = check_launch()) return s;
    TcBwdParams tp;
    tp.U = p.U;
    tp.LSE = p.LSE;
    tp.Dv = p.Dv;
    tp.dQacc = p.dQacc;
    tp.dU = p.dU;
    tp.dK = p.dK;
    tp.dV = p.dV;
    tp.Nq = p.Nq;
    tp.Nkv = p.Nkv;
    tp.h0 = p.h0;
    tp.H = p.H;
    tp.w = p.w;
    tp.sl2 = p.scale * kLog2e;
    tp.scale = p.scale;
    tp.ks0 = p.ks[0];
    tp.ks1 = p.ks[1];
    tp.ks2 = p.ks[2];
    tp.vs0 = p.vs[0];
    tp.vs1 = p.vs[1];
    tp.vs2 = p.vs[2];
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(bwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
        attr_set = true;
    }
    dim3 grid((unsigned)((p.Nkv + BN - 1) / BN), (unsigned)p.H, (unsigned)p.B);
    bwd_tc_kernel<<<grid, kThreads, kSmemBytes, st>>>(mq, mk, mv, mdo, tp);
    note_launch();
    if (gfwa_status_t s = check_launch()) return s;
    bwd_tc_post_kernel<<<rgrid, 256, 0, st>>>(p);
    note_launch();
    return check_launch();
}

}  // namespace gfwa
