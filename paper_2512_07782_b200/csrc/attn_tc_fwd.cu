// attn_tc_fwd.cu -- GatedFWA forward on the 5th-generation tensor cores
// (sm_100a): Alg. 2 re-designed for tcgen05/TMEM/TMA.
//
// One CTA owns one 128-row query tile of one (b, h) and streams the 128-key
// K/V tiles of its window, diagonal first (descending j).  TWO CTAs share an
// SM (98 KB smem, 256 TMEM columns each): while one runs its softmax the other's
// MMAs keep the tensor core busy, and one CTA's prologue (Q, K loads, first S)
// and epilogue overlap the other's main loop -- without a persistent scheduler.
//   warp 5      TMA producer: Q once, then K_j, V_j (one stage each: K_{j+1}
//               streams in during the softmax of step j, V_j during the S MMA);
//               128B swizzle, OOB rows zero-filled -> ragged tails for free
//   warp 4      MMA issuer (one elected lane): S = Q K_j^T (SS, fp32 in TMEM)
//               and O += P V_j (TS: bf16 P read from TMEM); tcgen05.commit
//               tracks all earlier MMAs, so S_full of step n also certifies
//               that PV of step n-1 has landed.
//   warps 0-3   softmax, one thread per query row holding its 128 S values in
//               registers (four tcgen05.ld, one wait; setmaxnreg gives this
//               warpgroup 224 registers): add the gate bias as an
//               outer difference of two u vectors (nothing N x w is
//               materialised), window-mask only on diagonal / window-edge tiles
//               (a per-row column range turned into bit masks), online
//               softmax in fp32 with packed f32x2 FMA/ADD, 3-input max and a lazy
//               rescale (the reference max moves only when it grows by > 2^8),
//               part of exp2 on the FMA pipe, bf16 P back over the S columns;
//               epilogue O / l staged in smem with the 128B swizzle and written
//               by TMA stores, LSE = m + ln l.
//   warps 6-7   training forward (O_f32 requested): convert each V tile to fp16
//               in place once it lands, so the PV product runs with P in fp16
//               (reading C-23: the fp32 O that the backward's D = rowsum(O dO)
//               is taken from carries 8x less P rounding than with bf16 P);
//               otherwise idle (they complete the second warpgroup for setmaxnreg)
// TMEM (256 columns per CTA): S [0,128), O [128,256) x 128 lanes.
// Key tiles outside every row's window are never loaded.
#include <vector>

#ifndef GFWA_FWD_POLY
#define GFWA_FWD_POLY 0
#endif

#include "attn_common.cuh"
#include "sm100.cuh"
#include "tma_host.cuh"

namespace gfwa {
namespace {

using namespace sm100;

constexpr int BM = 128;          // query rows per tile
constexpr int BN = 128;          // keys per tile
constexpr int D = 128;           // head dim
constexpr uint32_t kTileBytes = BM * D * 2;  // 32 KB bf16 tile
constexpr uint32_t kZeroBytes = 64 * 32 * 4;   // 8 KB: one {32 d, 64 rows} fp32 box of zeros
constexpr int kThreads = 256;    // softmax warpgroup + (MMA, TMA, 2 idle)
constexpr int kMmaWarp = 4, kTmaWarp = 5;
constexpr int kSoftmaxRegs = 224;  // CTA pool at (256, 2): 256 x 128; 128 x 224 + 128 x 32 fits it
constexpr int kOtherRegs = 32;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr int kPolyPairs = GFWA_FWD_POLY;  // of every 4 column pairs, how many use exp2_poly2

struct TcFwdParams {
    const float* U;
    float* LSE;
    int64_t Nq, Nkv, h0, H;
    int w;
    int store_f32;
    float* zero_acc;   // gfwa_fwd_train: the dQ accumulator [B, Nq, H, d] whose rows of this tile are zeroed
    unsigned long long* token;
    unsigned long long token_val;
    float sl2;         // scale * log2(e)
    long long* trace;  // diagnostics only (GFWA_TRACE_FWD): per-CTA clock64 stamps
};

#define GFWA_TR(slot)                                                                                         \
    do {                                                                                                      \
        if (p.trace)                                                                                          \
            p.trace[((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 64 + (slot)] = clock64(); \
    } while (0)

struct __align__(8) Bars {
    uint64_t q_full, k_full, k_empty, v_full, v_empty, v_conv, s_full, p_ready, o_full;
};

__device__ __forceinline__ int64_t kv_tile_lo(int64_t g_lo, int w) { return max64(0, g_lo - w + 1) / BN; }

// bits [lo, hi] (inclusive, clipped to the 32-bit word starting at column base)
__device__ __forceinline__ uint32_t range_bits(int lo, int hi, int base) {
    const int a = min(max(lo - base, 0), 32), z = min(max(hi - base + 1, 0), 32);
    const uint32_t upto_z = z >= 32 ? 0xffffffffu : ((1u << z) - 1u);
    const uint32_t below_a = a >= 32 ? 0xffffffffu : ((1u << a) - 1u);
    return upto_z & ~below_a;
}

template <bool kF16P>  // training forward: P, V in fp16 for the PV product (reading C-23)
__global__ void __launch_bounds__(kThreads, 2)
    fwd_tc_kernel(const __grid_constant__ CUtensorMap mzq, const __grid_constant__ CUtensorMap mq,
                  const __grid_constant__ CUtensorMap mk,
                  const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mo,
                  const __grid_constant__ CUtensorMap mo32, const TcFwdParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* Qs = smem;
    uint8_t* Ks = Qs + kTileBytes;
    uint8_t* Vs = Ks + kTileBytes;
    __shared__ __align__(16) float s_nbk[BN];  // negated key bias -(u_k - uref) log2e
    uint8_t* Zs = Vs + kTileBytes;  // 8 KB of zeros (gfwa_fwd_train)
    Bars* bars = (Bars*)(Zs + kZeroBytes);
    uint32_t* tmem_sh = (uint32_t*)(bars + 1);

    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        GFWA_TR(0);
        if (p.trace) {
            uint32_t smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            p.trace[((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 64 + 63] = smid;
        }
    }
    const int64_t b = blockIdx.z, h = blockIdx.y;
    const int64_t r0 = (int64_t)blockIdx.x * BM;
    // Alg. 2 l.7-9: key positions g = t + h0
    const int64_t glo = r0 + p.h0, ghi = min64(r0 + BM - 1, p.Nq - 1) + p.h0;
    const int64_t jlo = kv_tile_lo(glo, p.w), jhi = ghi / BN;

    if (threadIdx.x == 0) {
        mbar_init(&bars->q_full, 1);
        mbar_init(&bars->k_full, 1);
        mbar_init(&bars->k_empty, 1);
        mbar_init(&bars->v_full, 1);
        mbar_init(&bars->v_empty, 1);
        mbar_init(&bars->v_conv, 2);
        mbar_init(&bars->s_full, 1);
        mbar_init(&bars->p_ready, 4);
        mbar_init(&bars->o_full, 1);
        fence_barrier_init();
    }
    if (warp == kMmaWarp) {
        tmem_alloc(tmem_sh, 256);
        tmem_relinquish();
    }
    if (warp == kTmaWarp && elect_one()) {
        tma_prefetch(&mq);
        tma_prefetch(&mk);
        tma_prefetch(&mv);
        tma_prefetch(&mo);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_sh;
    if (threadIdx.x == 0) GFWA_TR(1);
    // registers move from the MMA/TMA warpgroup to the softmax warpgroup
    if (warp >= 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kOtherRegs));

    if (warp == kTmaWarp) {
        // ------------------------------------------------ TMA producer
        if (elect_one()) {
            const uint64_t pol_kv = policy_evict_last();  // K/V tiles are re-read by ~w/128 neighbours
            mbar_expect_tx(&bars->q_full, kTileBytes);
            for (int half = 0; half < 2; ++half)
                tma_load_4d(Qs + half * (kTileBytes / 2), &mq, &bars->q_full, half * 64, (int)h, (int)r0, (int)b);
            int k = 0;
            for (int64_t j = jhi; j >= jlo; --j, ++k) {
                mbar_wait(&bars->k_empty, (k & 1) ^ 1);
                mbar_expect_tx(&bars->k_full, kTileBytes);
                for (int half = 0; half < 2; ++half)
                    tma_load_4d_hint(Ks + half * (kTileBytes / 2), &mk, &bars->k_full, half * 64, (int)h,
                                     (int)(j * BN), (int)b, pol_kv);
                mbar_wait(&bars->v_empty, (k & 1) ^ 1);
                mbar_expect_tx(&bars->v_full, kTileBytes);
                for (int half = 0; half < 2; ++half)
                    tma_load_4d_hint(Vs + half * (kTileBytes / 2), &mv, &bars->v_full, half * 64, (int)h,
                                     (int)(j * BN), (int)b, pol_kv);
            }
        }
        __syncwarp();
        if (p.zero_acc) {
            // gfwa_fwd_train: this idle warp zeroes the tile's 128 rows of the backward's
            // fp32 dQ accumulator with TMA stores of an 8 KB zero box, while the
            // other warps finish the tile (the writes overlap the compute)
            const uint32_t zb = smem_u32(Zs) + (threadIdx.x & 31) * 256;
#pragma unroll
            for (int k2 = 0; k2 < 16; ++k2) sts128(zb + k2 * 16, make_uint4(0u, 0u, 0u, 0u));
            fence_proxy_async();
            __syncwarp();
            if ((threadIdx.x & 31) == 0) {
                for (int rh = 0; rh < 2; ++rh)
                    for (int c = 0; c < 4; ++c) tma_store_4d(&mzq, Zs, c * 32, (int)h, (int)(r0 + 64 * rh), (int)b);
                bulk_commit();
                if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) *p.token = p.token_val;
                bulk_wait_read0();  // the zero box stays valid until read
            }
            __syncwarp();
        }
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------ MMA issuer
        const uint32_t idesc_qk = idesc_bf16(BM, BN, false, false);
        // training forward: P and V in fp16 (A/B format F16 = 0), reading C-23
        const uint32_t idesc_pv = idesc_bf16(BM, D, false, true) & ~(kF16P ? (63u << 7) : 0u);
        uint64_t* v_ready = kF16P ? &bars->v_conv : &bars->v_full;
        const uint32_t qbase = smem_u32(Qs), kbase = smem_u32(Ks), vbase = smem_u32(Vs);
        mbar_wait(&bars->q_full, 0);
        int k = 0;
        for (int64_t j = jhi; j >= jlo; --j, ++k) {
            if (k > 0) {
                // O += P(k-1) V(k-1), then V's stage is free
                mbar_wait(&bars->p_ready, (k - 1) & 1);
                mbar_wait(v_ready, (k - 1) & 1);
                tc_fence_after();
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < BN / 16; ++kk)
                        mma_ts(tmem + 128, tmem + 8 * kk, sdesc_sw128(vbase + kk * 2048, kTileBytes / 2, 1024),
                               idesc_pv, (k > 1 || kk > 0) ? 1u : 0u);
                    tc_commit(&bars->v_empty);
                }
                __syncwarp();
            }
            // S = Q K_j^T (over the P just consumed: tcgen05 MMAs run in issue order)
            mbar_wait(&bars->k_full, k & 1);
            if (k < 8 && (threadIdx.x & 31) == 0) GFWA_TR(2 + k);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint32_t off = (kk >> 2) * (kTileBytes / 2) + (kk & 3) * 32;
                    mma_ss(tmem, sdesc_sw128(qbase + off, 16, 1024), sdesc_sw128(kbase + off, 16, 1024), idesc_qk,
                           kk > 0 ? 1u : 0u);
                }
                tc_commit(&bars->s_full);
                tc_commit(&bars->k_empty);
            }
            __syncwarp();
        }
        // last PV, then O is final
        mbar_wait(&bars->p_ready, (k - 1) & 1);
        mbar_wait(v_ready, (k - 1) & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BN / 16; ++kk)
                mma_ts(tmem + 128, tmem + 8 * kk, sdesc_sw128(vbase + kk * 2048, kTileBytes / 2, 1024), idesc_pv,
                       (k > 1 || kk > 0) ? 1u : 0u);
            tc_commit(&bars->o_full);
        }
        __syncwarp();
    } else if (kF16P && warp >= 6) {
        // ------------------------------------------------ V -> fp16 in place (training forward)
        // 2048 16-byte chunks per tile over 64 threads; the layout (128B swizzle) is
        // unchanged, only the element encoding: bf16 -> fp32 (exact) -> fp16 (RNE)
        const uint32_t vb = smem_u32(Vs) + (threadIdx.x - 192) * 16;
        int k = 0;
        for (int64_t j = jhi; j >= jlo; --j, ++k) {
            mbar_wait(&bars->v_full, k & 1);
#pragma unroll 4
            for (int c = 0; c < (int)(kTileBytes / 16 / 64); ++c) {
                const uint32_t a = vb + c * 64 * 16;
                uint4 x = lds128u(a);
                x.x = bf16x2_to_f16x2(x.x);
                x.y = bf16x2_to_f16x2(x.y);
                x.z = bf16x2_to_f16x2(x.z);
                x.w = bf16x2_to_f16x2(x.w);
                sts128(a, x);
            }
            fence_proxy_async();  // generic-proxy writes -> visible to the tensor core
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(&bars->v_conv);
        }
    } else if (warp < 4) {
        // ------------------------------------------------ softmax warpgroup
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kSoftmaxRegs));
        const int r = threadIdx.x & 127;
        const int64_t t = r0 + r;
        const bool valid = t < p.Nq;
        const int64_t g = t + p.h0;
        const float* Ubh = p.U + (b * p.H + h) * p.Nkv;
        // Bias in log2 units relative to a per-CTA reference u (reading C-18):
        // u_q - u_k = (u_q - uref) - (u_k - uref); each difference is formed in
        // fp32 before scaling, and the row constant (u_q - uref) cancels in the
        // softmax, so it only re-enters the LSE.
        const float uref = Ubh[glo];
        const float bq = valid ? (Ubh[g] - uref) * kLog2e : 0.f;
        const uint32_t lane_addr = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        const uint64_t sl2x2 = f2pack(p.sl2, p.sl2);
        float m_used = -INFINITY, l = 0.f;
        int n = 0;
        float u_next = jhi * BN + r < p.Nkv ? Ubh[jhi * BN + r] : 0.f;
        for (int64_t j = jhi; j >= jlo; --j, ++n) {
            // -(u_k - uref) log2e of this key tile -> smem (WG-cooperative); the
            // next tile's u is prefetched into a register meanwhile
            named_bar_sync(1, 128);
            s_nbk[r] = (uref - u_next) * kLog2e;
            if (j > jlo) u_next = (j - 1) * BN + r < p.Nkv ? Ubh[(j - 1) * BN + r] : 0.f;
            named_bar_sync(1, 128);
            mbar_wait(&bars->s_full, n & 1);
            if (n < 8 && r == 0) GFWA_TR(16 + n);
            tc_fence_after();
            const bool trw = (n == 1 && (r == 0 || r == 96));
            const bool interior = (j * BN + BN - 1 <= glo) && (j * BN >= ghi - p.w + 1);
            uint32_t keep[4] = {~0u, ~0u, ~0u, ~0u};
            if (!interior) {
                // keys in (g - w, g] and < N_kv, as columns of this tile
                const int64_t kb = j * BN;
                const int hi = (int)min64(min64(g - kb, (int64_t)BN - 1), p.Nkv - 1 - kb);
                const int lo = (int)max64(g - p.w + 1 - kb, (int64_t)0);
#pragma unroll
                for (int c = 0; c < 4; ++c) keep[c] = range_bits(lo, hi, 32 * c);
            }
            // the whole S row in registers: four loads, one wait, then the logits
            // x = scale*q.k - (u_k - uref) log2e (Alg. 2 l.12-15) in place as
            // packed pairs; max and exp both run from registers
            uint32_t raw[BN];
#pragma unroll
            for (int cb = 0; cb < BN; cb += 32)
                tmem_ld32(lane_addr + cb, *reinterpret_cast<uint32_t(*)[32]>(raw + cb));
            tmem_wait_ld();
            if (trw) GFWA_TR(10 + (r == 96));
            uint64_t xp[BN / 2];
#pragma unroll
            for (int e = 0; e < BN; e += 4) {
                const float4 nb = *reinterpret_cast<const float4*>(s_nbk + e);
                xp[e / 2] = ffma2(f2pack(__uint_as_float(raw[e]), __uint_as_float(raw[e + 1])), sl2x2,
                                  f2pack(nb.x, nb.y));
                xp[e / 2 + 1] = ffma2(f2pack(__uint_as_float(raw[e + 2]), __uint_as_float(raw[e + 3])), sl2x2,
                                      f2pack(nb.z, nb.w));
            }
            if (!interior) {
#pragma unroll
                for (int e = 0; e < BN / 2; ++e) {
                    const uint32_t kw = keep[e >> 4];
                    const int bit = 2 * (e & 15);
                    float a, z;
                    f2unpack(xp[e], a, z);
                    a = ((kw >> bit) & 1u) ? a : -INFINITY;
                    z = ((kw >> (bit + 1)) & 1u) ? z : -INFINITY;
                    xp[e] = f2pack(a, z);
                }
            }
            float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int e = 0; e < BN / 2; ++e) {
                float a, z;
                f2unpack(xp[e], a, z);
                mx[e & 3] = fmax3(mx[e & 3], a, z);
            }
            const float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
            if (trw) GFWA_TR(12 + (r == 96));
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
            const uint64_t nm2 = f2pack(-mref, -mref);
            uint64_t acc[4] = {0, 0, 0, 0};  // packed (0.f, 0.f)
#pragma unroll
            for (int cb = 0; cb < BN; cb += 32) {
                uint32_t pk[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const uint64_t d = fadd2(xp[cb / 2 + e], nm2);
                    float p0, p1;
                    if ((e & 3) < kPolyPairs) {
                        // part of the exponentials on the FMA pipe: MUFU.EX2 is
                        // co-critical with the tensor core on B200
                        f2unpack(exp2_poly2(d), p0, p1);
                    } else {
                        float d0, d1;
                        f2unpack(d, d0, d1);
                        p0 = ex2(d0);
                        p1 = ex2(d1);
                    }
                    acc[e & 3] = fadd2(acc[e & 3], f2pack(p0, p1));
                    pk[e] = kF16P ? pack_f16x2(p0, p1) : pack_bf16x2(p0, p1);
                }
                tmem_st16(lane_addr + cb / 2, pk);  // P (bf16, or fp16 when training) over the S columns
            }
            if (trw) GFWA_TR(14 + (r == 96));
            {
                const uint64_t a01 = fadd2(acc[0], acc[1]), a23 = fadd2(acc[2], acc[3]);
                float s0, s1;
                f2unpack(fadd2(a01, a23), s0, s1);
                l += s0 + s1;
            }
            // rescale O (PV of the previous step is complete: S_full certified it)
            if (__any_sync(0xffffffffu, need) && n > 0) {
                uint32_t ob[32];
#pragma unroll
                for (int c = 0; c < D; c += 32) {
                    tmem_ld32(lane_addr + 128 + c, ob);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) ob[e] = __float_as_uint(__uint_as_float(ob[e]) * corr);
                    tmem_st32(lane_addr + 128 + c, ob);
                }
            }
            tmem_wait_st();
            if (trw) GFWA_TR(34 + (r == 96));
            tc_fence_before();
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(&bars->p_ready);
            if (n < 8 && r == 0) GFWA_TR(24 + n);
            if (trw && r == 96) GFWA_TR(38);
        }
        // epilogue: O / l (Alg. 2 l.19-20) staged in smem (128B swizzle: bf16 in the
        // Q slot, fp32 in the K and V slots -- all idle once O_full fires) and
        // written with TMA stores
        mbar_wait(&bars->o_full, 0);
        if (r == 0) GFWA_TR(32);
        tc_fence_after();
        const float inv = l > 0.f ? 1.f / l : 0.f;
        const uint32_t sbf = smem_u32(Qs), sf = smem_u32(Ks);
        // two halves of 64 columns: both TMEM loads of a half in flight before one
        // wait, and the half's bulk stores issued as soon as it is staged, so the
        // second half's staging overlaps the first half's store read-out
#pragma unroll 1
        for (int hf = 0; hf < 2; ++hf) {
            uint32_t ob[2][32];
            tmem_ld32(lane_addr + 128 + 64 * hf, ob[0]);
            tmem_ld32(lane_addr + 128 + 64 * hf + 32, ob[1]);
            tmem_wait_ld();
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
            const int c = 2 * hf + cc;
            float v[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(ob[cc][e]) * inv;
            // bf16: columns [32c, 32c+32) = half c>>1, 16-B chunks (c&1)*4 + k
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int chunk = ((c & 1) * 4 + k) ^ (r & 7);
                uint4 pkv;
                pkv.x = pack_bf16x2(v[8 * k + 0], v[8 * k + 1]);
                pkv.y = pack_bf16x2(v[8 * k + 2], v[8 * k + 3]);
                pkv.z = pack_bf16x2(v[8 * k + 4], v[8 * k + 5]);
                pkv.w = pack_bf16x2(v[8 * k + 6], v[8 * k + 7]);
                sts128(sbf + (c >> 1) * (kTileBytes / 2) + r * 128 + chunk * 16, pkv);
            }
            if (p.store_f32) {
                // fp32: box c (32 columns, 128 B rows), 16-B pieces k
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int piece = k ^ (r & 7);
                    sts128(sf + c * 16384 + r * 128 + piece * 16,
                           make_uint4(__float_as_uint(v[4 * k]), __float_as_uint(v[4 * k + 1]),
                                      __float_as_uint(v[4 * k + 2]), __float_as_uint(v[4 * k + 3])));
                }
            }
            }
            fence_proxy_async();
            named_bar_sync(1, 128);
            if (r == 0) {
                tma_store_4d(&mo, Qs + hf * (kTileBytes / 2), hf * 64, (int)h, (int)r0, (int)b);
                if (p.store_f32)
                    for (int c = 2 * hf; c < 2 * hf + 2; ++c)
                        tma_store_4d(&mo32, Ks + c * 16384, c * 32, (int)h, (int)r0, (int)b);
                bulk_commit();
            }
        }
        if (valid) p.LSE[(b * p.H + h) * p.Nq + t] = (m_used + bq + __log2f(l)) * kLn2;
        if (r == 0) {
            bulk_wait_read0();  // smem must stay valid until the bulk stores have read it
            GFWA_TR(33);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

// dynamic smem: 1024 alignment slack + Q, K, V + barriers (2 CTAs per SM)
constexpr size_t kSmemBytes = 1024 + 3 * kTileBytes + kZeroBytes + sizeof(Bars) + 16;

}  // namespace

bool tc_fwd_supported(const AttnParams& p, gfwa_dtype_t dt) {
    if (dt != GFWA_BF16 || p.d != D) return false;
    if (p.Nkv >= ((int64_t)1 << 31) || p.H >= 65536 || p.B >= 65536) return false;
    if (const char* e = getenv("GFWA_FORCE_SIMT")) return e[0] == '0';
    return true;
}

gfwa_status_t tc_fwd(const AttnParams& p, cudaStream_t st) {
    CUtensorMap mq, mk, mv, mo, mo32, mzq;
    GFWA_REQUIRE(encode_bnhd_map(&mq, p.Q, p.B, p.Nq, p.H, D, p.qs, BM));
    if (p.zero_acc) {
        const int64_t acc_s[3] = {p.Nq * p.H * D, p.H * D, D};  // the backward's dQ accumulator layout
        GFWA_REQUIRE(encode_bnhd_map_f32(&mzq, p.zero_acc, p.B, p.Nq, p.H, D, acc_s, 64));
    } else {
        mzq = mq;  // unused
    }
    GFWA_REQUIRE(encode_bnhd_map(&mk, p.K, p.B, p.Nkv, p.H, D, p.ks, BN));
    GFWA_REQUIRE(encode_bnhd_map(&mv, p.V, p.B, p.Nkv, p.H, D, p.vs, BN));
    GFWA_REQUIRE(encode_bnhd_map(&mo, p.O, p.B, p.Nq, p.H, D, p.os, BM));
    if (p.O_f32)
        GFWA_REQUIRE(encode_bnhd_map_f32(&mo32, p.O_f32, p.B, p.Nq, p.H, D, p.os, BM));
    else
        mo32 = mo;  // unused
    TcFwdParams tp;
    tp.U = p.U;
    tp.LSE = p.LSE;
    tp.Nq = p.Nq;
    tp.Nkv = p.Nkv;
    tp.h0 = p.h0;
    tp.H = p.H;
    tp.w = p.w;
    tp.store_f32 = p.O_f32 != nullptr;
    tp.zero_acc = p.zero_acc;
    tp.token = p.token;
    tp.token_val = p.token_val;
    tp.sl2 = p.scale * kLog2e;
    // per launch: the attribute is per device (a process may drive several GPUs)
    auto kern = tp.store_f32 ? fwd_tc_kernel<true> : fwd_tc_kernel<false>;
    if (gfwa_status_t s = check_launch(
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes)))
        return s;
    dim3 grid((unsigned)((p.Nq + BM - 1) / BM), (unsigned)p.H, (unsigned)p.B);
    // diagnostics: GFWA_TRACE_FWD=<file> dumps per-CTA clock64 stamps (synchronous)
    const char* trace_file = getenv("GFWA_TRACE_FWD");
    const size_t n_cta = (size_t)grid.x * grid.y * grid.z;
    tp.trace = nullptr;
    if (trace_file) {
        cudaMalloc(&tp.trace, n_cta * 64 * sizeof(long long));
        cudaMemsetAsync(tp.trace, 0, n_cta * 64 * sizeof(long long), st);
    }
    kern<<<grid, kThreads, kSmemBytes, st>>>(mzq, mq, mk, mv, mo, mo32, tp);
    note_launch();
    if (trace_file) {
        std::vector<long long> hbuf(n_cta * 64);
        cudaStreamSynchronize(st);
        cudaMemcpy(hbuf.data(), tp.trace, hbuf.size() * sizeof(long long), cudaMemcpyDeviceToHost);
        cudaFree(tp.trace);
        if (FILE* f = fopen(trace_file, "wb")) {
            fwrite(hbuf.data(), sizeof(long long), hbuf.size(), f);
            fclose(f);
        }
    }
    return check_launch();
}

}  // namespace gfwa
