// attn_tc_bwd.cu -- GatedFWA backward on the 5th-generation tensor cores
// (sm_100a): Alg. E.2 with readings C-3, C-4, C-11, C-12.
//
// KV-major and persistent: one CTA per SM walks work items, each a 128-key
// tile of one (b, h) (K and V resident in smem) and the 64-query steps whose
// windows reach it.  The next item's K, V and first Q/dO stage
// are loaded into a rotating pool of shared-memory slots while the current
// item's last steps run, and its dK/dV epilogue overlaps the next item's
// first steps, so per-item prologue and epilogue latency is hidden.
// All five contractions run on tcgen05 with TMEM accumulators, pipelined
// across steps with two TMEM buffers (S^T/dP^T of step n are produced while
// the gradients of step n-1 are contracted):
//   S^T  = K Q^T          SS  M=128 keys, N=64 queries   -> buf[n&1] cols [0,64)
//   dP^T = V dO^T         SS                             -> buf[n&1] cols [64,128)
//   (softmax-grad, 2 warpgroups x 32 queries, thread = key: P^T = exp(S - L),
//    dS^T = P^T (dP^T - D); each warpgroup packs its P^T and dS^T back to TMEM
//    as bf16 over its own 32 S^T columns (P^T in the first 16, dS^T in the
//    next 16: no cross-warpgroup barrier), dS^T also to smem)
//   dQ^T = K^T dS^T       SS  M=128 (d), N=64             -> the freed [64,128)
//   dV  += P^T dO         TS  (A = P^T from TMEM)         -> TMEM [256,384)
//   dK  += dS^T Q         TS  (A = dS^T from TMEM)        -> TMEM [384,512)
// The dQ^T tile is drained by a third warpgroup (thread = head-dim lane) into
// an fp32 dQ accumulator with coalesced L2 reductions while the next step
// runs (the paper writes dQ back per tile).  du^k (column sum, C-4)
// accumulates per key thread; du^q (the paper's rowsum(dS), kept per
// C-11) is a cross-thread sum over keys done in fp32 with a warp butterfly
// transpose-reduce (after dS is handed to the MMA warp) and a cross-warp sum by
// the drain warpgroup, so both sums see the same fp32 dS and sum_m dU_m
// telescopes to zero.  dK, dV are read out of TMEM by the drain warpgroup
// (which then releases the accumulators) and stored as bf16 rows.
#include <type_traits>

#include "attn_common.cuh"
#include "sm100.cuh"
#include "tma_host.cuh"

namespace gfwa {
namespace {

using namespace sm100;

constexpr int BN = 128;   // keys per CTA
constexpr int BMQ = 64;   // queries per step
constexpr uint32_t kDQ = 32 * 128 * 4;    // 16 KB dQ staging: 4 warps x 2 x (16 queries x 32 d) fp32
constexpr uint32_t kDQW = 16 * 32 * 4;    // 2 KB: one drain warp's box
constexpr uint32_t kKVbox = 128 * 64 * 2;  // 16 KB: 128 key rows x 64 d (one 128-byte swizzle row)
constexpr uint32_t kQTbox = 64 * 64 * 2;   // 8 KB: 64 query rows x 64 d
// per head dim D in {64, 128}: the K slot is always 128 d wide (for D = 64 its
// second half is zeros, so K^T is the M = 128 A operand of dQ^T = K^T dS^T and
// dQ^T rows 64..127 come out zero); V, Q, dO tiles are D wide
template <int D>
struct BwdLay {
    static constexpr uint32_t kV = 128 * D * 2;
    static constexpr uint32_t kQT = 64 * D * 2;      // Q or dO tile
};
constexpr uint32_t kDS = 128 * 64 * 2;    // 16 KB dS^T tile
// bias folding (reading C-25): the per-query terms of the exponent and of dP - D enter
// the S^T and dP^T accumulators through one extra K = 16 slab each.  A side: one 1 KB
// 128B-swizzle atom whose 8 rows are identical (read with SBO = 0 for all 128 key rows);
// slab 0 = ones at k 0..2 (S^T), slab 1 = ones at k 3..5 (dP^T).  B side: per step g,
// slab g % 4 of a 64-row atom column holds [c'_hi, c'_mid, c'_lo, -D_hi, -D_mid, -D_lo, 0...]
// per query, c' = ((u_q - uref) - L_q) / scale split into three bf16 (24 bits), so that
// sl2 (S^T + c') = scale log2e q.k + (u_q - uref - L_q) log2e and dP^T + (-D) = dP - D.
constexpr uint32_t kAugA = 1024, kAugB = 64 * 128;
#ifndef GFWA_BWD_SWG
#define GFWA_BWD_SWG 2
#endif
constexpr int kSWG = GFWA_BWD_SWG;        // softmax-grad warpgroups, each owning QPW queries of a step
constexpr int QPW = 64 / kSWG;
constexpr int kDrainWarp0 = 4 * kSWG, kMmaWarp = kDrainWarp0 + 4, kTmaWarp = kMmaWarp + 1;
constexpr int kThreads = 32 * (kTmaWarp + 1);  // softmax-grad WGs, drain WG, MMA warp, TMA warp
#ifndef GFWA_BWD_NODQ
#define GFWA_BWD_NODQ 0  // experiment only: skip the dQ reductions
#endif
#ifndef GFWA_PRE_U
#define GFWA_PRE_U 4  // row groups in flight per warp in the backward's preprocess (2: 165, 4: 158 us at C2)
#endif
#ifndef GFWA_BWD_DQRED
#define GFWA_BWD_DQRED 0  // 1: dQ^T drained by per-query red.global.add instead of TMA bulk reductions
#endif
#ifndef GFWA_BWD_SFIRST
#define GFWA_BWD_SFIRST 1  // issue S^T(g) before waiting for the drain of dQ^T(g-2) (only dP^T(g) needs it)
#endif
#ifndef GFWA_BWD_NODUQ
#define GFWA_BWD_NODUQ 0  // experiment only: skip the du^q butterfly (wrong dU)
#endif
#ifndef GFWA_BWD_EXPT
#define GFWA_BWD_EXPT 0  // experiment only (wrong results): 1 no grad MMAs, 2 no S/dP MMAs, 3 ex2 -> fmul, 5 no softmax math,

#endif

struct TcBwdParams {
    const float* U;
    const float* LSE;
    const float* Dv;
    float* dQacc;  // [B, Nq, H, d] fp32, zeroed by the preprocess kernel (or gfwa_fwd_train)
    float* dU;     // [B, H, Nkv] fp32, zeroed before the launch
    __nv_bfloat16* dK;
    __nv_bfloat16* dV;
    int64_t ks[3], vs[3];  // dK / dV element strides over (b, n, h) (those of K / V)
    int64_t Nq, Nkv, h0, H, Hkv;
    int w;
    int G;              // query heads per K/V head (GQA; 1 = MHA)
    int n_kt, n_items;  // key tiles per (b, K/V head); work items = key tiles x Hkv x B
    int64_t B;
    // sequence sharding: fp32 copies of dK, dV for the first head_rows
    // and the last tail_rows key rows, [2 (dK, dV)][B][rows][Hkv][d] (null: none)
    float* f32_head;
    float* f32_tail;
    int64_t head_rows, tail_rows;
    float sl2, scale, inv_scale;
    unsigned long long* token;  // prepared-workspace token: consumed (cleared) by this kernel
    int hrows;                  // in-kernel halo: key tiles below hrows come from the halo maps
};

#ifndef GFWA_BWD_TRACE
#define GFWA_BWD_TRACE 0  // diagnostics build only: clock64 stamps per role into a device array
#endif
#if GFWA_BWD_TRACE
constexpr int kBTr = 512;  // stamps per (CTA, role), first 148 CTAs
__device__ long long g_bwd_trace[148 * 12 * kBTr];
#define BTR(role, k)                                                                        \
    do {                                                                                    \
        if ((k) < kBTr && blockIdx.x < 148) g_bwd_trace[(blockIdx.x * 12 + (role)) * kBTr + (k)] = clock64(); \
    } while (0)
#else
#define BTR(role, k) \
    do {             \
    } while (0)
#endif

// Shared-memory slot pool: five 32 KB slots hold the current item's K and V and
// the three Q/dO stages of its steps.  At an item boundary the roles rotate so
// the NEXT item's K, V and first Q/dO stage are loaded while the current item's
// last steps still run (its K is the last slot released, after the final
// gradient MMAs; V is released once the last dP^T MMA has read it):
//   K' = q[n % 3] (freed by step n-3), V' = V, q0' = q[(n+1) % 3] (step n-2),
//   q1' = q[(n+2) % 3] (step n-1), q2' = K
// Every role that touches the pool replays the same rotation, so no slot index
// is ever communicated.
constexpr int kPool = 5;
constexpr uint32_t kSlot = 32768;
struct Pool {
    uint32_t s = 0u | (1u << 3) | (2u << 6) | (3u << 9) | (4u << 12);  // K, V, q0, q1, q2 (3 bits each)
    __device__ __forceinline__ uint32_t f(int i) const { return (s >> (3 * i)) & 7u; }
    __device__ __forceinline__ uint32_t K() const { return f(0); }
    __device__ __forceinline__ uint32_t V() const { return f(1); }
    __device__ __forceinline__ uint32_t Q(int m) const { return f(2 + m % 3); }
    __device__ __forceinline__ void advance(int n) {
        const uint32_t k = K(), v = V(), a = Q(n), b = Q(n + 1), c = Q(n + 2);
        s = a | (v << 3) | (b << 6) | (c << 9) | (k << 12);
    }
};

struct __align__(8) Bars {
    uint64_t full[kPool], empty[kPool], aug_empty[4];
    uint64_t st_full[2], ds_ready[2], dq_full[2], dq_drained[2], red_ready[2], red_free[2];
    uint64_t dkdv_full, dkdv_free;
};

__device__ __forceinline__ void red_add(float* addr, float a) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(addr), "f"(a) : "memory");
}

__device__ __forceinline__ uint32_t range_bits(int lo, int hi, int base) {
    const int a = min(max(lo - base, 0), 32), z = min(max(hi - base + 1, 0), 32);
    const uint32_t upto_z = z >= 32 ? 0xffffffffu : ((1u << z) - 1u);
    const uint32_t below_a = a >= 32 ? 0xffffffffu : ((1u << a) - 1u);
    return upto_z & ~below_a;
}

// One work item: a 128-key tile of one (b, K/V head h) and the 64-query steps whose
// windows reach it (Alg. E.2 l.12-14), for each of the G query heads
// h G + gi reading that K/V head (GQA): tot = G nsteps steps, head-major, all
// accumulating into the same dK / dV
struct BItem {
    int b, h, j0, qt_lo, nsteps, tot;
};
__device__ __forceinline__ BItem make_bitem(const TcBwdParams& p, int idx) {
    BItem it;
    const int jt = idx % p.n_kt, bh = idx / p.n_kt;
    it.h = bh % (int)p.Hkv;
    it.b = bh / (int)p.Hkv;
    it.j0 = jt * BN;
    const int64_t j_last = min64((int64_t)it.j0 + BN, p.Nkv) - 1;
    const int64_t t_lo = max64(0, (int64_t)it.j0 - p.h0);
    const int64_t t_hi = min64(p.Nq - 1, j_last + p.w - 1 - p.h0);
    it.qt_lo = (int)(t_lo / BMQ);
    it.nsteps = t_lo <= t_hi ? (int)(t_hi / BMQ - it.qt_lo + 1) : 0;
    it.tot = it.nsteps * p.G;
    return it;
}

// Persistent: one CTA per SM walks work items idx = blockIdx.x + k * gridDim.x.
// kRows: also write the fp32 copies of the boundary rows' dK, dV (sequence sharding)
template <int D, bool kRows>
__global__ void __launch_bounds__(kThreads, 1)
    bwd_tc_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                  const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mdo,
                  const __grid_constant__ CUtensorMap mdk, const __grid_constant__ CUtensorMap mdv,
                  const __grid_constant__ CUtensorMap mdq, const __grid_constant__ CUtensorMap mkh,
                  const __grid_constant__ CUtensorMap mvh, const TcBwdParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    constexpr uint32_t kKV = BwdLay<D>::kV, kQT = BwdLay<D>::kQT;
    constexpr int kHalves = D / 64;      // 64-column TMA boxes per row
    uint8_t* pool_base = smem;           // kPool slots of kSlot bytes
    uint8_t* dSs = pool_base + kPool * kSlot;  // 2 x dS^T tile
    uint8_t* dQs = dSs + 2 * kDS;        // dQ staging: per drain warp 2 x [16 queries][32 d] fp32, 128B swizzle
    uint8_t* augA = dQs + kDQ;           // 1 KB, see kAugA
    uint8_t* augB = augA + kAugA;        // 8 KB: 64 query rows x 4 slabs (slab a = step g % 4)
    Bars* bars = (Bars*)(augB + kAugB);
    uint32_t* tmem_sh = (uint32_t*)(bars + 1);
    __shared__ float s_red[2][kSWG][4][QPW];          // [parity][wg][warp][query] du^q partials

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kPool; ++s) {
            mbar_init(&bars->full[s], 2);  // TMA bytes + the producer's own arrive (after its generic writes)
            mbar_init(&bars->empty[s], 1);
        }
        for (int a = 0; a < 4; ++a) mbar_init(&bars->aug_empty[a], 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->st_full[i], 1);
            mbar_init(&bars->ds_ready[i], 4 * kSWG);
            mbar_init(&bars->dq_full[i], 1);
            mbar_init(&bars->dq_drained[i], 4);
            mbar_init(&bars->red_ready[i], 4 * kSWG);
            mbar_init(&bars->red_free[i], 2);
        }
        mbar_init(&bars->dkdv_full, 1);
        mbar_init(&bars->dkdv_free, 4);
        fence_barrier_init();
    }
    {  // bias-folding slabs: B zero except the per-step chunk the producer writes; A constant
        for (uint32_t i = threadIdx.x; i < kAugB / 16; i += kThreads)
            sts128(smem_u32(augB) + i * 16, make_uint4(0u, 0u, 0u, 0u));
        if (threadIdx.x < 64) {  // A atom: row r = tid / 8, 16-B chunk c = tid % 8 (physical)
            const uint32_t r = threadIdx.x >> 3, c = threadIdx.x & 7, logical = c ^ r;
            const uint32_t one = 0x3F80u;  // bf16 1.0
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (logical == 0) v = make_uint4(one | (one << 16), one, 0u, 0u);                  // k 0..2
            if (logical == 2) v = make_uint4(0u, one << 16, one | (one << 16), 0u);            // k 16+3..16+5
            sts128(smem_u32(augA) + r * 128 + c * 16, v);
        }
    }
    fence_proxy_async();
    if (warp == kMmaWarp) {
        tmem_alloc(tmem_sh, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_sh;
    // the pre kernel has read the token (stream order): clear it, so the next backward
    // on this workspace zeroes its accumulator unless a new gfwa_fwd_train prepares it
    if (p.token && threadIdx.x == 0 && blockIdx.x == 0) *p.token = 0ull;

    if (warp == kTmaWarp) {
        // ------------------------------------------------ producer: TMA + per-step vectors
        Pool pool;
        uint32_t acq = 0;  // bit s: parity of the acquisitions of slot s so far
        auto acquire = [&](uint32_t s) {
            mbar_wait(&bars->empty[s], ((acq >> s) & 1u) ^ 1u);
            acq ^= 1u << s;
        };
        int g = 0;
        for (int idx = blockIdx.x; idx < p.n_items; idx += gridDim.x) {
            const BItem it = make_bitem(p, idx);
            if (it.nsteps == 0) continue;
            // K and V of the item
#pragma unroll 1
            for (int kv = 0; kv < 2; ++kv) {
                const uint32_t s = kv ? pool.V() : pool.K();
                acquire(s);
                uint8_t* dst = pool_base + s * kSlot;
                if (D < 128 && kv == 0) {  // K^T rows d >= D of the dQ^T MMA (M = 128): zeros
                    for (uint32_t i = lane; i < kKVbox / 16; i += 32)
                        sts128(smem_u32(dst + kKVbox) + i * 16, make_uint4(0u, 0u, 0u, 0u));
                    fence_proxy_async();
                }
                __syncwarp();
                if (elect_one()) {
                    mbar_expect_tx(&bars->full[s], kKV);
                    // in-kernel halo: key tiles below hrows from the halo's own (e.g. peer) memory
                    const bool hz = it.j0 < p.hrows;
                    const CUtensorMap* km = kv ? (hz ? &mvh : &mv) : (hz ? &mkh : &mk);
                    for (int half = 0; half < kHalves; ++half)
                        tma_load_4d(dst + half * kKVbox, km, &bars->full[s], half * 64, it.h,
                                    hz ? it.j0 : it.j0 - p.hrows, it.b);
                    mbar_arrive(&bars->full[s]);
                }
                __syncwarp();
            }
            // the per-query vectors of step f + 1 are loaded while step f's stage is
            // refilled (software pipelined: their global-load latency stays off the full barrier).
            // Step f = gi nsteps + m: query head h G + gi, query tile qt_lo + m
            float vu[2], vl[2], vd[2], vref = 0.f;
            auto fetch = [&](int f) {
                const int gi = f / it.nsteps, m = f - gi * it.nsteps;
                const int64_t bh = (int64_t)it.b * p.H + (int64_t)it.h * p.G + gi;
                const float* Ubh = p.U + bh * p.Nkv;
                if (f < it.tot) vref = Ubh[it.j0];  // per-(item, query head) bias reference (reading C-18)
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int64_t t = (int64_t)(it.qt_lo + m) * BMQ + lane + 32 * i;
                    const bool ok = f < it.tot && t < p.Nq;
                    const int64_t vi = bh * p.Nq + t;
                    vu[i] = ok ? Ubh[t + p.h0] : 0.f;
                    vl[i] = ok ? p.LSE[vi] : 0.f;
                    vd[i] = ok ? p.Dv[vi] : 0.f;
                }
            };
            fetch(0);
            for (int f = 0; f < it.tot; ++f, ++g) {
                const uint32_t s = pool.Q(f);
                const int gi = f / it.nsteps, m = f - gi * it.nsteps;
                const int hq = it.h * p.G + gi;
                const int t0 = (it.qt_lo + m) * BMQ;
                const float uref = vref;
                acquire(s);
                if (lane == 0) BTR(3, g);
                if (elect_one()) {
                    mbar_expect_tx(&bars->full[s], 2 * kQT);
                    uint8_t* qd = pool_base + s * kSlot;
                    for (int half = 0; half < kHalves; ++half) {
                        tma_load_4d(qd + half * kQTbox, &mq, &bars->full[s], half * 64, hq, t0, it.b);
                        tma_load_4d(qd + kQT + half * kQTbox, &mdo, &bars->full[s], half * 64, hq, t0, it.b);
                    }
                }
                // the bias slab of step g (slab g % 4, free once step g - 4's S^T/dP^T MMAs ran)
                const int a = g & 3;
                mbar_wait(&bars->aug_empty[a], ((g >> 2) & 1) ^ 1);
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int q = lane + 32 * i;
                    const bool ok = (int64_t)t0 + q < p.Nq;
                    const float c = ok ? ((vu[i] - uref) - vl[i]) * p.inv_scale : 0.f;
                    const float dv = ok ? -vd[i] : 0.f;
                    uint32_t ch, cm, cl, dh, dm, dl;
                    split3_bf16(c, ch, cm, cl);
                    split3_bf16(dv, dh, dm, dl);
                    // k 0..7 of the slab: [c_hi, c_mid, c_lo, -D_hi, -D_mid, -D_lo, 0, 0]
                    const uint4 v = make_uint4(ch | (cm << 16), cl | (dh << 16), dm | (dl << 16), 0u);
                    sts128(smem_u32(augB) + (q >> 3) * 1024 + (q & 7) * 128 + (((2 * a) ^ (q & 7)) * 16), v);
                }
                fence_proxy_async();  // generic-proxy writes -> the tensor core's async proxy
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->full[s]);
                fetch(f + 1);
            }
            pool.advance(it.tot);
        }
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------ MMA issuer
        const uint32_t id_st = idesc_bf16(128, BMQ, false, false);  // S^T, dP^T
        const uint32_t id_tm = idesc_bf16(128, D, false, true);     // dV, dK (A in TMEM, B MN-major)
        const uint32_t id_dq = idesc_bf16(128, BMQ, true, true);    // dQ^T (A, B MN-major)
        const uint32_t pb = smem_u32(pool_base);
        Pool pool;
        uint32_t fpar = 0;  // bit s: parity of the next fill of slot s to consume
        auto wait_full = [&](uint32_t s) {
            mbar_wait(&bars->full[s], (fpar >> s) & 1u);
            fpar ^= 1u << s;
        };
        // the previous step, whose gradient MMAs are issued after this step's S^T / dP^T
        int pg = -1, pm = 0, pn = 0, pitem = 0;
        uint32_t ps = 0, pk = 0;
        auto mma2 = [&]() {
            const int bm = pg & 1;
            mbar_wait(&bars->ds_ready[bm], (pg >> 1) & 1);
            // the item's first gradient MMAs overwrite dV / dK: the epilogue must have read the last item's
            if (pm == 0 && pitem > 0) mbar_wait(&bars->dkdv_free, (pitem - 1) & 1);
            if (lane == 0) BTR(5, pg);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t buf = tmem + 128 * bm;
                const uint32_t qb = pb + ps * kSlot, ob = qb + kQT, kb = pb + pk * kSlot;
                const uint32_t sb = smem_u32(dSs + bm * kDS);
                // dQ^T = K^T dS^T, one N = 64 chain into the freed columns [64,128)
#pragma unroll
                for (int kk = 0; kk < BN / 16 && GFWA_BWD_EXPT != 1; ++kk)
                    mma_ss(buf + 64, sdesc_sw128(kb + kk * 2048, kKVbox, 1024),
                           sdesc_sw128(sb + kk * 2048, 8192, 1024), id_dq, kk > 0 ? 1u : 0u);
                tc_commit(&bars->dq_full[bm]);
                // dV += P^T dO ; dK += dS^T Q   (P^T and dS^T of queries [32 g, 32 g + 32) in
                // columns [32 g, 32 g + 16) and [32 g + 16, 32 g + 32); 16 queries = 8 columns per K step)
#pragma unroll
                for (int kk = 0; kk < BMQ / 16 && GFWA_BWD_EXPT != 1; ++kk) {
                    const uint32_t acc = (pm > 0 || kk > 0) ? 1u : 0u;
                    // queries [16 kk, 16 kk + 16): warpgroup kk / 2's columns, half kk % 2
                    const uint32_t pc = QPW * ((16 * kk) / QPW) + 8 * (kk % (QPW / 16));
                    mma_ts(tmem + 256, buf + pc, sdesc_sw128(ob + kk * 2048, kQTbox, 1024), id_tm, acc);
                    mma_ts(tmem + 384, buf + pc + QPW / 2, sdesc_sw128(qb + kk * 2048, kQTbox, 1024), id_tm, acc);
                }
                tc_commit(&bars->empty[ps]);  // Q/dO stage free
                if (pm == pn - 1) {
                    tc_commit(&bars->dkdv_full);
                    tc_commit(&bars->empty[pk]);  // K free (its last reader was dQ^T)
                }
            }
            __syncwarp();
        };
        int g = 0, nitem = 0;
        for (int idx = blockIdx.x; idx < p.n_items; idx += gridDim.x) {
            const BItem it = make_bitem(p, idx);
            if (it.nsteps == 0) continue;
            const uint32_t sK = pool.K(), sV = pool.V();
            for (int m = 0; m < it.tot; ++m, ++g) {  // m: flat step (query head major)
                const uint32_t s = pool.Q(m);
                const int bn = g & 1;
                if (m == 0) {
                    wait_full(sK);
                    wait_full(sV);
                }
                wait_full(s);
#if GFWA_BWD_SFIRST
                // S^T(g) writes columns [0,64) of buffer g&1 (P^T / dS^T of step g-2, read by
                // gradient MMAs already issued ahead of it); only dP^T(g), in [64,128), needs
                // dQ^T(g-2) drained -- so S^T(g) runs on the tensor core during the drain
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t qb = pb + s * kSlot;
                    const uint32_t kb = pb + sK * kSlot;
                    const uint32_t buf = tmem + 128 * bn;
#pragma unroll
                    for (int kk = 0; kk < D / 16 && GFWA_BWD_EXPT != 2; ++kk) {
                        const uint32_t ka = (kk >> 2) * kKVbox + (kk & 3) * 32;
                        const uint32_t qa = (kk >> 2) * kQTbox + (kk & 3) * 32;
                        mma_ss(buf, sdesc_sw128(kb + ka, 16, 1024), sdesc_sw128(qb + qa, 16, 1024), id_st, kk > 0);
                    }
                    const uint64_t bslab = sdesc_sw128(smem_u32(augB) + 32 * (g & 3), 16, 1024);
                    mma_ss(buf, sdesc_sw128(smem_u32(augA), 16, 0), bslab, id_st, 1u);
                }
                __syncwarp();
                if (g >= 2) mbar_wait(&bars->dq_drained[bn], ((g - 2) >> 1) & 1);
                tc_fence_after();
                if (lane == 0) BTR(1, g);
                if (elect_one()) {
                    const uint32_t qb = pb + s * kSlot, ob = qb + kQT;
                    const uint32_t vb = pb + sV * kSlot;
                    const uint32_t buf = tmem + 128 * bn;
#pragma unroll
                    for (int kk = 0; kk < D / 16 && GFWA_BWD_EXPT != 2; ++kk) {
                        const uint32_t ka = (kk >> 2) * kKVbox + (kk & 3) * 32;
                        const uint32_t qa = (kk >> 2) * kQTbox + (kk & 3) * 32;
                        mma_ss(buf + 64, sdesc_sw128(vb + ka, 16, 1024), sdesc_sw128(ob + qa, 16, 1024), id_st, kk > 0);
                    }
                    const uint64_t bslab = sdesc_sw128(smem_u32(augB) + 32 * (g & 3), 16, 1024);
                    mma_ss(buf + 64, sdesc_sw128(smem_u32(augA) + 32, 16, 0), bslab, id_st, 1u);
                    tc_commit(&bars->st_full[bn]);
                    tc_commit(&bars->aug_empty[g & 3]);
                    if (m == it.tot - 1) tc_commit(&bars->empty[sV]);  // V's last reader was this dP^T
                }
                __syncwarp();
#else
                if (g >= 2) mbar_wait(&bars->dq_drained[bn], ((g - 2) >> 1) & 1);
                tc_fence_after();
                if (lane == 0) BTR(1, g);
                if (elect_one()) {
                    const uint32_t qb = pb + s * kSlot, ob = qb + kQT;
                    const uint32_t kb = pb + sK * kSlot, vb = pb + sV * kSlot;
                    const uint32_t buf = tmem + 128 * bn;
#pragma unroll
                    for (int kk = 0; kk < D / 16 && GFWA_BWD_EXPT != 2; ++kk) {
                        const uint32_t ka = (kk >> 2) * kKVbox + (kk & 3) * 32;
                        const uint32_t qa = (kk >> 2) * kQTbox + (kk & 3) * 32;
                        mma_ss(buf, sdesc_sw128(kb + ka, 16, 1024), sdesc_sw128(qb + qa, 16, 1024), id_st, kk > 0);
                        mma_ss(buf + 64, sdesc_sw128(vb + ka, 16, 1024), sdesc_sw128(ob + qa, 16, 1024), id_st, kk > 0);
                    }
                    // + the per-query bias slabs (C-25): A rows repeat (SBO = 0), B = step g's slab
                    const uint64_t bslab = sdesc_sw128(smem_u32(augB) + 32 * (g & 3), 16, 1024);
                    mma_ss(buf, sdesc_sw128(smem_u32(augA), 16, 0), bslab, id_st, 1u);
                    mma_ss(buf + 64, sdesc_sw128(smem_u32(augA) + 32, 16, 0), bslab, id_st, 1u);
                    tc_commit(&bars->st_full[bn]);
                    tc_commit(&bars->aug_empty[g & 3]);
                    if (m == it.tot - 1) tc_commit(&bars->empty[sV]);  // V's last reader was this dP^T
                }
                __syncwarp();
#endif
                if (pg >= 0) mma2();
                pg = g;
                pm = m;
                pn = it.tot;
                ps = s;
                pk = sK;
                pitem = nitem;
            }
            pool.advance(it.tot);
            ++nitem;
        }
        if (pg >= 0) mma2();
    } else if (warp < kDrainWarp0) {
        // ------------------------------------------------ softmax-grad: thread = key, QPW queries per WG
        const int wg = warp >> 2;  // query columns [QPW wg, QPW wg + QPW) of each step
        const int kr = threadIdx.x & 127;
        const uint64_t sl2x2 = f2pack(p.sl2, p.sl2);
        const uint32_t lane_addr = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        int g = 0;
        for (int idx = blockIdx.x; idx < p.n_items; idx += gridDim.x) {
            const BItem it = make_bitem(p, idx);
            if (it.nsteps == 0) continue;
            const int64_t j0 = it.j0, j = j0 + kr;
            const bool kvalid = j < p.Nkv;
#pragma unroll 1
            for (int gi = 0; gi < p.G; ++gi) {  // query heads of this K/V head (GQA)
            const int64_t bhq = (int64_t)it.b * p.H + (int64_t)it.h * p.G + gi;
            const float* Ubh = p.U + bhq * p.Nkv;
            const float uref = Ubh[j0];
            const float nuk = kvalid ? -(Ubh[j] - uref) * kLog2e : 0.f;
            const uint64_t nuk2 = f2pack(nuk, nuk);
            uint64_t colsum2 = 0;  // packed (0.f, 0.f)
            for (int m = 0; m < it.nsteps; ++m, ++g) {
                const int bn = g & 1;
                const int64_t t0 = (int64_t)(it.qt_lo + m) * BMQ;
                mbar_wait(&bars->st_full[bn], (g >> 1) & 1);
                if (threadIdx.x == 0) BTR(0, g);
                if (threadIdx.x == 128) BTR(9, g);
                tc_fence_after();
                const uint32_t scol = 128 * bn + QPW * wg;  // this WG's S^T columns (dP^T at +64)
                // keys in (g - w, g] of each query g = t + h0, as a column range
                const bool interior = (j0 + BN - 1 <= t0 + p.h0) && (j0 > t0 + BMQ - 1 + p.h0 - p.w) &&
                                      (t0 + BMQ <= p.Nq) && (j0 + BN <= p.Nkv);
                uint32_t keep = ~0u;
                if (!interior) {
                    const int64_t qlo = j - p.h0 - t0, qhi = min64(j - p.h0 - t0 + p.w - 1, p.Nq - 1 - t0);
                    keep = kvalid ? range_bits((int)max64(qlo, -1), (int)min64(qhi, (int64_t)BMQ), QPW * wg) : 0u;
                }
                float ds[QPW];
                uint32_t pk[QPW / 2], dk[QPW / 2];
                uint32_t sall[QPW], dall[QPW];  // both TMEM loads in flight before one wait
                if constexpr (QPW == 32) {
                    tmem_ld32(lane_addr + scol, *reinterpret_cast<uint32_t(*)[32]>(sall));
                    tmem_ld32(lane_addr + scol + 64, *reinterpret_cast<uint32_t(*)[32]>(dall));
                } else {
                    tmem_ld16(lane_addr + scol, *reinterpret_cast<uint32_t(*)[16]>(sall));
                    tmem_ld16(lane_addr + scol + 64, *reinterpret_cast<uint32_t(*)[16]>(dall));
                }
                tmem_wait_ld();
                // each warpgroup packs its P^T, dS^T over its own S^T columns (no
                // cross-warpgroup barrier); dQ^T then gets [64,128) whole.  Two copies of
                // the loop: interior steps (every (key, query) pair in the window) carry no
                // per-element mask instructions at all
                auto calc = [&](auto masked_tag) {
                    constexpr bool kMasked = decltype(masked_tag)::value;
#pragma unroll
                    for (int h16 = 0; h16 < QPW; h16 += 16) {
                        const uint32_t* s16 = sall + h16;
                        const uint32_t* d16 = dall + h16;
#pragma unroll
                        for (int a = 0; a < 16; a += 2) {
                            const int e2 = h16 + a;
                            // P = exp(scale q.k + (u_q - u_k) - L_q), log2 units: the
                            // per-query part is already in S^T (C-25), the per-key part is nuk
                            const uint64_t x = ffma2(f2pack(__uint_as_float(s16[a]), __uint_as_float(s16[a + 1])),
                                                     sl2x2, nuk2);
                            float x0, x1;
                            f2unpack(x, x0, x1);
                            if constexpr (kMasked) {
                                x0 = ((keep >> e2) & 1u) ? x0 : -INFINITY;
                                x1 = ((keep >> (e2 + 1)) & 1u) ? x1 : -INFINITY;
                            }
                            const uint64_t pr = GFWA_BWD_EXPT == 3 ? fmul2(f2pack(x0, x1), sl2x2)
                                                                   : f2pack(ex2(x0), ex2(x1));
                            // dS = P (dP - D); dP^T already holds dP - D (C-25)
                            const uint64_t dsv =
                                fmul2(pr, f2pack(__uint_as_float(d16[a]), __uint_as_float(d16[a + 1])));
                            colsum2 = fadd2(colsum2, dsv);  // du^k, fp32 (C-4)
                            float p0, p1;
                            f2unpack(pr, p0, p1);
                            f2unpack(dsv, ds[e2], ds[e2 + 1]);
                            pk[e2 / 2] = pack_bf16x2(p0, p1);
                            dk[e2 / 2] = pack_bf16x2(ds[e2], ds[e2 + 1]);
                        }
                    }
                };
                if (GFWA_BWD_EXPT == 5) {
#pragma unroll
                    for (int e = 0; e < QPW; ++e) ds[e] = __uint_as_float(sall[e] ^ dall[e]);
#pragma unroll
                    for (int e = 0; e < QPW / 2; ++e) pk[e] = dk[e] = sall[e];
                } else if (interior) {
                    calc(std::false_type{});
                } else {
                    calc(std::true_type{});
                }
                // P^T -> columns [QPW wg, QPW wg + QPW/2), dS^T -> [QPW wg + QPW/2, QPW wg + QPW)
                if constexpr (QPW == 32) {
                    tmem_st16(lane_addr + 128 * bn + QPW * wg, *reinterpret_cast<const uint32_t(*)[16]>(pk));
                    tmem_st16(lane_addr + 128 * bn + QPW * wg + QPW / 2, *reinterpret_cast<const uint32_t(*)[16]>(dk));
                } else {
                    tmem_st8(lane_addr + 128 * bn + QPW * wg, *reinterpret_cast<const uint32_t(*)[8]>(pk));
                    tmem_st8(lane_addr + 128 * bn + QPW * wg + QPW / 2, *reinterpret_cast<const uint32_t(*)[8]>(dk));
                }
                {  // dS^T row -> smem (128B-swizzled MN-major: row = key, 16-B chunk of 8 queries ^ key%8)
                    const uint32_t sb = smem_u32(dSs + bn * kDS) + kr * 128;
#pragma unroll
                    for (int c = 0; c < QPW / 8; ++c)
                        sts128(sb + ((((QPW / 8) * wg + c) ^ (kr & 7)) * 16),
                               make_uint4(dk[4 * c], dk[4 * c + 1], dk[4 * c + 2], dk[4 * c + 3]));
                }
                tmem_wait_st();
                fence_proxy_async();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->ds_ready[bn]);
                if (threadIdx.x == 0) BTR(6, g);
                if (threadIdx.x == 128) BTR(8, g);
                if (threadIdx.x == 96) BTR(10, g);
                if (threadIdx.x == 224) BTR(11, g);
                // du^q partial over this warp's 32 keys, off the MMA's critical path (the
                // gradient contractions of step g are already running): butterfly
                // transpose-reduce -> lane l holds query QPW wg + l; the drain warpgroup
                // sums the 4 warps' partials and issues the red.add (C-11)
#pragma unroll
                for (int sft = QPW / 2; sft >= 1 && !GFWA_BWD_NODUQ && GFWA_BWD_EXPT != 5; sft >>= 1) {
                    const bool up = lane & sft;
#pragma unroll
                    for (int e = 0; e < sft; ++e) {
                        const float send = up ? ds[e] : ds[e + sft];
                        const float keepv = up ? ds[e + sft] : ds[e];
                        ds[e] = keepv + __shfl_xor_sync(0xffffffffu, send, sft);
                    }
                }
                if (g >= 2) mbar_wait(&bars->red_free[bn], ((g - 2) >> 1) & 1);
                if (QPW < 32) ds[0] += __shfl_xor_sync(0xffffffffu, ds[0], QPW);  // lane halves hold the same query
                if (lane < QPW) s_red[bn][wg][warp & 3][lane] = ds[0];
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->red_ready[bn]);
            }
            float c0, c1;
            f2unpack(colsum2, c0, c1);
            if (kvalid) red_add(p.dU + bhq * p.Nkv + j, -(c0 + c1));  // du^k (C-4)
            }
        }
    } else if (warp < kMmaWarp) {
        // ------------------------------------------------ dQ drain + dK/dV epilogue: thread = TMEM lane
        // dQ^T (TMEM, lane = d) -> smem [16 queries][32 d] fp32 boxes (128B swizzle) ->
        // TMA bulk reduce-add into the fp32 dQ accumulator: the L2 does the adds, no
        // per-thread atomics.  Each drain warp stages its own 32 d (double-buffered
        // 2 KB boxes) and issues its own reduces, so no cross-warp barrier.  After an
        // item's last step the same threads (now lane = key) move dV, dK out of TMEM
        // (releasing it for the next item's first gradient MMAs) and store them.
        const int dl = threadIdx.x - 32 * kDrainWarp0;  // 0..127
        const uint32_t lane_addr = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        const uint32_t qcol[4] = {64, 80, 96, 112};  // dQ^T: columns [64,128) of the buffer
        uint8_t* wbox = dQs + (warp & 3) * 2 * kDQW;
        // du^q_t += rowsum(dS) at key position t + h0 (C-11): the 4 per-warp
        // partials of each softmax-grad warpgroup (threads dl < 64, one query each)
        auto combine_duq = [&](int mm, int64_t t0, int64_t bh) {
            if (dl < BMQ) {
                const int bq = mm & 1;
                mbar_wait(&bars->red_ready[bq], (mm >> 1) & 1);
                const int wq = dl / QPW, lq = dl % QPW;
                const float rs =
                    s_red[bq][wq][0][lq] + s_red[bq][wq][1][lq] + s_red[bq][wq][2][lq] + s_red[bq][wq][3][lq];
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->red_free[bq]);
                const int64_t t = t0 + dl;
                if (t < p.Nq) red_add(p.dU + bh * p.Nkv + t + p.h0, rs);
            }
        };
        // dV (mul 1) and dK (mul scale, C-3) rows of key j -> global, bf16
        auto store_row = [&](__nv_bfloat16* base, const uint32_t (&v)[32], int c0, float mul) {
            uint4* dst = reinterpret_cast<uint4*>(base + c0);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint4 o;
                o.x = pack_bf16x2(__uint_as_float(v[8 * k + 0]) * mul, __uint_as_float(v[8 * k + 1]) * mul);
                o.y = pack_bf16x2(__uint_as_float(v[8 * k + 2]) * mul, __uint_as_float(v[8 * k + 3]) * mul);
                o.z = pack_bf16x2(__uint_as_float(v[8 * k + 4]) * mul, __uint_as_float(v[8 * k + 5]) * mul);
                o.w = pack_bf16x2(__uint_as_float(v[8 * k + 6]) * mul, __uint_as_float(v[8 * k + 7]) * mul);
                dst[k] = o;
            }
        };
        // key j's row in the fp32 head / tail copy (the epilogue's tsr 0 is dV, 1 is dK; the
        // buffers hold [dK, dV]), or null when j is outside that range
        auto f32_row = [&](const BItem& it, int64_t j, int tsr, bool tail = false) -> float* {
            float* base = tail ? p.f32_tail : p.f32_head;
            const int64_t rows = tail ? p.tail_rows : p.head_rows;
            const int64_t r = tail ? j - (p.Nkv - p.tail_rows) : j;
            if (!base || r < 0 || r >= rows || j >= p.Nkv) return nullptr;
            const int64_t which = tsr ? 0 : 1;  // dK first, then dV
            return base + (((which * p.B + it.b) * rows + r) * p.Hkv + it.h) * D;
        };
        int g = 0, nitem = 0, pg = -1;
        int64_t pt0 = 0, pbh = 0;
        for (int idx = blockIdx.x; idx < p.n_items; idx += gridDim.x) {
            const BItem it = make_bitem(p, idx);
            const int64_t j = (int64_t)it.j0 + dl;
            __nv_bfloat16* dvrow = p.dV + (int64_t)it.b * p.vs[0] + j * p.vs[1] + (int64_t)it.h * p.vs[2];
            __nv_bfloat16* dkrow = p.dK + (int64_t)it.b * p.ks[0] + j * p.ks[1] + (int64_t)it.h * p.ks[2];
            if (it.nsteps == 0) {  // no query reaches these keys: dK = dV = 0
                if (j < p.Nkv) {
                    uint32_t z[32];
#pragma unroll
                    for (int e = 0; e < 32; ++e) z[e] = 0u;
#pragma unroll
                    for (int c = 0; c < D; c += 32) {
                        store_row(dvrow, z, c, 1.f);
                        store_row(dkrow, z, c, 1.f);
                    }
#pragma unroll 1
                    for (int tsr = 0; tsr < 2 && kRows; ++tsr)
                        for (int c = 0; c < D; c += 4) {
                            if (float* f = f32_row(it, j, tsr)) *reinterpret_cast<float4*>(f + c) = make_float4(0.f, 0.f, 0.f, 0.f);
                            if (float* f = f32_row(it, j, tsr, true)) *reinterpret_cast<float4*>(f + c) = make_float4(0.f, 0.f, 0.f, 0.f);
                        }
                }
                continue;
            }
#pragma unroll 1
            for (int gi = 0; gi < p.G; ++gi) {  // query heads of this K/V head (GQA)
            const int hq = it.h * p.G + gi;
            const int64_t bh = (int64_t)it.b * p.H + hq;
            for (int m = 0; m < it.nsteps; ++m, ++g) {
                const int bm = g & 1;
                const int64_t t0 = (int64_t)(it.qt_lo + m) * BMQ;
                mbar_wait(&bars->dq_full[bm], (g >> 1) & 1);
                if (dl == 0) BTR(2, g);
                tc_fence_after();
                const bool dlive = 32 * (warp & 3) < D;  // D = 64: dQ^T lanes 64..127 are the zero padding
                uint32_t v[4][16];
                if (dlive) {
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) tmem_ld16(lane_addr + 128 * bm + qcol[qq], v[qq]);
                    tmem_wait_ld();
                }
                // all 64 queries are in registers: release the TMEM buffer first
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->dq_drained[bm]);
                if (dl == 0) BTR(7, g);
                if (pg >= 0) combine_duq(pg, pt0, pbh);  // the previous step's partials are in smem by now
                if (GFWA_BWD_DQRED) {
                    // per query one coalesced 128-byte L2 reduction (lane = d): no staging
                    if (dlive && !GFWA_BWD_NODQ) {
                        float* acc = p.dQacc + (((int64_t)it.b * p.Nq + t0) * p.H + hq) * D + 32 * (warp & 3) + lane;
                        const int64_t qstride = p.H * D;
                        const int nq = (int)min64(BMQ, p.Nq - t0);
#pragma unroll
                        for (int r = 0; r < 4; ++r)
#pragma unroll
                            for (int e = 0; e < 16; ++e)
                                if (16 * r + e < nq) red_add(acc + (16 * r + e) * qstride, __uint_as_float(v[r][e]));
                    }
                } else {
                    // four rounds of 16 queries; row = query (128 B = this warp's 32 d),
                    // 16-B chunk (d%32)/4 ^ (query%8), word d%4
    #pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        if (!dlive) break;
                        if (lane == 0) bulk_wait_read1();  // the reduce two rounds back has read this box
                        __syncwarp();
                        const uint32_t sq = smem_u32(wbox + (r & 1) * kDQW);
    #pragma unroll
                        for (int e = 0; e < 16; ++e)
                            sts32(sq + e * 128 + ((((lane >> 2) ^ e) & 7) << 4) + (lane & 3) * 4, __uint_as_float(v[r][e]));
                        fence_proxy_async();
                        __syncwarp();
                        if (lane == 0 && !GFWA_BWD_NODQ) {
                            tma_reduce_add_4d(&mdq, wbox + (r & 1) * kDQW, 32 * (warp & 3), hq, (int)(t0 + 16 * r),
                                              it.b);
                            bulk_commit();
                        }
                    }
                }
                pg = g;
                pt0 = t0;
                pbh = bh;
            }
            }
            // epilogue of the item: dV, dK (TMEM lane = key) -> bf16 [32 keys][64 d] boxes,
            // staged one at a time in this warp's 4 KB of the dQ staging and written by TMA
            // stores (the item's K slot is released by the MMA warp right away, so the next
            // item's Q/dO loads do not wait for the epilogue)
            mbar_wait(&bars->dkdv_full, nitem & 1);
            if (dl == 0) BTR(4, nitem);
            tc_fence_after();
            const uint32_t stg = smem_u32(wbox);
#pragma unroll 1
            for (int tsr = 0; tsr < 2; ++tsr) {  // 0: dV (TMEM [256, 384)), 1: dK ([384, 512), times scale)
                const float mul = tsr ? p.scale : 1.f;
#pragma unroll 1
                for (int hf = 0; hf < kHalves; ++hf) {
                    uint32_t a[32], b[32];
                    tmem_ld32(lane_addr + 256 + 128 * tsr + 64 * hf, a);
                    tmem_ld32(lane_addr + 256 + 128 * tsr + 64 * hf + 32, b);
                    tmem_wait_ld();
                    if (tsr == 1 && hf == kHalves - 1) {  // every dV, dK column has been read: TMEM free
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&bars->dkdv_free);
                    }
                    if (kRows) {  // the boundary rows' fp32 copies (sequence sharding)
#pragma unroll 1
                        for (int ht = 0; ht < 2; ++ht)
                            if (float* f = f32_row(it, j, tsr, ht == 1)) {
                                f += 64 * hf;
#pragma unroll
                                for (int e = 0; e < 32; e += 4) {
                                    *reinterpret_cast<float4*>(f + e) =
                                        make_float4(__uint_as_float(a[e]) * mul, __uint_as_float(a[e + 1]) * mul,
                                                    __uint_as_float(a[e + 2]) * mul, __uint_as_float(a[e + 3]) * mul);
                                    *reinterpret_cast<float4*>(f + 32 + e) =
                                        make_float4(__uint_as_float(b[e]) * mul, __uint_as_float(b[e + 1]) * mul,
                                                    __uint_as_float(b[e + 2]) * mul, __uint_as_float(b[e + 3]) * mul);
                                }
                            }
                    }
                    if (lane == 0) bulk_wait_read0();  // earlier stores / reductions have read the staging
                    __syncwarp();
                    const uint32_t row = stg + lane * 128;  // 128B swizzle: chunk ^ (key % 8)
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint32_t* v = k < 4 ? a + 8 * k : b + 8 * (k - 4);
                        uint4 o;
                        o.x = pack_bf16x2(__uint_as_float(v[0]) * mul, __uint_as_float(v[1]) * mul);
                        o.y = pack_bf16x2(__uint_as_float(v[2]) * mul, __uint_as_float(v[3]) * mul);
                        o.z = pack_bf16x2(__uint_as_float(v[4]) * mul, __uint_as_float(v[5]) * mul);
                        o.w = pack_bf16x2(__uint_as_float(v[6]) * mul, __uint_as_float(v[7]) * mul);
                        sts128(row + ((k ^ (lane & 7)) << 4), o);
                    }
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_4d(tsr ? &mdk : &mdv, wbox, hf * 64, it.h, it.j0 + 32 * (warp & 3), it.b);
                        bulk_commit();
                    }
                }
            }
            if (lane == 0) bulk_wait_read0();  // the next step's dQ rounds reuse the staging
            __syncwarp();
            ++nitem;
        }
        if (pg >= 0) combine_duq(pg, pt0, pbh);
        if (lane == 0) bulk_wait0();  // reductions complete before the CTA exits
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <int D>
constexpr size_t smem_bytes() {
    return 1024 + kPool * kSlot + 2 * kDS + kDQ + kAugA + kAugB + sizeof(Bars) + 16;
}

// dQacc zeroing fused with D = rowsum(O dO)  (Alg. E.2 l.7; O + O_lo, C-12)
template <int D>
__global__ void __launch_bounds__(256) bwd_tc_pre_kernel(AttnParams p) {
    const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const int64_t total = p.B * p.Nq * p.H;
    if (row >= total) return;
    const int64_t h = row % p.H, t = (row / p.H) % p.Nq, b = row / (p.H * p.Nq);
    const int64_t oo = b * p.os[0] + t * p.os[1] + h * p.os[2];
    const __nv_bfloat16* dO = (const __nv_bfloat16*)p.dO + oo;
    float acc = 0.f;
    const int c = lane * 4;  // 4 elements per lane: lanes [0, D/4)
    const bool act = lane < D / 4;
    if (act) {
    const uint2 g2 = *reinterpret_cast<const uint2*>(dO + c);
    const float2 g01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&g2.x));
    const float2 g23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&g2.y));
    const uint2 o2 = *reinterpret_cast<const uint2*>((const __nv_bfloat16*)p.O + oo + c);
    float2 o01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&o2.x));
    float2 o23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&o2.y));
    if (p.Olo) {
        const uint2 l2 = *reinterpret_cast<const uint2*>((const __nv_bfloat16*)p.Olo + oo + c);
        const float2 l01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&l2.x));
        const float2 l23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&l2.y));
        o01.x += l01.x;
        o01.y += l01.y;
        o23.x += l23.x;
        o23.y += l23.y;
    }
    acc = o01.x * g01.x + o01.y * g01.y + o23.x * g23.x + o23.y * g23.y;
    }
    acc = warp_sum(acc);
    if (lane == 0) p.Dv[(b * p.H + h) * p.Nq + t] = acc;
    if (act && !(p.token && *p.token == p.token_val))  // not already zeroed by gfwa_fwd_train
        *reinterpret_cast<float4*>(p.dQacc + ((b * p.Nq + t) * p.H + h) * D + c) = make_float4(0.f, 0.f, 0.f, 0.f);
}

// D = rowsum((O + O_lo) dO) and zeroing of dQacc, fast path for contiguous O, O_lo, dO:
// each warp takes R rows per iteration (32 / (D / 8) lanes per row, 16-byte loads, all
// 3R loads in flight before any use), grid-stride, 32-bit index math; the zeroing as
// flat 16-byte stores
template <int D>
__global__ void __launch_bounds__(256) bwd_tc_pre_flat_kernel(const __nv_bfloat16* __restrict__ o,
                                                             const __nv_bfloat16* __restrict__ olo,
                                                             const __nv_bfloat16* __restrict__ dO,
                                                             float* __restrict__ Dv, float* __restrict__ acc,
                                                             uint32_t rows, uint32_t H, uint32_t Nq,
                                                             float* __restrict__ dU, uint32_t n_du,
                                                             const unsigned long long* __restrict__ token,
                                                             unsigned long long token_val) {
    constexpr int LPR = D / 8;           // lanes per row (8 bf16 = 16 B each)
    constexpr int RPW = 32 / LPR;        // rows per warp load
    constexpr int U = GFWA_PRE_U;        // loads unrolled: U * RPW rows per iteration
    const uint32_t lane = threadIdx.x & 31, sub = lane / LPR, cl = lane % LPR;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    // gfwa_fwd_train already zeroed the accumulator (its token is in the workspace)
    const bool zero = !(token && *token == token_val);
    // dU accumulates red.adds in the main kernel: zero it here (no separate memset launch)
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_du; i += gridDim.x * blockDim.x) dU[i] = 0.f;
    auto dot8 = [](uint4 a, uint4 l, uint4 g) {
        const uint32_t* av = &a.x;
        const uint32_t* lv = &l.x;
        const uint32_t* gv = &g.x;
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float2 fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(av + k));
            const float2 fl = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(lv + k));
            const float2 fg = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(gv + k));
            s = fmaf(fa.x + fl.x, fg.x, s);
            s = fmaf(fa.y + fl.y, fg.y, s);
        }
        return s;
    };
    for (uint32_t r0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * (U * RPW); r0 < rows; r0 += nw * U * RPW) {
        uint4 va[U], vl[U], vg[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t row = r0 + u * RPW + sub;
            ok[u] = row < rows;
            const size_t e = (size_t)(ok[u] ? row : 0) * D + cl * 8;
            va[u] = __ldcs(reinterpret_cast<const uint4*>(o + e));
            vl[u] = __ldcs(reinterpret_cast<const uint4*>(olo + e));
            vg[u] = __ldcs(reinterpret_cast<const uint4*>(dO + e));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            float a = dot8(va[u], vl[u], vg[u]);
#pragma unroll
            for (int m = LPR / 2; m >= 1; m >>= 1) a += __shfl_xor_sync(0xffffffffu, a, m);
            const uint32_t row = r0 + u * RPW + sub;
            if (ok[u]) {
                if (cl == 0) {
                    const uint32_t hh = row % H, bt = row / H, t = bt % Nq, b = bt / Nq;
                    Dv[((size_t)b * H + hh) * Nq + t] = a;
                }
                if (zero) {
                    float4* z = reinterpret_cast<float4*>(acc + (size_t)row * D) + 2 * cl;
                    z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
                    z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
        }
    }
}

// AttnLayer epilogue backward fused with the preprocess (reading C-27): per
// (b, t, h) row, from Y's gradient dY, the gate pre-activation g, gamma and the
// forward's rstd r (O~ = O + O_lo, the fp32 attention output):
//   dn = dY swish(g);  dg = dY n swish'(g) (n = gamma O~ r);  dgamma += dn O~ r
//   dO~ = r gamma dn - (r^3 O~ / d) sum_c gamma_c dn_c O~_c   -> bf16 (the dP MMA operand)
//   D = rowsum(O~ * bf16(dO~))   (C-12; the same dO values the main kernel contracts)
// plus the zeroing of dU (and of the dQ accumulator unless gfwa_fwd_train prepared it).
// Flat [rows, D] layouts; a warp takes 32 / (D / 8) rows per iteration (8 channels per
// lane); dgamma is reduced per block in smem, then one atomic per channel per block.
template <int D>
__global__ void __launch_bounds__(256) bwd_tc_pre_normgate_kernel(
    const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ olo, const __nv_bfloat16* __restrict__ g,
    const __nv_bfloat16* __restrict__ dY, const float* __restrict__ gamma, const float* __restrict__ rstd,
    __nv_bfloat16* __restrict__ dO, __nv_bfloat16* __restrict__ dg, float* __restrict__ dgamma,
    float* __restrict__ Dv, float* __restrict__ acc, uint32_t rows, uint32_t H, uint32_t Nq, float* __restrict__ dU,
    uint32_t n_du, const unsigned long long* __restrict__ token, unsigned long long token_val) {
    constexpr int LPR = D / 8, RPW = 32 / LPR;
    __shared__ float s_dg[8][D];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, sub = lane / LPR, cl = lane % LPR;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const bool zero = !(token && *token == token_val);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_du; i += gridDim.x * blockDim.x) dU[i] = 0.f;
    float gam[8], dga[8];
    {
        const float4 a = __ldg(reinterpret_cast<const float4*>(gamma + 8 * cl));
        const float4 b = __ldg(reinterpret_cast<const float4*>(gamma + 8 * cl) + 1);
        gam[0] = a.x; gam[1] = a.y; gam[2] = a.z; gam[3] = a.w;
        gam[4] = b.x; gam[5] = b.y; gam[6] = b.z; gam[7] = b.w;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) dga[c] = 0.f;
    auto unpack8 = [](uint4 v, float (&f)[8]) {
        const uint32_t* w = &v.x;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float2 t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(w + k));
            f[2 * k] = t.x;
            f[2 * k + 1] = t.y;
        }
    };
    for (uint32_t r0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * RPW; r0 < rows; r0 += nw * RPW) {
        const uint32_t row = r0 + sub;
        const bool ok = row < rows;
        const size_t e = (size_t)(ok ? row : 0) * D + cl * 8;
        const uint32_t hh = (ok ? row : 0) % H, bt = (ok ? row : 0) / H, t = bt % Nq, b = bt / Nq;
        const size_t vi = ((size_t)b * H + hh) * Nq + t;
        float ov[8], gv[8], yv[8], dn[8];
        unpack8(__ldcs(reinterpret_cast<const uint4*>(o + e)), ov);
        if (olo) {
            float lv[8];
            unpack8(__ldcs(reinterpret_cast<const uint4*>(olo + e)), lv);
#pragma unroll
            for (int c = 0; c < 8; ++c) ov[c] += lv[c];
        }
        unpack8(__ldcs(reinterpret_cast<const uint4*>(g + e)), gv);
        unpack8(__ldcs(reinterpret_cast<const uint4*>(dY + e)), yv);
        if (!ok)  // a dummy load of row 0: contributes nothing to dgamma
#pragma unroll
            for (int c = 0; c < 8; ++c) yv[c] = 0.f;
        const float r = __ldg(rstd + vi);
        float s1 = 0.f;
        uint32_t dgw[4];
#pragma unroll
        for (int c = 0; c < 8; c += 2) {
            float dgc[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const float sg = 1.f / (1.f + __expf(-gv[c + q]));
                const float G = gv[c + q] * sg;
                dn[c + q] = yv[c + q] * G;
                const float n = gam[c + q] * ov[c + q] * r;
                dgc[q] = yv[c + q] * n * (sg + G * (1.f - sg));
                dga[c + q] = fmaf(dn[c + q] * ov[c + q], r, dga[c + q]);
                s1 = fmaf(gam[c + q] * dn[c + q], ov[c + q], s1);
            }
            dgw[c / 2] = pack_bf16x2(dgc[0], dgc[1]);
        }
#pragma unroll
        for (int m = LPR / 2; m >= 1; m >>= 1) s1 += __shfl_xor_sync(0xffffffffu, s1, m);
        const float k3 = r * r * r * s1 * (1.f / D);
        uint32_t dow[4];
        float dsum = 0.f;
#pragma unroll
        for (int c = 0; c < 8; c += 2) {
            const float d0 = r * gam[c] * dn[c] - k3 * ov[c];
            const float d1 = r * gam[c + 1] * dn[c + 1] - k3 * ov[c + 1];
            dow[c / 2] = pack_bf16x2(d0, d1);
            const float2 rb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&dow[c / 2]));
            dsum = fmaf(ov[c], rb.x, fmaf(ov[c + 1], rb.y, dsum));
        }
#pragma unroll
        for (int m = LPR / 2; m >= 1; m >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, m);
        if (ok) {
            *reinterpret_cast<uint4*>(dO + e) = make_uint4(dow[0], dow[1], dow[2], dow[3]);
            *reinterpret_cast<uint4*>(dg + e) = make_uint4(dgw[0], dgw[1], dgw[2], dgw[3]);
            if (cl == 0) Dv[vi] = dsum;
            if (zero) {
                float4* z = reinterpret_cast<float4*>(acc + (size_t)row * D) + 2 * cl;
                z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
                z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    }
    // dgamma: the warp's sub-rows (lanes with the same cl), then the block, then global
#pragma unroll
    for (int c = 0; c < 8; ++c)
        for (int m = LPR; m < 32; m <<= 1) dga[c] += __shfl_xor_sync(0xffffffffu, dga[c], m);
    if (sub == 0)
#pragma unroll
        for (int c = 0; c < 8; ++c) s_dg[warp][8 * cl + c] = dga[c];
    __syncthreads();
    for (int c = threadIdx.x; c < D; c += blockDim.x) {
        float v = 0.f;
#pragma unroll
        for (int w8 = 0; w8 < 8; ++w8) v += s_dg[w8][c];
        atomicAdd(dgamma + c, v);
    }
}

// dQ = scale * dQacc -> bf16 (C-3), flat fast path for a contiguous dQ: 8 elements
// per thread (32-byte loads, 16-byte stores), grid-stride, no index division
__global__ void __launch_bounds__(256) bwd_tc_post_flat_kernel(const float* __restrict__ acc,
                                                              __nv_bfloat16* __restrict__ dq, int64_t n8, float scale) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 a = __ldcs(reinterpret_cast<const float4*>(acc) + 2 * i);
        const float4 c = __ldcs(reinterpret_cast<const float4*>(acc) + 2 * i + 1);
        uint4 o;
        o.x = pack_bf16x2(a.x * scale, a.y * scale);
        o.y = pack_bf16x2(a.z * scale, a.w * scale);
        o.z = pack_bf16x2(c.x * scale, c.y * scale);
        o.w = pack_bf16x2(c.z * scale, c.w * scale);
        reinterpret_cast<uint4*>(dq)[i] = o;
    }
}

// dQ = scale * dQacc -> bf16 (C-3), general strides
template <int D>
__global__ void __launch_bounds__(256) bwd_tc_post_kernel(AttnParams p) {
    const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const int64_t total = p.B * p.Nq * p.H;
    if (row >= total) return;
    const int64_t h = row % p.H, t = (row / p.H) % p.Nq, b = row / (p.H * p.Nq);
    const int c = lane * 4;
    if (lane >= D / 4) return;
    const float4 a = *reinterpret_cast<const float4*>(p.dQacc + ((b * p.Nq + t) * p.H + h) * D + c);
    uint2 o;
    o.x = pack_bf16x2(a.x * p.scale, a.y * p.scale);
    o.y = pack_bf16x2(a.z * p.scale, a.w * p.scale);
    *reinterpret_cast<uint2*>((__nv_bfloat16*)p.dQ + b * p.qs[0] + t * p.qs[1] + h * p.qs[2] + c) = o;
}

}  // namespace

bool tc_bwd_supported(const AttnParams& p, gfwa_dtype_t dt) {
    if (dt != GFWA_BF16 || (p.d != 64 && p.d != 128)) return false;
    if (p.Nkv >= ((int64_t)1 << 31) || p.H >= 65536 || p.B >= 65536) return false;
    if (const char* e = getenv("GFWA_FORCE_SIMT")) return e[0] == '0';
    return true;
}

size_t tc_bwd_workspace(const AttnParams& p) { return (size_t)p.B * p.Nq * p.H * p.d * sizeof(float); }

template <int D>
static gfwa_status_t tc_bwd_d(const AttnParams& pin, cudaStream_t st, void* ws) {
    AttnParams p = pin;
    p.dQacc = (float*)ws;
    CUtensorMap mq, mk, mv, mdo, mdk, mdv, mdq;
    GFWA_REQUIRE(encode_bnhd_map(&mq, p.Q, p.B, p.Nq, p.H, D, p.qs, BMQ));
    // K / V hold key rows [hrows, Nkv); rows [0, hrows) come from the halo maps (in-kernel halo)
    GFWA_REQUIRE(encode_bnhd_map(&mk, p.K, p.B, p.Nkv - p.hrows, p.Hkv, D, p.ks, BN));
    GFWA_REQUIRE(encode_bnhd_map(&mv, p.V, p.B, p.Nkv - p.hrows, p.Hkv, D, p.vs, BN));
    CUtensorMap mkh = mk, mvh = mv;
    if (p.hrows) {
        GFWA_REQUIRE(encode_bnhd_map(&mkh, p.Kh, p.B, p.hrows, p.Hkv, D, p.khs, BN));
        GFWA_REQUIRE(encode_bnhd_map(&mvh, p.Vh, p.B, p.hrows, p.Hkv, D, p.vhs, BN));
    }
    GFWA_REQUIRE(encode_bnhd_map(&mdo, p.dO, p.B, p.Nq, p.H, D, p.os, BMQ));
    GFWA_REQUIRE(encode_bnhd_map(&mdk, p.dK, p.B, p.Nkv, p.Hkv, D, p.ks, BN / 4));  // [32 keys][64 d] store boxes
    GFWA_REQUIRE(encode_bnhd_map(&mdv, p.dV, p.B, p.Nkv, p.Hkv, D, p.vs, BN / 4));
    const int64_t acc_s[3] = {p.Nq * p.H * D, p.H * D, D};  // dQacc [B, Nq, H, d] fp32
    GFWA_REQUIRE(encode_bnhd_map_f32(&mdq, p.dQacc, p.B, p.Nq, p.H, D, acc_s, 16));
    const int64_t rows = p.B * p.Nq * p.H;
    const unsigned rgrid = (unsigned)((rows + 7) / 8);
    int n_sm = 148, dev = 0;  // per call: the attribute is per device
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t n_du = p.B * p.H * p.Nkv;
    const bool o_flat = p.Olo && p.os[2] == D && p.os[1] == p.H * D && p.os[0] == p.Nq * p.H * D &&
                        rows < ((int64_t)1 << 31) && n_du < ((int64_t)1 << 31);
    if (p.ng_dY) {  // AttnLayer epilogue backward fused with the preprocess (C-27); layouts checked by the caller
        if (gfwa_status_t s = check_launch(cudaMemsetAsync(p.ng_dgamma, 0, D * sizeof(float), st))) return s;
        bwd_tc_pre_normgate_kernel<D><<<(unsigned)min64((rows + 8 * 256 / D - 1) / (8 * 256 / D), (int64_t)n_sm * 8), 256,
                                        0, st>>>(
            (const __nv_bfloat16*)p.O, (const __nv_bfloat16*)p.Olo, (const __nv_bfloat16*)p.ng_g,
            (const __nv_bfloat16*)p.ng_dY, p.ng_gamma, p.ng_rstd, (__nv_bfloat16*)p.dO, (__nv_bfloat16*)p.ng_dg,
            p.ng_dgamma, p.Dv, p.dQacc, (uint32_t)rows, (uint32_t)p.H, (uint32_t)p.Nq, p.dU, (uint32_t)n_du, p.token,
            p.token_val);
    } else if (o_flat) {
        bwd_tc_pre_flat_kernel<D><<<(unsigned)min64((rows + 8 * 256 * GFWA_PRE_U / D - 1) / (8 * 256 * GFWA_PRE_U / D), (int64_t)n_sm * 8), 256, 0, st>>>(
            (const __nv_bfloat16*)p.O, (const __nv_bfloat16*)p.Olo, (const __nv_bfloat16*)p.dO, p.Dv, p.dQacc, (uint32_t)rows, (uint32_t)p.H, (uint32_t)p.Nq, p.dU,
            (uint32_t)n_du, p.token, p.token_val);
    } else {
        if (gfwa_status_t s = check_launch(cudaMemsetAsync(p.dU, 0, (size_t)n_du * sizeof(float), st))) return s;
        bwd_tc_pre_kernel<D><<<rgrid, 256, 0, st>>>(p);
    }
    note_launch();
    if (gfwa_status_t s = check_launch()) return s;
    stage_event(0, st);  // measurement hook: after the preprocess kernel
    TcBwdParams tp;
    tp.U = p.U;
    tp.LSE = p.LSE;
    tp.Dv = p.Dv;
    tp.dQacc = p.dQacc;
    tp.dU = p.dU;
    tp.Nq = p.Nq;
    tp.Nkv = p.Nkv;
    tp.h0 = p.h0;
    tp.H = p.H;
    tp.Hkv = p.Hkv;
    tp.G = (int)(p.H / p.Hkv);
    tp.w = p.w;
    tp.sl2 = p.scale * kLog2e;
    tp.scale = p.scale;
    tp.inv_scale = 1.f / p.scale;
    tp.token = p.token;
    tp.hrows = (int)p.hrows;
    tp.dK = (__nv_bfloat16*)p.dK;
    tp.dV = (__nv_bfloat16*)p.dV;
    for (int i = 0; i < 3; ++i) {
        tp.ks[i] = p.ks[i];
        tp.vs[i] = p.vs[i];
    }
    tp.n_kt = (int)((p.Nkv + BN - 1) / BN);
    tp.B = p.B;
    tp.f32_head = p.f32_head;
    tp.f32_tail = p.f32_tail;
    tp.head_rows = p.f32_head_rows;
    tp.tail_rows = p.f32_tail_rows;
    const int64_t n_items = (int64_t)tp.n_kt * p.Hkv * p.B;
    if (n_items >= ((int64_t)1 << 31)) return GFWA_ERR_INVALID_ARGUMENT;
    tp.n_items = (int)n_items;
    // per launch: the attribute is per device (a process may drive several GPUs)
    constexpr size_t kSmemBytes = smem_bytes<D>();
    if (gfwa_status_t s = check_launch(
            cudaFuncSetAttribute(bwd_tc_kernel<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes)))
        return s;
    if (gfwa_status_t s = check_launch(
            cudaFuncSetAttribute(bwd_tc_kernel<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes)))
        return s;
    int64_t cap = n_sm;  // persistent: one CTA per SM
    if (const char* e = getenv("GFWA_BWD_GRID")) cap = max64(1, atoll(e));  // diagnostics: fewer CTAs, more items each
    const unsigned grid = (unsigned)min64(n_items, cap);
    auto kern = (tp.f32_head || tp.f32_tail) ? bwd_tc_kernel<D, true> : bwd_tc_kernel<D, false>;
    kern<<<grid, kThreads, kSmemBytes, st>>>(mq, mk, mv, mdo, mdk, mdv, mdq, mkh, mvh, tp);
    note_launch();
    if (gfwa_status_t s = check_launch()) return s;
    stage_event(1, st);  // measurement hook: after the main kernel
    const bool dq_flat = p.qs[2] == D && p.qs[1] == p.H * D && p.qs[0] == p.Nq * p.H * D;
    if (dq_flat) {
        const int64_t n8 = rows * D / 8;
        const unsigned g = (unsigned)min64((n8 + 255) / 256, (int64_t)n_sm * 8);
        bwd_tc_post_flat_kernel<<<g, 256, 0, st>>>(p.dQacc, (__nv_bfloat16*)p.dQ, n8, p.scale);
    } else {
        bwd_tc_post_kernel<D><<<rgrid, 256, 0, st>>>(p);
    }
    note_launch();
    return check_launch();
}

#if GFWA_BWD_TRACE
extern "C" int gfwa_debug_bwd_trace(long long* host, size_t n) {
    if (n > sizeof(g_bwd_trace) / sizeof(long long)) n = sizeof(g_bwd_trace) / sizeof(long long);
    return (int)cudaMemcpyFromSymbol(host, g_bwd_trace, n * sizeof(long long));
}
#endif

gfwa_status_t tc_bwd(const AttnParams& p, cudaStream_t st, void* ws) {
    return p.d == 64 ? tc_bwd_d<64>(p, st, ws) : tc_bwd_d<128>(p, st, ws);
}

}  // namespace gfwa
