// attn_tc_fwd.cu -- GatedFWA forward on the 5th-generation tensor cores
// (sm_100a): Alg. 2 re-designed for tcgen05/TMEM/TMA.
//
// Persistent, warp-specialised, one CTA per SM.  A work item is a PAIR of
// 128-row query tiles (A = rows [r0, r0+128), B = [r0+128, r0+256)) of one
// (b, h); both share every 128-key K/V tile of their (overlapping) windows, so
// each K/V tile is staged once per 256 query rows.  The key tiles of the item
// are walked diagonal-first (descending j); the first one only feeds B (its
// diagonal), the last only A (its window edge).
//
//   warp 21     TMA producer: Q_A, Q_B per item (a slot is refilled as soon as
//               the tile's last S MMA has read it), K_j and V_j through one ring
//               of three tile slots (evict-last: re-read by ~w/128 neighbouring
//               items);
//   warp 20     MMA issuer (one elected lane), ping-pong over the two tiles:
//                 O_A += P_A V_{n-1};  S_A = Q_A K_n^T;
//                 O_B += P_B V_{n-1};  S_B = Q_B K_n^T
//               (P lives over its S columns, so a tile's next S is issued after
//               its PV; while the tensor core runs one tile's pair the other
//               tile's softmax runs)
//   warps 0-7   softmax of tile A, warps 8-15 of tile B: two warpgroups per
//               tile, each owning one 64-column half of every S row (one thread
//               per row and half; the row max is exchanged through smem per key
//               tile, the row sum per item), two passes over TMEM, the
//               gate bias as an outer difference of two u vectors (P:377-380,
//               nothing N x w is materialised), window masks only on diagonal /
//               edge tiles with fully masked 32-key chunks skipped
//               (no exponentials), online softmax in fp32 with a lazy rescale
//               (the reference max moves only when it grows by > 2^8; the rare
//               rescale of O runs in TMEM by the row's own thread), 16-bit P
//               written back over the S columns.  LSE = m + ln l.
//   warps 16-19 epilogue: O / l -> bf16 O (staged per 64-column half) and, in
//               the training forward, its bf16 residual O_lo = bf16(O/l - O)
//               (staged in a 32 KB buffer; O + O_lo carries O to ~2^-17, which
//               is what the backward's D = rowsum(O dO) needs, reading C-12),
//               written by TMA stores; gfwa_fwd_train: it also zeroes the tile's
//               rows of the backward's dQ accumulator (coalesced 512-byte rows)
//   warps 22-23 training forward: the in-place fp16 conversion of every V tile
//               (reading C-23: P and V in fp16 for the PV product, so the fp32 O
//               that D = rowsum(O dO) is taken from carries 8x less P rounding
//               than with bf16 P)
// TMEM (512 columns): S_A [0,128), S_B [128,256), O_A [256,384), O_B [384,512).
// Key tiles outside every row's window are never loaded.
#include "attn_common.cuh"
#include "sm100.cuh"
#include "tma_host.cuh"

#ifndef GFWA_FWD_POLY
#define GFWA_FWD_POLY 0
#endif
#ifndef GFWA_FWD_LD16
#define GFWA_FWD_LD16 1  // softmax passes in 16-column chunks with the next TMEM load in flight
#endif
#ifndef GFWA_FWD_TRACE
#define GFWA_FWD_TRACE 0  // diagnostics build only: clock64 stamps per role into a device array
#endif

namespace gfwa {
namespace {

using namespace sm100;

constexpr int BM = 128;  // query rows per tile (two tiles per item)
constexpr int BN = 128;  // keys per tile
constexpr uint32_t kBox = BM * 64 * 2;  // one 16 KB TMA box: 128 rows x 64 bf16 (one 128-byte swizzle row)
// six warpgroups, 80 registers each (the CTA register file): softmax A (two
// warpgroups, one per 64-column half of the S row), softmax B (two), epilogue,
// {MMA, TMA, 2 V-convert warps}
// 512 x 128 = 64K): softmax A, softmax B, epilogue, {MMA, TMA, 2 V-convert warps}
constexpr int kThreads = 768;
constexpr int kEpiWarp0 = 16, kMmaWarp = 20, kTmaWarp = 21, kCvtWarp0 = 22;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr int kPolyPairs = GFWA_FWD_POLY;  // of every 4 column pairs, how many use exp2_poly2

// dynamic shared memory (1024-aligned base), per head dim D in {64, 128}
template <int D>
struct Lay {
    static constexpr uint32_t kTile = BM * D * 2;           // one bf16 Q/K/V/O tile
    static constexpr uint32_t kOffQ = 0;                    // Q_A, Q_B
    static constexpr uint32_t kOffKV = 2 * kTile;           // one K/V ring of 3 tile slots: K_0 V_0 K_1 V_1 ...
    static constexpr uint32_t kOffE = 5 * kTile;            // 32 KB: a 64-column box of O, then of O_lo
    // gate-bias slabs (reading C-26): B side one 128-key x 128 B swizzle region whose 32-B
    // column s holds ring slot s's per-key slab; A side one 1 KB atom of identical rows
    static constexpr uint32_t kOffSlabK = kOffE + 2 * kBox;  // 16 KB
    static constexpr uint32_t kOffSlabA = kOffSlabK + BN * 128;  // 1 KB
    static constexpr uint32_t kOffLinv = kOffSlabA + 1024;    // [2 tiles][128] 1/l
    static constexpr uint32_t kOffXch = kOffLinv + 2 * BM * 4;  // [2 tiles][2 parities][2 halves][128] row maxes
    static constexpr uint32_t kOffXchL = kOffXch + 8 * BM * 4;  // [2 tiles][128] half 1's row sum
    static constexpr uint32_t kOffBars = kOffXchL + 2 * BM * 4;
    static constexpr size_t kSmemBytes = kOffBars + 256;
};
constexpr int kSlots = 3;

struct __align__(8) Bars {
    uint64_t q_full[2], q_empty[2];
    // a slot alternates K and V fills: each kind completes its own barrier, so a
    // consumer of one kind never sees a phase of the other (parity aliasing)
    uint64_t k_full[kSlots], v_full[kSlots], kv_empty[kSlots], v_ready[kSlots];
    uint64_t s_full[2], p_ready[2], o_full[2], o_free[2], l_ready[2], l_free[2];
    uint32_t tmem;
};
static_assert(sizeof(Bars) <= 256, "barrier block");

struct TcFwdParams {
    const float* U;
    float* LSE;
    int64_t Nq, Nkv, h0, H, B;
    int w;
    int G;  // query heads per K/V head (GQA; 1 = MHA)
    int store_lo;
    int n_items, n_pairs;
    float* zero_acc;  // gfwa_fwd_train: the dQ accumulator [B, Nq, H, d] whose item rows are zeroed
    unsigned long long* token;
    unsigned long long token_val;
    float sl2;  // scale * log2(e)
    float inv_scale;
    // AttnLayer epilogue (reading C-27), active when ng_g is set
    const __nv_bfloat16* ng_g;
    __nv_bfloat16* ng_Y;
    const float* ng_gamma;
    float* ng_rstd;
    float ng_eps;
    int64_t os[3];  // O's (= g's, Y's) element strides over (b, n, h)
    int hrows;      // in-kernel halo: key tiles below hrows come from the halo maps
};

#if GFWA_FWD_TRACE
constexpr int kTrMax = 1024;  // stamps per (CTA, role)
__device__ long long g_fwd_trace[148 * 8 * kTrMax];
#define FTR(role, k)                                                                          \
    do {                                                                                      \
        if ((k) < kTrMax && blockIdx.x < 148)                                                 \
            g_fwd_trace[((int)blockIdx.x * 8 + (role)) * kTrMax + (k)] = clock64();          \
    } while (0)
#else
#define FTR(role, k) \
    do {             \
    } while (0)
#endif

// bits [lo, hi] (inclusive, clipped to the 32-bit word starting at column base)
__device__ __forceinline__ uint32_t range_bits(int lo, int hi, int base) {
    const int a = min(max(lo - base, 0), 32), z = min(max(hi - base + 1, 0), 32);
    const uint32_t upto_z = z >= 32 ? 0xffffffffu : ((1u << z) - 1u);
    const uint32_t below_a = a >= 32 ? 0xffffffffu : ((1u << a) - 1u);
    return upto_z & ~below_a;
}

// The geometry of one work item: rows of tiles A and B, their key-tile ranges
// (Alg. 2 l.7-9 with key positions g = t + h0), and the union walked by the item.
// 32-bit positions (N_kv < 2^31 is checked on the host); per-tile fields are
// read with explicit selects so nothing lands in local memory.
struct Item {
    int b, h, r0;
    int glo0, glo1, ghi0, ghi1;  // key positions of the tile's first / last valid query row
    int jlo0, jlo1, jhi0, jhi1;  // key tiles needed by tile X (empty tile: jlo > jhi)
    int jtop;                    // first key tile of the walk (descending)
    int nsteps;
    bool has0, has1;
    __device__ __forceinline__ bool has(int x) const { return x ? has1 : has0; }
    __device__ __forceinline__ int jlo(int x) const { return x ? jlo1 : jlo0; }
    __device__ __forceinline__ int jhi(int x) const { return x ? jhi1 : jhi0; }
    __device__ __forceinline__ int glo(int x) const { return x ? glo1 : glo0; }
    __device__ __forceinline__ int ghi(int x) const { return x ? ghi1 : ghi0; }
    __device__ __forceinline__ bool uses(int x, int j) const { return has(x) && j >= jlo(x) && j <= jhi(x); }
};

__device__ __forceinline__ Item make_item(const TcFwdParams& p, int idx) {
    Item it;
    const int pair = idx % p.n_pairs;
    const int bh = idx / p.n_pairs;
    it.h = bh % (int)p.H;
    it.b = bh / (int)p.H;
    it.r0 = pair * 2 * BM;
    const int Nq = (int)p.Nq, h0 = (int)p.h0;
    it.has0 = it.r0 < Nq;
    it.has1 = it.r0 + BM < Nq;
    it.glo0 = it.r0 + h0;
    it.glo1 = it.r0 + BM + h0;
    it.ghi0 = min(it.r0 + BM - 1, Nq - 1) + h0;
    it.ghi1 = min(it.r0 + 2 * BM - 1, Nq - 1) + h0;
    it.jlo0 = max(0, it.glo0 - p.w + 1) / BN;
    it.jlo1 = max(0, it.glo1 - p.w + 1) / BN;
    it.jhi0 = it.ghi0 / BN;
    it.jhi1 = it.ghi1 / BN;
    if (!it.has1) {
        it.jlo1 = 1;
        it.jhi1 = 0;
    }
    it.jtop = it.has1 ? it.jhi1 : it.jhi0;
    it.nsteps = it.jtop - it.jlo0 + 1;
    return it;
}

// softmax pass helpers on 16-column chunks (GFWA_FWD_LD16)
__device__ __forceinline__ void max_chunk16(const uint32_t (&raw)[16], uint32_t kw, bool interior, float (&mx)[4]) {
#pragma unroll
    for (int e = 0; e < 16; e += 4) {
        float a0 = __uint_as_float(raw[e]), a1 = __uint_as_float(raw[e + 1]);
        float a2 = __uint_as_float(raw[e + 2]), a3 = __uint_as_float(raw[e + 3]);
        if (!interior) {
            a0 = ((kw >> e) & 1u) ? a0 : -INFINITY;
            a1 = ((kw >> (e + 1)) & 1u) ? a1 : -INFINITY;
            a2 = ((kw >> (e + 2)) & 1u) ? a2 : -INFINITY;
            a3 = ((kw >> (e + 3)) & 1u) ? a3 : -INFINITY;
        }
        mx[(e >> 2) & 3] = fmax3(mx[(e >> 2) & 3], fmaxf(a0, a1), fmaxf(a2, a3));
    }
}
template <bool kF16P>
__device__ __forceinline__ void exp_chunk16(const uint32_t (&xr)[16], uint32_t kw, bool interior, uint64_t sl2x2,
                                            uint64_t nm2, float (&acc)[8], uint32_t (&pk)[8]) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const uint64_t dd = ffma2(f2pack(__uint_as_float(xr[2 * e]), __uint_as_float(xr[2 * e + 1])), sl2x2, nm2);
        float d0, d1;
        f2unpack(dd, d0, d1);
        if (!interior) {
            d0 = ((kw >> (2 * e)) & 1u) ? d0 : -INFINITY;
            d1 = ((kw >> (2 * e + 1)) & 1u) ? d1 : -INFINITY;
        }
        const float p0 = ex2(d0), p1 = ex2(d1);
        acc[(2 * e) & 7] += p0;
        acc[(2 * e + 1) & 7] += p1;
        pk[e] = kF16P ? pack_f16x2(p0, p1) : pack_bf16x2(p0, p1);
    }
}

// kF16P: training forward (O_lo wanted): P, V in fp16 for the PV product (reading C-23);
// kNG: the AttnLayer epilogue (reading C-27) is fused into the store rounds
template <int D, bool kF16P, bool kNG>
__global__ void __launch_bounds__(kThreads, 1)
    fwd_tc_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                  const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mo,
                  const __grid_constant__ CUtensorMap mol, const __grid_constant__ CUtensorMap mkh,
                  const __grid_constant__ CUtensorMap mvh, const TcFwdParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    using L = Lay<D>;
    constexpr uint32_t kTile = L::kTile, kOffQ = L::kOffQ, kOffKV = L::kOffKV, kOffE = L::kOffE,
 kOffLinv = L::kOffLinv;
    constexpr int kHalves = D / 64;  // 64-column TMA boxes per tile row
    Bars* bars = (Bars*)(smem + L::kOffBars);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        if (smem_u32(smem) & 1023u) __trap();  // the 128B-swizzle tiles need a 1024-aligned base
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->q_full[i], 1);
            mbar_init(&bars->q_empty[i], 1);  // the tile's last S MMA
            mbar_init(&bars->s_full[i], 1);
            mbar_init(&bars->p_ready[i], 8);  // both softmax warpgroups of the tile
            mbar_init(&bars->o_full[i], 1);
            mbar_init(&bars->o_free[i], 4);
            mbar_init(&bars->l_ready[i], 4);
            mbar_init(&bars->l_free[i], 4);  // the epilogue warps have read 1/l
        }
        for (int i = 0; i < kSlots; ++i) {
            mbar_init(&bars->k_full[i], 2);  // TMA bytes + the producer's bias slab
            mbar_init(&bars->v_full[i], 1);
            mbar_init(&bars->kv_empty[i], 1);
            mbar_init(&bars->v_ready[i], 2);  // the two convert warps
        }
        fence_barrier_init();
    }
    {  // bias slabs: B region zero (k 8..15 of every slab stay zero), A atom = ones at k 0..2
        for (uint32_t i = threadIdx.x; i < BN * 128 / 16; i += kThreads)
            sts128(smem_u32(smem + L::kOffSlabK) + i * 16, make_uint4(0u, 0u, 0u, 0u));
        if (threadIdx.x < 64) {  // row r = tid / 8, physical 16-B chunk c = tid % 8
            const uint32_t r = threadIdx.x >> 3, c = threadIdx.x & 7, one = 0x3F80u;
            sts128(smem_u32(smem + L::kOffSlabA) + r * 128 + c * 16,
                   (c ^ r) == 0 ? make_uint4(one | (one << 16), one, 0u, 0u) : make_uint4(0u, 0u, 0u, 0u));
        }
        fence_proxy_async();
    }
    if (warp == kMmaWarp) {
        tmem_alloc(&bars->tmem, 512);
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
    const uint32_t tmem = bars->tmem;


    if (warp == kTmaWarp) {
        // ------------------------------------------------------------ TMA producer
        const uint64_t pol_kv = policy_evict_last();
        uint32_t fq[2] = {0, 0}, kc = 0;
        for (int idx = blockIdx.x; idx < p.n_items; idx += gridDim.x) {
            const Item it = make_item(p, idx);
            bool q_loaded[2] = {false, false};
            const float* Ubh = p.U + ((int64_t)it.b * p.H + it.h) * p.Nkv;
            const float uref = Ubh[it.glo0];  // the item's bias reference (reading C-18)
            for (int n = 0; n < it.nsteps; ++n) {
                const int j = it.jtop - n;
#pragma unroll
                for (int x = 1; x >= 0; --x)
                    if (it.uses(x, j) && !q_loaded[x]) {  // Q_X just before its first key tile
                        mbar_wait_park(&bars->q_empty[x], (fq[x] & 1) ^ 1);
                        if (elect_one()) {
                            mbar_expect_tx(&bars->q_full[x], kTile);
                            uint8_t* dst = smem + kOffQ + x * kTile;
                            for (int half = 0; half < kHalves; ++half)
                                tma_load_4d(dst + half * kBox, &mq, &bars->q_full[x], half * 64, it.h,
                                            it.r0 + x * BM, it.b);
                        }
                        __syncwarp();
                        ++fq[x];
                        q_loaded[x] = true;
                    }
                // K_j then V_j into the next two ring slots (load m = 2g, 2g + 1 of step g)
#pragma unroll
                for (int kv = 0; kv < 2; ++kv) {
                    const uint32_t m = 2 * kc + kv, sl = m % kSlots;
                    mbar_wait_park(&bars->kv_empty[sl], ((m / kSlots) & 1) ^ 1);
                    if (kv == 0 && lane == 0) FTR(6, (int)kc);
                    if (elect_one()) {
                        uint64_t* full = kv ? &bars->v_full[sl] : &bars->k_full[sl];
                        mbar_expect_tx(full, kTile);
                        // in-kernel halo: tiles below hrows from the halo's own (e.g. peer) memory
                        const bool hz = j * BN < p.hrows;
                        const CUtensorMap* km = kv ? (hz ? &mvh : &mv) : (hz ? &mkh : &mk);
                        for (int half = 0; half < kHalves; ++half)
                            tma_load_4d_hint(smem + kOffKV + sl * kTile + half * kBox, km, full, half * 64,
                                             it.h / p.G, hz ? j * BN : j * BN - p.hrows, it.b, pol_kv);
                    }
                    if (kv == 0) {
                        // K_j's slab: b = (uref - u_k) / scale per key as hi + mid + lo bf16, so the
                        // S MMA yields q.k + b and sl2 (q.k + b) = scale log2e q.k - (u_k - uref) log2e
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int r = lane + 32 * i, key = j * BN + r;
                            const float bk = key < (int)p.Nkv ? (uref - Ubh[key]) * p.inv_scale : 0.f;
                            uint32_t bh, bm, bl;
                            split3_bf16(bk, bh, bm, bl);
                            sts128(smem_u32(smem + L::kOffSlabK) + r * 128 + (((2 * sl) ^ (r & 7)) << 4),
                                   make_uint4(bh | (bm << 16), bl, 0u, 0u));
                        }
                        fence_proxy_async();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&bars->k_full[sl]);
                    }
                    __syncwarp();
                }
                ++kc;
            }
        }
        if (p.zero_acc && blockIdx.x == 0 && lane == 0) *p.token = p.token_val;
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------------------ MMA issuer
        const uint32_t idesc_qk = idesc_bf16(BM, BN, false, false);
        const uint32_t idesc_pv = idesc_bf16(BM, D, false, true) & ~(kF16P ? (63u << 7) : 0u);

        uint32_t kc = 0, cp[2] = {0, 0}, nit[2] = {0, 0}, fq[2] = {0, 0};
        for (int idx = blockIdx.x; idx < p.n_items; idx += gridDim.x) {
            const Item it = make_item(p, idx);
            bool first_pv[2] = {true, true};
            for (int n = 0; n <= it.nsteps; ++n) {
                const int j = it.jtop - n;  // this step's key tile (n < nsteps)
                // this step's K is ring load 2 kc, the previous step's V is load 2 kc - 1
                const uint32_t mk_ = 2 * kc, mv_ = 2 * kc - 1;
                const uint32_t sk = mk_ % kSlots, sv = mv_ % kSlots;
                bool v_waited = false, k_waited = false;
#pragma unroll
                for (int x = 0; x < 2; ++x) {
                    // O_X += P_X V_{n-1} (Alg. 2 l.16-17)
                    if (n > 0 && it.uses(x, j + 1)) {
                        mbar_wait_park(&bars->p_ready[x], cp[x] & 1);
                        ++cp[x];
                        if (first_pv[x]) mbar_wait_park(&bars->o_free[x], (nit[x] & 1) ^ 1);  // epilogue read O_X
                        if (!v_waited) {
                            // one phase per V fill of the slot: V loads m = 2g + 1 land in slot
                            // m % 3 every 6 loads, so this is fill m / 6 of the slot
                            mbar_wait_park(kF16P ? &bars->v_ready[sv] : &bars->v_full[sv], (mv_ / (2 * kSlots)) & 1);
                            v_waited = true;
                        }
                        tc_fence_after();
                        if (lane == 0) FTR(2, (int)(2 * (cp[0] + cp[1])));
                        if (elect_one()) {
                            const uint32_t vb = smem_u32(smem + kOffKV + sv * kTile);
#pragma unroll
                            for (int kk = 0; kk < BN / 16; ++kk)
                                // P of keys [16 kk, 16 kk + 16): S-row half kk / 4 holds its
                                // 64 keys' P in its own first 32 columns
                                mma_ts(tmem + 256 + 128 * x, tmem + 128 * x + 64 * (kk >> 2) + 8 * (kk & 3),
                                       sdesc_sw128(vb + kk * 2048, kBox, 1024), idesc_pv,
                                       (!first_pv[x] || kk > 0) ? 1u : 0u);
                            if (j + 1 == it.jlo(x)) tc_commit(&bars->o_full[x]);
                        }
                        __syncwarp();
                        first_pv[x] = false;
                    }
                    // S_X = Q_X K_n^T (Alg. 2 l.11-12), over the P just consumed: tcgen05
                    // MMAs of one thread execute in issue order
                    if (n < it.nsteps && it.uses(x, j)) {
                        if (!k_waited) {
                            mbar_wait_park(&bars->k_full[sk], (mk_ / (2 * kSlots)) & 1);  // K fill m / 6 of the slot
                            k_waited = true;
                        }
                        if (j == it.jhi(x)) mbar_wait_park(&bars->q_full[x], fq[x]++ & 1);
                        tc_fence_after();
                        if (lane == 0) FTR(3 + x, (int)kc);
                        if (elect_one()) {
                            const uint32_t qb = smem_u32(smem + kOffQ + x * kTile);
                            const uint32_t kb = smem_u32(smem + kOffKV + sk * kTile);
#pragma unroll
                            for (int kk = 0; kk < D / 16; ++kk) {
                                const uint32_t off = (kk >> 2) * kBox + (kk & 3) * 32;
                                mma_ss(tmem + 128 * x, sdesc_sw128(qb + off, 16, 1024),
                                       sdesc_sw128(kb + off, 16, 1024), idesc_qk, kk > 0 ? 1u : 0u);
                            }
                            // + the per-key gate bias (C-26): ones (A, rows repeat: SBO = 0) x slab
                            mma_ss(tmem + 128 * x, sdesc_sw128(smem_u32(smem + L::kOffSlabA), 16, 0),
                                   sdesc_sw128(smem_u32(smem + L::kOffSlabK) + 32 * sk, 16, 1024), idesc_qk, 1u);
                            tc_commit(&bars->s_full[x]);
                            if (j == it.jlo(x)) tc_commit(&bars->q_empty[x]);
                        }
                        __syncwarp();
                    }
                }
                if (elect_one()) {
                    if (n < it.nsteps) tc_commit(&bars->kv_empty[sk]);  // both S of this step issued
                    if (n > 0) tc_commit(&bars->kv_empty[sv]);        // both PV of the previous step issued
                }
                __syncwarp();
                if (n < it.nsteps) ++kc;
            }
            for (int x = 0; x < 2; ++x)
                if (it.has(x)) ++nit[x];
        }
    } else if (warp >= kCvtWarp0) {
        // ------------------------------------------------------------ V -> fp16 in place (training)
        // the layout (128B swizzle) is unchanged, only the element encoding:
        // bf16 -> fp32 (exact) -> fp16 (RNE); 2048 16-byte chunks over 64 threads
        if (kF16P) {
            const int ct = threadIdx.x - kCvtWarp0 * 32;
            uint32_t kc = 0;
            for (int idx = blockIdx.x; idx < p.n_items; idx += gridDim.x) {
                const Item it = make_item(p, idx);
                for (int n = 0; n < it.nsteps; ++n, ++kc) {
                    const uint32_t m = 2 * kc + 1, sl = m % kSlots;  // this step's V: ring load 2 kc + 1
                    mbar_wait_park(&bars->v_full[sl], (m / (2 * kSlots)) & 1);
                    const uint32_t vb = smem_u32(smem + kOffKV + sl * kTile) + ct * 16;
#pragma unroll 8
                    for (int c = 0; c < (int)(kTile / 16 / 64); ++c) {
                        const uint32_t a = vb + c * 64 * 16;
                        uint4 q4 = lds128u(a);
                        q4.x = bf16x2_to_f16x2(q4.x);
                        q4.y = bf16x2_to_f16x2(q4.y);
                        q4.z = bf16x2_to_f16x2(q4.z);
                        q4.w = bf16x2_to_f16x2(q4.w);
                        sts128(a, q4);
                    }
                    fence_proxy_async();  // generic-proxy writes -> visible to the tensor core
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bars->v_ready[sl]);
                }
            }
        }
    } else if (warp < kEpiWarp0) {
        // ------------------------------------------------------------ softmax (tile x, half hh)
        // Two warpgroups per tile: half hh owns S columns [64 hh, 64 hh + 64) of every
        // row (warps of both halves reach the same TMEM lanes: lane quarter = warp % 4),
        // so each warp's serial chain per key tile is half as long.  The row max is
        // exchanged through smem once per key tile, the row sum once per item.
        const int x = warp >> 3, hh = (warp >> 2) & 1;
        const int r = threadIdx.x & 127;
        const uint32_t lane_addr = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        const uint32_t s_col = 128 * x + 64 * hh, o_col = 256 + 128 * x + (D / 2) * hh;
        float* linv = reinterpret_cast<float*>(smem + kOffLinv) + x * BM;
        float* xch = reinterpret_cast<float*>(smem + L::kOffXch) + x * 4 * BM;    // [parity][half][row]
        const uint32_t bar_tile = 5 + x;  // named barrier id of the tile's two softmax warpgroups
        const uint64_t sl2x2 = f2pack(p.sl2, p.sl2);
        uint32_t cs = 0, nit = 0;
        for (int idx = blockIdx.x; idx < p.n_items; idx += gridDim.x) {
            const Item it = make_item(p, idx);
            if (!it.has(x)) continue;
            const float* Ubh = p.U + ((int64_t)it.b * p.H + it.h) * p.Nkv;
            const int t = it.r0 + x * BM + r;
            const bool valid = t < (int)p.Nq;
            const int g = t + (int)p.h0;
            const int Nkv = (int)p.Nkv;
            const int glo_x = it.glo(x), ghi_x = it.ghi(x), jlo_x = it.jlo(x), jt = it.jhi(x);
            // bias in log2 units relative to the item's reference u (reading C-18): the
            // row constant (u_q - uref) cancels in the softmax and re-enters the LSE
            const float uref = Ubh[it.glo0];
            const float bq = valid ? (Ubh[g] - uref) * kLog2e : 0.f;
            float m_used = -INFINITY, l = 0.f;  // l: this half's partial row sum
            for (int j = jt; j >= jlo_x; --j, ++cs) {
                if (r == 0) FTR(x, 6 * (int)cs);
                mbar_wait_park(&bars->s_full[x], cs & 1);
                if (r == 0) FTR(x, 6 * (int)cs + 1);
                tc_fence_after();
                const bool interior = (j * BN + BN - 1 <= glo_x) && (j * BN >= ghi_x - p.w + 1) && (j * BN + BN <= Nkv);
                uint32_t keep[2] = {~0u, ~0u};
                bool live[2] = {true, true};  // warp-uniform: the 32-key chunk has a kept key in some row
                if (!interior) {
                    // keys in (g - w, g] and < N_kv, as columns of this tile
                    const int kb = j * BN;
                    const int hi = min(min(g - kb, BN - 1), Nkv - 1 - kb);
                    const int lo = max(g - p.w + 1 - kb, 0);
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        keep[c] = range_bits(lo, hi, 64 * hh + 32 * c);
                        live[c] = __any_sync(0xffffffffu, keep[c] != 0u);
                    }
                }
                // pass 1: the half-row max of S' = q.k - (u_k - uref) / scale (the gate bias is
                // already in the accumulator, C-26; masked to -inf outside the window, Alg. 2
                // l.12-15); x = sl2 S' is monotone in S', so the max is taken on S'
                float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#if GFWA_FWD_LD16
                {
                    // four 16-column chunks, the next chunk's TMEM load in flight while the
                    // current one is reduced (TMEM load latency under load is hundreds of cycles)
                    uint32_t ra[16], rb[16];
                    const uint32_t kw0 = keep[0], kw1 = keep[1];
                    const bool l0 = live[0], l1 = live[1];
                    // (loads of fully masked chunks are issued anyway: no data-dependent merges
                    // of the in-flight registers; only their reduction is skipped)
                    tmem_ld16(lane_addr + s_col, ra);
                    tmem_wait_ld();
                    tmem_ld16(lane_addr + s_col + 16, rb);
                    if (l0) max_chunk16(ra, kw0 & 0xffffu, interior, mx);
                    tmem_wait_ld();
                    tmem_ld16(lane_addr + s_col + 32, ra);
                    if (l0) max_chunk16(rb, kw0 >> 16, interior, mx);
                    tmem_wait_ld();
                    tmem_ld16(lane_addr + s_col + 48, rb);
                    if (l1) max_chunk16(ra, kw1 & 0xffffu, interior, mx);
                    tmem_wait_ld();
                    if (l1) max_chunk16(rb, kw1 >> 16, interior, mx);
                }
#else
#pragma unroll
                for (int cb = 0; cb < 2; ++cb) {
                    if (!(cb ? live[1] : live[0])) continue;  // masked for the whole warp: pass 2 skips it too
                    uint32_t raw[32];
                    tmem_ld32(lane_addr + s_col + 32 * cb, raw);
                    tmem_wait_ld();
                    const uint32_t kw = cb ? keep[1] : keep[0];
#pragma unroll
                    for (int e = 0; e < 32; e += 4) {
                        float a0 = __uint_as_float(raw[e]), a1 = __uint_as_float(raw[e + 1]);
                        float a2 = __uint_as_float(raw[e + 2]), a3 = __uint_as_float(raw[e + 3]);
                        if (!interior) {
                            a0 = ((kw >> e) & 1u) ? a0 : -INFINITY;
                            a1 = ((kw >> (e + 1)) & 1u) ? a1 : -INFINITY;
                            a2 = ((kw >> (e + 2)) & 1u) ? a2 : -INFINITY;
                            a3 = ((kw >> (e + 3)) & 1u) ? a3 : -INFINITY;
                        }
                        mx[(e >> 2) & 3] = fmax3(mx[(e >> 2) & 3], fmaxf(a0, a1), fmaxf(a2, a3));
                    }
                }
#endif
                if (r == 0) FTR(x, 6 * (int)cs + 2);
                // the row max over both halves (exchange through smem), in log2 units
                // (double-buffered by key-tile parity: a half may run one tile ahead of the other)
                float* xc = xch + (cs & 1) * 2 * BM;
                xc[hh * BM + r] = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
                named_bar_sync(bar_tile, 256);
                const float mraw = fmaxf(xc[r], xc[BM + r]);
                if (r == 0) FTR(x, 6 * (int)cs + 3);
                const float mt = mraw == -INFINITY ? -INFINITY : mraw * p.sl2;
                // lazy online softmax: move the reference max only when it grows by > 2^8
                // (both halves take the same decision from the same values)
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
                float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                // pass 2: exponentials 2^(sl2 S' - m), the half-row sum, 16-bit P of the half's 64
                // keys into its own first 32 S columns (chunk cb's P lands on columns that
                // chunk cb's S' already left: [16 cb, 16 cb + 16) <= [32 cb, 32 cb + 32))
#if GFWA_FWD_LD16
                {
                    // four 16-column chunks with the next chunk's load in flight; chunk q's P
                    // lands on columns [8 q, 8 q + 8), below every S' column still to be read
                    uint32_t xa[16], xb[16], pk[8];
                    const uint32_t kw0 = keep[0], kw1 = keep[1];
                    const bool l0 = live[0], l1 = live[1];
                    const uint32_t z8[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
                    tmem_ld16(lane_addr + s_col, xa);
                    tmem_wait_ld();
                    tmem_ld16(lane_addr + s_col + 16, xb);
                    if (l0) {
                        exp_chunk16<kF16P>(xa, kw0 & 0xffffu, interior, sl2x2, nm2, acc, pk);
                        tmem_st8(lane_addr + s_col, pk);
                    } else {
                        tmem_st8(lane_addr + s_col, z8);
                    }
                    tmem_wait_ld();
                    tmem_ld16(lane_addr + s_col + 32, xa);
                    if (l0) {
                        exp_chunk16<kF16P>(xb, kw0 >> 16, interior, sl2x2, nm2, acc, pk);
                        tmem_st8(lane_addr + s_col + 8, pk);
                    } else {
                        tmem_st8(lane_addr + s_col + 8, z8);
                    }
                    tmem_wait_ld();
                    tmem_ld16(lane_addr + s_col + 48, xb);
                    if (l1) {
                        exp_chunk16<kF16P>(xa, kw1 & 0xffffu, interior, sl2x2, nm2, acc, pk);
                        tmem_st8(lane_addr + s_col + 16, pk);
                    } else {
                        tmem_st8(lane_addr + s_col + 16, z8);
                    }
                    tmem_wait_ld();
                    if (l1) {
                        exp_chunk16<kF16P>(xb, kw1 >> 16, interior, sl2x2, nm2, acc, pk);
                        tmem_st8(lane_addr + s_col + 24, pk);
                    } else {
                        tmem_st8(lane_addr + s_col + 24, z8);
                    }
                }
#else
#pragma unroll
                for (int cb = 0; cb < 2; ++cb) {
                    uint32_t pk[16];
                    if (cb ? live[1] : live[0]) {
                        uint32_t xr[32];
                        tmem_ld32(lane_addr + s_col + 32 * cb, xr);
                        tmem_wait_ld();
                        const uint32_t kw = cb ? keep[1] : keep[0];
#pragma unroll
                        for (int e = 0; e < 16; ++e) {
                            const uint64_t d = ffma2(f2pack(__uint_as_float(xr[2 * e]), __uint_as_float(xr[2 * e + 1])),
                                                     sl2x2, nm2);
                            float d0, d1, p0, p1;
                            f2unpack(d, d0, d1);
                            if (!interior) {
                                d0 = ((kw >> (2 * e)) & 1u) ? d0 : -INFINITY;
                                d1 = ((kw >> (2 * e + 1)) & 1u) ? d1 : -INFINITY;
                            }
                            if ((e & 3) < kPolyPairs) {
                                f2unpack(exp2_poly2(f2pack(d0, d1)), p0, p1);
                            } else {
                                p0 = ex2(d0);
                                p1 = ex2(d1);
                            }
                            acc[(2 * e) & 7] += p0;
                            acc[(2 * e + 1) & 7] += p1;
                            pk[e] = kF16P ? pack_f16x2(p0, p1) : pack_bf16x2(p0, p1);
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < 16; ++e) pk[e] = 0u;
                    }
                    tmem_st16(lane_addr + s_col + 16 * cb, pk);
                }
#endif
                l += ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
                // rescale this half's O columns (the PV of the previous step is complete:
                // S_full certified it)
                if (__any_sync(0xffffffffu, need)) {
                    uint32_t ob[32];
#pragma unroll 1
                    for (int c = 0; c < D / 2; c += 32) {
                        tmem_ld32(lane_addr + o_col + c, ob);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 32; ++e) ob[e] = __float_as_uint(__uint_as_float(ob[e]) * corr);
                        tmem_st32(lane_addr + o_col + c, ob);
                    }
                }
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->p_ready[x]);
                if (r == 0) FTR(x, 6 * (int)cs + 5);
            }
            // Alg. 2 l.19-20: l = both halves' sums; 1/l for the epilogue, LSE = m + ln l
            // (natural log, bias included).  linv is reused per item: wait until the
            // epilogue has read the previous item's
            float* xl = reinterpret_cast<float*>(smem + L::kOffXchL) + x * BM;
            if (hh == 1) xl[r] = l;
            named_bar_sync(bar_tile, 256);
            if (hh == 0) {
                const float lt = l + xl[r];
                mbar_wait_park(&bars->l_free[x], (nit & 1) ^ 1);
                linv[r] = lt > 0.f ? 1.f / lt : 0.f;
                if (valid) p.LSE[((int64_t)it.b * p.H + it.h) * p.Nq + t] = (m_used + bq + __log2f(lt)) * kLn2;
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->l_ready[x]);
            }
            ++nit;
        }
    } else {
        // ------------------------------------------------------------ epilogue (+ V -> fp16)
        const int r = threadIdx.x & 127;
        const int ew = warp - kEpiWarp0;  // == warp & 3: TMEM lanes [32 ew, 32 ew + 32)
        const uint32_t lane_addr = tmem + ((uint32_t)(ew * 32) << 16);
        const float* linv_all = reinterpret_cast<const float*>(smem + kOffLinv);
        uint32_t nit0 = 0, nit1 = 0;
        auto epilogue = [&](const Item& it, int x) {
            const uint32_t ph = (x ? nit1 : nit0) & 1;
            if (r == 0) FTR(5, (int)(4 * (nit0 + nit1)));
            mbar_wait_park(&bars->o_full[x], ph);
            mbar_wait_park(&bars->l_ready[x], ph);
            if (r == 0) FTR(5, (int)(4 * (nit0 + nit1)) + 1);
            tc_fence_after();
            const float inv = linv_all[x * BM + r];
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->l_free[x]);
            uint8_t* ehi = smem + kOffE;  // [O box | O_lo box] of one 64-column half
            const uint32_t sbf = smem_u32(ehi), sf = smem_u32(ehi + kBox);
            const uint32_t o_col = 256 + 128 * x;
            constexpr bool ng = kNG;
            const int trow = it.r0 + x * BM + r;  // this thread's query row
            const bool rvalid = trow < (int)p.Nq;
            float rstd = 0.f;
            if (ng) {
                // AttnLayer epilogue (C-27): rstd = 1/sqrt(mean_c O_c^2 + eps) of
                // the fp32 output row, one read pass over TMEM before the store rounds
                float ss = 0.f;
#pragma unroll 1
                for (int cq = 0; cq < D / 32; ++cq) {
                    uint32_t ob[32];
                    tmem_ld32(lane_addr + o_col + 32 * cq, ob);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const float v = __uint_as_float(ob[e]) * inv;
                        ss = fmaf(v, v, ss);
                    }
                }
                rstd = rsqrtf(ss * (1.f / D) + p.ng_eps);
                if (rvalid) p.ng_rstd[((int64_t)it.b * p.H + it.h) * p.Nq + trow] = rstd;
            }
            // four rounds of 32 columns: O (bf16) into the Q slot, O_lo into E; each
            // 64-column half is stored as soon as it is staged
#pragma unroll 1
            for (int cq = 0; cq < D / 32; ++cq) {
                uint32_t ob[32];
                tmem_ld32(lane_addr + o_col + 32 * cq, ob);
                tmem_wait_ld();
                if (cq == D / 32 - 1) {  // all of O_X has been read: release its columns
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bars->o_free[x]);
                }
                const int hf = cq >> 1, cc = cq & 1;
                if (cc == 0 && hf > 0) {  // the previous half's stores must have read the staging
                    if (r == 0) bulk_wait_read0();
                    named_bar_sync(7, 128);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int chunk = (cc * 4 + k) ^ (r & 7);
                    uint32_t hw[4], lw[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float v0 = __uint_as_float(ob[8 * k + 2 * e]) * inv;
                        const float v1 = __uint_as_float(ob[8 * k + 2 * e + 1]) * inv;
                        hw[e] = pack_bf16x2(v0, v1);
                        if (p.store_lo) {
                            float h0, h1;
                            f2unpack(bf2_to_f2(hw[e]), h0, h1);
                            lw[e] = pack_bf16x2(v0 - h0, v1 - h1);
                        }
                    }
                    const uint32_t off = r * 128 + chunk * 16;
                    sts128(sbf + off, make_uint4(hw[0], hw[1], hw[2], hw[3]));
                    if (p.store_lo) sts128(sf + off, make_uint4(lw[0], lw[1], lw[2], lw[3]));
                }
                if (cc == 1) {
                    fence_proxy_async();
                    named_bar_sync(7, 128);
                    if (r == 0) {
                        const int row0 = it.r0 + x * BM;
                        tma_store_4d(&mo, ehi, hf * 64, it.h, row0, it.b);
                        if (p.store_lo) tma_store_4d(&mol, ehi + kBox, hf * 64, it.h, row0, it.b);
                        bulk_commit();
                    }
                }
            }
            if (p.zero_acc) {
                // gfwa_fwd_train: zero this tile's rows of the backward's fp32 dQ accumulator
                // [B, Nq, H, d] while the stores drain (one 512-byte row per warp store;
                // this warpgroup is otherwise idle between epilogues)
                const int r1 = min(it.r0 + x * BM + BM, (int)p.Nq);
                for (int t = it.r0 + x * BM + ew; t < r1; t += 4) {
                    float4* row = reinterpret_cast<float4*>(p.zero_acc + (((int64_t)it.b * p.Nq + t) * p.H + it.h) * D);
                    if (lane < D / 4) row[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
            if (r == 0) {
                bulk_wait_read0();  // the staging buffers are reusable once the stores have read them
                FTR(5, (int)(4 * (nit0 + nit1)) + 2);
            }
            named_bar_sync(7, 128);
            if (x)
                ++nit1;
            else
                ++nit0;
        };
        for (int idx = blockIdx.x; idx < p.n_items; idx += gridDim.x) {
            const Item it = make_item(p, idx);
            if (it.has1) epilogue(it, 1);  // B's last key tile comes before A's
            if (it.has0) epilogue(it, 0);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// AttnLayer epilogue, second half (reading C-27): Y = swish(g) gamma (O + O_lo)
// rstd, one streaming pass over the rows the forward just wrote (rstd came from the
// forward's epilogue, taken on the fp32 output in TMEM).  Packed [rows, D] layouts; a
// warp takes 32 / (D / 8) rows per load group (16 B per lane), U groups in flight.
template <int D>
__global__ void __launch_bounds__(256) normgate_y_kernel(const __nv_bfloat16* __restrict__ O,
                                                         const __nv_bfloat16* __restrict__ Olo,
                                                         const __nv_bfloat16* __restrict__ g,
                                                         const float* __restrict__ gamma,
                                                         const float* __restrict__ rstd,
                                                         __nv_bfloat16* __restrict__ Y, uint32_t rows, uint32_t H,
                                                         uint32_t Nq) {
    constexpr int LPR = D / 8, RPW = 32 / LPR, U = 4;
    const uint32_t lane = threadIdx.x & 31, sub = lane / LPR, cl = lane % LPR;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const float4 ga = __ldg(reinterpret_cast<const float4*>(gamma) + 2 * cl);
    const float4 gb = __ldg(reinterpret_cast<const float4*>(gamma) + 2 * cl + 1);
    const float gam[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
    for (uint32_t r0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * (U * RPW); r0 < rows; r0 += nw * U * RPW) {
        uint4 ov[U], lv[U], gv[U];
        float rs[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t row = min(r0 + u * RPW + sub, rows - 1);
            const size_t e = (size_t)row * D + cl * 8;
            ov[u] = __ldcs(reinterpret_cast<const uint4*>(O + e));
            lv[u] = Olo ? __ldcs(reinterpret_cast<const uint4*>(Olo + e)) : make_uint4(0u, 0u, 0u, 0u);
            gv[u] = __ldcs(reinterpret_cast<const uint4*>(g + e));
            const uint32_t hh = row % H, bt = row / H, t = bt % Nq, b = bt / Nq;
            rs[u] = __ldg(rstd + ((size_t)b * H + hh) * Nq + t);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t row = r0 + u * RPW + sub;
            const uint32_t* ow = &ov[u].x;
            const uint32_t* lw = &lv[u].x;
            const uint32_t* gw = &gv[u].x;
            uint32_t yw[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float o0, o1, l0, l1, g0, g1;
                f2unpack(bf2_to_f2(ow[e]), o0, o1);
                f2unpack(bf2_to_f2(lw[e]), l0, l1);
                f2unpack(bf2_to_f2(gw[e]), g0, g1);
                const float s0 = fmaf(0.5f, tanh_approx(0.5f * g0), 0.5f);
                const float s1 = fmaf(0.5f, tanh_approx(0.5f * g1), 0.5f);
                yw[e] = pack_bf16x2(g0 * s0 * gam[2 * e] * (o0 + l0) * rs[u], g1 * s1 * gam[2 * e + 1] * (o1 + l1) * rs[u]);
            }
            if (row < rows) __stcs(reinterpret_cast<uint4*>(Y + (size_t)row * D + cl * 8), make_uint4(yw[0], yw[1], yw[2], yw[3]));
        }
    }
}

}  // namespace

#if GFWA_FWD_TRACE
// diagnostics build only: copy the stamp array out (148 x 8 x kTrMax int64)
extern "C" int gfwa_debug_fwd_trace(long long* host, size_t n) {
    if (n > sizeof(g_fwd_trace) / sizeof(long long)) n = sizeof(g_fwd_trace) / sizeof(long long);
    return (int)cudaMemcpyFromSymbol(host, g_fwd_trace, n * sizeof(long long));
}
#endif

bool tc_fwd_supported(const AttnParams& p, gfwa_dtype_t dt) {
    if (dt != GFWA_BF16 || (p.d != 64 && p.d != 128)) return false;
    if (p.Nkv >= ((int64_t)1 << 31) || p.H >= 65536 || p.B >= 65536) return false;
    if (const char* e = getenv("GFWA_FORCE_SIMT")) return e[0] == '0';
    return true;
}

template <int D>
static gfwa_status_t tc_fwd_d(const AttnParams& p, cudaStream_t st) {
    CUtensorMap mq, mk, mv, mo, mol;
    GFWA_REQUIRE(encode_bnhd_map(&mq, p.Q, p.B, p.Nq, p.H, D, p.qs, BM));
    // K / V hold key rows [hrows, Nkv); rows [0, hrows) come from the halo maps (in-kernel halo)
    GFWA_REQUIRE(encode_bnhd_map(&mk, p.K, p.B, p.Nkv - p.hrows, p.Hkv, D, p.ks, BN));
    GFWA_REQUIRE(encode_bnhd_map(&mv, p.V, p.B, p.Nkv - p.hrows, p.Hkv, D, p.vs, BN));
    CUtensorMap mkh = mk, mvh = mv;
    if (p.hrows) {
        GFWA_REQUIRE(encode_bnhd_map(&mkh, p.Kh, p.B, p.hrows, p.Hkv, D, p.khs, BN));
        GFWA_REQUIRE(encode_bnhd_map(&mvh, p.Vh, p.B, p.hrows, p.Hkv, D, p.vhs, BN));
    }
    GFWA_REQUIRE(encode_bnhd_map(&mo, p.O, p.B, p.Nq, p.H, D, p.os, BM));
    if (p.O_lo)
        GFWA_REQUIRE(encode_bnhd_map(&mol, p.O_lo, p.B, p.Nq, p.H, D, p.os, BM));
    else
        mol = mo;  // unused
    TcFwdParams tp;
    tp.U = p.U;
    tp.LSE = p.LSE;
    tp.Nq = p.Nq;
    tp.Nkv = p.Nkv;
    tp.h0 = p.h0;
    tp.H = p.H;
    tp.B = p.B;
    tp.w = p.w;
    tp.G = (int)(p.H / p.Hkv);
    tp.store_lo = p.O_lo != nullptr;
    tp.zero_acc = p.zero_acc;
    tp.token = p.token;
    tp.token_val = p.token_val;
    tp.sl2 = p.scale * kLog2e;
    tp.inv_scale = 1.f / p.scale;
    tp.ng_g = (const __nv_bfloat16*)p.ng_g;
    tp.ng_Y = (__nv_bfloat16*)p.ng_Y;
    tp.ng_gamma = p.ng_gamma;
    tp.ng_rstd = p.ng_rstd;
    tp.ng_eps = p.ng_eps;
    for (int i = 0; i < 3; ++i) tp.os[i] = p.os[i];
    tp.hrows = (int)p.hrows;
    tp.n_pairs = (int)((p.Nq + 2 * BM - 1) / (2 * BM));
    const int64_t n_items = (int64_t)tp.n_pairs * p.H * p.B;
    if (n_items >= ((int64_t)1 << 31) || p.Nkv + 2 * BM >= ((int64_t)1 << 31)) return GFWA_ERR_INVALID_ARGUMENT;
    tp.n_items = (int)n_items;
    int dev = 0, n_sm = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    // per launch: the attribute is per device (a process may drive several GPUs)
    auto kern = tp.ng_g ? (tp.store_lo ? fwd_tc_kernel<D, true, true> : fwd_tc_kernel<D, false, true>)
                        : (tp.store_lo ? fwd_tc_kernel<D, true, false> : fwd_tc_kernel<D, false, false>);
    constexpr size_t kSmemBytes = Lay<D>::kSmemBytes;
    if (gfwa_status_t s = check_launch(
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes)))
        return s;
    int64_t cap = n_sm;
    if (const char* e = getenv("GFWA_FWD_GRID")) cap = max64(1, atoll(e));  // diagnostics: fewer CTAs, more items each
    const unsigned grid = (unsigned)min64(n_items, cap);
    kern<<<grid, kThreads, kSmemBytes, st>>>(mq, mk, mv, mo, mol, mkh, mvh, tp);
    note_launch();
    if (gfwa_status_t s = check_launch()) return s;
    if (!p.ng_g) return GFWA_OK;
    const int64_t rows = p.B * p.Nq * p.H;  // < 2^31, packed layout: checked by the caller
    constexpr int kRowsPerBlock = 8 * 4 * (256 / D);
    normgate_y_kernel<D><<<(unsigned)min64((rows + kRowsPerBlock - 1) / kRowsPerBlock, (int64_t)n_sm * 8), 256, 0, st>>>(
        (const __nv_bfloat16*)p.O, (const __nv_bfloat16*)p.O_lo, (const __nv_bfloat16*)p.ng_g, p.ng_gamma, p.ng_rstd,
        (__nv_bfloat16*)p.ng_Y, (uint32_t)rows, (uint32_t)p.H, (uint32_t)p.Nq);
    note_launch();
    return check_launch();
}

gfwa_status_t tc_fwd(const AttnParams& p, cudaStream_t st) {
    return p.d == 64 ? tc_fwd_d<64>(p, st) : tc_fwd_d<128>(p, st);
}

}  // namespace gfwa
