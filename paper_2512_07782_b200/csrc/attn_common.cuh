// attn_common.cuh -- parameter block shared by the attention kernels.
#pragma once
#include "common.cuh"

namespace gfwa {

struct AttnParams {
    // problem
    int64_t B, H, Nq, Nkv, h0;  // h0 = Nkv - Nq halo rows
    int64_t Hkv;                // K/V heads (GQA): query head h reads K/V head h / (H / Hkv)
    int d, w;
    float scale;
    // element strides over (b, n, h); d contiguous
    int64_t qs[3], ks[3], vs[3], os[3];
    // in-kernel halo: key rows [0, hrows) from Kh / Vh (strides khs / vhs), the rest from K / V
    int64_t hrows;
    const void* Kh;
    const void* Vh;
    int64_t khs[3], vhs[3];
    // forward
    const void* Q;
    const void* K;
    const void* V;
    const float* U;  // [B,H,Nkv]
    void* O;
    void* O_lo;         // bf16 residual of the output cast, bf16(O_exact - O) (nullable; C-12)
    float* LSE;      // [B,H,Nq]
    // backward
    const void* dO;
    const void* Olo;    // that residual for D = rowsum((O + O_lo) dO) (may be null -> use O)
    void* dQ;
    void* dK;
    void* dV;
    float* dU;          // [B,H,Nkv]
    float* Dv;          // [B,H,Nq] workspace: rowsum(O*dO)
    float* dQacc;       // fp32 dQ accumulator workspace (tensor-core path)
    // gfwa_fwd_train: the forward zeroes the backward's dQ accumulator in its
    // epilogue and marks the workspace (token) so the backward skips that pass
    float* zero_acc;               // [B, Nq, H, d] fp32 region to zero (null: none)
    unsigned long long* token;     // prepared-workspace token slot (device)
    unsigned long long token_val;  // value identifying this problem's preparation
    // AttnLayer output epilogue (reading C-27): Y = swish(g) * gamma * O * rstd,
    // rstd = 1/sqrt(mean_c O_c^2 + eps) per (b, t, h) row; g, Y, dY, dg share O's strides
    const void* ng_g;      // bf16 gate pre-activation (null: no epilogue)
    const float* ng_gamma; // [d]
    float ng_eps;
    float* ng_rstd;        // [B,H,Nq] (forward output, backward input)
    void* ng_Y;            // forward output
    const void* ng_dY;     // backward input
    void* ng_dg;           // backward output
    float* ng_dgamma;      // backward output [d] (zeroed and accumulated by the call)
    bool pre_done;         // backward: D, dO and the zeroing came from the fused epilogue pre kernel
    // sequence sharding: fp32 copies of dK, dV of the first / last key rows ([2][B][rows][H][d])
    float* f32_head;
    float* f32_tail;
    int64_t f32_head_rows, f32_tail_rows;
};

// token marking a backward workspace whose dQ accumulator the forward already zeroed
// the prepared-workspace token: a mix of the whole descriptor (never 0, the cleared value)
inline unsigned long long prep_token(const AttnParams& p) {
    unsigned long long x = 0x4746574174726E21ull;
    const long long f[6] = {p.B, p.H, p.Nq, p.Nkv, p.d, p.w};
    for (long long v : f) {
        x ^= (unsigned long long)v + 0x9E3779B97F4A7C15ull + (x << 6) + (x >> 2);
        x *= 0xBF58476D1CE4E5B9ull;
    }
    return x | 1ull;
}

__device__ __forceinline__ int64_t off3(const int64_t* s, int64_t b, int64_t n, int64_t h) {
    return b * s[0] + n * s[1] + h * s[2];
}

// Launchers implemented in attn_simt.cu / attn_tc_*.cu
gfwa_status_t simt_fwd(const AttnParams& p, gfwa_dtype_t dt, cudaStream_t st);
gfwa_status_t simt_bwd(const AttnParams& p, gfwa_dtype_t dt, cudaStream_t st);
gfwa_status_t bwd_preprocess(const AttnParams& p, gfwa_dtype_t dt, cudaStream_t st);

}  // namespace gfwa
