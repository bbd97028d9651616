/*
 * gfwa.h -- C ABI of libgfwa.so, the B200 (sm_100a) GatedFWA hot path.
 *
 * GatedFWA (arXiv 2512.07782) = sliding-window softmax attention whose logits
 * carry a cumulative decay bias B_tj = u_t - u_j built from a per-token,
 * per-head gate alpha.  Citations "P:<line>" refer to the paper's LaTeX
 * source, "S:<line>" to SPEC.md; "C-<n>" are the readings of
 * silent/ambiguous passages listed in DESIGN.md §3.
 *
 * Conventions shared by every call
 * --------------------------------
 *  - All tensor pointers are DEVICE pointers owned by the caller.  The
 *    library never allocates, frees or synchronises; every call is enqueued
 *    on `stream` (a cudaStream_t; NULL = legacy default stream) and returns
 *    as soon as the work is launched.  No host reads of device data.
 *  - Scratch memory is passed in (`ws`, `ws_bytes`), sized by the matching
 *    *_workspace_size() call, and must be 256-byte aligned.  Unless a call
 *    says otherwise the workspace needs no initialisation.
 *  - Errors are returned as gfwa_status_t; arguments are validated before
 *    any launch, so INVALID_ARGUMENT / UNSUPPORTED leave outputs untouched.
 *    GFWA_ERR_CUDA reports a launch error; gfwa_last_cuda_error() gives the
 *    cudaError_t of the calling thread's last failure.  No exception crosses
 *    the ABI.  There is no CPU fallback: a non-sm_100 device is UNSUPPORTED.
 *  - Token index t is 0-based.  Window (Alg. 2 line 14 P:382; C-2):
 *    query at key position g attends keys j with max(0, g-w+1) <= j <= g
 *    (w keys including itself, clipped at 0; w >= N is full causal).
 *  - Logit (Eq. 12; C-1): s_tj = scale * q_t.k_j + (u_t - u_j),
 *    scale defaults to 1/sqrt(d) and multiplies q.k only.
 *  - dtypes: Q/K/V/O/dO/dQ/dK/dV/caches are GFWA_BF16 (tensor-core path) or
 *    GFWA_F32 (exact parity path).  U, LSE, D, dU, dalpha are fp32; O_lo
 *    (the bf16 residual of O's output cast) is bf16;
 *    carries and totals are fp64.
 */
#ifndef GFWA_H_
#define GFWA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* gfwa_stream_t; /* == cudaStream_t */

typedef enum {
    GFWA_OK = 0,
    GFWA_ERR_INVALID_ARGUMENT = 1, /* null pointer, bad size, misaligned pointer/stride */
    GFWA_ERR_UNSUPPORTED = 2,      /* head dim / dtype combination / device not CC 10.0 */
    GFWA_ERR_CUDA = 3,             /* a CUDA launch failed; see gfwa_last_cuda_error() */
    GFWA_ERR_WORKSPACE = 4,        /* ws_bytes smaller than *_workspace_size() */
    GFWA_ERR_NONFINITE = 5         /* opt-in debug check found NaN/Inf (gfwa_check_finite) */
} gfwa_status_t;

typedef enum { GFWA_F32 = 0, GFWA_BF16 = 1 } gfwa_dtype_t;

/* Gate input kind for gfwa_gate_prefix / gfwa_decode.
 * HBETA: (h, beta) as in Alg. 1, alpha = softplus(beta*h)/(beta+eps).
 * ALPHA: alpha is given directly (beta ignored) -- lets callers bring their
 *        own gate and lets tests drive alpha = 0 (SWA) or constant alpha. */
typedef enum { GFWA_GATE_HBETA = 0, GFWA_GATE_ALPHA = 1 } gfwa_gate_kind_t;

/* ------------------------------------------------------------------------- */
/* Gate preprocessing: Alg. 1 "Fused Tiled Scan", Eq. 9-11.       */
/* ------------------------------------------------------------------------- */

/*
 * gfwa_gate_prefix -- one streaming pass over (h, beta):
 *   z = beta*h;  alpha = softplus(z)/(beta+eps)            (Alg. 1 l.5-7)
 *   U[b,hh,t] = carry_in[b,hh] - sum_{q<=t} alpha[b,q,hh]  (Alg. 1 l.8-10, Eq. 11,
 *                                                            inclusive prefix, C-8)
 *   total[b,hh] = sum_q alpha[b,q,hh]                       (for the cross-rank scan)
 * in_dtype   dtype of h/beta (GFWA_BF16 or GFWA_F32).
 * h, beta    [B, N, H] row-major (H contiguous).  beta unused for GATE_ALPHA
 *            (then h holds alpha).
 * carry_in   [B*H] fp64 device array or NULL (= 0).
 * U          [B, H, N] fp32 output (N contiguous, head-major for attention).
 * total      [B*H] fp64 output or NULL.
 * Accumulation: fp32 per element, fp64 across chunks (reading C-9).
 * ws         >= gfwa_gate_prefix_workspace_size(B, N, H) bytes; need not be
 *            initialised (the call clears what it uses, on `stream`).
 */
size_t gfwa_gate_prefix_workspace_size(int64_t B, int64_t N, int64_t H);
gfwa_status_t gfwa_gate_prefix(gfwa_gate_kind_t kind, gfwa_dtype_t in_dtype, const void* h,
                               const void* beta, int64_t B, int64_t N, int64_t H, float eps,
                               const double* carry_in, float* U, double* total, void* ws,
                               size_t ws_bytes, gfwa_stream_t stream);

/*
 * gfwa_gate_prefix_bwd -- backward of gfwa_gate_prefix ("gradients into U flow
 * through the same streamed scan"; chain rule of Eq. 9):
 *   dalpha[b,hh,t] = carry[b,hh] - sum_{t'>=t} dU[b,hh,t']       (reverse scan)
 *   dh    = dalpha * sigmoid(beta h) * beta/(beta+eps)
 *   dbeta = dalpha * (sigmoid(beta h) h (beta+eps) - softplus(beta h))/(beta+eps)^2
 * dU [B,H,N] fp32 in; dalpha [B,H,N] fp32 out (or NULL); dh, dbeta [B,N,H] in
 * in_dtype out (NULL to skip; ignored for GATE_ALPHA, where dh receives dalpha
 * in [B,N,H] layout if non-NULL).  carry [B*H] fp64 or NULL: the suffix sum
 * of later sequence shards (sequence sharding, north_star).
 * ws as for gfwa_gate_prefix.
 */
size_t gfwa_gate_prefix_bwd_workspace_size(int64_t B, int64_t N, int64_t H);
gfwa_status_t gfwa_gate_prefix_bwd(gfwa_gate_kind_t kind, gfwa_dtype_t in_dtype, const void* h,
                                   const void* beta, int64_t B, int64_t N, int64_t H, float eps,
                                   const float* dU, const double* carry, float* dalpha, void* dh,
                                   void* dbeta, void* ws, size_t ws_bytes, gfwa_stream_t stream);

/*
 * gfwa_gate_prefix_variant -- the two preprocessing designs the paper compares
 * its kernel with, for the benchmark of SURVEY §8(f) f2.  NOT
 * the product path: same output as gfwa_gate_prefix with GATE_HBETA and no
 * carry (U[b,hh,t] = -sum_{q<=t} alpha, fp32 in-run / fp64 across runs, C-9).
 *   variant 1  Alg. 1 as the paper launches it: one CTA per (b, head)
 *              walking the time axis in 1024-token chunks with an on-chip
 *              carry (serial across chunks); reads h, beta once.
 *   variant 2  Scan-Then-Propagate, App. E.1: chunk sums, a scan
 *              of the chunk sums, then a re-read of h, beta that writes U;
 *              H <= 32 (else GFWA_ERR_UNSUPPORTED).
 * h, beta    [B, N, H] in in_dtype (GFWA_BF16 or GFWA_F32); U [B, H, N] fp32.
 * ws         >= gfwa_gate_prefix_variant_workspace_size(variant, B, N, H)
 *            bytes (variant 2: chunk sums and offsets, fp64); caller-owned.
 * Errors: INVALID_ARGUMENT (variant not 1/2, null pointers, sizes < 1),
 * UNSUPPORTED (dtype, H > 32 for variant 2), WORKSPACE, CUDA.
 */
size_t gfwa_gate_prefix_variant_workspace_size(int variant, int64_t B, int64_t N, int64_t H);
gfwa_status_t gfwa_gate_prefix_variant(int variant, gfwa_dtype_t in_dtype, const void* h, const void* beta,
                                       int64_t B, int64_t N, int64_t H, float eps, float* U, void* ws,
                                       size_t ws_bytes, gfwa_stream_t stream);

/* ------------------------------------------------------------------------- */
/* Attention: Alg. 2 (forward) and Alg. E.2 (backward) */
/* ------------------------------------------------------------------------- */

/*
 * Problem descriptor.  Queries are the LAST N_q rows of the N_kv-row key
 * sequence: query t sits at key position g = t + (N_kv - N_q).  N_kv > N_q
 * carries a halo of earlier keys (sequence sharding); the U frame is the key
 * frame (U has N_kv entries per (b,h)).
 * Strides are in ELEMENTS over (b, n, h); the head dim d is contiguous.
 * Gradients share the layout of their primal: dQ uses q_stride, dK k_stride,
 * dV v_stride, dO and O use o_stride.  For the BF16 path every stride and
 * base pointer must be 16-byte aligned (TMA).
 * Grouped-query attention (the NSA configuration's GQA): with
 * H_kv > 0, K, V, dK, dV have H_kv heads and query head hh reads K/V head
 * hh / (H / H_kv); U, LSE, dU, dalpha stay per query head, so every query
 * head keeps its own gate (Eq. 7 is per head).  dK, dV of a K/V head sum
 * the gradients of its H / H_kv query heads.  H % H_kv == 0 is required;
 * H_kv != H runs on the BF16 tensor-core path only (UNSUPPORTED otherwise).
 * H_kv = 0 means H_kv = H (multi-head attention).
 */
typedef struct {
    int64_t B, H, N_q, N_kv;
    int32_t d;          /* head dim: 64 or 128 */
    int32_t w;          /* window, >= 1 */
    float scale;        /* <= 0 selects 1/sqrt(d) */
    gfwa_dtype_t dtype; /* dtype of Q, K, V, O, dO, dQ, dK, dV */
    int64_t q_stride[3], k_stride[3], v_stride[3], o_stride[3];
    int64_t H_kv;       /* K/V heads (GQA), H % H_kv == 0; 0 = H */
    /*
     * In-kernel halo (SURVEY 8(e)'s B200 refinement, 8(f) f3): halo_rows > 0 makes
     * the attention kernels TMA-load key rows [0, halo_rows) straight from K_halo /
     * V_halo -- typically the previous sequence shard's last rows in that rank's own
     * memory, mapped into this process (CUDA IPC / NVLink peer pointer), so the
     * halo never needs a copy or a send -- and rows [halo_rows, N_kv) from K / V,
     * which then hold N_kv - halo_rows rows ([B, N_kv - halo_rows, H_kv, d] with
     * k_stride / v_stride).  K_halo / V_halo are [B, halo_rows, H_kv, d] with
     * kh_stride / vh_stride (elements, 16-byte aligned) and must stay valid and
     * unchanged until the call's work completes on the stream.  Requirements:
     * BF16, the tensor-core path, halo_rows % 128 == 0, halo_rows <= N_kv - N_q
     * (the halo lies in front of every query); INVALID_ARGUMENT / UNSUPPORTED
     * otherwise.  Results equal the same call on one contiguous [halo; local] K / V;
     * gradients (dK, dV, dU) still cover all N_kv rows in the caller's buffers,
     * dK / dV with K's / V's strides (so with B > 1 the batch stride of K / V must
     * span N_kv rows, e.g. K / V views of the local rows of [B, N_kv, H_kv, d]
     * buffers).
     * halo_rows = 0 (a zero-initialised tail): K / V hold all N_kv rows.
     */
    int64_t halo_rows;
    const void* K_halo;
    const void* V_halo;
    int64_t kh_stride[3], vh_stride[3];
} gfwa_attn_desc_t;

/*
 * gfwa_fwd -- Eq. 12 via Alg. 2: for every (b, hh, t)
 *   O[b,t,hh,:] = sum_j softmax_j(s_tj) V[b,j,hh,:] over the window,
 *   LSE[b,hh,t] = log sum_j exp(s_tj)   (natural log, bias included, C-10)
 * Q [B,N_q,H,d], K, V [B,N_kv,H,d], U [B,H,N_kv] fp32 -> O [B,N_q,H,d],
 * LSE [B,H,N_q] fp32.  O_lo (nullable; BF16 dtype only, same layout and
 * strides as O) receives the bf16 residual of the output cast,
 * O_lo = bf16(O_fp32 - O), so O + O_lo carries the fp32 O to ~2^-17 relative;
 * pass it to gfwa_bwd so D = rowsum(O*dO) is taken from it (reading C-12;
 * SURVEY C-12's bf16-residual alternative to an fp32 O: half the bytes).
 * With O_lo the tensor-core path forms the PV product with P and V in fp16
 * (reading C-23; |v| < 65504 required), without it in bf16.  Key tiles
 * outside every row's window are never read.  INVALID_ARGUMENT if O_lo is
 * given with dtype F32 (an fp32 O is exact).
 */
gfwa_status_t gfwa_fwd(const gfwa_attn_desc_t* desc, const void* Q, const void* K, const void* V,
                       const float* U, void* O, void* O_lo, float* LSE, gfwa_stream_t stream);

/*
 * gfwa_bwd -- Alg. E.2 with readings C-3 (scale on dQ, dK),
 * C-4 (du^k is a column sum), C-11 (du^q row sum kept), C-12 (D from O + O_lo):
 *   D = rowsum(O*dO);  P = exp(s - LSE);  dS = P (dO V^T - D)
 *   dV = P^T dO;  dQ = scale dS K;  dK = scale dS^T Q
 *   dU[g] = sum_j dS_tj (g = t + h0)  -  sum_t dS_tj (key j)
 *   dalpha = dalpha_carry - reverse_cumsum(dU)     (NULL to skip)
 * D = rowsum((O + O_lo) * dO) when O_lo is given (BF16), else rowsum(O * dO);
 * O, O_lo and dO share O's strides.  dK, dV, dU cover all N_kv
 * key rows (halo rows included); dQ covers N_q rows.  dalpha [B,H,N_kv] fp32,
 * dalpha_carry [B*H] fp64 or NULL.
 * ws >= gfwa_bwd_workspace_size(desc); need not be initialised.
 */
/*
 * gfwa_fwd_train -- gfwa_fwd for a training step whose backward will run on
 * bwd_ws (>= gfwa_bwd_workspace_size(desc) bytes, 256-byte aligned): on the
 * tensor-core path the forward (its TMA producer warp, once its loads are
 * issued) also zeroes the backward's fp32 dQ accumulator inside bwd_ws and
 * marks bwd_ws (a token of the whole descriptor in its first 256 bytes), so
 * the next gfwa_bwd on it with the same desc skips that zeroing pass (268 MB
 * at BASELINE configs[1]).  Every gfwa_fwd_train overwrites the token and every
 * tensor-core gfwa_bwd clears it, so only the latest prepared descriptor is
 * honoured: a gfwa_bwd with another descriptor (or after an intervening
 * backward) zeroes its own accumulator, and interleaving shapes on one
 * workspace is safe.  When O_lo is given, the PV product runs with P and V in
 * fp16 (reading C-23: the O + O_lo that D is taken from then carries 8x less
 * P rounding than with bf16 P); V must then lie in the fp16 range
 * (|v| < 65504; larger values overflow to inf).  Calls sharing a workspace
 * must be ordered on one stream.  Other paths: exactly gfwa_fwd.  Errors as
 * gfwa_fwd, plus WORKSPACE.
 */
gfwa_status_t gfwa_fwd_train(const gfwa_attn_desc_t* desc, const void* Q, const void* K, const void* V,
                             const float* U, void* O, void* O_lo, float* LSE, void* bwd_ws,
                             size_t bwd_ws_bytes, gfwa_stream_t stream);

size_t gfwa_bwd_workspace_size(const gfwa_attn_desc_t* desc);
gfwa_status_t gfwa_bwd(const gfwa_attn_desc_t* desc, const void* Q, const void* K, const void* V,
                       const float* U, const void* O, const void* O_lo, const float* LSE,
                       const void* dO, void* dQ, void* dK, void* dV, float* dU, float* dalpha,
                       const double* dalpha_carry, void* ws, size_t ws_bytes, gfwa_stream_t stream);

/*
 * gfwa_bwd_rows_f32 -- gfwa_bwd that also writes fp32 copies of dK and dV (before
 * their bf16 rounding) for the first head_rows and the last tail_rows key rows:
 * dKV_head [2][B][head_rows][H_kv][d] and dKV_tail [2][B][tail_rows][H_kv][d] (dK
 * in [0], dV in [1]; contiguous, 16-byte aligned; H_kv = H without GQA).  Sequence sharding (SURVEY
 * 8(e) step 2; BASELINE north_star): rank r's partial gradients of its w halo
 * rows (its head rows) travel to rank r-1 in fp32 and are added there to that
 * rank's fp32 tail rows, so the boundary rows are rounded to bf16 once.  The
 * bf16 dK/dV of those rows are written as by gfwa_bwd.  Tensor-core path only
 * (UNSUPPORTED otherwise); a count of 0 disables that side.
 */
gfwa_status_t gfwa_bwd_rows_f32(const gfwa_attn_desc_t* desc, const void* Q, const void* K, const void* V,
                                const float* U, const void* O, const void* O_lo, const float* LSE,
                                const void* dO, void* dQ, void* dK, void* dV, float* dU, float* dalpha,
                                const double* dalpha_carry, int64_t head_rows, float* dKV_head,
                                int64_t tail_rows, float* dKV_tail, void* ws, size_t ws_bytes,
                                gfwa_stream_t stream);

/* ------------------------------------------------------------------------- */
/* NSA extension with GatedFWA as the local branch (App. B)          */
/* ------------------------------------------------------------------------- */
typedef struct {
    int64_t B, H, N;
    int32_t d;          /* 64 or 128 */
    int32_t w;          /* window of the local (GatedFWA) branch */
    int32_t block;      /* compression / selection block length (length = stride), 1..64 */
    int32_t n_sel;      /* selected blocks besides the query's own block */
    float scale;        /* <= 0 selects 1/sqrt(d) */
    gfwa_dtype_t dtype; /* GFWA_BF16 */
} gfwa_nsa_desc_t;

/* Tensors the forward keeps for the backward (caller-owned; NULL members are
 * kept in the workspace, i.e. not available to a later gfwa_nsa_bwd). */
typedef struct {
    float* O_cmp;   /* [B,N,H,d] fp32 compressed-branch output */
    float* O_slc;   /* [B,N,H,d] fp32 selected-branch output */
    float* LSE_cmp; /* [B,H,N] fp32 (-inf where no block is complete) */
    float* LSE_slc; /* [B,H,N] fp32 */
    int32_t* sel;   /* [B,H,N,n_sel+1] selected blocks: own block first, -1 pads */
    void* O_loc;    /* [B,N,H,d] bf16 local (GatedFWA) branch output */
    void* O_loc_lo; /* [B,N,H,d] bf16 residual of O_loc's cast (C-12) */
    float* LSE_loc; /* [B,H,N] fp32 */
} gfwa_nsa_saved_t;

/*
 * gfwa_nsa_fwd -- forward of the hybrid:
 *   O = sigmoid(g0) o_cmp + sigmoid(g1) o_slc + sigmoid(g2) o_loc
 * with o_loc = gfwa_fwd(Q, K, V, U, w) (the GatedFWA local branch),
 * o_cmp = softmax attention of q_t over the block means (reading C-28: the
 * compression map phi is the block mean, block length = stride = `block`) of
 * the blocks that end at or before t (0 for t < block - 1), and o_slc = softmax
 * attention over the tokens <= t of the selected blocks: the query's own block
 * plus the n_sel complete blocks with the largest compressed-attention scores
 * scale q.Kc_i (reading C-29; ties to the lower index).  Q, K, V, O [B,N,H,d]
 * bf16 packed; U [B,H,N] fp32; gates [B,N,H,3] fp32 logits.  `saved`
 * (nullable) receives the tensors gfwa_nsa_bwd needs.  N / block <= 512.  The
 * compressed and selected branches run on CUDA-core kernels.
 */
size_t gfwa_nsa_workspace_size(const gfwa_nsa_desc_t* desc);
gfwa_status_t gfwa_nsa_fwd(const gfwa_nsa_desc_t* desc, const void* Q, const void* K, const void* V,
                           const float* U, const float* gates, void* O, const gfwa_nsa_saved_t* saved, void* ws,
                           size_t ws_bytes, gfwa_stream_t stream);

/*
 * gfwa_nsa_bwd -- the chain rule of gfwa_nsa_fwd for its (fixed) selection:
 * dgates [B,N,H,3] fp32 (sigmoid'(g_c) dO . o_c), the local branch by
 * gfwa_bwd on sigmoid(g2) dO (dU [B,H,N] from it alone), the compressed branch
 * (query side per query, block side per block, spread back through the block
 * mean) and the selected branch (dK, dV of the selected tokens by fp32
 * atomics); dQ, dK, dV [B,N,H,d] bf16 are the sums.  `saved` must hold every
 * member, as written by gfwa_nsa_fwd on the same inputs.
 */
gfwa_status_t gfwa_nsa_bwd(const gfwa_nsa_desc_t* desc, const void* Q, const void* K, const void* V,
                           const float* U, const float* gates, const void* dO, const gfwa_nsa_saved_t* saved,
                           void* dQ, void* dK, void* dV, float* dU, float* dgates, void* ws, size_t ws_bytes,
                           gfwa_stream_t stream);

/* ------------------------------------------------------------------------- */
/* AttnLayer output epilogue fused into the attention kernels:     */
/*   O~ = concat_h norm(GatedFWA_h),  G = swish(linear(X)),  out = (G . O~) W_O */
/* Reading C-27: norm = RMSNorm over the head dim with a per-channel weight    */
/* gamma[d] shared by the heads; swish(x) = x sigmoid(x) is applied to the     */
/* gate pre-activation g = linear(X) given by the caller; the W_O GEMM stays   */
/* the caller's.  Per (b, t, h) row:                                            */
/*   rstd = 1 / sqrt(mean_c O_c^2 + eps),  Y_c = g_c sigmoid(g_c) gamma_c O_c rstd */
/* ------------------------------------------------------------------------- */
typedef struct {
    const void* g;      /* [B,N_q,H,d] bf16, O's (packed) layout: gate pre-activation */
    const float* gamma; /* [d] fp32 RMSNorm weight, shared by the heads */
    float eps;          /* RMSNorm epsilon, > 0 */
    float* rstd;        /* [B,H,N_q] fp32: written by the forward, read by the backward */
} gfwa_normgate_t;

/*
 * gfwa_fwd_normgate -- gfwa_fwd (bwd_ws == NULL) or gfwa_fwd_train (bwd_ws given)
 * whose epilogue also takes rstd from the fp32 attention output in TMEM (one
 * extra read pass before the output is released), followed by one streaming
 * pass that writes Y [B,N_q,H,d] bf16 (O's layout) from O + O_lo (the fp32
 * output to ~2^-17; O alone when O_lo is NULL), g and gamma: the layer output
 * in one pass over the rows instead of an RMSNorm and a gate kernel chain.
 * O (the attention output O~, needed by the backward) and O_lo are written as
 * by gfwa_fwd.  (Computing Y inside the forward's epilogue warps was measured
 * slower: their global traffic delays the release of the output accumulator.)
 * BF16 tensor-core path only
 * (UNSUPPORTED otherwise); O's layout must be packed [B,N_q,H,d]
 * (INVALID_ARGUMENT otherwise); g, Y 16-byte aligned.
 */
gfwa_status_t gfwa_fwd_normgate(const gfwa_attn_desc_t* desc, const void* Q, const void* K, const void* V,
                                const float* U, const gfwa_normgate_t* ng, void* O, void* O_lo, float* LSE,
                                void* Y, void* bwd_ws, size_t bwd_ws_bytes, gfwa_stream_t stream);

/*
 * gfwa_bwd_normgate -- the layer backward from dY (the gradient of Y): the
 * epilogue's chain rule runs inside the backward's preprocess pass,
 *   dO~ = rstd gamma dn - (rstd^3 O~ / d) sum_c gamma_c dn_c O~_c,  dn = dY swish(g)
 *   dg = dY n swish'(g) (n = gamma O~ rstd),  dgamma = sum over rows of dn O~ rstd
 * with O~ = O + O_lo; dO~ is written to dO (bf16, O's layout: an OUTPUT here)
 * and D = rowsum(O~ * dO~) is taken from those bf16 values (C-12), then Alg.
 * E.2 proceeds exactly as gfwa_bwd.  dg [B,N_q,H,d] bf16; dgamma [d] fp32 is
 * overwritten (zeroed, then accumulated by the call).  Layout and path
 * requirements as gfwa_fwd_normgate; the other arguments as gfwa_bwd.
 */
gfwa_status_t gfwa_bwd_normgate(const gfwa_attn_desc_t* desc, const void* Q, const void* K, const void* V,
                                const float* U, const void* O, const void* O_lo, const float* LSE,
                                const gfwa_normgate_t* ng, const void* dY, void* dO, void* dg, float* dgamma,
                                void* dQ, void* dK, void* dV, float* dU, float* dalpha,
                                const double* dalpha_carry, void* ws, size_t ws_bytes, gfwa_stream_t stream);

/* ------------------------------------------------------------------------- */
/* Decode: one new token per sequence over a rolling w-entry cache.           */
/* The paper claims O(wd) per step with a KV cache but gives no  */
/* algorithm; reading C-16: decode(t) == row t of Eq. 12.                     */
/* ------------------------------------------------------------------------- */

typedef struct {
    int64_t B, H;
    int32_t d;                  /* 64 or 128 */
    int32_t w;                  /* cache length = window */
    float scale;                /* <= 0 selects 1/sqrt(d) */
    float eps;                  /* gate eps for GATE_HBETA */
    gfwa_dtype_t dtype;         /* dtype of q, k_new, v_new, caches, o */
    gfwa_gate_kind_t gate_kind; /* gate_a/gate_b are (h, beta) or (alpha, NULL), fp32 [B,H] */
    int64_t H_kv;               /* K/V heads (GQA): H % H_kv == 0, H/H_kv in {1,2,4,8}; 0 = H */
} gfwa_decode_desc_t;

/*
 * gfwa_decode -- for every (b, hh), with t = pos[b] (tokens already cached
 * before this one) and slot s = t mod w.  U_cache holds gate sums RELATIVE
 * to the newest cached token: U_cache[b,hh,slot(tau)] = u_tau - u_{t-1} >= 0
 * for each cached token tau (so the newest token's slot holds 0; build it from
 * a prefill's U as U[tau] - U[t-1]).  With u_t = u_{t-1} - alpha_t (Eq. 11):
 *   o[b,hh] = sum_i softmax_i(scale q.k_i + u_t - u_i) v_i over the
 *             min(t+1, w) valid slots (ring order is irrelevant), where
 *             u_t - u_i = -(U_cache[i] + alpha_t) and 0 for the new token
 *   K_cache[b,kv(hh),s] = k_new, V_cache[b,kv(hh),s] = v_new, and every valid
 *   U_cache entry becomes relative to u_t (U_cache[i] + alpha_t; slot s: 0).
 * The relative frame keeps the stored values bounded by the window's gate sum
 * at any position, so fp32 storage never swallows small gates (an absolute
 * running u loses them once its ulp exceeds alpha).
 * GQA (heads_per_gqa_group): query head hh reads
 * K/V head hh / (H / H_kv); the gate and U stay per query head.
 * q, o [B,H,d]; k_new, v_new [B,H_kv,d]; K_cache, V_cache [B,H_kv,w,d];
 * U_cache [B,H,w] fp32;
 * pos [B] int64 DEVICE array (graph-capturable).  The caches are updated in
 * place.  ws >= gfwa_decode_workspace_size(desc) bytes; it must be ZEROED once
 * by the caller before first use (the call leaves it zeroed again).
 */
size_t gfwa_decode_workspace_size(const gfwa_decode_desc_t* desc);
gfwa_status_t gfwa_decode(const gfwa_decode_desc_t* desc, const void* q, const void* k_new,
                          const void* v_new, const float* gate_a, const float* gate_b,
                          void* K_cache, void* V_cache, float* U_cache, const int64_t* pos, void* o,
                          void* ws, size_t ws_bytes, gfwa_stream_t stream);

/* ------------------------------------------------------------------------- */
/* Helpers                                                                    */
/* ------------------------------------------------------------------------- */
const char* gfwa_status_string(gfwa_status_t s);
/*
 * gfwa_check_finite -- debug check (SURVEY 8(b) NONFINITE; SPEC's "NaN/Inf is an
 * error surfaced"): GFWA_ERR_NONFINITE if any of the n elements of x (device,
 * dtype F32 or BF16) is NaN or +-Inf, else GFWA_OK.  Unlike every other call it
 * SYNCHRONISES `stream` (it reads a device flag back), so it is opt-in: call it
 * directly, or set GFWA_CHECK_FINITE=1 in the environment to have gfwa_fwd check
 * O and LSE and gfwa_bwd check dQ, dK, dV and dU after their launches.
 */
gfwa_status_t gfwa_check_finite(gfwa_dtype_t dtype, const void* x, int64_t n, gfwa_stream_t stream);

int gfwa_last_cuda_error(void); /* cudaError_t of this thread's last GFWA_ERR_CUDA */
const char* gfwa_version(void);
/* Number of kernel launches the calling thread has issued through this library
 * (monotonic; bench.py reads it to report gpu_launches). */
uint64_t gfwa_launch_count(void);
/* Measurement hook (bench.py's per-kernel roofline): registers up to 4 CUDA
 * events (cudaEvent_t handles, NULL entries allowed) for the calling thread's
 * NEXT tensor-core gfwa_bwd, which records events[0] after its preprocess
 * kernel and events[1] after its main kernel on the call's stream, then
 * forgets them.  Never synchronises; no effect on results. */
void gfwa_debug_stage_events(void* const* events, int n);
/* Which forward/backward implementation a descriptor routes to:
 * 0 = SIMT (fp32 parity path), 1 = tcgen05/TMA tensor-core path. */
int gfwa_attn_path(const gfwa_attn_desc_t* desc);

/* Diagnostic: one 128x128x128 tile through the tensor-core primitives the
 * attention kernels use (TMA 128B-swizzle loads, tcgen05 SS MMA S = Q K^T,
 * bf16 P = S written to TMEM, tcgen05 TS MMA O = P V).  Q, K, V: [128,128]
 * bf16 row-major device arrays; S_out, O_out: [128,128] fp32 device arrays. */
gfwa_status_t gfwa_debug_tc_selftest(const void* Q, const void* K, const void* V, float* S_out, float* O_out,
                                     gfwa_stream_t stream);
/* As above; flags bit 0: P is written to TMEM as fp16 and the TS MMA reads it
 * with A format F16 against the bf16 V (mixed-format kind::f16 probe). */
gfwa_status_t gfwa_debug_tc_selftest_ex(const void* Q, const void* K, const void* V, float* S_out, float* O_out,
                                        int flags, gfwa_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* GFWA_H_ */
