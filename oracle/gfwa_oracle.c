/*
 * gfwa_oracle.c -- plain, slow, fp64 CPU oracle for the GatedFWA hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or helper with the CUDA path under
 * paper_2512_07782_b200/ and never includes or links it.
 *
 * Citations: "P:<line>" is /root/reference/PAPER.md (arXiv 2512.07782, LaTeX
 * source) at that line; "S:<line>" is SPEC.md.  Readings of silent or garbled
 * passages are listed as C-<n> in DESIGN.md §3 and cited here by number.
 *
 * Every function is the plain definition written out, in the paper's order
 * and notation, with no blocking, fusion or reordering:
 *   gate          Eq. 9-11, Alg. 1 lines 5-10
 *   forward       Eq. 12, LSE as Alg. 2 line 19
 *   backward      Alg. E.2 written densely per row
 *   d-alpha       reverse cumsum of dU ("gradients into U flow
 *                 through the same streamed scan")
 *   gate chain    chain rule through Eq. 9-10
 *   attend_row    one query over an explicit key list (decode, C-16)
 *
 * Array layouts (all row-major, fp64):
 *   h, beta, dh, dbeta       [B][N][H]
 *   alpha, U, dU, dalpha     [B][H][N]
 *   Q, O, dO, dQ             [B][Nq][H][d]
 *   K, V, dK, dV             [B][Nkv][H][d]
 *   LSE                      [B][H][Nq]
 * Query t (0 <= t < Nq) sits at key index t + h0, h0 = Nkv - Nq (halo rows,
 * BASELINE.json north_star sequence sharding); its window is the key set
 * W(t) = { j : max(0, t+h0-w+1) <= j <= t+h0 } (Alg. 2 line 14 P:382).
 *
 * Parity status: every function here is pinned by tests/test_oracle_pins.py
 * (closed forms, worked examples, library routines, finite differences and
 * the brute-force Prop. 2 recurrence); see DESIGN.md §4 for the pin table.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* thread count for the OpenMP loops (benchmark plumbing; no arithmetic) */
void oracle_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* softplus(z) = log(1 + e^z).  Alg. 1 line 6 writes
 * nu + log(e^{z-nu} + e^{-nu}), nu = max(z,0); reading C-6: the same value
 * written as max(z,0) + log1p(exp(-|z|)) so that z << 0 keeps relative
 * accuracy. */
static double softplus(double z) { return fmax(z, 0.0) + log1p(exp(-fabs(z))); }

static double sigmoid(double z) { return 1.0 / (1.0 + exp(-z)); }

/* Gate alpha, Eq. 9 with the kernel's eps (Alg. 1 line 7, P:229,
 * reading C-5: eps = caller's value, default 1e-6):
 *   alpha = softplus(beta * h) / (beta + eps). */
static double gate_alpha(double h, double beta, double eps) {
    double z = beta * h;                 /* Alg. 1 line 5 */
    return softplus(z) / (beta + eps);   /* Alg. 1 lines 6-7 */
}

/*
 * oracle_gate_alpha: alpha[b][hh][t] from h, beta (Eq. 9-10).
 */
void oracle_gate_alpha(const double* h, const double* beta, int64_t B, int64_t N, int64_t H,
                       double eps, double* alpha) {
    for (int64_t b = 0; b < B; ++b)
        for (int64_t t = 0; t < N; ++t)
            for (int64_t hh = 0; hh < H; ++hh) {
                int64_t i = (b * N + t) * H + hh;
                alpha[(b * H + hh) * N + t] = gate_alpha(h[i], beta[i], eps);
            }
}

/*
 * oracle_gate_prefix: Eq. 11 u_t = sum_{q<=t} -alpha_q, an inclusive
 * prefix (reading C-8), plus an optional carry (the exclusive prefix of the
 * previous shards, BASELINE.json north_star "cross-rank exclusive scan"):
 *   U[b][h][t] = carry[b][h] - sum_{q=0..t} alpha[b][h][q]
 * alpha is given directly ([B][H][N]).  total[b][h] = sum_q alpha (may be NULL).
 * Sequential fp64 accumulation, Alg. 1 lines 8 and 10 with B_t = 1.
 */
void oracle_gate_prefix(const double* alpha, int64_t B, int64_t N, int64_t H,
                        const double* carry, double* U, double* total) {
    for (int64_t b = 0; b < B; ++b)
        for (int64_t hh = 0; hh < H; ++hh) {
            const double* a = alpha + (b * H + hh) * N;
            double* u = U + (b * H + hh) * N;
            double acc = carry ? carry[b * H + hh] : 0.0;
            double s = 0.0;
            for (int64_t t = 0; t < N; ++t) {
                acc -= a[t];
                s += a[t];
                u[t] = acc;
            }
            if (total) total[b * H + hh] = s;
        }
}

/* Window of query t (at key index g = t + h0): keys j in [lo, g],
 * lo = max(0, g - w + 1)  ("i-w < j <= i"; "q-w+1 <= g <= q";
 * reading C-2: clipped at key 0). */
static int64_t win_lo(int64_t g, int64_t w) { return g - w + 1 > 0 ? g - w + 1 : 0; }

/* Logit of Eq. 12: Phi_tj + B_tj with Phi = scale * q.k (Eq. 1; reading
 * C-1: scale on q.k only) and B_tj = u_t - u_j (Eq. 11). */
static double logit(const double* q, const double* k, int64_t d, double scale, double ut, double uj) {
    double dot = 0.0;
    for (int64_t c = 0; c < d; ++c) dot += q[c] * k[c];
    return scale * dot + (ut - uj);
}

/*
 * One forward row: Eq. 12 for query t of slice (b, hh).
 * Writes o[d] and returns LSE = m + log(l) (Alg. 2 line 19; reading
 * C-10: natural log, bias included).  s[] is caller scratch of >= w entries.
 */
static double fwd_row(const double* Q, const double* K, const double* V, const double* U,
                      int64_t Nq, int64_t Nkv, int64_t H, int64_t d, int64_t w, double scale,
                      int64_t b, int64_t hh, int64_t t, double* o, double* s) {
    const int64_t h0 = Nkv - Nq;
    const int64_t g = t + h0;
    const int64_t lo = win_lo(g, w);
    const double* q = Q + ((b * Nq + t) * H + hh) * d;
    const double* u = U + (b * H + hh) * Nkv;
    double m = -INFINITY;
    for (int64_t j = lo; j <= g; ++j) {
        s[j - lo] = logit(q, K + ((b * Nkv + j) * H + hh) * d, d, scale, u[g], u[j]);
        if (s[j - lo] > m) m = s[j - lo];
    }
    double l = 0.0;
    for (int64_t j = lo; j <= g; ++j) l += exp(s[j - lo] - m);
    for (int64_t c = 0; c < d; ++c) o[c] = 0.0;
    for (int64_t j = lo; j <= g; ++j) {
        double p = exp(s[j - lo] - m) / l;   /* S~_tj of Eq. 12 */
        const double* v = V + ((b * Nkv + j) * H + hh) * d;
        for (int64_t c = 0; c < d; ++c) o[c] += p * v[c];
    }
    return m + log(l);
}

/*
 * oracle_fwd: O = S~ V with S~ from Eq. 12, LSE per Alg. 2.
 */
void oracle_fwd(int64_t B, int64_t H, int64_t Nq, int64_t Nkv, int64_t d, int64_t w, double scale,
                const double* Q, const double* K, const double* V, const double* U,
                double* O, double* LSE) {
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int64_t b = 0; b < B; ++b)
        for (int64_t hh = 0; hh < H; ++hh) {
            double* s = (double*)malloc(sizeof(double) * (size_t)(w < Nkv ? w : Nkv));
            for (int64_t t = 0; t < Nq; ++t) {
                double lse = fwd_row(Q, K, V, U, Nq, Nkv, H, d, w, scale, b, hh, t,
                                     O + ((b * Nq + t) * H + hh) * d, s);
                if (LSE) LSE[(b * H + hh) * Nq + t] = lse;
            }
            free(s);
        }
}

/*
 * oracle_fwd_rows: the same definition evaluated only for n listed rows
 * (b, hh, t) = (rows[3i], rows[3i+1], rows[3i+2]); outputs o_out[n][d],
 * lse_out[n].  Used to check sampled rows at full benchmark sizes.
 */
void oracle_fwd_rows(int64_t B, int64_t H, int64_t Nq, int64_t Nkv, int64_t d, int64_t w, double scale,
                     const double* Q, const double* K, const double* V, const double* U,
                     int64_t n, const int64_t* rows, double* o_out, double* lse_out) {
    (void)B;
#pragma omp parallel for schedule(dynamic)
    for (int64_t i = 0; i < n; ++i) {
        double* s = (double*)malloc(sizeof(double) * (size_t)(w < Nkv ? w : Nkv));
        double lse = fwd_row(Q, K, V, U, Nq, Nkv, H, d, w, scale, rows[3 * i], rows[3 * i + 1],
                             rows[3 * i + 2], o_out + i * d, s);
        if (lse_out) lse_out[i] = lse;
        free(s);
    }
}

/*
 * oracle_attend_row: one query over an explicit ordered key list (decode,
 * reading C-16: decode(t) == row t of Eq. 12 over the last min(t+1,w) tokens).
 *   o = sum_i softmax_i(scale*q.k_i + (u_t - u_i)) v_i,  i = 0..n-1
 * keys [n][d], vals [n][d], u[n] (the u of each key token), ut = u of the query.
 * Returns the natural-log LSE.
 */
double oracle_attend_row(int64_t d, double scale, const double* q, int64_t n, const double* keys,
                         const double* vals, const double* u, double ut, double* o) {
    double m = -INFINITY;
    double* s = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
        s[i] = logit(q, keys + i * d, d, scale, ut, u[i]);
        if (s[i] > m) m = s[i];
    }
    double l = 0.0;
    for (int64_t i = 0; i < n; ++i) l += exp(s[i] - m);
    for (int64_t c = 0; c < d; ++c) o[c] = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double p = exp(s[i] - m) / l;
        for (int64_t c = 0; c < d; ++c) o[c] += p * vals[i * d + c];
    }
    free(s);
    return m + log(l);
}

/*
 * oracle_bwd: Alg. E.2 written densely, one (b, hh) slice at a
 * time, with readings C-3 (sm_scale on dQ and dK), C-4 ("du^k -= rowsum(ds)"
 * is the sum over queries of column j), C-11 (dU^q = rowsum(dS) is kept):
 *   P_tj  = exp(s_tj - LSE_t)
 *   dP_tj = dO_t . v_j
 *   D_t   = O_t . dO_t                              (O is this
 *                                                     oracle's own fp64 O)
 *   dS_tj = P_tj (dP_tj - D_t)
 *   dV_j += P_tj dO_t
 *   dQ_t += scale dS_tj k_j                         (C-3)
 *   dK_j += scale dS_tj q_t                         (C-3)
 *   dU^q_t += sum_j dS_tj ; dU^k_j -= sum_t dS_tj   (C-4)
 *   dU = dU^q + dU^k
 * dU is indexed by key position (Nkv rows); query t contributes its row sum
 * at key index t + h0.
 * If dalpha != NULL: dalpha[m] = carry - sum_{m' >= m} dU[m'] (reverse cumsum,
 * P:276; d/dalpha of Eq. 11 with the carry of later shards).
 */
void oracle_bwd(int64_t B, int64_t H, int64_t Nq, int64_t Nkv, int64_t d, int64_t w, double scale,
                const double* Q, const double* K, const double* V, const double* U,
                const double* dO, double* dQ, double* dK, double* dV, double* dU,
                double* dalpha, const double* dalpha_carry) {
    const int64_t h0 = Nkv - Nq;
    memset(dQ, 0, sizeof(double) * (size_t)(B * Nq * H * d));
    memset(dK, 0, sizeof(double) * (size_t)(B * Nkv * H * d));
    memset(dV, 0, sizeof(double) * (size_t)(B * Nkv * H * d));
    memset(dU, 0, sizeof(double) * (size_t)(B * H * Nkv));
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int64_t b = 0; b < B; ++b)
        for (int64_t hh = 0; hh < H; ++hh) {
            int64_t wmax = w < Nkv ? w : Nkv;
            double* s = (double*)malloc(sizeof(double) * (size_t)wmax);
            double* o = (double*)malloc(sizeof(double) * (size_t)d);
            double* du = dU + (b * H + hh) * Nkv;
            for (int64_t t = 0; t < Nq; ++t) {
                const int64_t g = t + h0;
                const int64_t lo = win_lo(g, w);
                const double* q = Q + ((b * Nq + t) * H + hh) * d;
                const double* dot = dO + ((b * Nq + t) * H + hh) * d;
                double* dq = dQ + ((b * Nq + t) * H + hh) * d;
                /* forward quantities of this row (recompute, as P:1095-1100) */
                double lse = fwd_row(Q, K, V, U, Nq, Nkv, H, d, w, scale, b, hh, t, o, s);
                double D = 0.0;
                for (int64_t c = 0; c < d; ++c) D += o[c] * dot[c];
                double rowsum = 0.0;
                for (int64_t j = lo; j <= g; ++j) {
                    const double* k = K + ((b * Nkv + j) * H + hh) * d;
                    const double* v = V + ((b * Nkv + j) * H + hh) * d;
                    double* dk = dK + ((b * Nkv + j) * H + hh) * d;
                    double* dv = dV + ((b * Nkv + j) * H + hh) * d;
                    double P = exp(s[j - lo] - lse);
                    double dP = 0.0;
                    for (int64_t c = 0; c < d; ++c) dP += dot[c] * v[c];
                    double dS = P * (dP - D);
                    for (int64_t c = 0; c < d; ++c) {
                        dv[c] += P * dot[c];
                        dq[c] += scale * dS * k[c];
                        dk[c] += scale * dS * q[c];
                    }
                    rowsum += dS;
                    du[j] -= dS;          /* dU^k, column sum (C-4) */
                }
                du[g] += rowsum;          /* dU^q, row sum (C-11) */
            }
            if (dalpha) {
                double* da = dalpha + (b * H + hh) * Nkv;
                double acc = dalpha_carry ? dalpha_carry[b * H + hh] : 0.0;
                for (int64_t m = Nkv - 1; m >= 0; --m) {
                    acc -= du[m];
                    da[m] = acc;
                }
            }
            free(s);
            free(o);
        }
}

/*
 * oracle_dalpha: dalpha[b][h][m] = carry[b][h] - sum_{m'>=m} dU[b][h][m']
 * (derivative of Eq. 11, through the reverse scan of P:276).
 */
void oracle_dalpha(const double* dU, int64_t B, int64_t H, int64_t N, const double* carry,
                   double* dalpha) {
    for (int64_t bh = 0; bh < B * H; ++bh) {
        double acc = carry ? carry[bh] : 0.0;
        for (int64_t m = N - 1; m >= 0; --m) {
            acc -= dU[bh * N + m];
            dalpha[bh * N + m] = acc;
        }
    }
}

/*
 * oracle_gate_chain: chain rule of Eq. 9 with the kernel eps
 * (S:134-142 gives the same derivatives):
 *   d alpha / d h    = sigmoid(beta h) beta / (beta + eps)
 *   d alpha / d beta = [sigmoid(beta h) h (beta + eps) - softplus(beta h)] / (beta + eps)^2
 * dalpha [B][H][N] -> dh, dbeta [B][N][H].
 */
void oracle_gate_chain(const double* h, const double* beta, const double* dalpha, int64_t B,
                       int64_t N, int64_t H, double eps, double* dh, double* dbeta) {
    for (int64_t b = 0; b < B; ++b)
        for (int64_t t = 0; t < N; ++t)
            for (int64_t hh = 0; hh < H; ++hh) {
                int64_t i = (b * N + t) * H + hh;
                double z = beta[i] * h[i];
                double be = beta[i] + eps;
                double da = dalpha[(b * H + hh) * N + t];
                dh[i] = da * sigmoid(z) * beta[i] / be;
                dbeta[i] = da * (sigmoid(z) * h[i] * be - softplus(z)) / (be * be);
            }
}

/*
 * AttnLayer output epilogue (§3 "(3) Block Structure"):
 *   O~ = concat_h norm(O~^(h)),  G = swish(linear(X)),  out = (G (.) O~) W_O
 * Reading C-27: norm is an RMSNorm over the head dim d with a per-channel
 * weight gamma[d] shared by the heads, swish(x) = x sigmoid(x) is applied to
 * the gate pre-activation g = linear(X) (given), and the W_O product is the
 * caller's GEMM.  Per row (b, t, h) of O [B][Nq][H][d]:
 *   r   = 1 / sqrt( (1/d) sum_c O_c^2 + eps )
 *   n_c = gamma_c O_c r
 *   Y_c = g_c sigmoid(g_c) n_c
 * rstd [B][H][Nq] receives r.
 */
void oracle_normgate_fwd(const double* O, const double* g, const double* gamma, int64_t B, int64_t Nq,
                         int64_t H, int64_t d, double eps, double* Y, double* rstd) {
    for (int64_t b = 0; b < B; ++b)
        for (int64_t t = 0; t < Nq; ++t)
            for (int64_t hh = 0; hh < H; ++hh) {
                const int64_t row = ((b * Nq + t) * H + hh) * d;
                double ms = 0.0;
                for (int64_t c = 0; c < d; ++c) ms += O[row + c] * O[row + c];
                ms /= (double)d;
                double r = 1.0 / sqrt(ms + eps);
                rstd[(b * H + hh) * Nq + t] = r;
                for (int64_t c = 0; c < d; ++c) {
                    double n = gamma[c] * O[row + c] * r;
                    double G = g[row + c] * sigmoid(g[row + c]);
                    Y[row + c] = G * n;
                }
            }
}

/*
 * Chain rule of oracle_normgate_fwd (C-27), given dY [B][Nq][H][d]:
 *   dn_c     = dY_c G_c                     (n_c = gamma_c O_c r)
 *   dg_c     = dY_c n_c (sigmoid(g_c) + g_c sigmoid(g_c) (1 - sigmoid(g_c)))
 *   dgamma_c = sum over every row of dn_c O_c r
 *   dO_k     = r gamma_k dn_k - (r^3 O_k / d) sum_c gamma_c dn_c O_c
 * (dr/dO_k = -r^3 O_k / d).  dO feeds Alg. E.2 as the attention output's gradient.
 */
void oracle_normgate_bwd(const double* O, const double* g, const double* gamma, const double* dY, int64_t B,
                         int64_t Nq, int64_t H, int64_t d, double eps, double* dO, double* dg, double* dgamma) {
    for (int64_t c = 0; c < d; ++c) dgamma[c] = 0.0;
    for (int64_t b = 0; b < B; ++b)
        for (int64_t t = 0; t < Nq; ++t)
            for (int64_t hh = 0; hh < H; ++hh) {
                const int64_t row = ((b * Nq + t) * H + hh) * d;
                double ms = 0.0;
                for (int64_t c = 0; c < d; ++c) ms += O[row + c] * O[row + c];
                ms /= (double)d;
                double r = 1.0 / sqrt(ms + eps);
                double s = 0.0; /* sum_c gamma_c dn_c O_c */
                for (int64_t c = 0; c < d; ++c) {
                    double sg = sigmoid(g[row + c]);
                    double G = g[row + c] * sg;
                    double n = gamma[c] * O[row + c] * r;
                    double dn = dY[row + c] * G;
                    dg[row + c] = dY[row + c] * n * (sg + g[row + c] * sg * (1.0 - sg));
                    dgamma[c] += dn * O[row + c] * r;
                    s += gamma[c] * dn * O[row + c];
                }
                for (int64_t k = 0; k < d; ++k) {
                    double dn = dY[row + k] * g[row + k] * sigmoid(g[row + k]);
                    dO[row + k] = r * gamma[k] * dn - r * r * r * O[row + k] / (double)d * s;
                }
            }
}

/*
 * NSA extension with GatedFWA as the local branch (App. B; readings
 * C-28, C-29).  Token compression: phi = the block MEAN (C-28: the
 * learnable MLP replaced by its parameter-free mean, block length = stride =
 * blk); compressed attention over the blocks that end at or before t; block
 * selection by the compressed-attention score, top n_sel of those
 * blocks plus the query's own block (C-29); selected attention over the tokens
 * <= t of the selected blocks; output sum_c sigmoid(g_c) o_c.
 */
/* Kc, Vc [B][nb][H][d], nb = N / blk (complete blocks) */
void oracle_nsa_compress(const double* K, const double* V, int64_t B, int64_t N, int64_t H, int64_t d, int64_t blk,
                         double* Kc, double* Vc) {
    const int64_t nb = N / blk;
    for (int64_t b = 0; b < B; ++b)
        for (int64_t i = 0; i < nb; ++i)
            for (int64_t hh = 0; hh < H; ++hh)
                for (int64_t c = 0; c < d; ++c) {
                    double sk = 0.0, sv = 0.0;
                    for (int64_t j = i * blk; j < (i + 1) * blk; ++j) {
                        sk += K[((b * N + j) * H + hh) * d + c];
                        sv += V[((b * N + j) * H + hh) * d + c];
                    }
                    Kc[((b * nb + i) * H + hh) * d + c] = sk / (double)blk;
                    Vc[((b * nb + i) * H + hh) * d + c] = sv / (double)blk;
                }
}

/* o_cmp [B][N][H][d]: softmax over the blocks i with (i+1) blk - 1 <= t of
 * scale q.Kc_i (0 when t < blk - 1); scores [B][H][N][nb] (-inf for blocks not complete) */
void oracle_nsa_cmp(const double* Q, const double* Kc, const double* Vc, int64_t B, int64_t N, int64_t H, int64_t d,
                    int64_t blk, double scale, double* Ocmp, double* scores) {
    const int64_t nb = N / blk;
    for (int64_t b = 0; b < B; ++b)
        for (int64_t hh = 0; hh < H; ++hh)
            for (int64_t t = 0; t < N; ++t) {
                const double* q = Q + ((b * N + t) * H + hh) * d;
                double* sc = scores + ((b * H + hh) * N + t) * nb;
                const int64_t nc = (t + 1) / blk;
                double m = -INFINITY;
                for (int64_t i = 0; i < nb; ++i) {
                    sc[i] = -INFINITY;
                    if (i >= nc) continue;
                    double s = 0.0;
                    for (int64_t c = 0; c < d; ++c) s += q[c] * Kc[((b * nb + i) * H + hh) * d + c];
                    sc[i] = scale * s;
                    if (sc[i] > m) m = sc[i];
                }
                double* o = Ocmp + ((b * N + t) * H + hh) * d;
                for (int64_t c = 0; c < d; ++c) o[c] = 0.0;
                if (nc == 0) continue;
                double l = 0.0;
                for (int64_t i = 0; i < nc; ++i) l += exp(sc[i] - m);
                for (int64_t i = 0; i < nc; ++i) {
                    const double p = exp(sc[i] - m) / l;
                    for (int64_t c = 0; c < d; ++c) o[c] += p * Vc[((b * nb + i) * H + hh) * d + c];
                }
            }
}

/* sel [B][H][N][nsel + 1]: the query's own block t / blk first, then the n_sel
 * complete blocks (other than its own) with the largest scores, ties to the lower
 * index; -1 where fewer exist */
void oracle_nsa_select(const double* scores, int64_t B, int64_t H, int64_t N, int64_t blk, int64_t nsel,
                       int64_t* sel) {
    const int64_t nb = N / blk;
    for (int64_t bh = 0; bh < B * H; ++bh)
        for (int64_t t = 0; t < N; ++t) {
            const double* sc = scores + (bh * N + t) * nb;
            int64_t* out = sel + (bh * N + t) * (nsel + 1);
            const int64_t own = t / blk;
            out[0] = own;
            for (int64_t k = 1; k <= nsel; ++k) {
                int64_t best = -1;
                for (int64_t i = 0; i < nb; ++i) {
                    if (i == own || sc[i] == -INFINITY) continue;
                    int taken = 0;
                    for (int64_t q = 1; q < k; ++q) taken |= out[q] == i;
                    if (taken) continue;
                    if (best < 0 || sc[i] > sc[best]) best = i;
                }
                out[k] = best;
            }
        }
}

/* o_slc [B][N][H][d]: softmax of scale q.k_j over the tokens j <= t of the selected blocks */
void oracle_nsa_slc(const double* Q, const double* K, const double* V, const int64_t* sel, int64_t B, int64_t N,
                    int64_t H, int64_t d, int64_t blk, int64_t nsel, double scale, double* Oslc) {
    for (int64_t b = 0; b < B; ++b)
        for (int64_t hh = 0; hh < H; ++hh)
            for (int64_t t = 0; t < N; ++t) {
                const double* q = Q + ((b * N + t) * H + hh) * d;
                const int64_t* sl = sel + ((b * H + hh) * N + t) * (nsel + 1);
                double m = -INFINITY;
                for (int64_t k = 0; k <= nsel; ++k) {
                    if (sl[k] < 0) continue;
                    for (int64_t j = sl[k] * blk; j < (sl[k] + 1) * blk && j <= t; ++j) {
                        double s = 0.0;
                        for (int64_t c = 0; c < d; ++c) s += q[c] * K[((b * N + j) * H + hh) * d + c];
                        if (scale * s > m) m = scale * s;
                    }
                }
                double l = 0.0;
                double* o = Oslc + ((b * N + t) * H + hh) * d;
                for (int64_t c = 0; c < d; ++c) o[c] = 0.0;
                for (int64_t k = 0; k <= nsel; ++k) {
                    if (sl[k] < 0) continue;
                    for (int64_t j = sl[k] * blk; j < (sl[k] + 1) * blk && j <= t; ++j) {
                        double s = 0.0;
                        for (int64_t c = 0; c < d; ++c) s += q[c] * K[((b * N + j) * H + hh) * d + c];
                        const double e = exp(scale * s - m);
                        l += e;
                        for (int64_t c = 0; c < d; ++c) o[c] += e * V[((b * N + j) * H + hh) * d + c];
                    }
                }
                for (int64_t c = 0; c < d; ++c) o[c] /= l;
            }
}

/* o = sigmoid(g0) o_cmp + sigmoid(g1) o_slc + sigmoid(g2) o_loc; g [B][N][H][3] */
void oracle_nsa_combine(const double* Ocmp, const double* Oslc, const double* Oloc, const double* g, int64_t B,
                        int64_t N, int64_t H, int64_t d, double* O) {
    for (int64_t r = 0; r < B * N * H; ++r) {
        const double a = sigmoid(g[3 * r]), s = sigmoid(g[3 * r + 1]), l = sigmoid(g[3 * r + 2]);
        for (int64_t c = 0; c < d; ++c) O[r * d + c] = a * Ocmp[r * d + c] + s * Oslc[r * d + c] + l * Oloc[r * d + c];
    }
}

/*
 * Chain rule of the NSA hybrid for a FIXED selection sel (the top-n
 * choice is piecewise constant, C-29): with dO_c = sigmoid(g_c) dO,
 *   dg_c   = sigmoid(g_c) (1 - sigmoid(g_c)) dO . o_c
 *   local  = Alg. E.2 on dO_loc (oracle_bwd), dU from it alone
 *   cmp    p_i softmax over complete blocks, dS_i = p_i (dO_cmp . Vc_i - D),
 *          D = sum_i p_i dO_cmp . Vc_i;  dq += scale dS_i Kc_i;  dKc_i += scale dS_i q;
 *          dVc_i += p_i dO_cmp;  dK_j, dV_j += dKc_i / blk, dVc_i / blk for j in block i
 *   slc    the same over the tokens <= t of the selected blocks, into dQ, dK, dV
 * dQ, dK, dV, dg [B][N][H][3] overwritten; dU [B][H][N].
 */
void oracle_nsa_bwd(const double* Q, const double* K, const double* V, const double* U, const double* g,
                    const double* dO, const int64_t* sel, int64_t B, int64_t N, int64_t H, int64_t d, int64_t w,
                    int64_t blk, int64_t nsel, double scale, double* dQ, double* dK, double* dV, double* dU,
                    double* dg) {
    const int64_t nb = N / blk, rows = B * N * H, n = rows * d;
    double* Kc = (double*)calloc((size_t)(B * (nb > 0 ? nb : 1) * H * d), sizeof(double));
    double* Vc = (double*)calloc((size_t)(B * (nb > 0 ? nb : 1) * H * d), sizeof(double));
    double* dKc = (double*)calloc((size_t)(B * (nb > 0 ? nb : 1) * H * d), sizeof(double));
    double* dVc = (double*)calloc((size_t)(B * (nb > 0 ? nb : 1) * H * d), sizeof(double));
    double* Oc = (double*)malloc(sizeof(double) * (size_t)n);
    double* Os = (double*)malloc(sizeof(double) * (size_t)n);
    double* Ol = (double*)malloc(sizeof(double) * (size_t)n);
    double* L = (double*)malloc(sizeof(double) * (size_t)rows);
    double* sc = (double*)malloc(sizeof(double) * (size_t)(B * H * N * (nb > 0 ? nb : 1)));
    double* dOl = (double*)malloc(sizeof(double) * (size_t)n);
    double* dQl = (double*)malloc(sizeof(double) * (size_t)n);
    double* dKl = (double*)malloc(sizeof(double) * (size_t)n);
    double* dVl = (double*)malloc(sizeof(double) * (size_t)n);
    if (nb > 0) oracle_nsa_compress(K, V, B, N, H, d, blk, Kc, Vc);
    oracle_nsa_cmp(Q, Kc, Vc, B, N, H, d, blk, scale, Oc, sc);
    oracle_nsa_slc(Q, K, V, sel, B, N, H, d, blk, nsel, scale, Os);
    oracle_fwd(B, H, N, N, d, w, scale, Q, K, V, U, Ol, L);
    memset(dQ, 0, sizeof(double) * (size_t)n);
    memset(dK, 0, sizeof(double) * (size_t)n);
    memset(dV, 0, sizeof(double) * (size_t)n);
    /* combination */
    for (int64_t r = 0; r < rows; ++r) {
        const double* o[3] = {Oc + r * d, Os + r * d, Ol + r * d};
        for (int cix = 0; cix < 3; ++cix) {
            const double sg = sigmoid(g[3 * r + cix]);
            double dot = 0.0;
            for (int64_t c = 0; c < d; ++c) dot += dO[r * d + c] * o[cix][c];
            dg[3 * r + cix] = sg * (1.0 - sg) * dot;
        }
        const double sl = sigmoid(g[3 * r + 2]);
        for (int64_t c = 0; c < d; ++c) dOl[r * d + c] = sl * dO[r * d + c];
    }
    /* local branch: Alg. E.2 */
    oracle_bwd(B, H, N, N, d, w, scale, Q, K, V, U, dOl, dQl, dKl, dVl, dU, NULL, NULL);
    for (int64_t e = 0; e < n; ++e) {
        dQ[e] += dQl[e];
        dK[e] += dKl[e];
        dV[e] += dVl[e];
    }
    /* compressed and selected branches */
    for (int64_t b = 0; b < B; ++b)
        for (int64_t hh = 0; hh < H; ++hh)
            for (int64_t t = 0; t < N; ++t) {
                const int64_t r = (b * N + t) * H + hh;
                const double* q = Q + r * d;
                const double sgc = sigmoid(g[3 * r]), sgs = sigmoid(g[3 * r + 1]);
                /* cmp */
                const int64_t nc = (t + 1) / blk;
                if (nc > 0) {
                    const double* s = sc + ((b * H + hh) * N + t) * nb;
                    double m = -INFINITY, l = 0.0, D = 0.0;
                    for (int64_t i = 0; i < nc; ++i) m = s[i] > m ? s[i] : m;
                    for (int64_t i = 0; i < nc; ++i) l += exp(s[i] - m);
                    for (int64_t i = 0; i < nc; ++i) {
                        double dp = 0.0;
                        for (int64_t c = 0; c < d; ++c) dp += sgc * dO[r * d + c] * Vc[((b * nb + i) * H + hh) * d + c];
                        D += exp(s[i] - m) / l * dp;
                    }
                    for (int64_t i = 0; i < nc; ++i) {
                        const double p = exp(s[i] - m) / l;
                        double dp = 0.0;
                        for (int64_t c = 0; c < d; ++c) dp += sgc * dO[r * d + c] * Vc[((b * nb + i) * H + hh) * d + c];
                        const double ds = p * (dp - D);
                        for (int64_t c = 0; c < d; ++c) {
                            dQ[r * d + c] += scale * ds * Kc[((b * nb + i) * H + hh) * d + c];
                            dKc[((b * nb + i) * H + hh) * d + c] += scale * ds * q[c];
                            dVc[((b * nb + i) * H + hh) * d + c] += p * sgc * dO[r * d + c];
                        }
                    }
                }
                /* slc */
                const int64_t* sl = sel + ((b * H + hh) * N + t) * (nsel + 1);
                double m = -INFINITY, l = 0.0, D = 0.0;
                for (int64_t k = 0; k <= nsel; ++k)
                    for (int64_t j = sl[k] * blk; sl[k] >= 0 && j < (sl[k] + 1) * blk && j <= t; ++j) {
                        double s = 0.0;
                        for (int64_t c = 0; c < d; ++c) s += q[c] * K[((b * N + j) * H + hh) * d + c];
                        m = scale * s > m ? scale * s : m;
                    }
                for (int64_t k = 0; k <= nsel; ++k)
                    for (int64_t j = sl[k] * blk; sl[k] >= 0 && j < (sl[k] + 1) * blk && j <= t; ++j) {
                        double s = 0.0, dp = 0.0;
                        for (int64_t c = 0; c < d; ++c) {
                            s += q[c] * K[((b * N + j) * H + hh) * d + c];
                            dp += sgs * dO[r * d + c] * V[((b * N + j) * H + hh) * d + c];
                        }
                        l += exp(scale * s - m);
                        D += exp(scale * s - m) * dp;
                    }
                D /= l;
                for (int64_t k = 0; k <= nsel; ++k)
                    for (int64_t j = sl[k] * blk; sl[k] >= 0 && j < (sl[k] + 1) * blk && j <= t; ++j) {
                        double s = 0.0, dp = 0.0;
                        for (int64_t c = 0; c < d; ++c) {
                            s += q[c] * K[((b * N + j) * H + hh) * d + c];
                            dp += sgs * dO[r * d + c] * V[((b * N + j) * H + hh) * d + c];
                        }
                        const double p = exp(scale * s - m) / l, ds = p * (dp - D);
                        for (int64_t c = 0; c < d; ++c) {
                            dQ[r * d + c] += scale * ds * K[((b * N + j) * H + hh) * d + c];
                            dK[((b * N + j) * H + hh) * d + c] += scale * ds * q[c];
                            dV[((b * N + j) * H + hh) * d + c] += p * sgs * dO[r * d + c];
                        }
                    }
            }
    /* compression: block means spread back */
    for (int64_t b = 0; b < B; ++b)
        for (int64_t i = 0; i < nb; ++i)
            for (int64_t hh = 0; hh < H; ++hh)
                for (int64_t c = 0; c < d; ++c)
                    for (int64_t j = i * blk; j < (i + 1) * blk; ++j) {
                        dK[((b * N + j) * H + hh) * d + c] += dKc[((b * nb + i) * H + hh) * d + c] / (double)blk;
                        dV[((b * N + j) * H + hh) * d + c] += dVc[((b * nb + i) * H + hh) * d + c] / (double)blk;
                    }
    free(Kc); free(Vc); free(dKc); free(dVc); free(Oc); free(Os); free(Ol); free(L); free(sc);
    free(dOl); free(dQl); free(dKl); free(dVl);
}
