#include <initializer_list>
// capi.cu -- argument validation, dispatch and helpers of the libgfwa C ABI
// (include/gfwa.h).  No allocation, no synchronisation, no host reads of
// device data; every launch goes onto the caller's stream.
#include <atomic>
#include <cmath>

#include "attn_common.cuh"
#include "driver_api.cuh"

namespace gfwa {

static std::atomic<uint64_t> g_launches{0};
static thread_local int g_last_cuda_error = 0;

void note_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

static thread_local cudaEvent_t g_stage_ev[4] = {nullptr, nullptr, nullptr, nullptr};
void stage_event(int stage, cudaStream_t st) {
    if (stage < 0 || stage >= 4 || !g_stage_ev[stage]) return;
    cudaEventRecord(g_stage_ev[stage], st);
    g_stage_ev[stage] = nullptr;
}

gfwa_status_t check_launch(cudaError_t err) {
    if (err == cudaSuccess) return GFWA_OK;
    g_last_cuda_error = (int)err;
    return GFWA_ERR_CUDA;
}

// Tensor-core (tcgen05) path hooks; defined in attn_tc_fwd.cu / attn_tc_bwd.cu.
bool tc_fwd_supported(const AttnParams& p, gfwa_dtype_t dt);
gfwa_status_t tc_fwd(const AttnParams& p, cudaStream_t st);
bool tc_bwd_supported(const AttnParams& p, gfwa_dtype_t dt);
size_t tc_bwd_workspace(const AttnParams& p);
gfwa_status_t tc_bwd(const AttnParams& p, cudaStream_t st, void* ws);

// reverse scan dU -> dalpha (gate_scan.cu internals via the public call)
}  // namespace gfwa

using namespace gfwa;

namespace {

// [B, N, H, d] with no gaps (the debug finite check walks such tensors flat)
bool packed(const int64_t* st, const AttnParams& p) {
    return st[2] == p.d && st[1] == p.H * p.d && st[0] == p.Nq * p.H * p.d;
}
bool packed_kv(const int64_t* st, const AttnParams& p) {
    return st[2] == p.d && st[1] == p.Hkv * p.d && st[0] == p.Nkv * p.Hkv * p.d;
}
bool check_finite_env();

// gfwa_fwd_train hands its preparation to the shared gfwa_fwd body (per thread)
struct Prepare {
    float* zero_acc = nullptr;
    unsigned long long* token = nullptr;
    unsigned long long token_val = 0;
};
thread_local Prepare g_prepare;

// gfwa_fwd_normgate / gfwa_bwd_normgate hand the AttnLayer epilogue (C-27) to the shared
// gfwa_fwd / gfwa_bwd bodies (per thread)
struct NormGate {
    const gfwa_normgate_t* ng = nullptr;
    void* Y = nullptr;         // forward output
    const void* dY = nullptr;  // backward input
    void* dg = nullptr;
    float* dgamma = nullptr;
};
thread_local NormGate g_normgate;

// gfwa_bwd_rows_f32 hands its fp32 boundary-row outputs to the shared gfwa_bwd body
struct RowsF32 {
    float* head = nullptr;
    float* tail = nullptr;
    int64_t head_rows = 0, tail_rows = 0;
};
thread_local RowsF32 g_rows;

// per device (a process may drive several GPUs), race-free (relaxed atomics:
// every thread computes the same value)
constexpr int kMaxDev = 64;
std::atomic<int> g_is_sm100[kMaxDev];  // 0 unknown, 1 yes, 2 no

bool device_is_sm100() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return false;
    if (dev < kMaxDev) {
        const int c = g_is_sm100[dev].load(std::memory_order_relaxed);
        if (c) return c == 1;
    }
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    const bool ok = major == 10 && minor == 0;
    if (dev < kMaxDev) g_is_sm100[dev].store(ok ? 1 : 2, std::memory_order_relaxed);
    return ok;
}

gfwa_status_t make_params(const gfwa_attn_desc_t* d, AttnParams& p) {
    if (!d) return GFWA_ERR_INVALID_ARGUMENT;
    if (d->B < 1 || d->H < 1 || d->N_q < 1 || d->N_kv < d->N_q || d->w < 1) return GFWA_ERR_INVALID_ARGUMENT;
    if (d->d != 64 && d->d != 128) return GFWA_ERR_UNSUPPORTED;
    if (d->dtype != GFWA_F32 && d->dtype != GFWA_BF16) return GFWA_ERR_UNSUPPORTED;
    if (!(d->scale == d->scale)) return GFWA_ERR_INVALID_ARGUMENT;
    if (d->B * d->H > 65535 * 65535LL || d->N_kv > ((int64_t)1 << 31)) return GFWA_ERR_INVALID_ARGUMENT;
    if (!device_is_sm100()) return GFWA_ERR_UNSUPPORTED;
    p = AttnParams{};
    p.B = d->B;
    p.H = d->H;
    if (d->H_kv < 0 || (d->H_kv > 0 && d->H % d->H_kv != 0)) return GFWA_ERR_INVALID_ARGUMENT;
    p.Hkv = d->H_kv > 0 ? d->H_kv : d->H;
    p.Nq = d->N_q;
    p.Nkv = d->N_kv;
    p.h0 = d->N_kv - d->N_q;
    p.d = d->d;
    p.w = d->w;
    p.scale = d->scale > 0.f ? d->scale : 1.f / std::sqrt((float)d->d);
    for (int i = 0; i < 3; ++i) {
        p.qs[i] = d->q_stride[i];
        p.ks[i] = d->k_stride[i];
        p.vs[i] = d->v_stride[i];
        p.os[i] = d->o_stride[i];
    }
    if (d->H > 65535 || d->B > 65535) return GFWA_ERR_INVALID_ARGUMENT;
    p.hrows = d->halo_rows;
    if (p.hrows != 0) {  // in-kernel halo: BF16 tensor-core path (checked at dispatch)
        if (p.hrows < 0 || p.hrows % 128 != 0 || p.hrows > p.h0 || d->dtype != GFWA_BF16 || !d->K_halo ||
            !d->V_halo || ((uintptr_t)d->K_halo % 16) || ((uintptr_t)d->V_halo % 16))
            return GFWA_ERR_INVALID_ARGUMENT;
        p.Kh = d->K_halo;
        p.Vh = d->V_halo;
        for (int i = 0; i < 3; ++i) {
            p.khs[i] = d->kh_stride[i];
            p.vhs[i] = d->vh_stride[i];
            if (p.khs[i] < 0 || p.vhs[i] < 0 || (p.khs[i] * 2) % 16 || (p.vhs[i] * 2) % 16)
                return GFWA_ERR_INVALID_ARGUMENT;
        }
    }
    return GFWA_OK;
}

// A thread that has only used another CUDA runtime (e.g. torch's autograd
// worker) may have no current driver context; the TMA descriptor encoder is a
// driver call, so bind the context that owns the caller's data first.
void bind_context(const void* dev_ptr) {
    CUcontext cur = nullptr;
    if (drv::ctxGetCurrent(&cur) == CUDA_SUCCESS && cur) return;
    CUcontext ctx = nullptr;
    if (drv::pointerGetAttribute(&ctx, CU_POINTER_ATTRIBUTE_CONTEXT, (CUdeviceptr)dev_ptr) == CUDA_SUCCESS && ctx)
        drv::ctxSetCurrent(ctx);
}

bool strides_ok(const int64_t* s, size_t esize) {
    for (int i = 0; i < 3; ++i)
        if (s[i] < 0 || ((s[i] * (int64_t)esize) % 16) != 0) return false;
    return true;
}

bool al16(const void* p) { return ((uintptr_t)p % 16) == 0; }

// in-kernel halo on another GPU's memory (a peer-mapped pointer): the kernels' TMA reads
// it over NVLink, which needs peer access from the current device (IPC mappings opened
// with lazy peer access have it already; "already enabled" is not an error)
void ensure_peer_access(const void* ptr) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    int cur = 0, can = 0;
    if (cudaGetDevice(&cur) != cudaSuccess || a.device < 0 || a.device == cur) return;
    if (cudaDeviceCanAccessPeer(&can, cur, a.device) == cudaSuccess && can &&
        cudaDeviceEnablePeerAccess(a.device, 0) != cudaSuccess)
        cudaGetLastError();  // cudaErrorPeerAccessAlreadyEnabled
}

}  // namespace

extern "C" gfwa_status_t gfwa_fwd(const gfwa_attn_desc_t* desc, const void* Q, const void* K, const void* V,
                                  const float* U, void* O, void* O_lo, float* LSE, gfwa_stream_t stream) {
    AttnParams p;
    if (gfwa_status_t s = make_params(desc, p)) return s;
    if (!Q || !K || !V || !U || !O || !LSE) return GFWA_ERR_INVALID_ARGUMENT;
    const size_t es = desc->dtype == GFWA_BF16 ? 2 : 4;
    if (!strides_ok(p.qs, es) || !strides_ok(p.ks, es) || !strides_ok(p.vs, es) || !strides_ok(p.os, es))
        return GFWA_ERR_INVALID_ARGUMENT;
    if (!al16(Q) || !al16(K) || !al16(V) || !al16(O) || (O_lo && !al16(O_lo))) return GFWA_ERR_INVALID_ARGUMENT;
    if (O_lo && desc->dtype != GFWA_BF16) return GFWA_ERR_INVALID_ARGUMENT;  // an fp32 O is exact already
    bind_context(Q);
    if (p.hrows) {
        ensure_peer_access(p.Kh);
        ensure_peer_access(p.Vh);
    }
    p.Q = Q;
    p.K = K;
    p.V = V;
    p.U = U;
    p.O = O;
    p.O_lo = O_lo;
    p.LSE = LSE;
    p.zero_acc = g_prepare.zero_acc;
    p.token = g_prepare.token;
    p.token_val = g_prepare.token_val;
    if (g_normgate.ng) {  // gfwa_fwd_normgate (validated there; tensor-core path only)
        if (!tc_fwd_supported(p, desc->dtype)) return GFWA_ERR_UNSUPPORTED;
        p.ng_g = g_normgate.ng->g;
        p.ng_gamma = g_normgate.ng->gamma;
        p.ng_eps = g_normgate.ng->eps;
        p.ng_rstd = g_normgate.ng->rstd;
        p.ng_Y = g_normgate.Y;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if ((p.Hkv != p.H || p.hrows) && !tc_fwd_supported(p, desc->dtype))
        return GFWA_ERR_UNSUPPORTED;  // GQA, in-kernel halo: tensor-core path
    gfwa_status_t s = tc_fwd_supported(p, desc->dtype) ? tc_fwd(p, st) : simt_fwd(p, desc->dtype, st);
    if (s != GFWA_OK || !check_finite_env()) return s;
    // opt-in debug check (GFWA_CHECK_FINITE=1): LSE, and O when it is packed
    if ((s = gfwa_check_finite(GFWA_F32, LSE, p.B * p.H * p.Nq, stream)) != GFWA_OK) return s;
    if (packed(p.os, p)) s = gfwa_check_finite(desc->dtype, O, p.B * p.Nq * p.H * p.d, stream);
    return s;
}

// [token | D | dalpha scan | dQ accumulator]; the token (a fixed 256-byte slot at
// the start, whatever the shape) marks a workspace whose accumulator the latest
// gfwa_fwd_train already zeroed for exactly this descriptor (tensor-core path
// only).  Every gfwa_fwd_train overwrites it and every tensor-core gfwa_bwd
// clears it, so interleaved shapes on one workspace stay correct: a backward
// whose descriptor does not match the token zeroes its own accumulator.
extern "C" gfwa_status_t gfwa_fwd_train(const gfwa_attn_desc_t* desc, const void* Q, const void* K,
                                        const void* V, const float* U, void* O, void* O_lo, float* LSE,
                                        void* bwd_ws, size_t bwd_ws_bytes, gfwa_stream_t stream);

static size_t bwd_ws_layout(const AttnParams& p, gfwa_dtype_t dt, size_t* off_D, size_t* off_scan,
                            size_t* off_tc, size_t* off_tok = nullptr) {
    size_t off = 256;
    if (off_tok) *off_tok = 0;
    *off_D = off;
    off += ((size_t)p.B * p.H * p.Nq * sizeof(float) + 255) & ~(size_t)255;
    *off_scan = off;
    off += gfwa_gate_prefix_bwd_workspace_size(p.B * p.H, p.Nkv, 1);  // the dalpha scan below
    *off_tc = off;
    if (tc_bwd_supported(p, dt)) off += (tc_bwd_workspace(p) + 255) & ~(size_t)255;
    return off;
}

// gfwa_fwd plus the preparation of the backward's workspace: on the tensor-core
// path the forward's epilogue zeroes the dQ accumulator (the writes overlap the
// compute-bound forward) and sets the token, so gfwa_bwd skips its zeroing pass.
extern "C" gfwa_status_t gfwa_fwd_train(const gfwa_attn_desc_t* desc, const void* Q, const void* K,
                                        const void* V, const float* U, void* O, void* O_lo, float* LSE,
                                        void* bwd_ws, size_t bwd_ws_bytes, gfwa_stream_t stream) {
    AttnParams p;
    if (gfwa_status_t s = make_params(desc, p)) return s;
    if (!bwd_ws || (uintptr_t)bwd_ws % 256) return GFWA_ERR_INVALID_ARGUMENT;
    size_t off_D, off_scan, off_tc, off_tok;
    const size_t need = bwd_ws_layout(p, desc->dtype, &off_D, &off_scan, &off_tc, &off_tok);
    if (bwd_ws_bytes < need) return GFWA_ERR_WORKSPACE;
    if (!tc_bwd_supported(p, desc->dtype) || !tc_fwd_supported(p, desc->dtype))  // nothing to prepare
        return gfwa_fwd(desc, Q, K, V, U, O, O_lo, LSE, stream);
    g_prepare.zero_acc = (float*)((char*)bwd_ws + off_tc);
    g_prepare.token = (unsigned long long*)((char*)bwd_ws + off_tok);
    g_prepare.token_val = prep_token(p);
    const gfwa_status_t s = gfwa_fwd(desc, Q, K, V, U, O, O_lo, LSE, stream);
    g_prepare = Prepare{};
    return s;
}

extern "C" size_t gfwa_bwd_workspace_size(const gfwa_attn_desc_t* desc) {
    AttnParams p;
    if (make_params(desc, p) != GFWA_OK) return 256;
    size_t a, b, c;
    return bwd_ws_layout(p, desc->dtype, &a, &b, &c);
}

// The dU -> dalpha reverse scan runs as a [B, Nkv, H=H] gate backward with
// kind ALPHA: it only needs dU in [B, H, Nkv] layout, which is exactly dU.
extern "C" gfwa_status_t gfwa_bwd(const gfwa_attn_desc_t* desc, const void* Q, const void* K, const void* V,
                                  const float* U, const void* O, const void* O_lo, const float* LSE,
                                  const void* dO, void* dQ, void* dK, void* dV, float* dU, float* dalpha,
                                  const double* dalpha_carry, void* ws, size_t ws_bytes, gfwa_stream_t stream) {
    AttnParams p;
    if (gfwa_status_t s = make_params(desc, p)) return s;
    GFWA_REQUIRE(Q && K && V && U && LSE && dO && dQ && dK && dV && dU && ws);
    GFWA_REQUIRE(O);
    GFWA_REQUIRE(!O_lo || (desc->dtype == GFWA_BF16 && al16(O_lo)));
    const size_t es = desc->dtype == GFWA_BF16 ? 2 : 4;
    GFWA_REQUIRE(strides_ok(p.qs, es) && strides_ok(p.ks, es) && strides_ok(p.vs, es) && strides_ok(p.os, es));
    const void* ptrs[] = {Q, K, V, dO, dQ, dK, dV};
    for (const void* pp : ptrs) GFWA_REQUIRE(al16(pp));
    GFWA_REQUIRE((uintptr_t)ws % 256 == 0);
    size_t off_D, off_scan, off_tc, off_tok;
    const size_t need = bwd_ws_layout(p, desc->dtype, &off_D, &off_scan, &off_tc, &off_tok);
    if (ws_bytes < need) return GFWA_ERR_WORKSPACE;
    p.token = tc_bwd_supported(p, desc->dtype) ? (unsigned long long*)((char*)ws + off_tok) : nullptr;
    p.token_val = prep_token(p);
    bind_context(Q);
    if (p.hrows) {
        ensure_peer_access(p.Kh);
        ensure_peer_access(p.Vh);
    }
    p.Q = Q;
    p.K = K;
    p.V = V;
    p.U = U;
    p.O = const_cast<void*>(O);
    p.Olo = O_lo;
    p.LSE = const_cast<float*>(LSE);
    p.dO = dO;
    p.dQ = dQ;
    p.dK = dK;
    p.dV = dV;
    p.dU = dU;
    p.Dv = (float*)((char*)ws + off_D);
    if (g_normgate.ng) {  // gfwa_bwd_normgate: the fused epilogue backward replaces the preprocess
        if (!tc_bwd_supported(p, desc->dtype)) return GFWA_ERR_UNSUPPORTED;
        p.ng_g = g_normgate.ng->g;
        p.ng_gamma = g_normgate.ng->gamma;
        p.ng_eps = g_normgate.ng->eps;
        p.ng_rstd = g_normgate.ng->rstd;
        p.ng_dY = g_normgate.dY;
        p.ng_dg = g_normgate.dg;
        p.ng_dgamma = g_normgate.dgamma;
    }
    if (g_rows.head || g_rows.tail) {  // gfwa_bwd_rows_f32 (tensor-core path only)
        if (!tc_bwd_supported(p, desc->dtype)) return GFWA_ERR_UNSUPPORTED;
        GFWA_REQUIRE(g_rows.head_rows <= p.Nkv && g_rows.tail_rows <= p.Nkv);
        p.f32_head = g_rows.head_rows > 0 ? g_rows.head : nullptr;
        p.f32_tail = g_rows.tail_rows > 0 ? g_rows.tail : nullptr;
        p.f32_head_rows = g_rows.head_rows;
        p.f32_tail_rows = g_rows.tail_rows;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if ((p.Hkv != p.H || p.hrows) && !tc_bwd_supported(p, desc->dtype))
        return GFWA_ERR_UNSUPPORTED;  // GQA, in-kernel halo: tensor-core path
    gfwa_status_t s;
    if (tc_bwd_supported(p, desc->dtype)) {
        s = tc_bwd(p, st, (char*)ws + off_tc);  // D, dQ/dU zeroing fused in its own pre kernel
    } else {
        if ((s = bwd_preprocess(p, desc->dtype, st)) != GFWA_OK) return s;
        s = simt_bwd(p, desc->dtype, st);
    }
    if (s != GFWA_OK) return s;
    if (check_finite_env()) {  // opt-in debug check (GFWA_CHECK_FINITE=1)
        if ((s = gfwa_check_finite(GFWA_F32, dU, p.B * p.H * p.Nkv, stream)) != GFWA_OK) return s;
        if (packed(p.qs, p) && (s = gfwa_check_finite(desc->dtype, dQ, p.B * p.Nq * p.H * p.d, stream)) != GFWA_OK)
            return s;
        const int64_t nkv = p.B * p.Nkv * p.Hkv * p.d;
        if (packed_kv(p.ks, p) && (s = gfwa_check_finite(desc->dtype, dK, nkv, stream)) != GFWA_OK) return s;
        if (packed_kv(p.vs, p) && (s = gfwa_check_finite(desc->dtype, dV, nkv, stream)) != GFWA_OK) return s;
    }
    if (!dalpha) return GFWA_OK;
    // dalpha = carry - reverse_cumsum(dU) over the N_kv key rows
    return gfwa_gate_prefix_bwd(GFWA_GATE_ALPHA, GFWA_F32, nullptr, nullptr, p.B * p.H, p.Nkv, 1, 0.f, dU,
                                dalpha_carry, dalpha, nullptr, nullptr, (char*)ws + off_scan,
                                gfwa_gate_prefix_bwd_workspace_size(p.B * p.H, p.Nkv, 1), stream);
}

extern "C" int gfwa_attn_path(const gfwa_attn_desc_t* desc) {
    AttnParams p;
    if (make_params(desc, p) != GFWA_OK) return -1;
    return tc_fwd_supported(p, desc->dtype) ? 1 : 0;
}

// ---------------------------------------------------------------- debug: non-finite check
namespace {
__device__ unsigned g_nonfinite;

template <typename T>
__global__ void nonfinite_kernel(const T* __restrict__ x, int64_t n) {
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(to_f32<T>(x[i]));
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&g_nonfinite, 1u);
}

bool check_finite_env() {
    static const int on = [] {
        const char* e = getenv("GFWA_CHECK_FINITE");
        return e && e[0] == '1' ? 1 : 0;
    }();
    return on != 0;
}
}  // namespace

extern "C" gfwa_status_t gfwa_check_finite(gfwa_dtype_t dtype, const void* x, int64_t n, gfwa_stream_t stream) {
    if (!x || n < 0) return GFWA_ERR_INVALID_ARGUMENT;
    if (dtype != GFWA_F32 && dtype != GFWA_BF16) return GFWA_ERR_UNSUPPORTED;
    if (n == 0) return GFWA_OK;
    cudaStream_t st = (cudaStream_t)stream;
    void* flag = nullptr;
    if (gfwa_status_t s = check_launch(cudaGetSymbolAddress(&flag, g_nonfinite))) return s;
    if (gfwa_status_t s = check_launch(cudaMemsetAsync(flag, 0, sizeof(unsigned), st))) return s;
    const unsigned grid = (unsigned)min64((n + 255) / 256, 148 * 8);
    if (dtype == GFWA_F32)
        nonfinite_kernel<float><<<grid, 256, 0, st>>>((const float*)x, n);
    else
        nonfinite_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)x, n);
    note_launch();
    if (gfwa_status_t s = check_launch()) return s;
    unsigned h = 0;
    if (gfwa_status_t s = check_launch(cudaMemcpyAsync(&h, flag, sizeof(unsigned), cudaMemcpyDeviceToHost, st)))
        return s;
    if (gfwa_status_t s = check_launch(cudaStreamSynchronize(st))) return s;
    return h ? GFWA_ERR_NONFINITE : GFWA_OK;
}

extern "C" const char* gfwa_status_string(gfwa_status_t s) {
    switch (s) {
        case GFWA_OK: return "GFWA_OK";
        case GFWA_ERR_INVALID_ARGUMENT: return "GFWA_ERR_INVALID_ARGUMENT";
        case GFWA_ERR_UNSUPPORTED: return "GFWA_ERR_UNSUPPORTED";
        case GFWA_ERR_CUDA: return "GFWA_ERR_CUDA";
        case GFWA_ERR_WORKSPACE: return "GFWA_ERR_WORKSPACE";
        case GFWA_ERR_NONFINITE: return "GFWA_ERR_NONFINITE";
    }
    return "GFWA_ERR_UNKNOWN";
}

extern "C" int gfwa_last_cuda_error(void) { return g_last_cuda_error; }
extern "C" const char* gfwa_version(void) { return "gfwa 0.1.0 (sm_100a)"; }
extern "C" void gfwa_debug_stage_events(void* const* events, int n) {
    for (int i = 0; i < 4; ++i) g_stage_ev[i] = (events && i < n) ? (cudaEvent_t)events[i] : nullptr;
}
extern "C" uint64_t gfwa_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

// ---------------------------------------------------------------------------
// AttnLayer output epilogue (reading C-27)
namespace {
gfwa_status_t check_normgate(const gfwa_attn_desc_t* desc, const gfwa_normgate_t* ng, const void* O,
                             const void* O_lo, std::initializer_list<const void*> bf16_rows) {
    AttnParams p;
    if (gfwa_status_t s = make_params(desc, p)) return s;
    GFWA_REQUIRE(ng && ng->g && ng->gamma && ng->rstd && O);
    GFWA_REQUIRE(ng->eps > 0.f && ng->eps == ng->eps);
    if (desc->dtype != GFWA_BF16) return GFWA_ERR_UNSUPPORTED;
    // every row tensor shares O's layout, which must be packed [B, N_q, H, d]
    GFWA_REQUIRE(packed(p.os, p) && p.B * p.Nq * p.H < ((int64_t)1 << 31));
    GFWA_REQUIRE(al16(ng->g) && al16(O) && (!O_lo || al16(O_lo)) && al16(ng->gamma));
    for (const void* q : bf16_rows) GFWA_REQUIRE(q && al16(q));
    return GFWA_OK;
}
}  // namespace

extern "C" gfwa_status_t gfwa_fwd_normgate(const gfwa_attn_desc_t* desc, const void* Q, const void* K,
                                           const void* V, const float* U, const gfwa_normgate_t* ng, void* O,
                                           void* O_lo, float* LSE, void* Y, void* bwd_ws, size_t bwd_ws_bytes,
                                           gfwa_stream_t stream) {
    if (gfwa_status_t s = check_normgate(desc, ng, O, O_lo, {Y})) return s;
    g_normgate = NormGate{};
    g_normgate.ng = ng;
    g_normgate.Y = Y;
    const gfwa_status_t s = bwd_ws ? gfwa_fwd_train(desc, Q, K, V, U, O, O_lo, LSE, bwd_ws, bwd_ws_bytes, stream)
                                   : gfwa_fwd(desc, Q, K, V, U, O, O_lo, LSE, stream);
    g_normgate = NormGate{};
    return s;
}

extern "C" gfwa_status_t gfwa_bwd_normgate(const gfwa_attn_desc_t* desc, const void* Q, const void* K,
                                           const void* V, const float* U, const void* O, const void* O_lo,
                                           const float* LSE, const gfwa_normgate_t* ng, const void* dY, void* dO,
                                           void* dg, float* dgamma, void* dQ, void* dK, void* dV, float* dU,
                                           float* dalpha, const double* dalpha_carry, void* ws, size_t ws_bytes,
                                           gfwa_stream_t stream) {
    if (gfwa_status_t s = check_normgate(desc, ng, O, O_lo, {dY, dO, dg})) return s;
    GFWA_REQUIRE(dgamma);
    g_normgate = NormGate{};
    g_normgate.ng = ng;
    g_normgate.dY = dY;
    g_normgate.dg = dg;
    g_normgate.dgamma = dgamma;
    const gfwa_status_t s = gfwa_bwd(desc, Q, K, V, U, O, O_lo, LSE, dO, dQ, dK, dV, dU, dalpha, dalpha_carry, ws,
                                     ws_bytes, stream);
    g_normgate = NormGate{};
    return s;
}

// sequence sharding: gfwa_bwd plus fp32 copies of the boundary rows' dK, dV
extern "C" gfwa_status_t gfwa_bwd_rows_f32(const gfwa_attn_desc_t* desc, const void* Q, const void* K,
                                           const void* V, const float* U, const void* O, const void* O_lo,
                                           const float* LSE, const void* dO, void* dQ, void* dK, void* dV,
                                           float* dU, float* dalpha, const double* dalpha_carry,
                                           int64_t head_rows, float* dKV_head, int64_t tail_rows, float* dKV_tail,
                                           void* ws, size_t ws_bytes, gfwa_stream_t stream) {
    GFWA_REQUIRE(head_rows >= 0 && tail_rows >= 0);
    GFWA_REQUIRE((head_rows == 0 || dKV_head) && (tail_rows == 0 || dKV_tail));
    GFWA_REQUIRE((!dKV_head || al16(dKV_head)) && (!dKV_tail || al16(dKV_tail)));
    g_rows = RowsF32{};
    g_rows.head = dKV_head;
    g_rows.tail = dKV_tail;
    g_rows.head_rows = head_rows;
    g_rows.tail_rows = tail_rows;
    const gfwa_status_t s = gfwa_bwd(desc, Q, K, V, U, O, O_lo, LSE, dO, dQ, dK, dV, dU, dalpha, dalpha_carry, ws,
                                     ws_bytes, stream);
    g_rows = RowsF32{};
    return s;
}

// ---------------------------------------------------------------------------
// NSA extension (App. B; readings C-28, C-29)
namespace gfwa {
size_t nsa_workspace(int64_t B, int64_t N, int64_t H, int d, int blk, int nsel);
gfwa_status_t nsa_fwd_branches(const void* Q, const void* K, const void* V, const float* g, int64_t B, int64_t N,
                               int64_t H, int d, int blk, int nsel, float scale, float* Kc, float* Vc, float* Ocmp,
                               float* Oslc, float* Lcmp, float* Lslc, int* sel, const void* Oloc, void* O,
                               cudaStream_t st, bool compress_only = false);
gfwa_status_t nsa_bwd_combine(const void* dO, const float* g, const float* Ocmp, const float* Oslc, const void* Oloc,
                              const void* Ololo, float* dOc, float* dOs, void* dOl, float* dg, float* Dc, float* Ds,
                              int64_t B, int64_t N, int64_t H, int d, cudaStream_t st);
gfwa_status_t nsa_bwd_branches(const void* Q, const void* K, const void* V, const int* sel, const float* Kc,
                               const float* Vc, const float* dOc, const float* dOs, const float* Lc, const float* Ls,
                               const float* Dc, const float* Ds, float* dQacc, float* dKacc, float* dVacc, float* dKc,
                               float* dVc, const void* dQl, const void* dKl, const void* dVl, void* dQ, void* dK,
                               void* dV, int64_t B, int64_t N, int64_t H, int d, int blk, int nsel, float scale,
                               int* scnt, int* soff, int* scur, int* slist, cudaStream_t st);
bool nsa_blocks_ok(int64_t N, int blk);
}  // namespace gfwa

namespace {
bool nsa_desc_ok(const gfwa_nsa_desc_t* d) {
    return d && d->B >= 1 && d->H >= 1 && d->N >= 1 && d->w >= 1 && d->block >= 1 && d->block <= 64 && d->n_sel >= 0 &&
           (d->d == 64 || d->d == 128) && d->dtype == GFWA_BF16 && nsa_blocks_ok(d->N, d->block) &&
           d->B * d->N * d->H < ((int64_t)1 << 31) && d->scale == d->scale;
}
gfwa_attn_desc_t nsa_local_desc(const gfwa_nsa_desc_t* d) {
    gfwa_attn_desc_t ad{};
    ad.B = d->B;
    ad.H = d->H;
    ad.N_q = d->N;
    ad.N_kv = d->N;
    ad.d = d->d;
    ad.w = d->w;
    ad.scale = d->scale;
    ad.dtype = GFWA_BF16;
    const int64_t st3[3] = {d->N * d->H * d->d, d->H * d->d, d->d};
    for (int i = 0; i < 3; ++i) ad.q_stride[i] = ad.k_stride[i] = ad.v_stride[i] = ad.o_stride[i] = st3[i];
    return ad;
}
// bump allocator over the caller's workspace (256-byte aligned pieces)
struct Carve {
    char* p;
    void* take(size_t bytes) {
        char* r = p;
        p += (bytes + 255) & ~(size_t)255;
        return r;
    }
};
size_t nsa_bwd_bytes(const gfwa_nsa_desc_t* d) {
    const size_t n = (size_t)d->B * d->N * d->H * d->d, rows = (size_t)d->B * d->N * d->H;
    const size_t nbk = (size_t)d->B * (d->N / d->block) * d->H * d->d;
    auto r = [](size_t b) { return (b + 255) & ~(size_t)255; };
    gfwa_attn_desc_t ad = nsa_local_desc(d);
    const size_t nbp = (size_t)d->B * d->H * ((d->N + d->block - 1) / d->block);
    return r(nbk * 4) * 4 + r(n * 4) * 5 + r(n * 2) * 4 + r(rows * 4) * 2 + r(gfwa_bwd_workspace_size(&ad)) +
           r(nbp * 4) * 3 + r(rows * (d->n_sel + 1) * 4);
}
}  // namespace

extern "C" size_t gfwa_nsa_workspace_size(const gfwa_nsa_desc_t* d) {
    if (!nsa_desc_ok(d)) return 256;
    const size_t f = nsa_workspace(d->B, d->N, d->H, d->d, d->block, d->n_sel);
    const size_t b = nsa_bwd_bytes(d);
    return (f > b ? f : b) + 256;
}

extern "C" gfwa_status_t gfwa_nsa_fwd(const gfwa_nsa_desc_t* d, const void* Q, const void* K, const void* V,
                                      const float* U, const float* gates, void* O, const gfwa_nsa_saved_t* saved,
                                      void* ws, size_t ws_bytes, gfwa_stream_t stream) {
    if (!d) return GFWA_ERR_INVALID_ARGUMENT;
    if (d->d != 64 && d->d != 128) return GFWA_ERR_UNSUPPORTED;
    if (d->dtype != GFWA_BF16) return GFWA_ERR_UNSUPPORTED;
    GFWA_REQUIRE(nsa_desc_ok(d));
    GFWA_REQUIRE(Q && K && V && U && gates && O && ws && (uintptr_t)ws % 256 == 0);
    GFWA_REQUIRE(al16(Q) && al16(K) && al16(V) && al16(O));
    if (ws_bytes < gfwa_nsa_workspace_size(d)) return GFWA_ERR_WORKSPACE;
    const int64_t B = d->B, N = d->N, H = d->H, nb = N / d->block;
    Carve cv{(char*)ws};
    float* Kc = (float*)cv.take((size_t)B * nb * H * d->d * 4 * 2);
    float* Vc = Kc + (size_t)B * nb * H * d->d;
    float* oc = (float*)cv.take((size_t)B * N * H * d->d * 4 * 2);
    float* os = oc + (size_t)B * N * H * d->d;
    int* sl = (int*)cv.take((size_t)B * H * N * (d->n_sel + 1) * 4);
    void* ol = cv.take((size_t)B * N * H * d->d * 2);
    float* lse = (float*)cv.take((size_t)B * H * N * 4 * 3);
    float *lc = lse + B * H * N, *ls = lc + B * H * N;
    void* olo = nullptr;
    if (saved) {
        if (saved->O_cmp) oc = saved->O_cmp;
        if (saved->O_slc) os = saved->O_slc;
        if (saved->sel) sl = saved->sel;
        if (saved->O_loc) ol = saved->O_loc;
        if (saved->LSE_loc) lse = saved->LSE_loc;
        if (saved->LSE_cmp) lc = saved->LSE_cmp;
        if (saved->LSE_slc) ls = saved->LSE_slc;
        olo = saved->O_loc_lo;
        GFWA_REQUIRE(al16(ol) && (!olo || al16(olo)));
    }
    // the local branch: GatedFWA itself (gfwa_fwd)
    gfwa_attn_desc_t ad = nsa_local_desc(d);
    if (gfwa_status_t s = gfwa_fwd(&ad, Q, K, V, U, ol, olo, lse, stream)) return s;
    const float scale = d->scale > 0.f ? d->scale : 1.f / std::sqrt((float)d->d);
    return nsa_fwd_branches(Q, K, V, gates, B, N, H, d->d, d->block, d->n_sel, scale, Kc, Vc, oc, os, lc, ls, sl, ol,
                            O, (cudaStream_t)stream);
}

extern "C" gfwa_status_t gfwa_nsa_bwd(const gfwa_nsa_desc_t* d, const void* Q, const void* K, const void* V,
                                      const float* U, const float* gates, const void* dO,
                                      const gfwa_nsa_saved_t* sv, void* dQ, void* dK, void* dV, float* dU,
                                      float* dgates, void* ws, size_t ws_bytes, gfwa_stream_t stream) {
    if (!d) return GFWA_ERR_INVALID_ARGUMENT;
    if (d->d != 64 && d->d != 128) return GFWA_ERR_UNSUPPORTED;
    if (d->dtype != GFWA_BF16) return GFWA_ERR_UNSUPPORTED;
    GFWA_REQUIRE(nsa_desc_ok(d));
    GFWA_REQUIRE(Q && K && V && U && gates && dO && sv && dQ && dK && dV && dU && dgates && ws);
    GFWA_REQUIRE(sv->O_cmp && sv->O_slc && sv->LSE_cmp && sv->LSE_slc && sv->sel && sv->O_loc && sv->LSE_loc);
    GFWA_REQUIRE((uintptr_t)ws % 256 == 0 && al16(Q) && al16(K) && al16(V) && al16(dO) && al16(dQ) && al16(dK) &&
                 al16(dV) && al16(sv->O_loc) && (!sv->O_loc_lo || al16(sv->O_loc_lo)));
    if (ws_bytes < gfwa_nsa_workspace_size(d)) return GFWA_ERR_WORKSPACE;
    const int64_t B = d->B, N = d->N, H = d->H, nb = N / d->block;
    const size_t n = (size_t)B * N * H * d->d, rows = (size_t)B * N * H, nbk = (size_t)B * nb * H * d->d;
    cudaStream_t st = (cudaStream_t)stream;
    Carve cv{(char*)ws};
    float* Kc = (float*)cv.take(nbk * 4);
    float* Vc = (float*)cv.take(nbk * 4);
    float* dKc = (float*)cv.take(nbk * 4);
    float* dVc = (float*)cv.take(nbk * 4);
    float* dOc = (float*)cv.take(n * 4);
    float* dOs = (float*)cv.take(n * 4);
    float* dQacc = (float*)cv.take(n * 4);
    float* dKacc = (float*)cv.take(n * 4);
    float* dVacc = (float*)cv.take(n * 4);
    void* dOl = cv.take(n * 2);
    void* dQl = cv.take(n * 2);
    void* dKl = cv.take(n * 2);
    void* dVl = cv.take(n * 2);
    float* Dc = (float*)cv.take(rows * 4);
    float* Ds = (float*)cv.take(rows * 4);
    gfwa_attn_desc_t ad = nsa_local_desc(d);
    const size_t lws = gfwa_bwd_workspace_size(&ad);
    void* lw = cv.take(lws);
    const size_t nbp = (size_t)B * H * ((N + d->block - 1) / d->block);
    int* scnt = (int*)cv.take(nbp * 4);
    int* soff = (int*)cv.take(nbp * 4);
    int* scur = (int*)cv.take(nbp * 4);
    int* slist = (int*)cv.take(rows * (d->n_sel + 1) * 4);
    const float scale = d->scale > 0.f ? d->scale : 1.f / std::sqrt((float)d->d);
    gfwa_status_t s;
    if ((s = nsa_bwd_combine(dO, gates, sv->O_cmp, sv->O_slc, sv->O_loc, sv->O_loc_lo, dOc, dOs, dOl, dgates, Dc, Ds,
                             B, N, H, d->d, st)))
        return s;
    // the local branch: Alg. E.2 on sigmoid(g2) dO
    if ((s = gfwa_bwd(&ad, Q, K, V, U, sv->O_loc, sv->O_loc_lo, sv->LSE_loc, dOl, dQl, dKl, dVl, dU, nullptr, nullptr,
                      lw, lws, stream)))
        return s;
    // block means of K, V again (the compressed branch's keys and values)
    if (nb > 0) {
        if ((s = nsa_fwd_branches(Q, K, V, gates, B, N, H, d->d, d->block, 0, scale, Kc, Vc, nullptr, nullptr, nullptr,
                                  nullptr, nullptr, nullptr, nullptr, st, true)))
            return s;
    }
    return nsa_bwd_branches(Q, K, V, sv->sel, Kc, Vc, dOc, dOs, sv->LSE_cmp, sv->LSE_slc, Dc, Ds, dQacc, dKacc, dVacc,
                            dKc, dVc, dQl, dKl, dVl, dQ, dK, dV, B, N, H, d->d, d->block, d->n_sel, scale, scnt,
                            soff, scur, slist, st);
}
