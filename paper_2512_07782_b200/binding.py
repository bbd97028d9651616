"""Thin ctypes binding of libgfwa.so (include/gfwa.h).

Argument marshalling only: every function takes torch CUDA tensors, checks
shapes/dtypes, passes raw device pointers plus the current CUDA stream to the
C ABI call of the same name, and raises ``GfwaError`` on a non-OK status.
Nothing here computes any part of the method; there is no CPU fallback --
if the library is missing or the device is not sm_100 the call fails loudly.
"""
from __future__ import annotations

import ctypes
import math
import os
import threading

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GFWA_LIB") or os.path.join(_PKG, "libgfwa.so")  # GFWA_LIB: experiment variants

GFWA_F32, GFWA_BF16 = 0, 1
GATE_HBETA, GATE_ALPHA = 0, 1
_STATUS = {
    0: "GFWA_OK",
    1: "GFWA_ERR_INVALID_ARGUMENT",
    2: "GFWA_ERR_UNSUPPORTED",
    3: "GFWA_ERR_CUDA",
    4: "GFWA_ERR_WORKSPACE",
    5: "GFWA_ERR_NONFINITE",
}


class GfwaError(RuntimeError):
    pass


class AttnDesc(ctypes.Structure):
    _fields_ = [
        ("B", ctypes.c_int64),
        ("H", ctypes.c_int64),
        ("N_q", ctypes.c_int64),
        ("N_kv", ctypes.c_int64),
        ("d", ctypes.c_int32),
        ("w", ctypes.c_int32),
        ("scale", ctypes.c_float),
        ("dtype", ctypes.c_int32),
        ("q_stride", ctypes.c_int64 * 3),
        ("k_stride", ctypes.c_int64 * 3),
        ("v_stride", ctypes.c_int64 * 3),
        ("o_stride", ctypes.c_int64 * 3),
        ("H_kv", ctypes.c_int64),
        ("halo_rows", ctypes.c_int64),
        ("K_halo", ctypes.c_void_p),
        ("V_halo", ctypes.c_void_p),
        ("kh_stride", ctypes.c_int64 * 3),
        ("vh_stride", ctypes.c_int64 * 3),
    ]


class DecodeDesc(ctypes.Structure):
    _fields_ = [
        ("B", ctypes.c_int64),
        ("H", ctypes.c_int64),
        ("d", ctypes.c_int32),
        ("w", ctypes.c_int32),
        ("scale", ctypes.c_float),
        ("eps", ctypes.c_float),
        ("dtype", ctypes.c_int32),
        ("gate_kind", ctypes.c_int32),
        ("H_kv", ctypes.c_int64),
    ]


class NsaDesc(ctypes.Structure):
    """gfwa_nsa_desc_t (include/gfwa.h): the NSA hybrid with GatedFWA as its local branch."""
    _fields_ = [("B", ctypes.c_int64), ("H", ctypes.c_int64), ("N", ctypes.c_int64), ("d", ctypes.c_int32),
                ("w", ctypes.c_int32), ("block", ctypes.c_int32), ("n_sel", ctypes.c_int32), ("scale", ctypes.c_float),
                ("dtype", ctypes.c_int32)]


class NsaSaved(ctypes.Structure):
    """gfwa_nsa_saved_t: the tensors gfwa_nsa_fwd keeps for gfwa_nsa_bwd."""
    _fields_ = [(n, ctypes.c_void_p) for n in ("O_cmp", "O_slc", "LSE_cmp", "LSE_slc", "sel", "O_loc", "O_loc_lo",
                                               "LSE_loc")]


class NormGate(ctypes.Structure):
    """gfwa_normgate_t (include/gfwa.h): the AttnLayer epilogue's inputs (C-27)."""
    _fields_ = [("g", ctypes.c_void_p), ("gamma", ctypes.c_void_p), ("eps", ctypes.c_float),
                ("rstd", ctypes.c_void_p)]


_lib = None
_lock = threading.Lock()
_VP = ctypes.c_void_p
_I64 = ctypes.c_int64

EXPORTED = (
    "gfwa_gate_prefix",
    "gfwa_gate_prefix_variant",
    "gfwa_gate_prefix_variant_workspace_size",
    "gfwa_gate_prefix_workspace_size",
    "gfwa_gate_prefix_bwd",
    "gfwa_gate_prefix_bwd_workspace_size",
    "gfwa_debug_tc_selftest_ex",
    "gfwa_debug_stage_events",
    "gfwa_fwd",
    "gfwa_fwd_train",
    "gfwa_bwd",
    "gfwa_bwd_workspace_size",
    "gfwa_decode",
    "gfwa_decode_workspace_size",
    "gfwa_check_finite",
    "gfwa_status_string",
    "gfwa_last_cuda_error",
    "gfwa_version",
    "gfwa_launch_count",
    "gfwa_attn_path",
    "gfwa_fwd_normgate",
    "gfwa_bwd_normgate",
    "gfwa_bwd_rows_f32",
    "gfwa_nsa_fwd",
    "gfwa_nsa_bwd",
    "gfwa_nsa_workspace_size",
)


def load() -> ctypes.CDLL:
    """Load libgfwa.so (fails loudly if it was not built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise GfwaError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(LIB_PATH)
        sz = ctypes.c_size_t
        lib.gfwa_gate_prefix_workspace_size.restype = sz
        lib.gfwa_gate_prefix_workspace_size.argtypes = [_I64, _I64, _I64]
        lib.gfwa_gate_prefix_bwd_workspace_size.restype = sz
        lib.gfwa_gate_prefix_bwd_workspace_size.argtypes = [_I64, _I64, _I64]
        lib.gfwa_gate_prefix.restype = ctypes.c_int
        lib.gfwa_gate_prefix.argtypes = [ctypes.c_int, ctypes.c_int, _VP, _VP, _I64, _I64, _I64, ctypes.c_float,
                                         _VP, _VP, _VP, _VP, sz, _VP]
        lib.gfwa_gate_prefix_bwd.restype = ctypes.c_int
        lib.gfwa_gate_prefix_bwd.argtypes = [ctypes.c_int, ctypes.c_int, _VP, _VP, _I64, _I64, _I64,
                                             ctypes.c_float, _VP, _VP, _VP, _VP, _VP, _VP, sz, _VP]
        lib.gfwa_gate_prefix_variant_workspace_size.restype = sz
        lib.gfwa_gate_prefix_variant_workspace_size.argtypes = [ctypes.c_int, _I64, _I64, _I64]
        lib.gfwa_gate_prefix_variant.restype = ctypes.c_int
        lib.gfwa_gate_prefix_variant.argtypes = [ctypes.c_int, ctypes.c_int, _VP, _VP, _I64, _I64, _I64,
                                                 ctypes.c_float, _VP, _VP, sz, _VP]
        lib.gfwa_fwd.restype = ctypes.c_int
        lib.gfwa_fwd.argtypes = [ctypes.POINTER(AttnDesc), _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP]
        lib.gfwa_fwd_train.restype = ctypes.c_int
        lib.gfwa_fwd_train.argtypes = [ctypes.POINTER(AttnDesc), _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, sz, _VP]
        lib.gfwa_bwd_workspace_size.restype = sz
        lib.gfwa_bwd_workspace_size.argtypes = [ctypes.POINTER(AttnDesc)]
        lib.gfwa_bwd.restype = ctypes.c_int
        lib.gfwa_bwd.argtypes = [ctypes.POINTER(AttnDesc)] + [_VP] * 15 + [sz, _VP]
        lib.gfwa_nsa_workspace_size.restype = sz
        lib.gfwa_nsa_workspace_size.argtypes = [ctypes.POINTER(NsaDesc)]
        lib.gfwa_nsa_fwd.restype = ctypes.c_int
        lib.gfwa_nsa_fwd.argtypes = [ctypes.POINTER(NsaDesc)] + [_VP] * 6 + [ctypes.POINTER(NsaSaved), _VP, sz, _VP]
        lib.gfwa_nsa_bwd.restype = ctypes.c_int
        lib.gfwa_nsa_bwd.argtypes = [ctypes.POINTER(NsaDesc)] + [_VP] * 6 + [ctypes.POINTER(NsaSaved)] + [_VP] * 6 + \
            [sz, _VP]
        lib.gfwa_bwd_rows_f32.restype = ctypes.c_int
        lib.gfwa_bwd_rows_f32.argtypes = [ctypes.POINTER(AttnDesc)] + [_VP] * 14 + [_I64, _VP, _I64, _VP, _VP, sz, _VP]
        lib.gfwa_fwd_normgate.restype = ctypes.c_int
        lib.gfwa_fwd_normgate.argtypes = [ctypes.POINTER(AttnDesc)] + [_VP] * 4 + [ctypes.POINTER(NormGate)] + \
            [_VP] * 5 + [sz, _VP]
        lib.gfwa_bwd_normgate.restype = ctypes.c_int
        lib.gfwa_bwd_normgate.argtypes = [ctypes.POINTER(AttnDesc)] + [_VP] * 7 + [ctypes.POINTER(NormGate)] + \
            [_VP] * 11 + [sz, _VP]
        lib.gfwa_decode_workspace_size.restype = sz
        lib.gfwa_decode_workspace_size.argtypes = [ctypes.POINTER(DecodeDesc)]
        lib.gfwa_decode.restype = ctypes.c_int
        lib.gfwa_decode.argtypes = [ctypes.POINTER(DecodeDesc)] + [_VP] * 11 + [sz, _VP]
        lib.gfwa_check_finite.restype = ctypes.c_int
        lib.gfwa_check_finite.argtypes = [ctypes.c_int, _VP, _I64, _VP]
        lib.gfwa_status_string.restype = ctypes.c_char_p
        lib.gfwa_last_cuda_error.restype = ctypes.c_int
        lib.gfwa_version.restype = ctypes.c_char_p
        lib.gfwa_launch_count.restype = ctypes.c_uint64
        lib.gfwa_attn_path.restype = ctypes.c_int
        lib.gfwa_attn_path.argtypes = [ctypes.POINTER(AttnDesc)]
        _lib = lib
        return lib


def _check(status: int, what: str):
    if status != 0:
        extra = ""
        if status == 3:
            extra = f" (cudaError {load().gfwa_last_cuda_error()})"
        raise GfwaError(f"{what}: {_STATUS.get(status, status)}{extra}")


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return GFWA_BF16
    if t.dtype == torch.float32:
        return GFWA_F32
    raise GfwaError(f"unsupported dtype {t.dtype} (bf16 or fp32)")


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise GfwaError("libgfwa takes CUDA tensors only (no CPU fallback)")


_ws_cache: dict = {}


def workspace(nbytes: int, device, tag: str = "scratch", zero: bool = False) -> torch.Tensor:
    """Cached device scratch (caller-owned per the ABI); `zero` tensors are
    zeroed once at allocation (decode's self-resetting counters).  Keyed by
    (tag, device, current stream): calls on one stream are ordered, so they may
    share a workspace; calls on different streams get their own."""
    dev = torch.device(device).index if torch.device(device).index is not None else torch.cuda.current_device()
    key = (tag, dev, torch.cuda.current_stream(dev).cuda_stream)
    t = _ws_cache.get(key)
    if t is None or t.numel() < nbytes:
        t = (torch.zeros if zero else torch.empty)(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        _ws_cache[key] = t
    return t


def _bnh_strides(t: torch.Tensor):
    """(b, n, h) element strides of a [B,N,H,d] tensor with d contiguous."""
    if t.dim() != 4 or t.stride(3) != 1:
        raise GfwaError("attention tensors must be [B,N,H,d] with the head dim contiguous")
    return (t.stride(0), t.stride(1), t.stride(2))


def _grad_kv(K, V, Nkv: int):
    """dK, dV over all Nkv key rows: K's layout when K holds them all, else contiguous
    [B, Nkv, H_kv, d] (the in-kernel halo: K holds only the local rows)."""
    if K.shape[1] == Nkv:
        return (torch.empty_strided(K.shape, K.stride(), dtype=K.dtype, device=K.device),
                torch.empty_strided(V.shape, V.stride(), dtype=V.dtype, device=V.device))
    # the ABI gives dK / dV K's / V's strides: a batch stride must cover all Nkv rows
    # (B = 1, or K a view of the local rows of a [B, Nkv, H_kv, d] buffer)
    shp = (K.shape[0], Nkv, K.shape[2], K.shape[3])
    out = []
    for T in (K, V):
        if T.shape[0] > 1 and T.stride(0) < Nkv * T.stride(1):
            raise GfwaError("kv_halo with B > 1: K / V must be views of [B, N_kv, H_kv, d] buffers")
        out.append(torch.empty_strided(shp, T.stride(), dtype=T.dtype, device=T.device))
    return out[0], out[1]


def make_desc(Q, K, V, O_like, w: int, scale: float | None, kv_halo=None) -> AttnDesc:
    """kv_halo = (K_halo, V_halo): the in-kernel halo (include/gfwa.h): key rows
    [0, halo) are read from these tensors (e.g. CUDA-IPC / peer-mapped views of the
    previous shard's last rows) and K, V hold the remaining rows."""
    B, Nq, H, d = Q.shape
    hr = 0 if kv_halo is None else kv_halo[0].shape[1]
    Nkv = K.shape[1] + hr
    dsc = AttnDesc()
    dsc.B, dsc.H, dsc.N_q, dsc.N_kv, dsc.d, dsc.w = B, H, Nq, Nkv, d, int(w)
    dsc.scale = float(scale) if scale is not None else 0.0
    dsc.dtype = _dt(Q)
    dsc.q_stride[:] = _bnh_strides(Q)
    dsc.k_stride[:] = _bnh_strides(K)
    dsc.v_stride[:] = _bnh_strides(V)
    dsc.o_stride[:] = _bnh_strides(O_like)
    dsc.H_kv = K.shape[2] if K.shape[2] != H else 0  # GQA: K/V heads (0 = H)
    if kv_halo is not None:
        Kh, Vh = kv_halo
        if Kh.shape != Vh.shape or Kh.shape[0] != B or Kh.shape[2:] != K.shape[2:] or Kh.dtype != K.dtype:
            raise GfwaError("kv_halo tensors must be [B, halo_rows, H_kv, d] like K")
        dsc.halo_rows = hr
        dsc.K_halo, dsc.V_halo = Kh.data_ptr(), Vh.data_ptr()
        dsc.kh_stride[:] = _bnh_strides(Kh)
        dsc.vh_stride[:] = _bnh_strides(Vh)
    return dsc


# --------------------------------------------------------------------------- gate


def gfwa_gate_prefix(h: torch.Tensor, beta: torch.Tensor | None = None, eps: float = 1e-6,
                     carry_in: torch.Tensor | None = None, want_total: bool = False, alpha_input: bool = False):
    """U [B,H,N] fp32 (and total [B,H] fp64) from h, beta [B,N,H] (Alg. 1).

    alpha_input=True: ``h`` holds alpha directly (GFWA_GATE_ALPHA)."""
    lib = load()
    _need_cuda(h, beta, carry_in)
    h = h.contiguous()
    beta = None if beta is None else beta.to(h.dtype).contiguous()  # one in_dtype for both
    B, N, H = h.shape
    U = torch.empty(B, H, N, dtype=torch.float32, device=h.device)
    total = torch.empty(B, H, dtype=torch.float64, device=h.device) if want_total else None
    if carry_in is not None:
        carry_in = carry_in.to(torch.float64).contiguous()
    nbytes = lib.gfwa_gate_prefix_workspace_size(B, N, H)
    ws = workspace(nbytes, h.device, "gate")
    kind = GATE_ALPHA if alpha_input else GATE_HBETA
    st = lib.gfwa_gate_prefix(kind, _dt(h), _ptr(h), _ptr(beta), B, N, H, float(eps), _ptr(carry_in), _ptr(U),
                              _ptr(total), _ptr(ws), nbytes, _stream(h.device))
    _check(st, "gfwa_gate_prefix")
    return (U, total) if want_total else U


def gfwa_gate_prefix_variant(variant: int, h: torch.Tensor, beta: torch.Tensor, eps: float = 1e-6):
    """U [B,H,N] by one of the paper's comparison designs:
    1 = one program per head with an on-chip carry, 2 = Scan-Then-Propagate
    (App. E.1).  Benchmark/parity use only; the product call is
    gfwa_gate_prefix."""
    lib = load()
    _need_cuda(h, beta)
    h = h.contiguous()
    beta = beta.to(h.dtype).contiguous()
    B, N, H = h.shape
    U = torch.empty(B, H, N, dtype=torch.float32, device=h.device)
    nbytes = lib.gfwa_gate_prefix_variant_workspace_size(variant, B, N, H)
    ws = workspace(nbytes, h.device, f"gate_v{variant}")
    st = lib.gfwa_gate_prefix_variant(variant, _dt(h), _ptr(h), _ptr(beta), B, N, H, float(eps), _ptr(U), _ptr(ws),
                                      nbytes, _stream(h.device))
    _check(st, "gfwa_gate_prefix_variant")
    return U


def gfwa_gate_prefix_bwd(dU: torch.Tensor, h: torch.Tensor | None = None, beta: torch.Tensor | None = None,
                         eps: float = 1e-6, carry: torch.Tensor | None = None, want_dalpha: bool = True,
                         want_dh: bool = True):
    """dalpha [B,H,N] (reverse scan) and dh, dbeta [B,N,H] (chain rule of Eq. 9)."""
    lib = load()
    _need_cuda(dU, h, beta, carry)
    dU = dU.to(torch.float32).contiguous()
    B, H, N = dU.shape
    dev = dU.device
    io_dt = h.dtype if h is not None else torch.float32  # dh, dbeta in the dtype of h, beta
    dalpha = torch.empty(B, H, N, dtype=torch.float32, device=dev) if want_dalpha else None
    dh = dbeta = None
    if want_dh and h is not None:
        h = h.contiguous()
        beta = beta.to(io_dt).contiguous()
        dh = torch.empty(B, N, H, dtype=io_dt, device=dev)
        dbeta = torch.empty(B, N, H, dtype=io_dt, device=dev)
    if carry is not None:
        carry = carry.to(torch.float64).contiguous()
    nbytes = lib.gfwa_gate_prefix_bwd_workspace_size(B, N, H)
    ws = workspace(nbytes, dev, "gate")
    in_dt = GFWA_BF16 if io_dt == torch.bfloat16 else GFWA_F32
    st = lib.gfwa_gate_prefix_bwd(GATE_HBETA, in_dt, _ptr(h), _ptr(beta), B, N, H, float(eps), _ptr(dU),
                                  _ptr(carry), _ptr(dalpha), _ptr(dh), _ptr(dbeta), _ptr(ws), nbytes,
                                  _stream(dev))
    _check(st, "gfwa_gate_prefix_bwd")
    return dalpha, dh, dbeta


# --------------------------------------------------------------------------- attention


def gfwa_fwd(Q, K, V, U, w: int, scale: float | None = None, want_o_lo: bool = False, out=None, out_lo=None,
             prepare_bwd: bool = False, kv_halo=None):
    """O [B,Nq,H,d], LSE [B,H,Nq] (+ O_lo) per Eq. 12 / Alg. 2.
    O_lo (bf16 only; None for fp32, whose O is exact): the bf16 residual of the
    output cast, bf16(O_exact - O), for the backward's D (reading C-12).
    out / out_lo: caller tensors (views allowed) receiving O and O_lo; O_lo must
    share O's element strides (the ABI's one stride set).
    prepare_bwd: gfwa_fwd_train on the workspace gfwa_bwd will use (the forward
    zeroes the backward's dQ accumulator; the next gfwa_bwd skips that pass).
    kv_halo = (K_halo, V_halo): the first key rows come from these tensors (the
    in-kernel halo of include/gfwa.h); K, V hold the rest and U covers all rows."""
    lib = load()
    _need_cuda(Q, K, V, U)
    U = U.contiguous()
    B, Nq, H, d = Q.shape
    O = out if out is not None else torch.empty(B, Nq, H, d, dtype=Q.dtype, device=Q.device)
    O_lo = None
    if Q.dtype == torch.bfloat16:
        if out_lo is not None:
            if out_lo.stride() != O.stride() or out_lo.dtype != torch.bfloat16:
                raise GfwaError("out_lo must be bf16 with the strides of O")
            O_lo = out_lo
        elif want_o_lo:
            O_lo = torch.empty_strided(O.shape, O.stride(), dtype=torch.bfloat16, device=Q.device)
    LSE = torch.empty(B, H, Nq, dtype=torch.float32, device=Q.device)
    dsc = make_desc(Q, K, V, O, w, scale, kv_halo)
    if prepare_bwd:
        nbytes = lib.gfwa_bwd_workspace_size(ctypes.byref(dsc))
        ws = workspace(nbytes, Q.device, "bwd")  # the tensor gfwa_bwd below takes
        st = lib.gfwa_fwd_train(ctypes.byref(dsc), _ptr(Q), _ptr(K), _ptr(V), _ptr(U), _ptr(O), _ptr(O_lo),
                                _ptr(LSE), _ptr(ws), nbytes, _stream(Q.device))
        _check(st, "gfwa_fwd_train")
        return O, LSE, O_lo
    st = lib.gfwa_fwd(ctypes.byref(dsc), _ptr(Q), _ptr(K), _ptr(V), _ptr(U), _ptr(O), _ptr(O_lo), _ptr(LSE),
                      _stream(Q.device))
    _check(st, "gfwa_fwd")
    return O, LSE, O_lo


def gfwa_bwd(Q, K, V, U, O, LSE, dO, w: int, scale: float | None = None, O_lo=None, want_dalpha: bool = True,
             dalpha_carry=None, kv_halo=None):
    """dQ, dK, dV, dU (+ dalpha) per Alg. E.2; D = rowsum((O + O_lo) dO).
    kv_halo: as in gfwa_fwd; dK, dV then cover all N_kv rows (halo rows first)."""
    lib = load()
    _need_cuda(Q, K, V, U, O, LSE, dO)
    if dO.stride() != O.stride() or (O_lo is not None and O_lo.stride() != O.stride()):
        # O, dO and O_lo share one (b, n, h) stride set in the ABI
        O, dO = O.contiguous(), dO.contiguous()
        O_lo = None if O_lo is None else O_lo.contiguous()
    B, Nq, H, d = Q.shape
    dev = Q.device
    dsc = make_desc(Q, K, V, O, w, scale, kv_halo)
    Nkv = dsc.N_kv
    dQ = torch.empty_strided(Q.shape, Q.stride(), dtype=Q.dtype, device=dev)
    dK, dV = _grad_kv(K, V, Nkv)
    dU = torch.empty(B, H, Nkv, dtype=torch.float32, device=dev)
    dalpha = torch.empty(B, H, Nkv, dtype=torch.float32, device=dev) if want_dalpha else None
    if dalpha_carry is not None:
        dalpha_carry = dalpha_carry.to(torch.float64).contiguous()
    nbytes = lib.gfwa_bwd_workspace_size(ctypes.byref(dsc))
    ws = workspace(nbytes, dev, "bwd")
    st = lib.gfwa_bwd(ctypes.byref(dsc), _ptr(Q), _ptr(K), _ptr(V), _ptr(U.contiguous()), _ptr(O), _ptr(O_lo),
                      _ptr(LSE), _ptr(dO), _ptr(dQ), _ptr(dK), _ptr(dV), _ptr(dU), _ptr(dalpha),
                      _ptr(dalpha_carry), _ptr(ws), nbytes, _stream(dev))
    _check(st, "gfwa_bwd")
    return dQ, dK, dV, dU, dalpha


def gfwa_fwd_normgate(Q, K, V, U, g, gamma, w: int, eps: float = 1e-5, scale: float | None = None,
                      want_o_lo: bool = True, prepare_bwd: bool = False):
    """AttnLayer forward (reading C-27): the attention of gfwa_fwd plus, in
    its epilogue, Y = swish(g) * gamma * O * rstd per (b, t, h) row, rstd =
    1/sqrt(mean_c O_c^2 + eps).  g [B,Nq,H,d] bf16 (the gate pre-activation
    linear(X)); gamma [d] fp32.  Returns (Y, O, LSE, O_lo, rstd)."""
    lib = load()
    _need_cuda(Q, K, V, U, g, gamma)
    B, Nq, H, d = Q.shape
    dev = Q.device
    O = torch.empty(B, Nq, H, d, dtype=Q.dtype, device=dev)
    Y = torch.empty_like(O)
    O_lo = torch.empty_like(O) if want_o_lo else None
    LSE = torch.empty(B, H, Nq, dtype=torch.float32, device=dev)
    rstd = torch.empty(B, H, Nq, dtype=torch.float32, device=dev)
    g = g.contiguous()
    gamma = gamma.to(torch.float32).contiguous()
    ng = NormGate(_ptr(g), _ptr(gamma), float(eps), _ptr(rstd))
    dsc = make_desc(Q, K, V, O, w, scale)
    ws, nbytes = None, 0
    if prepare_bwd:
        nbytes = lib.gfwa_bwd_workspace_size(ctypes.byref(dsc))
        ws = workspace(nbytes, dev, "bwd")
    st = lib.gfwa_fwd_normgate(ctypes.byref(dsc), _ptr(Q), _ptr(K), _ptr(V), _ptr(U.contiguous()), ctypes.byref(ng),
                               _ptr(O), _ptr(O_lo), _ptr(LSE), _ptr(Y), _ptr(ws), nbytes, _stream(dev))
    _check(st, "gfwa_fwd_normgate")
    return Y, O, LSE, O_lo, rstd


def gfwa_bwd_normgate(Q, K, V, U, O, LSE, g, gamma, rstd, dY, w: int, eps: float = 1e-5,
                      scale: float | None = None, O_lo=None, want_dalpha: bool = True, dalpha_carry=None):
    """AttnLayer backward from dY: the epilogue's chain rule (dO~, dg, dgamma) fused into
    the backward's preprocess, then Alg. E.2 on dO~.  Returns
    (dQ, dK, dV, dU, dalpha, dg, dgamma, dO~)."""
    lib = load()
    _need_cuda(Q, K, V, U, O, LSE, g, gamma, rstd, dY)
    B, Nq, H, d = Q.shape
    Nkv = K.shape[1]
    dev = Q.device
    O = O.contiguous()
    O_lo = None if O_lo is None else O_lo.contiguous()
    g, dY = g.contiguous(), dY.contiguous()
    gamma = gamma.to(torch.float32).contiguous()
    dO = torch.empty_like(O)
    dg = torch.empty_like(O)
    dgamma = torch.empty(d, dtype=torch.float32, device=dev)
    dQ = torch.empty_strided(Q.shape, Q.stride(), dtype=Q.dtype, device=dev)
    dK = torch.empty_strided(K.shape, K.stride(), dtype=K.dtype, device=dev)
    dV = torch.empty_strided(V.shape, V.stride(), dtype=V.dtype, device=dev)
    dU = torch.empty(B, H, Nkv, dtype=torch.float32, device=dev)
    dalpha = torch.empty(B, H, Nkv, dtype=torch.float32, device=dev) if want_dalpha else None
    if dalpha_carry is not None:
        dalpha_carry = dalpha_carry.to(torch.float64).contiguous()
    ng = NormGate(_ptr(g), _ptr(gamma), float(eps), _ptr(rstd.contiguous()))
    dsc = make_desc(Q, K, V, O, w, scale)
    nbytes = lib.gfwa_bwd_workspace_size(ctypes.byref(dsc))
    ws = workspace(nbytes, dev, "bwd")
    st = lib.gfwa_bwd_normgate(ctypes.byref(dsc), _ptr(Q), _ptr(K), _ptr(V), _ptr(U.contiguous()), _ptr(O),
                               _ptr(O_lo), _ptr(LSE), ctypes.byref(ng), _ptr(dY), _ptr(dO), _ptr(dg), _ptr(dgamma),
                               _ptr(dQ), _ptr(dK), _ptr(dV), _ptr(dU), _ptr(dalpha), _ptr(dalpha_carry), _ptr(ws),
                               nbytes, _stream(dev))
    _check(st, "gfwa_bwd_normgate")
    return dQ, dK, dV, dU, dalpha, dg, dgamma, dO


def gfwa_bwd_rows_f32(Q, K, V, U, O, LSE, dO, w: int, head_rows: int, tail_rows: int,
                      scale: float | None = None, O_lo=None, kv_halo=None):
    """gfwa_bwd plus fp32 copies [2 (dK, dV), B, rows, H_kv, d] of dK, dV for the first
    head_rows and last tail_rows key rows (sequence sharding: the halo's partial
    gradients travel and are added in fp32).  Returns (dQ, dK, dV, dU, head, tail)."""
    lib = load()
    _need_cuda(Q, K, V, U, O, LSE, dO)
    if dO.stride() != O.stride() or (O_lo is not None and O_lo.stride() != O.stride()):
        O, dO = O.contiguous(), dO.contiguous()
        O_lo = None if O_lo is None else O_lo.contiguous()
    B, Nq, H, d = Q.shape
    dev = Q.device
    dsc = make_desc(Q, K, V, O, w, scale, kv_halo)
    Nkv = dsc.N_kv
    dQ = torch.empty_strided(Q.shape, Q.stride(), dtype=Q.dtype, device=dev)
    dK, dV = _grad_kv(K, V, Nkv)
    dU = torch.empty(B, H, Nkv, dtype=torch.float32, device=dev)
    Hkv = K.shape[2]  # GQA: the copies have K's heads
    head = torch.empty(2, B, head_rows, Hkv, d, dtype=torch.float32, device=dev) if head_rows > 0 else None
    tail = torch.empty(2, B, tail_rows, Hkv, d, dtype=torch.float32, device=dev) if tail_rows > 0 else None
    nbytes = lib.gfwa_bwd_workspace_size(ctypes.byref(dsc))
    ws = workspace(nbytes, dev, "bwd")
    st = lib.gfwa_bwd_rows_f32(ctypes.byref(dsc), _ptr(Q), _ptr(K), _ptr(V), _ptr(U.contiguous()), _ptr(O),
                               _ptr(O_lo), _ptr(LSE), _ptr(dO), _ptr(dQ), _ptr(dK), _ptr(dV), _ptr(dU), None, None,
                               int(head_rows), _ptr(head), int(tail_rows), _ptr(tail), _ptr(ws), nbytes,
                               _stream(dev))
    _check(st, "gfwa_bwd_rows_f32")
    return dQ, dK, dV, dU, head, tail


def gfwa_nsa_fwd(Q, K, V, U, gates, w: int, block: int = 64, n_sel: int = 16, scale: float | None = None):
    """NSA hybrid forward with GatedFWA as the local branch (App. B; readings
    C-28, C-29): O = sigmoid(g0) o_cmp + sigmoid(g1) o_slc + sigmoid(g2) o_gatedfwa.
    Q, K, V [B,N,H,d] bf16; U [B,H,N]; gates [B,N,H,3] fp32 logits.  Returns (O, saved):
    saved is a dict of the tensors gfwa_nsa_bwd needs (o_cmp, o_slc, the LSEs, the
    selection, the local branch's output and residual)."""
    lib = load()
    _need_cuda(Q, K, V, U, gates)
    B, N, H, d = Q.shape
    dev = Q.device
    Q, K, V = Q.contiguous(), K.contiguous(), V.contiguous()
    U, gates = U.contiguous(), gates.float().contiguous()
    O = torch.empty_like(Q)
    f32 = lambda *sh: torch.empty(*sh, dtype=torch.float32, device=dev)  # noqa: E731
    sv = {"O_cmp": f32(B, N, H, d), "O_slc": f32(B, N, H, d), "LSE_cmp": f32(B, H, N), "LSE_slc": f32(B, H, N),
          "sel": torch.empty(B, H, N, n_sel + 1, dtype=torch.int32, device=dev), "O_loc": torch.empty_like(Q),
          "O_loc_lo": torch.empty_like(Q), "LSE_loc": f32(B, H, N)}
    saved = NsaSaved(*[_ptr(sv[n]) for n, _ in NsaSaved._fields_])
    dsc = NsaDesc(B, H, N, d, w, block, n_sel, -1.0 if scale is None else float(scale), GFWA_BF16)
    nbytes = lib.gfwa_nsa_workspace_size(ctypes.byref(dsc))
    ws = workspace(nbytes, dev, "nsa")
    st = lib.gfwa_nsa_fwd(ctypes.byref(dsc), _ptr(Q), _ptr(K), _ptr(V), _ptr(U), _ptr(gates), _ptr(O),
                          ctypes.byref(saved), _ptr(ws), nbytes, _stream(dev))
    _check(st, "gfwa_nsa_fwd")
    return O, sv


def gfwa_nsa_bwd(Q, K, V, U, gates, dO, saved, w: int, block: int = 64, n_sel: int = 16,
                 scale: float | None = None):
    """The NSA hybrid's backward (fixed selection): (dQ, dK, dV, dU, dgates)."""
    lib = load()
    _need_cuda(Q, K, V, U, gates, dO)
    B, N, H, d = Q.shape
    dev = Q.device
    Q, K, V, dO = Q.contiguous(), K.contiguous(), V.contiguous(), dO.contiguous()
    U, gates = U.contiguous(), gates.float().contiguous()
    dQ, dK, dV = torch.empty_like(Q), torch.empty_like(K), torch.empty_like(V)
    dU = torch.empty(B, H, N, dtype=torch.float32, device=dev)
    dg = torch.empty(B, N, H, 3, dtype=torch.float32, device=dev)
    sv = NsaSaved(*[_ptr(saved[n]) for n, _ in NsaSaved._fields_])
    dsc = NsaDesc(B, H, N, d, w, block, n_sel, -1.0 if scale is None else float(scale), GFWA_BF16)
    nbytes = lib.gfwa_nsa_workspace_size(ctypes.byref(dsc))
    ws = workspace(nbytes, dev, "nsa")
    st = lib.gfwa_nsa_bwd(ctypes.byref(dsc), _ptr(Q), _ptr(K), _ptr(V), _ptr(U), _ptr(gates), _ptr(dO),
                          ctypes.byref(sv), _ptr(dQ), _ptr(dK), _ptr(dV), _ptr(dU), _ptr(dg), _ptr(ws), nbytes,
                          _stream(dev))
    _check(st, "gfwa_nsa_bwd")
    return dQ, dK, dV, dU, dg


def gfwa_attn_path(Q, K, V, w: int) -> int:
    """0 = SIMT parity path, 1 = tcgen05 tensor-core path (for this shape/dtype)."""
    dsc = make_desc(Q, K, V, Q, w, None)
    return int(load().gfwa_attn_path(ctypes.byref(dsc)))


# --------------------------------------------------------------------------- decode


def gfwa_decode(q, k_new, v_new, gate_a, K_cache, V_cache, U_cache, pos, gate_b=None, eps: float = 1e-6,
                scale: float | None = None, out=None):
    """One decode step (reading C-16); caches are updated in place.  gate_b=None
    means gate_a holds alpha directly; else (gate_a, gate_b) = (h, beta)."""
    lib = load()
    _need_cuda(q, k_new, v_new, gate_a, K_cache, V_cache, U_cache, pos)
    B, H, d = q.shape
    Hkv, w = K_cache.shape[1], K_cache.shape[2]  # Hkv < H: GQA groups of H // Hkv query heads
    for t in (q, k_new, v_new, K_cache, V_cache, U_cache):
        if not t.is_contiguous():
            raise GfwaError("decode tensors must be contiguous")
    dsc = DecodeDesc()
    dsc.B, dsc.H, dsc.d, dsc.w, dsc.H_kv = B, H, d, w, Hkv
    dsc.scale = float(scale) if scale is not None else 0.0
    dsc.eps = float(eps)
    dsc.dtype = _dt(q)
    dsc.gate_kind = GATE_ALPHA if gate_b is None else GATE_HBETA
    o = out if out is not None else torch.empty_like(q)
    ga = gate_a.float().contiguous()
    gb = None if gate_b is None else gate_b.float().contiguous()
    nbytes = lib.gfwa_decode_workspace_size(ctypes.byref(dsc))
    ws = workspace(nbytes, q.device, f"decode{B}x{H}x{Hkv}x{w}x{d}", zero=True)
    st = lib.gfwa_decode(ctypes.byref(dsc), _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(ga),
                         _ptr(gb), _ptr(K_cache),
                         _ptr(V_cache), _ptr(U_cache), _ptr(pos), _ptr(o), _ptr(ws), nbytes, _stream(q.device))
    _check(st, "gfwa_decode")
    return o


def gfwa_check_finite(x: torch.Tensor) -> bool:
    """Debug check (synchronises the stream): True if every element is finite.
    GFWA_CHECK_FINITE=1 makes gfwa_fwd / gfwa_bwd run it on their outputs and
    raise GFWA_ERR_NONFINITE."""
    lib = load()
    _need_cuda(x)
    x = x.contiguous()
    st = lib.gfwa_check_finite(_dt(x), _ptr(x), x.numel(), _stream(x.device))
    if st == 5:
        return False
    _check(st, "gfwa_check_finite")
    return True


def gfwa_debug_tc_selftest(Q, K, V, flags: int = 0):
    """S = Q K^T and O = bf16(S) V (flags & 1: fp16(S) V) on one 128x128 tile through the tcgen05 path."""
    lib = load()
    _need_cuda(Q, K, V)
    S = torch.empty(128, 128, dtype=torch.float32, device=Q.device)
    O = torch.empty_like(S)
    f = lib.gfwa_debug_tc_selftest_ex
    f.restype = ctypes.c_int
    f.argtypes = [_VP] * 5 + [ctypes.c_int, _VP]
    _check(f(_ptr(Q), _ptr(K), _ptr(V), _ptr(S), _ptr(O), int(flags), _stream(Q.device)), "gfwa_debug_tc_selftest")
    return S, O


def debug_stage_events(events) -> None:
    """Register torch.cuda.Event objects for the next tensor-core gfwa_bwd on this
    thread: events[0] after its preprocess kernel, events[1] after its main kernel."""
    lib = load()
    arr = (ctypes.c_void_p * 4)(*([e.cuda_event if e is not None else None for e in events] + [None] * 4)[:4])
    f = lib.gfwa_debug_stage_events
    f.restype = None
    f.argtypes = [ctypes.c_void_p, ctypes.c_int]
    f(ctypes.cast(arr, ctypes.c_void_p), len(events))


def launch_count() -> int:
    return int(load().gfwa_launch_count())


def version() -> str:
    return load().gfwa_version().decode()


def default_scale(d: int) -> float:
    return 1.0 / math.sqrt(d)
