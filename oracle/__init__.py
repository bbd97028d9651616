"""fp64 CPU oracle for the GatedFWA hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` leg may import this package.  It wraps
``oracle/gfwa_oracle.c`` (plain C, fp64 loops, OpenMP over (b, h)) through
ctypes and shares no code with ``paper_2512_07782_b200`` (neither imports the
other).  Inputs are numpy/torch arrays; they are converted to float64 (the
exact values the GPU saw, upcast) before the call.

See ``gfwa_oracle.c`` for the paper citations of every function.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gfwa_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.c_int64


def build(force: bool = False) -> str:
    """Compile gfwa_oracle.c -> liboracle.so with gcc -O2 -fopenmp."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.oracle_num_threads.restype = ctypes.c_int
        lib.oracle_attend_row.restype = ctypes.c_double
        _lib = lib
    return _lib


def _f64(x) -> np.ndarray:
    """Exact upcast of a torch tensor / numpy array to contiguous float64."""
    try:
        import torch

        if isinstance(x, torch.Tensor):
            x = x.detach().to("cpu", torch.float64).numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def _p(a: np.ndarray | None):
    if a is None:
        return ctypes.cast(None, _D)
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_D)


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def set_num_threads(n: int) -> None:
    """OpenMP threads of the oracle loops (torchrun exports OMP_NUM_THREADS=1)."""
    _load().oracle_set_num_threads(ctypes.c_int(int(n)))


def gate_alpha(h, beta, eps: float = 1e-6) -> np.ndarray:
    """alpha [B,H,N] from h, beta [B,N,H] (Eq. 9; Alg. 1 l.5-7)."""
    h, beta = _f64(h), _f64(beta)
    B, N, H = h.shape
    out = np.empty((B, H, N))
    _load().oracle_gate_alpha(_p(h), _p(beta), _I64(B), _I64(N), _I64(H), ctypes.c_double(eps), _p(out))
    return out


def gate_prefix(alpha, carry=None):
    """U [B,H,N] = carry - cumsum(alpha) (Eq. 11), total [B,H] = sum alpha."""
    alpha = _f64(alpha)
    B, H, N = alpha.shape
    U = np.empty((B, H, N))
    total = np.empty((B, H))
    c = None if carry is None else _f64(carry).reshape(B, H)
    _load().oracle_gate_prefix(_p(alpha), _I64(B), _I64(N), _I64(H), _p(c), _p(U), _p(total))
    return U, total


def gate_prefix_hbeta(h, beta, eps: float = 1e-6, carry=None):
    """Alg. 1 end to end: (h, beta) -> (U, total, alpha)."""
    alpha = gate_alpha(h, beta, eps)
    U, total = gate_prefix(alpha, carry)
    return U, total, alpha


def fwd(Q, K, V, U, w: int, scale: float | None = None):
    """O [B,Nq,H,d], LSE [B,H,Nq] per Eq. 12 / Alg. 2.

    Q [B,Nq,H,d]; K, V [B,Nkv,H,d]; U [B,H,Nkv]; queries are the last Nq keys.
    """
    Q, K, V, U = _f64(Q), _f64(K), _f64(V), _f64(U)
    B, Nq, H, d = Q.shape
    Nkv = K.shape[1]
    scale = 1.0 / np.sqrt(d) if scale is None else scale
    O = np.empty_like(Q)
    LSE = np.empty((B, H, Nq))
    _load().oracle_fwd(_I64(B), _I64(H), _I64(Nq), _I64(Nkv), _I64(d), _I64(w), ctypes.c_double(scale),
                       _p(Q), _p(K), _p(V), _p(U), _p(O), _p(LSE))
    return O, LSE


def fwd_rows(Q, K, V, U, w: int, rows, scale: float | None = None):
    """Eq. 12 evaluated only for the listed (b, h, t) rows -> (o [n,d], lse [n])."""
    Q, K, V, U = _f64(Q), _f64(K), _f64(V), _f64(U)
    B, Nq, H, d = Q.shape
    Nkv = K.shape[1]
    scale = 1.0 / np.sqrt(d) if scale is None else scale
    r = np.ascontiguousarray(np.asarray(rows, dtype=np.int64).reshape(-1, 3))
    n = r.shape[0]
    o = np.empty((n, d))
    lse = np.empty((n,))
    _load().oracle_fwd_rows(_I64(B), _I64(H), _I64(Nq), _I64(Nkv), _I64(d), _I64(w), ctypes.c_double(scale),
                            _p(Q), _p(K), _p(V), _p(U), _I64(n),
                            r.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _p(o), _p(lse))
    return o, lse


def attend_row(q, keys, vals, u, ut: float, scale: float | None = None):
    """One query over an explicit key list (decode, reading C-16) -> (o [d], lse)."""
    q, keys, vals, u = _f64(q), _f64(keys), _f64(vals), _f64(u)
    d = q.shape[-1]
    n = keys.shape[0]
    scale = 1.0 / np.sqrt(d) if scale is None else scale
    o = np.empty((d,))
    lse = _load().oracle_attend_row(_I64(d), ctypes.c_double(scale), _p(q), _I64(n), _p(keys), _p(vals),
                                    _p(u), ctypes.c_double(ut), _p(o))
    return o, float(lse)


def bwd(Q, K, V, U, dO, w: int, scale: float | None = None, dalpha_carry=None, want_dalpha: bool = True):
    """Alg. E.2 densely -> dict(dQ, dK, dV, dU, dalpha)."""
    Q, K, V, U, dO = _f64(Q), _f64(K), _f64(V), _f64(U), _f64(dO)
    B, Nq, H, d = Q.shape
    Nkv = K.shape[1]
    scale = 1.0 / np.sqrt(d) if scale is None else scale
    dQ = np.empty_like(Q)
    dK = np.empty_like(K)
    dV = np.empty_like(V)
    dU = np.empty((B, H, Nkv))
    dalpha = np.empty((B, H, Nkv)) if want_dalpha else None
    c = None if dalpha_carry is None else _f64(dalpha_carry).reshape(B, H)
    _load().oracle_bwd(_I64(B), _I64(H), _I64(Nq), _I64(Nkv), _I64(d), _I64(w), ctypes.c_double(scale),
                       _p(Q), _p(K), _p(V), _p(U), _p(dO), _p(dQ), _p(dK), _p(dV), _p(dU), _p(dalpha), _p(c))
    return {"dQ": dQ, "dK": dK, "dV": dV, "dU": dU, "dalpha": dalpha}


def dalpha_scan(dU, carry=None) -> np.ndarray:
    """dalpha = carry - reverse_cumsum(dU) over the last axis."""
    dU = _f64(dU)
    B, H, N = dU.shape
    out = np.empty_like(dU)
    c = None if carry is None else _f64(carry).reshape(B, H)
    _load().oracle_dalpha(_p(dU), _I64(B), _I64(H), _I64(N), _p(c), _p(out))
    return out


def gate_chain(h, beta, dalpha, eps: float = 1e-6):
    """(dh, dbeta) [B,N,H] from dalpha [B,H,N] (chain rule of Eq. 9)."""
    h, beta, dalpha = _f64(h), _f64(beta), _f64(dalpha)
    B, N, H = h.shape
    dh = np.empty_like(h)
    db = np.empty_like(h)
    _load().oracle_gate_chain(_p(h), _p(beta), _p(dalpha), _I64(B), _I64(N), _I64(H), ctypes.c_double(eps),
                              _p(dh), _p(db))
    return dh, db


def normgate_fwd(O, g, gamma, eps: float = 1e-5):
    """AttnLayer epilogue (reading C-27): Y = swish(g) * gamma * O * rstd
    per (b, t, h) row, rstd = 1/sqrt(mean_c O_c^2 + eps).  O, g [B,Nq,H,d];
    gamma [d].  Returns (Y [B,Nq,H,d], rstd [B,H,Nq])."""
    O, g, gamma = _f64(O), _f64(g), _f64(gamma)
    B, Nq, H, d = O.shape
    Y = np.empty_like(O)
    rstd = np.empty((B, H, Nq))
    _load().oracle_normgate_fwd(_p(O), _p(g), _p(gamma), _I64(B), _I64(Nq), _I64(H), _I64(d),
                                ctypes.c_double(eps), _p(Y), _p(rstd))
    return Y, rstd


def normgate_bwd(O, g, gamma, dY, eps: float = 1e-5):
    """Chain rule of normgate_fwd: (dO, dg [B,Nq,H,d], dgamma [d])."""
    O, g, gamma, dY = _f64(O), _f64(g), _f64(gamma), _f64(dY)
    B, Nq, H, d = O.shape
    dO = np.empty_like(O)
    dg = np.empty_like(O)
    dgamma = np.empty(d)
    _load().oracle_normgate_bwd(_p(O), _p(g), _p(gamma), _p(dY), _I64(B), _I64(Nq), _I64(H), _I64(d),
                                ctypes.c_double(eps), _p(dO), _p(dg), _p(dgamma))
    return dO, dg, dgamma


# --- NSA extension with GatedFWA as the local branch (App. B, C-28, C-29)


def nsa_compress(K, V, blk: int):
    """Block means Kc, Vc [B, N // blk, H, d] (C-28)."""
    K, V = _f64(K), _f64(V)
    B, N, H, d = K.shape
    nb = N // blk
    Kc, Vc = np.empty((B, nb, H, d)), np.empty((B, nb, H, d))
    _load().oracle_nsa_compress(_p(K), _p(V), _I64(B), _I64(N), _I64(H), _I64(d), _I64(blk), _p(Kc), _p(Vc))
    return Kc, Vc


def nsa_cmp(Q, Kc, Vc, blk: int, scale: float | None = None):
    """Compressed attention (O_cmp [B,N,H,d], scores [B,H,N,nb])."""
    Q, Kc, Vc = _f64(Q), _f64(Kc), _f64(Vc)
    B, N, H, d = Q.shape
    nb = N // blk
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    O = np.empty_like(Q)
    sc = np.empty((B, H, N, max(nb, 1)))
    _load().oracle_nsa_cmp(_p(Q), _p(Kc), _p(Vc), _I64(B), _I64(N), _I64(H), _I64(d), _I64(blk),
                           ctypes.c_double(scale), _p(O), _p(sc))
    return O, sc[..., :nb]


def nsa_select(scores, N: int, blk: int, nsel: int):
    """Selected blocks [B,H,N,nsel+1] (own block first, then top-nsel complete blocks; -1 pads)."""
    sc = _f64(scores)
    B, H = sc.shape[:2]
    sel = np.empty((B, H, N, nsel + 1), dtype=np.int64)
    _load().oracle_nsa_select(_p(sc), _I64(B), _I64(H), _I64(N), _I64(blk), _I64(nsel),
                              sel.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    return sel


def nsa_slc(Q, K, V, sel, blk: int, scale: float | None = None):
    """Selected-block attention O_slc [B,N,H,d] over the given selection."""
    Q, K, V = _f64(Q), _f64(K), _f64(V)
    sel = np.ascontiguousarray(np.asarray(sel, dtype=np.int64))
    B, N, H, d = Q.shape
    nsel = sel.shape[-1] - 1
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    O = np.empty_like(Q)
    _load().oracle_nsa_slc(_p(Q), _p(K), _p(V), sel.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _I64(B),
                           _I64(N), _I64(H), _I64(d), _I64(blk), _I64(nsel), ctypes.c_double(scale), _p(O))
    return O


def nsa_combine(Ocmp, Oslc, Oloc, g):
    """O = sigmoid(g0) O_cmp + sigmoid(g1) O_slc + sigmoid(g2) O_loc."""
    Ocmp, Oslc, Oloc, g = _f64(Ocmp), _f64(Oslc), _f64(Oloc), _f64(g)
    B, N, H, d = Ocmp.shape
    O = np.empty_like(Ocmp)
    _load().oracle_nsa_combine(_p(Ocmp), _p(Oslc), _p(Oloc), _p(g), _I64(B), _I64(N), _I64(H), _I64(d), _p(O))
    return O


def nsa_bwd(Q, K, V, U, g, dO, sel, w: int, blk: int, scale: float | None = None):
    """Chain rule of the NSA hybrid for a fixed selection: (dQ, dK, dV, dU, dgates)."""
    Q, K, V, U, g, dO = (_f64(x) for x in (Q, K, V, U, g, dO))
    sel = np.ascontiguousarray(np.asarray(sel, dtype=np.int64))
    B, N, H, d = Q.shape
    nsel = sel.shape[-1] - 1
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    dQ, dK, dV = np.empty_like(Q), np.empty_like(K), np.empty_like(V)
    dU = np.empty((B, H, N))
    dg = np.empty_like(g)
    _load().oracle_nsa_bwd(_p(Q), _p(K), _p(V), _p(U), _p(g), _p(dO), sel.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                           _I64(B), _I64(N), _I64(H), _I64(d), _I64(w), _I64(blk), _I64(nsel), ctypes.c_double(scale),
                           _p(dQ), _p(dK), _p(dV), _p(dU), _p(dg))
    return dQ, dK, dV, dU, dg


def nsa_fwd_fixed(Q, K, V, U, g, sel, w: int, blk: int, scale: float | None = None):
    """The NSA hybrid's output for a fixed selection (for finite differences)."""
    Kc, Vc = nsa_compress(K, V, blk)
    Oc, _ = nsa_cmp(Q, Kc, Vc, blk, scale)
    Os = nsa_slc(Q, K, V, sel, blk, scale)
    Ol, _ = fwd(Q, K, V, U, w, scale)
    return nsa_combine(Oc, Os, Ol, g)
