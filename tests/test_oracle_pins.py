"""Pins for the fp64 oracle (oracle/gfwa_oracle.c) against what the paper and
the mathematics fix -- never against the oracle's own formula retyped.

Each test names the passage it pins.  A plausible mistake anywhere in the
oracle (dropped term, wrong sign or index, transposed operand, wrong window
edge, wrong scale placement) fails at least one of them:

  gate     worked examples (S:104, S:124 -> tests/golden), softplus closed forms
           (S:49-51), library softplus, carry/total invariants
  fwd      torch fp64 SDPA (library routine) for alpha=0/w>=N (full causal),
           alpha=0 (SWA), and arbitrary U via a dense float mask; the
           constant-alpha closed form -a(t-j); the 2-token example;
           w=1 / N=1 special cases; shift invariance; the brute-force Prop. 2
           recurrence (P:189-198 with reading C-13); halo frame
  bwd      central finite differences (fp64) for dQ, dK, dV, dU, dalpha;
           torch fp64 autograd through the dense formulation; rowsum(dS)=0
           consequences (sum dU = 0, dalpha_0 = 0); dO=0, N=1, constant-dU
  chain    finite differences of alpha(h, beta)
"""
import math
import os

import numpy as np
import pytest
import torch

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
EPS = 1e-6


def _rand(shape, seed, scale=1.0):
    return np.random.default_rng(seed).standard_normal(shape) * scale


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def _read_golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                rows.append([float(x) for x in line.split()])
    return rows


# ----------------------------------------------------------------------------- gate


def test_gate_worked_example_h0_beta1():
    """S:104 / S:124: h=0, beta=1 => alpha = ln2/(1+eps), U_t = -(t+1) ln2/(1+eps)."""
    (eps, N), (alpha_ref,), U_ref = _read_golden("gate_h0_beta1.txt")
    N = int(N)
    h = np.zeros((1, N, 1))
    beta = np.ones((1, N, 1))
    U, total, alpha = oracle.gate_prefix_hbeta(h, beta, eps)
    assert np.allclose(alpha[0, 0], alpha_ref, rtol=1e-15, atol=0)
    assert np.allclose(U[0, 0], U_ref, rtol=1e-15, atol=0)
    assert total[0, 0] == pytest.approx(N * alpha_ref, rel=1e-15)


def test_softplus_closed_forms():
    """softplus(0)=ln2, softplus(100)~100 without overflow, softplus(-50)~e^-50;
    S:63: softplus(z) - softplus(-z) = z.  Probed through alpha with beta=1."""
    z = np.array([0.0, 100.0, -50.0, 3.0, -3.0, 700.0, -700.0])
    h = z.reshape(1, -1, 1)
    a = oracle.gate_alpha(h, np.ones_like(h), EPS)[0, 0] * (1 + EPS)
    assert a[0] == pytest.approx(math.log(2.0), rel=1e-15)
    assert a[1] == pytest.approx(100.0 + math.exp(-100.0), rel=1e-15)
    assert a[2] == pytest.approx(math.exp(-50.0) - math.exp(-100.0) / 2, rel=1e-14)
    assert np.isfinite(a).all() and (a > 0).all()
    assert a[3] - a[4] == pytest.approx(3.0, rel=1e-14)
    assert a[5] == pytest.approx(700.0, rel=1e-15)
    assert 0 <= a[6] < 1e-300 or a[6] == 0.0


def test_gate_alpha_vs_library_softplus():
    """Eq. 9: alpha = softplus(beta*h)/(beta+eps), vs torch's fp64 softplus."""
    h = _rand((2, 37, 3), 1, 3.0)
    beta = 1.0 + torch.nn.functional.elu(torch.from_numpy(_rand((2, 37, 3), 2, 0.5))).numpy()
    a = oracle.gate_alpha(h, beta, EPS)
    ref = torch.nn.functional.softplus(torch.from_numpy(beta * h), beta=1.0, threshold=1e9).numpy() / (beta + EPS)
    assert _rel(a, ref.transpose(0, 2, 1)) < 1e-14


def test_gate_prefix_invariants():
    """Eq. 11: U strictly decreasing (alpha>0), U_{N-1} = -sum(alpha),
    carry adds a constant (north_star exclusive scan), constant alpha -> linear."""
    alpha = np.abs(_rand((2, 3, 101), 3)) + 1e-3
    U, total = oracle.gate_prefix(alpha)
    assert (np.diff(U, axis=-1) < 0).all()
    assert np.allclose(U[..., -1], -alpha.sum(-1), rtol=1e-13)
    assert np.allclose(total, alpha.sum(-1), rtol=1e-13)
    carry = _rand((2, 3), 4)
    U2, _ = oracle.gate_prefix(alpha, carry)
    assert np.allclose(U2 - carry[..., None], U, rtol=0, atol=1e-12)
    Uc, _ = oracle.gate_prefix(np.full((1, 1, 10), 0.3))
    assert np.allclose(Uc[0, 0], -0.3 * np.arange(1, 11), rtol=1e-14)


# ----------------------------------------------------------------------------- forward


def _sdpa(Q, K, V, mask):
    """torch fp64 SDPA; Q [B,N,H,d] -> [B,N,H,d]; mask [B,H,N,N] float (additive)."""
    q, k, v = (torch.from_numpy(np.ascontiguousarray(x.transpose(0, 2, 1, 3))) for x in (Q, K, V))
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v, attn_mask=torch.from_numpy(mask))
    return o.numpy().transpose(0, 2, 1, 3)


def _window_mask(N, w):
    t = np.arange(N)[:, None]
    j = np.arange(N)[None, :]
    return (j <= t) & (j > t - w)


def _qkv(B, N, H, d, seed):
    return _rand((B, N, H, d), seed), _rand((B, N, H, d), seed + 1), _rand((B, N, H, d), seed + 2)


@pytest.mark.parametrize("N,w", [(13, 13), (13, 40), (1, 1), (24, 24)])
def test_fwd_alpha0_full_causal_is_sdpa(N, w):
    """north_star / S:205: alpha=0 and w>=N reduces to full causal softmax attention."""
    B, H, d = 2, 3, 8
    Q, K, V = _qkv(B, N, H, d, 10)
    O, _ = oracle.fwd(Q, K, V, np.zeros((B, H, N)), w)
    q, k, v = (torch.from_numpy(np.ascontiguousarray(x.transpose(0, 2, 1, 3))) for x in (Q, K, V))
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True).numpy().transpose(0, 2, 1, 3)
    assert _rel(O, ref) < 1e-13


@pytest.mark.parametrize("N,w", [(17, 1), (17, 3), (17, 5), (33, 8)])
def test_fwd_alpha0_is_swa(N, w):
    """north_star / S:204: alpha=0 reduces to SWA with window {j: t-w < j <= t}."""
    B, H, d = 1, 2, 8
    Q, K, V = _qkv(B, N, H, d, 20)
    O, _ = oracle.fwd(Q, K, V, np.zeros((B, H, N)), w)
    mask = np.where(_window_mask(N, w), 0.0, -np.inf)[None, None].repeat(H, 1)
    assert _rel(O, _sdpa(Q, K, V, mask)) < 1e-13


@pytest.mark.parametrize("N,w", [(19, 4), (19, 19), (30, 7)])
def test_fwd_general_U_is_dense_masked_sdpa(N, w):
    """Eq. 12: softmax(qk/sqrt(d) + u_t - u_j) over the window, as
    torch fp64 SDPA with a dense float mask B + (-inf outside the window)."""
    B, H, d = 2, 2, 8
    Q, K, V = _qkv(B, N, H, d, 30)
    alpha = np.abs(_rand((B, H, N), 33))
    U = -np.cumsum(alpha, axis=-1)
    bias = U[..., :, None] - U[..., None, :]
    mask = np.where(_window_mask(N, w)[None, None], bias, -np.inf)
    O, LSE = oracle.fwd(Q, K, V, U, w)
    assert _rel(O, _sdpa(Q, K, V, mask)) < 1e-13
    # LSE: natural log of the masked biased partition function.
    s = np.einsum("bthc,bjhc->bhtj", Q, K) / math.sqrt(d) + mask
    ref = np.log(np.exp(s - s.max(-1, keepdims=True)).sum(-1)) + s.max(-1)
    assert np.allclose(LSE, ref, rtol=1e-13, atol=1e-13)


def test_fwd_constant_alpha_closed_form():
    """north_star: constant alpha=a gives the closed-form bias -a(t-j) (ALiBi-like);
    the mask is built from the closed form, not from U."""
    B, N, H, d, w, a = 1, 21, 2, 8, 6, 0.3
    Q, K, V = _qkv(B, N, H, d, 40)
    U, _ = oracle.gate_prefix(np.full((B, H, N), a))
    t = np.arange(N)[:, None]
    j = np.arange(N)[None, :]
    mask = np.where(_window_mask(N, w), -a * (t - j), -np.inf)[None, None].repeat(H, 1)
    O, _ = oracle.fwd(Q, K, V, U, w)
    assert _rel(O, _sdpa(Q, K, V, mask)) < 1e-13


def test_fwd_two_token_worked_example():
    """N=2, w=2, equal logits, u1-u0 = -ln3 => weights (1/4, 3/4)."""
    ((w0, w1),) = _read_golden("two_token_weights.txt")
    d = 4
    Q = np.zeros((1, 2, 1, d))
    Q[0, 1, 0, 0] = 1.0
    K = np.zeros((1, 2, 1, d))
    K[0, :, 0, 0] = 0.7  # equal logits for query 1
    V = np.zeros((1, 2, 1, d))
    V[0, 0, 0, 0] = 1.0  # o[0] = weight on key 0
    V[0, 1, 0, 1] = 1.0  # o[1] = weight on key 1
    U = np.array([[[0.0, -math.log(3.0)]]])
    O, _ = oracle.fwd(Q, K, V, U, 2)
    assert O[0, 1, 0, 0] == pytest.approx(w0, rel=1e-14)
    assert O[0, 1, 0, 1] == pytest.approx(w1, rel=1e-14)


def test_fwd_special_cases():
    """w=1 => O=V; N=1 => O=v0 and LSE = scale q0.k0;
    U + c leaves O and LSE unchanged."""
    B, N, H, d = 2, 9, 2, 8
    Q, K, V = _qkv(B, N, H, d, 50)
    U = -np.cumsum(np.abs(_rand((B, H, N), 51)), -1)
    O, _ = oracle.fwd(Q, K, V, U, 1)
    assert np.allclose(O, V, rtol=0, atol=1e-15)
    O1, L1 = oracle.fwd(Q[:, :1], K[:, :1], V[:, :1], U[..., :1], 5)
    assert np.allclose(O1, V[:, :1], atol=1e-15)
    assert np.allclose(L1[:, :, 0], np.einsum("bhc,bhc->bh", Q[:, 0], K[:, 0]) / math.sqrt(d), rtol=1e-14)
    Oa, La = oracle.fwd(Q, K, V, U, 4)
    Ob, Lb = oracle.fwd(Q, K, V, U + 123.25, 4)
    assert np.allclose(Oa, Ob, atol=1e-13) and np.allclose(La, Lb, atol=1e-12)


@pytest.mark.parametrize("w,t", [(16, 40), (5, 30), (1, 12), (3, 2)])
def test_fwd_brute_force_gated_recurrence(w, t):
    """Prop. 2 (proof P:927-969) with reading C-13: for a fixed query
    q_t, run the gated memory recurrence over s = 0..t
        A_s = e^{-alpha_s} A_{s-1} + e^{x_s} v_s - [s>=w] (prod_{j=s-w+1}^{s} e^{-alpha_j}) e^{x_{s-w}} v_{s-w}
    (x_i = q_t.k_i/sqrt(d), Z the same with v=1).  Then A_t/Z_t = O_t exactly.
    The leaving coefficient is built from alpha directly, not from U."""
    B, H, N, d = 1, 1, 64, 8
    Q, K, V = _qkv(B, N, H, d, 60 + w)
    alpha = 0.05 + 0.05 * np.abs(_rand((N,), 61))  # small alpha keeps C-13 sharp
    U, _ = oracle.gate_prefix(alpha.reshape(1, 1, N))
    O, _ = oracle.fwd(Q, K, V, U, w)
    q = Q[0, t, 0]
    x = K[0, :, 0] @ q / math.sqrt(d)
    A = np.zeros(d)
    Z = 0.0
    A_paper = np.zeros(d)
    Z_paper = 0.0
    for s in range(t + 1):
        decay = math.exp(-alpha[s])
        A = decay * A + math.exp(x[s]) * V[0, s, 0]
        Z = decay * Z + math.exp(x[s])
        A_paper = decay * A_paper + math.exp(x[s]) * V[0, s, 0]
        Z_paper = decay * Z_paper + math.exp(x[s])
        if s >= w:
            leave = math.exp(-alpha[s - w + 1 : s + 1].sum())  # exact: e^{B_{s,s-w}} (C-13)
            leave_paper = math.exp(-alpha[s - w + 1 : s].sum())  # Eq. 13 as printed: c_s
            A -= leave * math.exp(x[s - w]) * V[0, s - w, 0]
            Z -= leave * math.exp(x[s - w])
            A_paper -= leave_paper * math.exp(x[s - w]) * V[0, s - w, 0]
            Z_paper -= leave_paper * math.exp(x[s - w])
    assert np.allclose(A / Z, O[0, t, 0], rtol=1e-11, atol=1e-12)
    if t >= w:  # the printed c_t misses by e^{-alpha_t}: documents reading C-13
        assert np.max(np.abs(A_paper / Z_paper - O[0, t, 0])) > 1e-9


def test_fwd_halo_frame_matches_full_run():
    """north_star sequence sharding: queries are the last Nq of Nkv keys (h0 = Nkv-Nq
    halo rows); the result equals the matching rows of the unsharded run, and a
    constant shift of the halo frame's U changes nothing."""
    B, N, H, d, w = 1, 40, 2, 8, 7
    Q, K, V = _qkv(B, N, H, d, 70)
    U = -np.cumsum(np.abs(_rand((B, H, N), 71)), -1)
    O, L = oracle.fwd(Q, K, V, U, w)
    s, h0 = 24, 7  # shard starts at 24, halo of w rows
    Os, Ls = oracle.fwd(Q[:, s:], K[:, s - h0 :], V[:, s - h0 :], U[..., s - h0 :] - U[..., s - 1 : s], w)
    assert np.allclose(Os, O[:, s:], atol=1e-13) and np.allclose(Ls, L[..., s:], atol=1e-12)
    rows = [(0, 1, 3), (0, 0, 39), (0, 1, 0)]
    o, lse = oracle.fwd_rows(Q, K, V, U, w, rows)
    for i, (b, hh, t) in enumerate(rows):
        assert np.allclose(o[i], O[b, t, hh], atol=1e-15) and lse[i] == pytest.approx(L[b, hh, t], abs=1e-14)


def test_attend_row_is_fwd_row():
    """Decode reading C-16: one query over its explicit window list == fwd row t."""
    B, N, H, d, w = 1, 30, 1, 8, 6
    Q, K, V = _qkv(B, N, H, d, 80)
    U = -np.cumsum(np.abs(_rand((B, H, N), 81)), -1)
    O, L = oracle.fwd(Q, K, V, U, w)
    for t in (0, 3, 5, 29):
        lo = max(0, t - w + 1)
        perm = np.random.default_rng(t).permutation(t + 1 - lo)  # ring order is irrelevant
        idx = np.arange(lo, t + 1)[perm]
        o, lse = oracle.attend_row(Q[0, t, 0], K[0, idx, 0], V[0, idx, 0], U[0, 0, idx], U[0, 0, t])
        assert np.allclose(o, O[0, t, 0], atol=1e-14) and lse == pytest.approx(L[0, 0, t], abs=1e-13)


# ----------------------------------------------------------------------------- backward


def _loss(Q, K, V, U, dO, w):
    O, _ = oracle.fwd(Q, K, V, U, w)
    return float(np.sum(O * dO))


def _fd(f, x, idx, h=1e-6):
    xp = x.copy()
    xm = x.copy()
    xp[idx] += h
    xm[idx] -= h
    return (f(xp) - f(xm)) / (2 * h)


@pytest.mark.parametrize("N,d,w", [(7, 4, 1), (9, 8, 3), (8, 4, 8), (12, 4, 5)])
def test_bwd_finite_differences(N, d, w):
    """S:215/S:278/S:583: central FD in fp64 of L = sum(O*dO) w.r.t. Q, K, V, U and
    alpha (U = -cumsum(alpha)) matches dQ, dK, dV, dU, dalpha (readings C-3, C-4)."""
    B, H = 1, 2
    Q, K, V = _qkv(B, N, H, d, 90)
    dO = _rand((B, N, H, d), 93)
    alpha = 0.1 + np.abs(_rand((B, H, N), 94))
    U, _ = oracle.gate_prefix(alpha)
    g = oracle.bwd(Q, K, V, U, dO, w)
    rng = np.random.default_rng(95)
    for name, x, grad in (("Q", Q, g["dQ"]), ("K", K, g["dK"]), ("V", V, g["dV"])):
        for _ in range(6):
            idx = tuple(int(rng.integers(0, s)) for s in x.shape)

            def f(xx, name=name):
                args = {"Q": Q, "K": K, "V": V}
                args[name] = xx
                return _loss(args["Q"], args["K"], args["V"], U, dO, w)

            assert _fd(f, x, idx) == pytest.approx(grad[idx], rel=1e-6, abs=1e-8), name
    for m in range(N):
        idx = (0, 1, m)
        assert _fd(lambda uu: _loss(Q, K, V, uu, dO, w), U, idx) == pytest.approx(g["dU"][idx], rel=1e-6, abs=1e-8)
        fa = lambda aa: _loss(Q, K, V, oracle.gate_prefix(aa)[0], dO, w)  # noqa: E731
        assert _fd(fa, alpha, idx) == pytest.approx(g["dalpha"][idx], rel=1e-6, abs=1e-8)


def test_bwd_vs_torch_autograd():
    """Library routine: torch fp64 autograd through the dense masked formulation
    of Eq. 12 with alpha as the leaf (U = -cumsum(alpha))."""
    B, N, H, d, w = 2, 23, 2, 8, 6
    Q, K, V = _qkv(B, N, H, d, 100)
    dO = _rand((B, N, H, d), 101)
    alpha = 0.05 + np.abs(_rand((B, H, N), 102))
    U, _ = oracle.gate_prefix(alpha)
    g = oracle.bwd(Q, K, V, U, dO, w)
    tq, tk, tv, ta = (torch.from_numpy(x.copy()).requires_grad_(True) for x in (Q, K, V, alpha))
    tu = -torch.cumsum(ta, -1)
    bias = tu[..., :, None] - tu[..., None, :]
    win = torch.from_numpy(_window_mask(N, w))
    mask = torch.where(win, bias, torch.tensor(-float("inf"), dtype=torch.float64))
    o = torch.nn.functional.scaled_dot_product_attention(
        tq.transpose(1, 2), tk.transpose(1, 2), tv.transpose(1, 2), attn_mask=mask
    ).transpose(1, 2)
    (o * torch.from_numpy(dO)).sum().backward()
    assert _rel(g["dQ"], tq.grad.numpy()) < 1e-12
    assert _rel(g["dK"], tk.grad.numpy()) < 1e-12
    assert _rel(g["dV"], tv.grad.numpy()) < 1e-12
    assert _rel(g["dalpha"], ta.grad.numpy()) < 1e-12


def test_bwd_invariants_and_special_cases():
    """Appendix A.1 of SURVEY: rowsum(dS)=0 => sum_m dU_m = 0 and dalpha_0 = 0;
    S:213-214: dO=0 => zero grads; N=1 => dV=dO, others 0; constant dU=c
    => dalpha_q = -c (N-q)."""
    B, N, H, d, w = 1, 31, 2, 8, 5
    Q, K, V = _qkv(B, N, H, d, 110)
    dO = _rand((B, N, H, d), 111)
    U = -np.cumsum(0.2 + np.abs(_rand((B, H, N), 112)), -1)
    g = oracle.bwd(Q, K, V, U, dO, w)
    assert np.allclose(g["dU"].sum(-1), 0.0, atol=1e-12)
    assert np.allclose(g["dalpha"][..., 0], 0.0, atol=1e-12)
    z = oracle.bwd(Q, K, V, U, np.zeros_like(dO), w)
    assert all(np.abs(z[k]).max() == 0.0 for k in ("dQ", "dK", "dV", "dU", "dalpha"))
    g1 = oracle.bwd(Q[:, :1], K[:, :1], V[:, :1], U[..., :1], dO[:, :1], w)
    assert np.allclose(g1["dV"], dO[:, :1], atol=1e-15)
    assert np.abs(g1["dQ"]).max() < 1e-15 and np.abs(g1["dK"]).max() < 1e-15 and np.abs(g1["dU"]).max() < 1e-15
    c = 0.37
    da = oracle.dalpha_scan(np.full((1, 1, 10), c))
    assert np.allclose(da[0, 0], -c * (10 - np.arange(10)), rtol=1e-14)
    da2 = oracle.dalpha_scan(np.full((1, 1, 10), c), carry=np.array([[2.0]]))
    assert np.allclose(da2[0, 0], 2.0 - c * (10 - np.arange(10)), rtol=1e-14)


def test_bwd_halo_shard_sums_to_full():
    """north_star sequence sharding, backward: rank r's dK/dV/dU over [halo; local]
    plus rank r+1's halo part equals the full run; the dalpha carry equals
    +sum(dU_halo of r+1)."""
    B, N, H, d, w = 1, 36, 1, 4, 6
    Q, K, V = _qkv(B, N, H, d, 120)
    dO = _rand((B, N, H, d), 121)
    U = -np.cumsum(0.1 + np.abs(_rand((B, H, N), 122)), -1)
    full = oracle.bwd(Q, K, V, U, dO, w)
    S = 18  # two shards of 18 rows; shard 1 has a w-row halo
    g0 = oracle.bwd(Q[:, :S], K[:, :S], V[:, :S], U[..., :S], dO[:, :S], w, want_dalpha=False)
    g1 = oracle.bwd(Q[:, S:], K[:, S - w :], V[:, S - w :], U[..., S - w :], dO[:, S:], w, want_dalpha=False)
    dK0 = g0["dK"].copy()
    dK0[:, S - w :] += g1["dK"][:, :w]
    dU0 = g0["dU"].copy()
    dU0[..., S - w :] += g1["dU"][..., :w]
    assert np.allclose(dK0, full["dK"][:, :S], atol=1e-13)
    assert np.allclose(g1["dK"][:, w:], full["dK"][:, S:], atol=1e-13)
    assert np.allclose(dU0, full["dU"][..., :S], atol=1e-13)
    carry = g1["dU"][..., :w].sum(-1)
    da0 = oracle.dalpha_scan(dU0, carry=carry)
    assert np.allclose(da0, full["dalpha"][..., :S], atol=1e-12)
    da1 = oracle.dalpha_scan(g1["dU"][..., w:])
    assert np.allclose(da1, full["dalpha"][..., S:], atol=1e-12)


def test_gate_chain_finite_differences():
    """Chain rule of Eq. 9: dh, dbeta vs central FD of sum(alpha*dalpha)."""
    B, N, H = 1, 6, 2
    h = _rand((B, N, H), 130, 2.0)
    beta = 1.0 + torch.nn.functional.elu(torch.from_numpy(_rand((B, N, H), 131, 0.5))).numpy()
    da = _rand((B, H, N), 132)
    dh, db = oracle.gate_chain(h, beta, da, EPS)
    f_h = lambda x: float(np.sum(oracle.gate_alpha(x, beta, EPS) * da))  # noqa: E731
    f_b = lambda x: float(np.sum(oracle.gate_alpha(h, x, EPS) * da))  # noqa: E731
    for idx in [(0, t, hh) for t in range(N) for hh in range(H)]:
        assert _fd(f_h, h, idx) == pytest.approx(dh[idx], rel=1e-6, abs=1e-9)
        assert _fd(f_b, beta, idx) == pytest.approx(db[idx], rel=1e-6, abs=1e-9)


# --- AttnLayer epilogue (reading C-27): RMSNorm per head, swish gate ---


def test_normgate_closed_forms():
    """Constant rows: O_c = a for all c gives n_c = gamma_c a / sqrt(a^2 + eps); g = 0
    gives Y = 0 (swish(0) = 0) and dg = dY n / 2 (sigmoid(0) = 1/2); with eps = 0
    and gamma = 1 every row of n has mean square exactly 1."""
    B, N, H, d = 1, 3, 2, 8
    a = np.array([0.5, -2.0, 3.0]).reshape(1, N, 1, 1) * np.ones((B, N, H, d))
    gamma = 1.0 + 0.1 * np.arange(d)
    g = np.full((B, N, H, d), 40.0)  # swish(40) = 40 (sigmoid(40) = 1 - 4e-18)
    Y, rstd = oracle.normgate_fwd(a, g, gamma, eps=1e-5)
    expect = 40.0 * gamma * a / np.sqrt(a ** 2 + 1e-5)
    assert np.allclose(Y, expect, rtol=1e-14)
    assert np.allclose(rstd, 1.0 / np.sqrt(a[:, :, :, 0].transpose(0, 2, 1) ** 2 + 1e-5), rtol=1e-14)
    O = _rand((B, N, H, d), 140)
    dY = _rand((B, N, H, d), 141)
    Y0, _ = oracle.normgate_fwd(O, np.zeros_like(O), gamma, eps=1e-5)
    assert np.all(Y0 == 0.0)
    _, dg0, _ = oracle.normgate_bwd(O, np.zeros_like(O), gamma, dY, eps=1e-5)
    n = gamma * O / np.sqrt(np.mean(O ** 2, -1, keepdims=True) + 1e-5)
    assert np.allclose(dg0, 0.5 * dY * n, rtol=1e-13, atol=1e-15)
    Yn, _ = oracle.normgate_fwd(O, np.full_like(O, 40.0), np.ones(d), eps=0.0)
    assert np.allclose(np.mean((Yn / 40.0) ** 2, -1), 1.0, rtol=1e-13)


def test_normgate_bwd_finite_differences():
    """dO, dg, dgamma of the epilogue vs central FD of sum(Y * dY)."""
    B, N, H, d = 1, 2, 2, 5
    O = _rand((B, N, H, d), 142)
    g = _rand((B, N, H, d), 143, 2.0)
    gamma = 1.0 + _rand((d,), 144, 0.3)
    dY = _rand((B, N, H, d), 145)
    dO, dg, dgamma = oracle.normgate_bwd(O, g, gamma, dY, eps=1e-3)
    loss = lambda o, gg, ga: float(np.sum(oracle.normgate_fwd(o, gg, ga, eps=1e-3)[0] * dY))  # noqa: E731
    for idx in [(0, t, hh, c) for t in range(N) for hh in range(H) for c in range(d)]:
        assert _fd(lambda x: loss(x, g, gamma), O, idx) == pytest.approx(dO[idx], rel=1e-6, abs=1e-9)
        assert _fd(lambda x: loss(O, x, gamma), g, idx) == pytest.approx(dg[idx], rel=1e-6, abs=1e-9)
    for c in range(d):
        assert _fd(lambda x: loss(O, g, x), gamma, (c,)) == pytest.approx(dgamma[c], rel=1e-6, abs=1e-9)


def test_normgate_matches_torch_autograd():
    """The same epilogue through torch's fp64 ops and autograd (a library routine,
    independent of the oracle's loops): RMSNorm * weight, times g * sigmoid(g)."""
    B, N, H, d = 2, 3, 2, 16
    O = torch.from_numpy(_rand((B, N, H, d), 146)).requires_grad_(True)
    g = torch.from_numpy(_rand((B, N, H, d), 147, 2.0)).requires_grad_(True)
    gamma = torch.from_numpy(1.0 + _rand((d,), 148, 0.3)).requires_grad_(True)
    dY = torch.from_numpy(_rand((B, N, H, d), 149))
    Yt = torch.nn.functional.rms_norm(O, (d,), weight=gamma, eps=1e-5) * torch.nn.functional.silu(g)
    Yt.backward(dY)
    Y, rstd = oracle.normgate_fwd(O.detach(), g.detach(), gamma.detach(), eps=1e-5)
    dO, dg, dgamma = oracle.normgate_bwd(O.detach(), g.detach(), gamma.detach(), dY, eps=1e-5)
    assert np.allclose(Y, Yt.detach().numpy(), rtol=1e-12, atol=1e-14)
    assert np.allclose(dO, O.grad.numpy(), rtol=1e-11, atol=1e-13)
    assert np.allclose(dg, g.grad.numpy(), rtol=1e-11, atol=1e-13)
    assert np.allclose(dgamma, gamma.grad.numpy(), rtol=1e-11, atol=1e-13)


# --- NSA extension (App. B; readings C-28 block-mean compression, C-29 selection) ---


def _sdpa_causal(Q, K, V):
    """fp64 torch SDPA, causal (a library routine independent of the oracle's loops)."""
    q, k, v = (torch.from_numpy(np.ascontiguousarray(x)).permute(0, 2, 1, 3) for x in (Q, K, V))
    return torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True).permute(0, 2, 1, 3).numpy()


def test_nsa_compress_is_block_mean():
    K, V = _rand((2, 40, 3, 8), 160), _rand((2, 40, 3, 8), 161)
    Kc, Vc = oracle.nsa_compress(K, V, 8)
    assert Kc.shape == (2, 5, 3, 8)
    assert np.allclose(Kc, K.reshape(2, 5, 8, 3, 8).mean(2), atol=1e-15)
    assert np.allclose(Vc, V.reshape(2, 5, 8, 3, 8).mean(2), atol=1e-15)


def test_nsa_branches_reduce_to_causal_attention():
    """blk = 1: every token is its own compressed block, so compressed attention is full
    causal attention (but for the first row, whose own block is its only one, and
    complete); with n_sel >= N the selection keeps every earlier block as well, so
    selected attention is full causal attention too (torch SDPA, fp64)."""
    B, N, H, d = 1, 12, 2, 8
    Q, K, V = _rand((B, N, H, d), 162), _rand((B, N, H, d), 163), _rand((B, N, H, d), 164)
    ref = _sdpa_causal(Q, K, V)
    Kc, Vc = oracle.nsa_compress(K, V, 1)
    Ocmp, sc = oracle.nsa_cmp(Q, Kc, Vc, 1)
    assert np.allclose(Ocmp, ref, atol=1e-12)
    sel = oracle.nsa_select(sc, N, 1, N)
    Oslc = oracle.nsa_slc(Q, K, V, sel, 1)
    assert np.allclose(Oslc, ref, atol=1e-12)


def test_nsa_select_and_slc_by_hand():
    """Selection = own block + the top n_sel complete blocks by compressed score (ties to
    the lower index, C-29), checked against a direct argsort; o_slc of a selection that
    is only the own block is causal attention inside that block."""
    B, N, H, d, blk, nsel = 1, 64, 1, 4, 8, 2
    rng = np.random.default_rng(165)
    sc = rng.standard_normal((B, H, N, N // blk))
    for t in range(N):  # blocks ending after t are not complete
        sc[0, 0, t, (t + 1) // blk:] = -np.inf
    sel = oracle.nsa_select(sc, N, blk, nsel)
    for t in range(N):
        own = t // blk
        cand = [i for i in range((t + 1) // blk) if i != own]
        top = sorted(cand, key=lambda i: (-sc[0, 0, t, i], i))[:nsel]
        assert list(sel[0, 0, t]) == [own] + top + [-1] * (nsel - len(top))
    Q, K, V = _rand((B, N, H, d), 166), _rand((B, N, H, d), 167), _rand((B, N, H, d), 168)
    only_own = np.full((B, H, N, nsel + 1), -1, dtype=np.int64)
    only_own[..., 0] = np.arange(N)[None, None, :] // blk
    O = oracle.nsa_slc(Q, K, V, only_own, blk)
    for i0 in range(0, N, blk):
        blkref = _sdpa_causal(Q[:, i0:i0 + blk], K[:, i0:i0 + blk], V[:, i0:i0 + blk])
        assert np.allclose(O[:, i0:i0 + blk], blkref, atol=1e-12)


def test_nsa_combine_gates():
    """sigmoid gates: g -> -inf removes a branch, g = 0 weighs it 1/2."""
    shape = (1, 5, 2, 4)
    a, s, l = _rand(shape, 169), _rand(shape, 170), _rand(shape, 171)
    g = np.zeros(shape[:3] + (3,))
    g[..., 0], g[..., 1], g[..., 2] = -800.0, 0.0, 800.0
    assert np.allclose(oracle.nsa_combine(a, s, l, g), 0.5 * s + l, atol=1e-14)


def test_nsa_bwd_finite_differences():
    """NSA chain rule for a fixed selection vs central FD of sum(O * W): dQ, dK, dV, dU
    (through the local branch's gate), dgates."""
    B, N, H, d, w, blk, nsel = 1, 12, 1, 4, 5, 3, 2
    Q, K, V = _rand((B, N, H, d), 180), _rand((B, N, H, d), 181), _rand((B, N, H, d), 182)
    U = -np.cumsum(0.2 + np.abs(_rand((B, H, N), 183)), -1)
    g = _rand((B, N, H, 3), 184)
    W = _rand((B, N, H, d), 185)
    Kc, Vc = oracle.nsa_compress(K, V, blk)
    _, sc = oracle.nsa_cmp(Q, Kc, Vc, blk)
    sel = oracle.nsa_select(sc, N, blk, nsel)
    dQ, dK, dV, dU, dg = oracle.nsa_bwd(Q, K, V, U, g, W, sel, w, blk)
    loss = lambda q, k, v, u, gg: float(np.sum(oracle.nsa_fwd_fixed(q, k, v, u, gg, sel, w, blk) * W))  # noqa: E731
    for idx in [(0, t, 0, c) for t in range(N) for c in range(d)]:
        assert _fd(lambda x: loss(x, K, V, U, g), Q, idx) == pytest.approx(dQ[idx], rel=1e-6, abs=1e-8)
        assert _fd(lambda x: loss(Q, x, V, U, g), K, idx) == pytest.approx(dK[idx], rel=1e-6, abs=1e-8)
        assert _fd(lambda x: loss(Q, K, x, U, g), V, idx) == pytest.approx(dV[idx], rel=1e-6, abs=1e-8)
    for idx in [(0, 0, t) for t in range(N)]:
        assert _fd(lambda x: loss(Q, K, V, x, g), U, idx) == pytest.approx(dU[idx], rel=1e-6, abs=1e-8)
    for idx in [(0, t, 0, c) for t in range(N) for c in range(3)]:
        assert _fd(lambda x: loss(Q, K, V, U, x), g, idx) == pytest.approx(dg[idx], rel=1e-6, abs=1e-8)
