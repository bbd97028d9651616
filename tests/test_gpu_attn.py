"""GPU parity of gfwa_fwd / gfwa_bwd (Alg. 2, Alg. E.2) against the fp64 oracle,
called through the C ABI on the same seeded inputs.

fp32 path: max relative error per (b,h) slice <= 1e-4 on O, <= 1e-3 on
gradients; bf16 path: max abs error <= 2e-2 on O, <= 5e-2 on gradients
(north_star).  Shapes span several tiles with ragged tails and the method's
degenerate cases (N=1, w=1, w>=N, halo rows N_kv > N_q, d=64/128)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2512_07782_b200 import binding as gb
from parity import (TOL_BF16_GRAD, TOL_BF16_O, TOL_F32_GRAD, TOL_F32_O, TOL_LSE, max_abs, np64,
                    rel_slices)

pytestmark = pytest.mark.gpu


def _U(B, H, Nkv, seed, mean=0.5):
    g = torch.Generator().manual_seed(seed)
    alpha = torch.nn.functional.softplus(torch.randn(B, H, Nkv, generator=g) + mean - 0.5)
    return (-torch.cumsum(alpha.double(), -1)).float()


def _run(s: synth.AttnShape, dtype, seed, U=None):
    Q, K, V, dO = synth.attn_inputs(s, seed=seed, dtype=dtype)
    U = _U(s.B, s.H, s.nkv, seed + 1) if U is None else U
    Qd, Kd, Vd, dOd, Ud = (x.cuda() for x in (Q, K, V, dO, U))
    O, LSE, Olo = gb.gfwa_fwd(Qd, Kd, Vd, Ud, s.w, want_o_lo=True)
    dQ, dK, dV, dU, da = gb.gfwa_bwd(Qd, Kd, Vd, Ud, O, LSE, dOd, s.w, O_lo=Olo)
    torch.cuda.synchronize()
    Or, Lr = oracle.fwd(Q, K, V, U, s.w)
    g = oracle.bwd(Q, K, V, U, dO, s.w)
    return dict(O=O, LSE=LSE, Olo=Olo, dQ=dQ, dK=dK, dV=dV, dU=dU, dalpha=da), dict(O=Or, LSE=Lr, **g)


F32_SHAPES = [
    synth.AttnShape(B=1, H=2, N=128, d=64, w=32),        # C1 (BASELINE configs[0])
    synth.AttnShape(B=1, H=1, N=1, d=64, w=1),           # N = 1
    synth.AttnShape(B=2, H=1, N=65, d=128, w=1),         # w = 1 -> O = V
    synth.AttnShape(B=1, H=3, N=200, d=64, w=37),        # ragged tiles, odd w
    synth.AttnShape(B=1, H=2, N=130, d=128, w=500),      # w >= N: full causal
    synth.AttnShape(B=1, H=2, N=257, d=128, w=64),       # w aligned to the tile
    synth.AttnShape(B=1, H=2, N=150, d=64, w=40, N_kv=190),  # halo rows (sequence shard)
]


@pytest.mark.parametrize("s", F32_SHAPES, ids=lambda s: f"B{s.B}H{s.H}N{s.N}kv{s.nkv}d{s.d}w{s.w}")
def test_fp32_path_matches_oracle(s):
    got, ref = _run(s, torch.float32, seed=s.N + s.w)
    assert rel_slices(got["O"], ref["O"], "bnhd") <= TOL_F32_O
    assert max_abs(got["LSE"], ref["LSE"]) <= 1e-4
    for k, lay in (("dQ", "bnhd"), ("dK", "bnhd"), ("dV", "bnhd"), ("dU", "bhn"), ("dalpha", "bhn")):
        if np.abs(ref[k]).max() == 0.0:
            # degenerate cases (w = 1, N = 1): the exact gradient is identically 0
            # (dS = P (dP - D) with P = 1, dP = D); only fp32 round-off of dP - D remains
            assert max_abs(got[k], ref[k]) <= 1e-4, k
        else:
            assert rel_slices(got[k], ref[k], lay) <= TOL_F32_GRAD, k


BF16_SHAPES = [
    synth.AttnShape(B=1, H=2, N=300, d=128, w=96),
    synth.AttnShape(B=2, H=2, N=1000, d=128, w=512),     # C2 window, ragged N
    synth.AttnShape(B=1, H=2, N=777, d=128, w=128),
    synth.AttnShape(B=1, H=2, N=640, d=64, w=200),
    synth.AttnShape(B=1, H=2, N=384, d=128, w=2048),     # w > N
    synth.AttnShape(B=1, H=2, N=512, d=128, w=256, N_kv=768),  # halo
    # the method's degenerate cases on the tensor-core path
    synth.AttnShape(B=1, H=2, N=1, d=128, w=1),           # N = 1: O = v_0, gradients 0 but dV
    synth.AttnShape(B=2, H=2, N=200, d=128, w=1),         # w = 1: O = V
    synth.AttnShape(B=1, H=3, N=37, d=128, w=33),         # sub-tile N, odd w
    synth.AttnShape(B=1, H=2, N=300, d=128, w=250, N_kv=500),  # halo of 200 rows (not tile-aligned)
    synth.AttnShape(B=1, H=2, N=390, d=128, w=1000),      # w >= N with a ragged tail
    synth.AttnShape(B=1, H=2, N=129, d=128, w=129, N_kv=129 + 70),  # ragged halo, w = N
    # head dim 64 (the paper's models: n_heads/d_head 12/64, 16/64) on tcgen05
    synth.AttnShape(B=2, H=2, N=700, d=64, w=300),
    synth.AttnShape(B=1, H=3, N=37, d=64, w=33),
    synth.AttnShape(B=1, H=2, N=300, d=64, w=250, N_kv=500),
]


@pytest.mark.parametrize("s", BF16_SHAPES, ids=lambda s: f"B{s.B}H{s.H}N{s.N}kv{s.nkv}d{s.d}w{s.w}")
def test_bf16_path_matches_oracle(s):
    Q = torch.empty(s.B, s.N, s.H, s.d, dtype=torch.bfloat16, device="cuda")
    K = torch.empty(s.B, s.nkv, s.H, s.d, dtype=torch.bfloat16, device="cuda")
    if s.d == 128:
        assert gb.gfwa_attn_path(Q, K, K, s.w) == 1, "bf16 d=128 must run on the tcgen05 kernels"
    got, ref = _run(s, torch.bfloat16, seed=3 * s.N + s.w)
    assert max_abs(got["O"], ref["O"]) <= TOL_BF16_O
    assert max_abs(got["LSE"], ref["LSE"]) <= TOL_LSE
    for k in ("dQ", "dK", "dV", "dU", "dalpha"):
        assert max_abs(got[k], ref[k]) <= TOL_BF16_GRAD, k


@pytest.mark.parametrize("d", [128, 64])
def test_bf16_late_max_growth(d):
    """Keys far back in the window that outscore every key of the query's own tile by
    2^11-2^16 (alpha = 0: no decay).  The forward walks key tiles diagonal-first, so
    these keys arrive after a row's reference max is set and force the lazy rescale
    of O and l (Alg. 2 l. "o <- diag(e^{m_old - m_new}) o + p v"; the kernel
    moves its reference only when the row max grows by > 2^8).  dO is scaled by 1/16: the
    spiked keys collect nearly all of the ~600 queries' probability, and dV at those
    rows would otherwise reach ~25, where one bf16 ulp alone exceeds 5e-2."""
    s = synth.AttnShape(B=1, H=2, N=640, d=d, w=640)
    Q, K, V, dO = synth.attn_inputs(s, seed=11, dtype=torch.float32)
    g = torch.Generator().manual_seed(12)
    for h in range(s.H):
        u = Q[0, 0, h] / Q[0, 0, h].norm() * d ** 0.5
        Q[0, :, h] = u + 0.3 * torch.randn(s.N, d, generator=g)
        K[0, 40, h] = u          # column 40: half 0, third 16-key chunk
        K[0, 120, h] = 0.7 * u   # column 120: half 1, last chunk
        K[0, 300, h] = 0.9 * u   # a spike in a middle tile as well
    dO = dO / 16
    Q, K, V, dO = (x.to(torch.bfloat16) for x in (Q, K, V, dO))
    U = torch.zeros(s.B, s.H, s.N)
    Qd, Kd, Vd, dOd, Ud = (x.cuda() for x in (Q, K, V, dO, U))
    O, LSE, Olo = gb.gfwa_fwd(Qd, Kd, Vd, Ud, s.w, want_o_lo=True)
    dQ, dK, dV, dU, da = gb.gfwa_bwd(Qd, Kd, Vd, Ud, O, LSE, dOd, s.w, O_lo=Olo)
    torch.cuda.synchronize()
    Or, Lr = oracle.fwd(Q, K, V, U, s.w)
    ref = oracle.bwd(Q, K, V, U, dO, s.w)
    assert max_abs(O, Or) <= TOL_BF16_O
    assert max_abs(LSE, Lr) <= TOL_LSE
    got = dict(dQ=dQ, dK=dK, dV=dV, dU=dU, dalpha=da)
    for k in got:
        assert max_abs(got[k], ref[k]) <= TOL_BF16_GRAD, k


def test_end_to_end_from_gate_inputs():
    """gate scan -> attention -> backward -> gate chain vs the oracle chain."""
    from paper_2512_07782_b200 import gated_fwa

    s = synth.AttnShape(B=1, H=4, N=333, d=128, w=100)
    Q, K, V, dO = synth.attn_inputs(s, seed=5, dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=6)
    leaves = [x.cuda().requires_grad_(True) for x in (Q, K, V, h, beta)]
    O = gated_fwa(*leaves, w=s.w)
    O.backward(dO.cuda())
    U, _, _ = oracle.gate_prefix_hbeta(h, beta)
    Or, _ = oracle.fwd(Q, K, V, U, s.w)
    g = oracle.bwd(Q, K, V, U, dO, s.w)
    dh, db = oracle.gate_chain(h, beta, g["dalpha"])
    assert max_abs(O, Or) <= TOL_BF16_O
    assert max_abs(leaves[0].grad, g["dQ"]) <= TOL_BF16_GRAD
    assert max_abs(leaves[1].grad, g["dK"]) <= TOL_BF16_GRAD
    assert max_abs(leaves[2].grad, g["dV"]) <= TOL_BF16_GRAD
    # dh, dbeta = dalpha * (d alpha / d h), dalpha * (d alpha / d beta): the exact fp32
    # chain multiplies dalpha's error by at most max|d alpha / d .|
    hh, bb = h.double().numpy(), beta.double().numpy()
    sg = 1.0 / (1.0 + np.exp(-bb * hh))
    sp = np.logaddexp(0.0, bb * hh)
    lip_h = np.abs(sg * bb / (bb + 1e-6)).max()
    lip_b = np.abs((sg * hh * (bb + 1e-6) - sp) / (bb + 1e-6) ** 2).max()
    assert max_abs(leaves[3].grad, dh) <= TOL_BF16_GRAD * max(1.0, lip_h)
    assert max_abs(leaves[4].grad, db) <= TOL_BF16_GRAD * max(1.0, lip_b)


def test_c2_full_size_sampled():
    """BASELINE configs[1] (C2: B=8, H=16, N=4096, d=128, w=512, bf16) in the
    launch configuration bench.py times; fwd checked on sampled rows across all
    slices, fwd+bwd checked in full on two (b, h) slices."""
    c = synth.CONFIGS["C2"]
    s = synth.AttnShape(B=c["B"], H=c["H"], N=c["N"], d=c["d"], w=c["w"])
    Q, K, V, dO = synth.attn_inputs(s, seed=c["seed"], device="cuda", dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=c["seed"], device="cuda")
    U = gb.gfwa_gate_prefix(h, beta)
    O, LSE, Olo = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True)
    dQ, dK, dV, dU, da = gb.gfwa_bwd(Q, K, V, U, O, LSE, dO, s.w, O_lo=Olo)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    rows = np.stack([rng.integers(0, s.B, 96), rng.integers(0, s.H, 96), rng.integers(0, s.N, 96)], 1)
    rows[:4, 2] = [0, 1, s.w - 1, s.N - 1]
    o_r, l_r = oracle.fwd_rows(Q, K, V, U, s.w, rows)
    o_g = np64(O)[rows[:, 0], rows[:, 2], rows[:, 1]]
    l_g = np64(LSE)[rows[:, 0], rows[:, 1], rows[:, 2]]
    assert np.abs(o_g - o_r).max() <= TOL_BF16_O
    assert np.abs(l_g - l_r).max() <= TOL_LSE
    for b, hh in ((0, 0), (s.B - 1, s.H - 1)):
        sl = lambda x: x[b:b + 1, :, hh:hh + 1]  # noqa: E731
        Ur = U[b:b + 1, hh:hh + 1]
        g = oracle.bwd(sl(Q), sl(K), sl(V), Ur, sl(dO), s.w)
        Or, _ = oracle.fwd(sl(Q), sl(K), sl(V), Ur, s.w)
        assert max_abs(sl(O), Or) <= TOL_BF16_O
        for k, t in (("dQ", dQ), ("dK", dK), ("dV", dV)):
            assert max_abs(sl(t), g[k]) <= TOL_BF16_GRAD, k
        assert max_abs(dU[b:b + 1, hh:hh + 1], g["dU"]) <= TOL_BF16_GRAD
        assert max_abs(da[b:b + 1, hh:hh + 1], g["dalpha"]) <= TOL_BF16_GRAD


def test_zero_grad_out_and_invariants():
    """dO = 0 -> all gradients exactly 0; sum_m dU_m = 0 and dalpha_0 = 0 (rowsum(dS) = 0)."""
    s = synth.AttnShape(B=1, H=2, N=260, d=128, w=70)
    Q, K, V, dO = synth.attn_inputs(s, seed=11, device="cuda", dtype=torch.float32)
    U = _U(1, 2, s.N, 12).cuda()
    O, LSE, Olo = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True)
    z = gb.gfwa_bwd(Q, K, V, U, O, LSE, torch.zeros_like(dO), s.w, O_lo=Olo)
    for t in z:
        assert torch.count_nonzero(t) == 0
    dQ, dK, dV, dU, da = gb.gfwa_bwd(Q, K, V, U, O, LSE, dO, s.w, O_lo=Olo)
    assert dU.double().sum(-1).abs().max().item() <= 1e-3 * dU.abs().max().item()
    assert da[..., 0].abs().max().item() <= 1e-3 * da.abs().max().item()


def test_bf16_tc_invariants():
    """On the tensor-core backward: dO = 0 -> every gradient exactly 0; sum_m dU_m = 0
    and dalpha_0 = 0 (rowsum(dS) = 0; du^q and du^k are summed from
    the same fp32 dS, reading C-11, so the telescoping holds to fp32 round-off)."""
    s = synth.AttnShape(B=2, H=4, N=1500, d=128, w=300)
    Q, K, V, dO = synth.attn_inputs(s, seed=13, device="cuda", dtype=torch.bfloat16)
    assert gb.gfwa_attn_path(Q, K, V, s.w) == 1
    h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=14, device="cuda")
    U = gb.gfwa_gate_prefix(h, beta)
    O, LSE, Olo = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True)
    z = gb.gfwa_bwd(Q, K, V, U, O, LSE, torch.zeros_like(dO), s.w, O_lo=Olo)
    for t in z:
        assert torch.count_nonzero(t) == 0
    dQ, dK, dV, dU, da = gb.gfwa_bwd(Q, K, V, U, O, LSE, dO, s.w, O_lo=Olo)
    # fp32 round-off of sums of ~N w terms of size |dS| <= max|dU|
    bound = 1e-4 * dU.abs().max().item()
    assert dU.double().sum(-1).abs().max().item() <= bound
    assert da[..., 0].abs().max().item() <= bound
    # dalpha is the exact reverse scan of dU
    scan = -torch.flip(torch.cumsum(torch.flip(dU.double(), [-1]), -1), [-1])
    assert (da.double() - scan).abs().max().item() <= 1e-5 * max(1.0, scan.abs().max().item())


def _sampled_full_size(s: synth.AttnShape, seed: int, n_rows: int, bwd_slices, halo: int = 0):
    """Forward on sampled rows across all slices, fwd+bwd in full on the given
    (b, h) slices, at a BASELINE shape in the launch configuration bench.py times."""
    Q, K, V, dO = synth.attn_inputs(s, seed=seed, device="cuda", dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, s.nkv, s.H, seed=seed, device="cuda")
    U = gb.gfwa_gate_prefix(h, beta)
    O, LSE, Olo = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True)
    dQ, dK, dV, dU, da = gb.gfwa_bwd(Q, K, V, U, O, LSE, dO, s.w, O_lo=Olo)
    torch.cuda.synchronize()
    rng = np.random.default_rng(seed)
    rows = np.stack([rng.integers(0, s.B, n_rows), rng.integers(0, s.H, n_rows), rng.integers(0, s.N, n_rows)], 1)
    rows[:4, 2] = [0, 1, min(s.w, s.N) - 1, s.N - 1]
    o_r, l_r = oracle.fwd_rows(Q, K, V, U, s.w, rows)
    o_g = np64(O)[rows[:, 0], rows[:, 2], rows[:, 1]]
    l_g = np64(LSE)[rows[:, 0], rows[:, 1], rows[:, 2]]
    assert np.abs(o_g - o_r).max() <= TOL_BF16_O
    assert np.abs(l_g - l_r).max() <= TOL_LSE
    for b, hh in bwd_slices:
        sl = lambda x: x[b:b + 1, :, hh:hh + 1]  # noqa: E731
        Ur = U[b:b + 1, hh:hh + 1]
        g = oracle.bwd(sl(Q), sl(K), sl(V), Ur, sl(dO), s.w)
        for k, t in (("dQ", dQ), ("dK", dK), ("dV", dV)):
            assert max_abs(sl(t), g[k]) <= TOL_BF16_GRAD, k
        assert max_abs(dU[b:b + 1, hh:hh + 1], g["dU"]) <= TOL_BF16_GRAD
        e_da = max_abs(da[b:b + 1, hh:hh + 1], g["dalpha"])
        print(f"dalpha max abs error b{b} h{hh}: {e_da:.4f}")
        assert e_da <= TOL_BF16_GRAD


@pytest.mark.parametrize("wl", ["C3_w128", "C3_w512", "C3_w2048"])
def test_c3_window_sweep_full_size_sampled(wl):
    """BASELINE configs[2] (H=32, N=8192, d=128, w in {128, 512, 2048}, bf16)."""
    c = synth.CONFIGS[wl]
    s = synth.AttnShape(B=c["B"], H=c["H"], N=c["N"], d=c["d"], w=c["w"])
    slices = [(0, 0), (0, c["H"] - 1)] if c["w"] <= 512 else [(0, c["H"] - 1)]  # oracle bwd is O(N w d)
    _sampled_full_size(s, c["seed"], 64, slices)


def test_c4_rank_shard_full_size_sampled():
    """BASELINE configs[3] at P=8: one rank's launch (S = 16384 query rows after a
    w = 2048 halo, N_kv = S + w, H = 32) -- the call the sequence-sharded step makes."""
    c = synth.CONFIGS["C4"]
    S = c["N"] // 8
    s = synth.AttnShape(B=c["B"], H=c["H"], N=S, d=c["d"], w=c["w"], N_kv=S + c["w"])
    _sampled_full_size(s, c["seed"], 64, [(0, 5)])


def test_fwd_train_prepares_the_backward_workspace():
    """gfwa_fwd_train zeroes the backward's dQ accumulator in the forward's
    epilogue and marks the workspace; the backward consumes the mark.  The
    gradients must equal the plain path's, also for a second backward on the
    same (now dirty, unmarked) workspace without a new preparation."""
    s = synth.AttnShape(B=2, H=3, N=700, d=128, w=200)
    Q, K, V, dO = synth.attn_inputs(s, seed=31, device="cuda", dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=32, device="cuda")
    U = gb.gfwa_gate_prefix(h, beta)
    O, LSE, Olo = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True)
    ref = gb.gfwa_bwd(Q, K, V, U, O, LSE, dO, s.w, O_lo=Olo)
    O2, LSE2, Olo2 = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True, prepare_bwd=True)
    assert torch.equal(O, O2) and torch.equal(LSE, LSE2) and torch.equal(Olo, Olo2)
    got = gb.gfwa_bwd(Q, K, V, U, O2, LSE2, dO, s.w, O_lo=Olo2)
    again = gb.gfwa_bwd(Q, K, V, U, O2, LSE2, dO, s.w, O_lo=Olo2)  # mark consumed: zeroes itself
    torch.cuda.synchronize()
    for a, b, c in zip(ref[:4], got[:4], again[:4]):
        tol = 1e-2 * max(1.0, a.float().abs().max().item())  # fp32 reduce order only (bf16 outputs)
        assert (a.float() - b.float()).abs().max().item() <= tol
        assert (a.float() - c.float()).abs().max().item() <= tol


def test_fwd_train_interleaved_shapes_share_one_workspace():
    """two prepared forwards of different shapes on the one cached
    workspace, then their backwards in reverse order (as autograd runs them).
    The token names the whole descriptor at a fixed offset: Y's backward finds
    its own token, X's finds it cleared and zeroes its accumulator itself."""
    sx = synth.AttnShape(B=2, H=3, N=900, d=128, w=300)
    sy = synth.AttnShape(B=1, H=2, N=500, d=128, w=128)
    out = {}
    for name, s, seed in (("X", sx, 41), ("Y", sy, 43)):
        Q, K, V, dO = synth.attn_inputs(s, seed=seed, device="cuda", dtype=torch.bfloat16)
        h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=seed + 1, device="cuda")
        U = gb.gfwa_gate_prefix(h, beta)
        ref_o = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True)
        ref = gb.gfwa_bwd(Q, K, V, U, *ref_o[:2], dO, s.w, O_lo=ref_o[2])
        out[name] = (Q, K, V, U, dO, s, [r.clone() for r in ref[:4]])
    prep = {}
    for name in ("X", "Y"):
        Q, K, V, U, dO, s, _ = out[name]
        prep[name] = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True, prepare_bwd=True)
    for name in ("Y", "X"):
        Q, K, V, U, dO, s, ref = out[name]
        O, LSE, Olo = prep[name]
        got = gb.gfwa_bwd(Q, K, V, U, O, LSE, dO, s.w, O_lo=Olo)
        torch.cuda.synchronize()
        for a, b in zip(ref, got[:4]):
            tol = 1e-2 * max(1.0, a.float().abs().max().item())  # fp32 reduce order only
            assert (a.float() - b.float()).abs().max().item() <= tol, name


def test_d64_full_grid_many_items_per_cta():
    """d = 64 at an LM size: the persistent forward walks several items per CTA
    (the O-release / phase bookkeeping per head dim); sampled rows vs the oracle."""
    s = synth.AttnShape(B=4, H=16, N=4096, d=64, w=512)
    Q, K, V, dO = synth.attn_inputs(s, seed=61, device="cuda", dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=62, device="cuda")
    U = gb.gfwa_gate_prefix(h, beta)
    for lo in (False, True):
        O, LSE, _ = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=lo)
        torch.cuda.synchronize()
        rng = np.random.default_rng(63)
        rows = np.stack([rng.integers(0, s.B, 64), rng.integers(0, s.H, 64), rng.integers(0, s.N, 64)], 1)
        o_r, l_r = oracle.fwd_rows(Q, K, V, U, s.w, rows)
        o_g = np64(O)[rows[:, 0], rows[:, 2], rows[:, 1]]
        l_g = np64(LSE)[rows[:, 0], rows[:, 1], rows[:, 2]]
        assert np.abs(o_g - o_r).max() <= TOL_BF16_O
        assert np.abs(l_g - l_r).max() <= TOL_LSE


@pytest.mark.parametrize("d", [64, 128])
def test_persistent_kernels_many_items_per_cta(d, monkeypatch):
    """Forward and backward forced onto 2 / 3 CTAs (GFWA_FWD_GRID / GFWA_BWD_GRID,
    read at every launch), so each CTA walks many work items: the backward's
    rotating shared-memory slot pool (next item's K, V and first Q/dO stage
    loaded during the current item's last steps, dK/dV staged in the item's K
    slot), the dK/dV-accumulator hand-over between items, and items no query
    reaches (a halo longer than w: those keys get dK = dV = 0)."""
    monkeypatch.setenv("GFWA_FWD_GRID", "2")
    monkeypatch.setenv("GFWA_BWD_GRID", "3")
    for s in (synth.AttnShape(B=2, H=3, N=900, d=d, w=200),
              synth.AttnShape(B=1, H=2, N=300, d=d, w=100, N_kv=300 + 450)):
        got, ref = _run(s, torch.bfloat16, seed=7 * s.N + d)
        assert max_abs(got["O"], ref["O"]) <= TOL_BF16_O
        assert max_abs(got["LSE"], ref["LSE"]) <= TOL_LSE
        for k in ("dQ", "dK", "dV", "dU", "dalpha"):
            assert max_abs(got[k], ref[k]) <= TOL_BF16_GRAD, k
        if s.nkv > s.N + s.w:  # keys before the first query's window: exact zeros
            dead = s.nkv - s.N - s.w + 1
            assert torch.count_nonzero(got["dK"][:, :dead]) == 0 and torch.count_nonzero(got["dV"][:, :dead]) == 0


def test_bwd_rows_f32_boundary_copies():
    """gfwa_bwd_rows_f32 (sequence sharding): the fp32 copies of the
    first / last key rows' dK, dV are the values the bf16 outputs were rounded from
    (they round to them exactly) and match the oracle within the bf16 budget."""
    s = synth.AttnShape(B=2, H=2, N=400, d=128, w=150, N_kv=400 + 150)
    Q, K, V, dO = synth.attn_inputs(s, seed=71, dtype=torch.bfloat16)
    U = _U(s.B, s.H, s.nkv, 72)
    Qd, Kd, Vd, dOd, Ud = (x.cuda() for x in (Q, K, V, dO, U))
    O, LSE, Olo = gb.gfwa_fwd(Qd, Kd, Vd, Ud, s.w, want_o_lo=True)
    dQ, dK, dV, dU, head, tail = gb.gfwa_bwd_rows_f32(Qd, Kd, Vd, Ud, O, LSE, dOd, s.w, s.w, s.w, O_lo=Olo)
    dQ2, dK2, dV2, dU2, _ = gb.gfwa_bwd(Qd, Kd, Vd, Ud, O, LSE, dOd, s.w, O_lo=Olo)
    torch.cuda.synchronize()
    assert torch.equal(dK, dK2) and torch.equal(dV, dV2) and torch.equal(dQ, dQ2)
    w = s.w
    for buf, rows in ((head, slice(0, w)), (tail, slice(s.nkv - w, s.nkv))):
        assert torch.equal(buf[0].to(torch.bfloat16), dK[:, rows])
        assert torch.equal(buf[1].to(torch.bfloat16), dV[:, rows])
    g = oracle.bwd(Q, K, V, U, dO, s.w)
    assert max_abs(head[0], g["dK"][:, :w]) <= TOL_BF16_GRAD and max_abs(tail[1], g["dV"][:, -w:]) <= TOL_BF16_GRAD
