"""GPU parity of the fused AttnLayer epilogue (reading C-27: per-head
RMSNorm with a shared weight gamma, swish gate on the pre-activation g) against
the fp64 oracle, through the C ABI (gfwa_fwd_normgate / gfwa_bwd_normgate).

Tolerances follow north_star's bf16 budget propagated through the epilogue: Y =
swish(g) gamma O rstd multiplies O's error (2e-2 abs) by L = max|swish(g) gamma
rstd| and adds Y's own bf16 output rounding (2^-8 relative); the backward is
linear in dY, so the attention-gradient tolerance (5e-2 abs for dO ~ N(0,1))
scales with max|dO~|, the exact gradient fed to Alg. E.2."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2512_07782_b200 import binding as gb
from parity import TOL_BF16_GRAD, TOL_BF16_O, TOL_LSE, max_abs, np64

pytestmark = pytest.mark.gpu
EPS = 1e-5


def _U(B, H, Nkv, seed):
    g = torch.Generator().manual_seed(seed)
    alpha = torch.nn.functional.softplus(torch.randn(B, H, Nkv, generator=g))
    return (-torch.cumsum(alpha.double(), -1)).float()


@pytest.mark.parametrize("s", [synth.AttnShape(B=1, H=2, N=300, d=128, w=96),
                               synth.AttnShape(B=2, H=3, N=700, d=64, w=300),
                               synth.AttnShape(B=1, H=2, N=513, d=128, w=512, N_kv=513 + 200)],
                         ids=lambda s: f"B{s.B}H{s.H}N{s.N}kv{s.nkv}d{s.d}w{s.w}")
def test_normgate_fwd_bwd_matches_oracle(s):
    Q, K, V, dO_unused = synth.attn_inputs(s, seed=s.N + s.d, dtype=torch.bfloat16)
    gen = torch.Generator().manual_seed(s.N)
    g = torch.randn(s.B, s.N, s.H, s.d, generator=gen).to(torch.bfloat16)
    gamma = (1.0 + 0.1 * torch.randn(s.d, generator=gen)).float()
    dY = torch.randn(s.B, s.N, s.H, s.d, generator=gen).to(torch.bfloat16)
    U = _U(s.B, s.H, s.nkv, s.N + 1)
    dev = [x.cuda() for x in (Q, K, V, U, g, gamma, dY)]
    Qd, Kd, Vd, Ud, gd, gmd, dYd = dev
    Y, O, LSE, Olo, rstd = gb.gfwa_fwd_normgate(Qd, Kd, Vd, Ud, gd, gmd, s.w, eps=EPS, prepare_bwd=True)
    dQ, dK, dV, dU, da, dg, dgamma, dOt = gb.gfwa_bwd_normgate(Qd, Kd, Vd, Ud, O, LSE, gd, gmd, rstd, dYd, s.w,
                                                               eps=EPS, O_lo=Olo)
    torch.cuda.synchronize()
    # oracle chain: Eq. 12 -> epilogue (C-27) -> its chain rule -> Alg. E.2 on dO~
    Or, Lr = oracle.fwd(Q, K, V, U, s.w)
    Yr, rr = oracle.normgate_fwd(Or, g, gamma, eps=EPS)
    dOr, dgr, dgamr = oracle.normgate_bwd(Or, g, gamma, dY, eps=EPS)
    gr = oracle.bwd(Q, K, V, U, dOr, s.w)
    gf = np64(g)
    sw = gf / (1.0 + np.exp(-gf))
    L = float(np.max(np.abs(sw * np64(gamma) * rr.transpose(0, 2, 1)[..., None])))
    assert max_abs(O, Or) <= TOL_BF16_O
    assert max_abs(LSE, Lr) <= TOL_LSE
    assert np.max(np.abs(np64(rstd) - rr) / rr) <= 1e-2
    assert max_abs(Y, Yr) <= TOL_BF16_O * max(1.0, L) + 2.0 ** -8 * np.abs(Yr).max()
    scale = max(1.0, float(np.abs(dOr).max()))
    assert max_abs(dOt, dOr) <= TOL_BF16_GRAD * scale
    for k, t in (("dQ", dQ), ("dK", dK), ("dV", dV), ("dU", dU), ("dalpha", da)):
        assert max_abs(t, gr[k]) <= TOL_BF16_GRAD * scale, k
    assert max_abs(dg, dgr) <= TOL_BF16_GRAD * max(1.0, float(np.abs(dgr).max()))
    assert max_abs(dgamma, dgamr) <= 1e-2 * float(np.abs(dgamr).max())


def test_normgate_plain_forward_is_unchanged():
    """The epilogue only adds outputs: O, LSE of gfwa_fwd_normgate equal gfwa_fwd's bit for bit."""
    s = synth.AttnShape(B=1, H=2, N=400, d=128, w=200)
    Q, K, V, _ = synth.attn_inputs(s, seed=9, device="cuda", dtype=torch.bfloat16)
    U = _U(1, 2, s.N, 10).cuda()
    g = torch.randn(1, s.N, 2, s.d, device="cuda").to(torch.bfloat16)
    gamma = torch.ones(s.d, device="cuda")
    Y, O, LSE, Olo, _ = gb.gfwa_fwd_normgate(Q, K, V, U, g, gamma, s.w)
    O2, LSE2, Olo2 = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True)
    assert torch.equal(O, O2) and torch.equal(LSE, LSE2) and torch.equal(Olo, Olo2)


def test_normgate_inference_without_residual():
    """Inference form (no O_lo, no backward workspace): Y from the bf16 O alone stays
    within the same budget at d = 64."""
    s = synth.AttnShape(B=1, H=2, N=333, d=64, w=128)
    Q, K, V, _ = synth.attn_inputs(s, seed=91, dtype=torch.bfloat16)
    gen = torch.Generator().manual_seed(92)
    g = torch.randn(1, s.N, 2, s.d, generator=gen).to(torch.bfloat16)
    gamma = (1.0 + 0.1 * torch.randn(s.d, generator=gen)).float()
    U = _U(1, 2, s.N, 93)
    Y, O, LSE, Olo, rstd = gb.gfwa_fwd_normgate(Q.cuda(), K.cuda(), V.cuda(), U.cuda(), g.cuda(), gamma.cuda(), s.w,
                                               eps=EPS, want_o_lo=False)
    torch.cuda.synchronize()
    assert Olo is None
    Or, _ = oracle.fwd(Q, K, V, U, s.w)
    Yr, rr = oracle.normgate_fwd(Or, g, gamma, eps=EPS)
    gf = np64(g)
    L = float(np.max(np.abs(gf / (1.0 + np.exp(-gf)) * np64(gamma) * rr.transpose(0, 2, 1)[..., None])))
    assert max_abs(Y, Yr) <= TOL_BF16_O * max(1.0, L) + 2.0 ** -7 * np.abs(Yr).max()
