"""GPU parity of grouped-query attention (GQA) on the tensor-core forward and
backward (gfwa_attn_desc_t.H_kv; the NSA configuration shares
one K/V head among a group of query heads).

The definition checked: query head hh attends with K/V head hh // G
(G = H / H_kv) and its own gate U[b, hh]; the fp64 oracle runs the same
problem as multi-head attention on K/V repeated G times per head, and the
gradient of a shared K/V head is the sum of its G query heads' gradients.
Tolerances: O, LSE, dQ, dU, dalpha as the MHA bf16 test (north_star);
dK, dV sum G per-head gradients, each within TOL_BF16_GRAD, so G x that bound
(triangle inequality; the kernel accumulates the sum in fp32 TMEM and rounds
once)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2512_07782_b200 import binding as gb
from parity import TOL_BF16_GRAD, TOL_BF16_O, TOL_LSE, max_abs

pytestmark = pytest.mark.gpu


def _U(B, H, Nkv, seed):
    g = torch.Generator().manual_seed(seed)
    alpha = torch.nn.functional.softplus(torch.randn(B, H, Nkv, generator=g))
    return (-torch.cumsum(alpha.double(), -1)).float()


def _inputs(s: synth.AttnShape, Hkv: int, seed: int):
    Q, K, V, dO = synth.attn_inputs(s, seed=seed, dtype=torch.bfloat16)
    K, V = K[:, :, :Hkv].contiguous(), V[:, :, :Hkv].contiguous()
    return Q, K, V, dO, _U(s.B, s.H, s.nkv, seed + 1)


CASES = [  # (shape, H_kv)
    (synth.AttnShape(B=1, H=4, N=300, d=128, w=96), 1),
    (synth.AttnShape(B=2, H=4, N=1000, d=128, w=512), 2),
    (synth.AttnShape(B=1, H=8, N=640, d=64, w=200), 2),
    (synth.AttnShape(B=1, H=6, N=512, d=128, w=256, N_kv=768), 3),  # halo rows
    (synth.AttnShape(B=1, H=4, N=37, d=128, w=33), 1),              # sub-tile N
    (synth.AttnShape(B=2, H=4, N=200, d=64, w=1), 2),               # w = 1: O = V
    (synth.AttnShape(B=1, H=16, N=260, d=128, w=2048), 1),          # G = 16, w > N
]


@pytest.mark.parametrize("s,Hkv", CASES, ids=lambda c: str(c) if isinstance(c, int) else
                         f"B{c.B}H{c.H}N{c.N}kv{c.nkv}d{c.d}w{c.w}")
def test_gqa_matches_oracle(s, Hkv):
    G = s.H // Hkv
    Q, K, V, dO, U = _inputs(s, Hkv, seed=5 * s.N + s.w + Hkv)
    Qd, Kd, Vd, dOd, Ud = (x.cuda() for x in (Q, K, V, dO, U))
    assert gb.gfwa_attn_path(Qd, Kd, Vd, s.w) == 1
    O, LSE, Olo = gb.gfwa_fwd(Qd, Kd, Vd, Ud, s.w, want_o_lo=True)
    dQ, dK, dV, dU, da = gb.gfwa_bwd(Qd, Kd, Vd, Ud, O, LSE, dOd, s.w, O_lo=Olo)
    torch.cuda.synchronize()
    assert dK.shape == K.shape and dV.shape == V.shape and dU.shape == (s.B, s.H, s.nkv)
    Ke, Ve = K.repeat_interleave(G, dim=2), V.repeat_interleave(G, dim=2)  # head hh -> K/V head hh // G
    Or, Lr = oracle.fwd(Q, Ke, Ve, U, s.w)
    g = oracle.bwd(Q, Ke, Ve, U, dO, s.w)
    assert max_abs(O, Or) <= TOL_BF16_O
    assert max_abs(LSE, Lr) <= TOL_LSE
    for k in ("dQ", "dU", "dalpha"):
        assert max_abs({"dQ": dQ, "dU": dU, "dalpha": da}[k], g[k]) <= TOL_BF16_GRAD, k
    B, Nkv, _, d = K.shape
    for k, got in (("dK", dK), ("dV", dV)):
        ref = np.asarray(g[k]).reshape(B, Nkv, Hkv, G, d).sum(3)
        assert max_abs(got, ref) <= G * TOL_BF16_GRAD, k


def test_gqa_forward_equals_mha_on_repeated_kv():
    """The forward reads K/V head hh // G in place: bit-identical to the MHA call on
    K/V repeated per group (same kernel, same tiles, same arithmetic)."""
    s, Hkv = synth.AttnShape(B=2, H=8, N=700, d=128, w=300), 2
    Q, K, V, _, U = _inputs(s, Hkv, seed=11)
    Qd, Kd, Vd, Ud = (x.cuda() for x in (Q, K, V, U))
    O1, L1, _ = gb.gfwa_fwd(Qd, Kd, Vd, Ud, s.w, want_o_lo=True)
    O2, L2, _ = gb.gfwa_fwd(Qd, Kd.repeat_interleave(4, 2), Vd.repeat_interleave(4, 2), Ud, s.w, want_o_lo=True)
    torch.cuda.synchronize()
    assert torch.equal(O1, O2) and torch.equal(L1, L2)


def test_gqa_rejects_bad_groups_and_fp32():
    Q = torch.zeros(1, 64, 6, 128, dtype=torch.bfloat16, device="cuda")
    K = torch.zeros(1, 64, 4, 128, dtype=torch.bfloat16, device="cuda")  # 6 % 4 != 0
    U = torch.zeros(1, 6, 64, device="cuda")
    with pytest.raises(RuntimeError, match="INVALID_ARGUMENT"):
        gb.gfwa_fwd(Q, K, K, U, 16)
    Qf, Kf = Q.float(), K[:, :, :2].float()  # fp32 GQA: the SIMT path has none
    with pytest.raises(RuntimeError, match="UNSUPPORTED"):
        gb.gfwa_fwd(Qf, Kf, Kf, U, 16)
