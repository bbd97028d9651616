"""Seeded random shapes on the tensor-core path (bf16, d = 64 / 128) against the
fp64 oracle: batch, heads, ragged N (1 .. 700), any window (1 .. 1200, often
w >= N), halo rows (0 .. 300, often not tile-aligned) and forced small
persistent grids (many work items per CTA).  Tolerances are north_star's bf16
budget (2e-2 abs on O, 5e-2 abs on gradients)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2512_07782_b200 import binding as gb
from parity import TOL_BF16_GRAD, TOL_BF16_O, TOL_LSE, max_abs

pytestmark = pytest.mark.gpu


def _case(k):
    r = np.random.default_rng(9000 + k)
    N = int(r.choice([1, 2, 63, 64, 65, 127, 129, 200, 255, 257, 383, 511, 700]))
    w = int(r.choice([1, 2, 17, 64, 100, 128, 300, 513, 1200]))
    halo = int(r.choice([0, 0, 1, 37, 128, 300]))
    d = int(r.choice([64, 128]))
    B, H = int(r.integers(1, 3)), int(r.integers(1, 4))
    grids = [None, ("2", "3"), ("1", "1")][int(r.integers(0, 3))]
    return synth.AttnShape(B=B, H=H, N=N, d=d, w=w, N_kv=N + halo), grids


@pytest.mark.parametrize("k", range(16))
def test_random_shapes_match_oracle(k, monkeypatch):
    s, grids = _case(k)
    if grids is not None:
        monkeypatch.setenv("GFWA_FWD_GRID", grids[0])
        monkeypatch.setenv("GFWA_BWD_GRID", grids[1])
    Q, K, V, dO = synth.attn_inputs(s, seed=100 + k, dtype=torch.bfloat16)
    g = torch.Generator().manual_seed(200 + k)
    U = (-torch.cumsum(torch.nn.functional.softplus(torch.randn(s.B, s.H, s.nkv, generator=g)).double(), -1)).float()
    Qd, Kd, Vd, dOd, Ud = (x.cuda() for x in (Q, K, V, dO, U))
    assert gb.gfwa_attn_path(Qd, Kd, Vd, s.w) == 1
    O, LSE, Olo = gb.gfwa_fwd(Qd, Kd, Vd, Ud, s.w, want_o_lo=True, prepare_bwd=bool(k % 2))
    dQ, dK, dV, dU, da = gb.gfwa_bwd(Qd, Kd, Vd, Ud, O, LSE, dOd, s.w, O_lo=Olo)
    torch.cuda.synchronize()
    Or, Lr = oracle.fwd(Q, K, V, U, s.w)
    ref = oracle.bwd(Q, K, V, U, dO, s.w)
    assert max_abs(O, Or) <= TOL_BF16_O
    assert max_abs(LSE, Lr) <= TOL_LSE
    for name, t in (("dQ", dQ), ("dK", dK), ("dV", dV), ("dU", dU), ("dalpha", da)):
        assert max_abs(t, ref[name]) <= TOL_BF16_GRAD, name


@pytest.mark.parametrize("k", range(8))
def test_random_shapes_kv_halo_match_oracle(k, monkeypatch):
    """The in-kernel halo (gfwa_attn_desc_t.halo_rows) on random shapes: the first
    halo_rows (a multiple of 128, <= the halo in front of the queries) key rows come
    from a separate buffer, the rest of the halo (if any) from K / V; forced small grids."""
    r = np.random.default_rng(9500 + k)
    N = int(r.choice([1, 65, 200, 257, 511]))
    hr = 128 * int(r.integers(1, 4))
    extra = int(r.choice([0, 0, 37, 128]))  # halo rows beyond the in-kernel part, read from K
    w = int(r.choice([1, 100, 300, 513, 1200]))
    d = int(r.choice([64, 128]))
    B, H = int(r.integers(1, 3)), int(r.integers(1, 4))
    if r.integers(0, 2):
        monkeypatch.setenv("GFWA_FWD_GRID", "2")
        monkeypatch.setenv("GFWA_BWD_GRID", "3")
    s = synth.AttnShape(B=B, H=H, N=N, d=d, w=w, N_kv=N + hr + extra)
    Q, K, V, dO = synth.attn_inputs(s, seed=300 + k, dtype=torch.bfloat16)
    g = torch.Generator().manual_seed(400 + k)
    U = (-torch.cumsum(torch.nn.functional.softplus(torch.randn(s.B, s.H, s.nkv, generator=g)).double(), -1)).float()
    Qd, Kd, Vd, dOd, Ud = (x.cuda() for x in (Q, K, V, dO, U))
    halo = (Kd[:, :hr].clone(), Vd[:, :hr].clone())
    O, LSE, Olo = gb.gfwa_fwd(Qd, Kd[:, hr:], Vd[:, hr:], Ud, s.w, want_o_lo=True, prepare_bwd=bool(k % 2),
                              kv_halo=halo)
    dQ, dK, dV, dU, da = gb.gfwa_bwd(Qd, Kd[:, hr:], Vd[:, hr:], Ud, O, LSE, dOd, s.w, O_lo=Olo, kv_halo=halo)
    torch.cuda.synchronize()
    Or, Lr = oracle.fwd(Q, K, V, U, s.w)
    ref = oracle.bwd(Q, K, V, U, dO, s.w)
    assert max_abs(O, Or) <= TOL_BF16_O
    assert max_abs(LSE, Lr) <= TOL_LSE
    for name, t in (("dQ", dQ), ("dK", dK), ("dV", dV), ("dU", dU), ("dalpha", da)):
        assert max_abs(t, ref[name]) <= TOL_BF16_GRAD, name
