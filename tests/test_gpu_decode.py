"""GPU parity of gfwa_decode (reading C-16: decode(t) == row t of Eq. 12)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2512_07782_b200 import binding as gb
from parity import TOL_BF16_O, TOL_F32_O, np64

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype,d,w,steps", [(torch.float32, 64, 16, 40), (torch.bfloat16, 128, 33, 70),
                                             (torch.float32, 128, 1, 5), (torch.bfloat16, 64, 700, 30)])
def test_decode_sequence_equals_prefill_rows(dtype, d, w, steps):
    """Run `steps` decode steps from an empty ring (wrapping when steps > w) and
    compare every output with the oracle forward row over the whole sequence.
    Gates enter as (h, beta) (GATE_HBETA)."""
    B, H = 2, 3
    s = synth.AttnShape(B=B, H=H, N=steps, d=d, w=w)
    Q, K, V, _ = synth.attn_inputs(s, seed=steps + w, dtype=dtype, with_grad_out=False)
    h, beta = synth.gate_inputs(B, steps, H, seed=w)
    Kc = torch.zeros(B, H, w, d, dtype=dtype, device="cuda")
    Vc = torch.zeros_like(Kc)
    Uc = torch.zeros(B, H, w, dtype=torch.float32, device="cuda")
    outs = []
    for t in range(steps):
        pos = torch.full((B,), t, dtype=torch.int64, device="cuda")
        o = gb.gfwa_decode(Q[:, t].cuda().contiguous(), K[:, t].cuda().contiguous(), V[:, t].cuda().contiguous(),
                           h[:, t].cuda(), Kc, Vc, Uc, pos, gate_b=beta[:, t].cuda())
        outs.append(np64(o))
    got = np.stack(outs, 1)  # [B, steps, H, d]
    U, _, _ = oracle.gate_prefix_hbeta(h, beta)
    ref, _ = oracle.fwd(Q, K, V, U, w)
    if dtype == torch.float32:
        num = np.abs(got - ref).max()
        assert num / np.abs(ref).max() <= TOL_F32_O
    else:
        assert np.abs(got - ref).max() <= TOL_BF16_O
    # the ring now holds the last min(steps, w) tokens at slot t mod w
    t_last = steps - 1
    for t in range(max(0, steps - w), steps):
        assert torch.equal(Kc[:, :, t % w].cpu(), K[:, t].to(dtype).permute(0, 1, 2))
    # U_cache is relative to the newest token: u_tau - u_{t_last} per slot
    for t in range(max(0, steps - w), steps):
        assert np.allclose(np64(Uc[:, :, t % w]), U[:, :, t] - U[:, :, t_last], rtol=1e-5, atol=1e-5)


def test_decode_C5_full_size_sampled():
    """BASELINE configs[4] (C5: B=64, H=32, d=128, w=2048, bf16) with a wrapped,
    pre-filled ring (pos = w + 17); 48 sampled (b, h) rows vs the oracle over
    their token-ordered window."""
    c = synth.CONFIGS["C5"]
    B, H, d, w = c["B"], c["H"], c["d"], c["w"]
    Kc, Vc, a_hist, q, k, v, a_new = synth.decode_inputs(B, H, d, w, seed=c["seed"], device="cuda")
    t = w + 17
    # history tokens t-w .. t-1 live at slot (token mod w); their u from the oracle scan,
    # stored relative to the newest cached token (the U_cache convention)
    U_hist, _ = oracle.gate_prefix(a_hist)            # u of tokens t-w..t-1 (frame: u_{t-w-1} = 0)
    slots = np.arange(t - w, t) % w
    Uc = np.zeros((B, H, w))
    Uc[:, :, slots] = U_hist - U_hist[:, :, -1:]
    Kc_ring = torch.empty_like(Kc)
    Vc_ring = torch.empty_like(Vc)
    Kc_ring[:, :, torch.from_numpy(slots).cuda()] = Kc
    Vc_ring[:, :, torch.from_numpy(slots).cuda()] = Vc
    Uc_t = torch.from_numpy(Uc).float().cuda()
    Uc_used = np64(Uc_t)  # the fp32 values the kernel reads
    pos = torch.full((B,), t, dtype=torch.int64, device="cuda")
    o = gb.gfwa_decode(q, k, v, a_new, Kc_ring, Vc_ring, Uc_t, pos)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    a_new_np = np64(a_new)
    for _ in range(48):
        b, hh = int(rng.integers(0, B)), int(rng.integers(0, H))
        order = [(tok % w) for tok in range(t - w + 1, t)]  # window of token t: t-w+1 .. t
        keys = np.concatenate([np64(Kc_ring[b, hh, order]), np64(k[b, hh])[None]])
        vals = np.concatenate([np64(Vc_ring[b, hh, order]), np64(v[b, hh])[None]])
        ut = -a_new_np[b, hh]  # frame u_{t-1} = 0
        u = np.concatenate([Uc_used[b, hh, order], [ut]])
        o_ref, _ = oracle.attend_row(np64(q[b, hh]), keys, vals, u, ut)
        assert np.abs(np64(o[b, hh]) - o_ref).max() <= TOL_BF16_O
    # the replaced slot now holds the new token
    assert torch.equal(Kc_ring[:, :, t % w], k) and torch.equal(Vc_ring[:, :, t % w], v)


@pytest.mark.parametrize("dtype,d,w,steps,G", [(torch.bfloat16, 128, 33, 50, 4), (torch.float32, 64, 16, 30, 2),
                                               (torch.bfloat16, 64, 20, 25, 8), (torch.bfloat16, 128, 1, 4, 4)])
def test_decode_gqa_sequence_equals_prefill_rows(dtype, d, w, steps, G):
    """GQA decode: query head hh reads K/V head hh // G; every
    step equals the oracle forward row with K/V expanded to the query heads
    (the definition of grouped-query attention), gates per query head."""
    B, H = 2, 8
    Hk = H // G
    s = synth.AttnShape(B=B, H=Hk, N=steps, d=d, w=w)
    _, K, V, _ = synth.attn_inputs(s, seed=steps + 3 * w, dtype=dtype, with_grad_out=False)
    sq = synth.AttnShape(B=B, H=H, N=steps, d=d, w=w)
    Q, _, _, _ = synth.attn_inputs(sq, seed=steps + 5 * w, dtype=dtype, with_grad_out=False)
    h, beta = synth.gate_inputs(B, steps, H, seed=w + G)
    Kc = torch.zeros(B, Hk, w, d, dtype=dtype, device="cuda")
    Vc = torch.zeros_like(Kc)
    Uc = torch.zeros(B, H, w, dtype=torch.float32, device="cuda")
    outs = []
    for t in range(steps):
        pos = torch.full((B,), t, dtype=torch.int64, device="cuda")
        o = gb.gfwa_decode(Q[:, t].cuda().contiguous(), K[:, t].cuda().contiguous(), V[:, t].cuda().contiguous(),
                           h[:, t].cuda(), Kc, Vc, Uc, pos, gate_b=beta[:, t].cuda())
        outs.append(np64(o))
    got = np.stack(outs, 1)  # [B, steps, H, d]
    U, _, _ = oracle.gate_prefix_hbeta(h, beta)
    ref, _ = oracle.fwd(Q, K.repeat_interleave(G, dim=2), V.repeat_interleave(G, dim=2), U, w)
    if dtype == torch.float32:
        assert np.abs(got - ref).max() / np.abs(ref).max() <= TOL_F32_O
    else:
        assert np.abs(got - ref).max() <= TOL_BF16_O
    for t in range(max(0, steps - w), steps):
        assert torch.equal(Kc[:, :, t % w].cpu(), K[:, t].to(dtype))


def test_decode_C5_gqa4_full_size_sampled():
    """C5 with GQA groups of 4 (B=64, H=32, H_kv=8, d=128, w=2048, bf16), wrapped
    ring (pos = w + 17); 48 sampled (b, h) rows vs the oracle."""
    c = synth.CONFIGS["C5_gqa4"]
    B, H, Hk, d, w = c["B"], c["H"], c["H_kv"], c["d"], c["w"]
    G = H // Hk
    Kc, Vc, a_hist, q, k, v, a_new = synth.decode_inputs(B, H, d, w, seed=c["seed"], device="cuda", H_kv=Hk)
    t = w + 17
    U_hist, _ = oracle.gate_prefix(a_hist)
    slots = np.arange(t - w, t) % w
    Uc = np.zeros((B, H, w))
    Uc[:, :, slots] = U_hist - U_hist[:, :, -1:]
    idx = torch.from_numpy(slots).cuda()
    Kc_ring, Vc_ring = torch.empty_like(Kc), torch.empty_like(Vc)
    Kc_ring[:, :, idx] = Kc
    Vc_ring[:, :, idx] = Vc
    Uc_t = torch.from_numpy(Uc).float().cuda()
    Uc_used = np64(Uc_t)
    pos = torch.full((B,), t, dtype=torch.int64, device="cuda")
    o = gb.gfwa_decode(q, k, v, a_new, Kc_ring, Vc_ring, Uc_t, pos)
    torch.cuda.synchronize()
    rng = np.random.default_rng(2)
    a_new_np = np64(a_new)
    order = [(tok % w) for tok in range(t - w + 1, t)]
    for _ in range(48):
        b, hh = int(rng.integers(0, B)), int(rng.integers(0, H))
        kh = hh // G
        keys = np.concatenate([np64(Kc_ring[b, kh, order]), np64(k[b, kh])[None]])
        vals = np.concatenate([np64(Vc_ring[b, kh, order]), np64(v[b, kh])[None]])
        ut = -a_new_np[b, hh]  # frame u_{t-1} = 0
        u = np.concatenate([Uc_used[b, hh, order], [ut]])
        o_ref, _ = oracle.attend_row(np64(q[b, hh]), keys, vals, u, ut)
        assert np.abs(np64(o[b, hh]) - o_ref).max() <= TOL_BF16_O
    assert torch.equal(Kc_ring[:, :, t % w], k) and torch.equal(Vc_ring[:, :, t % w], v)
    # every query head's ring is now relative to its own u_t: the new slot holds 0,
    # the others u_tau - u_t = U_cache + alpha_t
    after = np64(Uc_t)
    assert np.all(after[:, :, t % w] == 0.0)
    keep = [s for s in range(w) if s != t % w]
    assert np.allclose(after[:, :, keep], Uc_used[:, :, keep] + a_new_np[:, :, None], rtol=1e-6, atol=1e-5)


def test_decode_long_position_no_gate_drift():
    """3000 consecutive decode steps at a position past 10^6 with small
    gates (alpha ~ 5e-3).  An fp32 running absolute u would be ~1e4 there and
    swallow such alphas; the relative ring keeps every bias exact to fp32 of the
    window's gate sum.  After the run each slot must hold u_tau - u_last of the
    fp64 scan of the alphas the kernel saw, and the last output must equal the
    oracle row over the window."""
    B, H, d, w, steps, t0 = 1, 2, 64, 512, 3000, 1_000_003
    s = synth.AttnShape(B=B, H=H, N=steps, d=d, w=w)
    Q, K, V, _ = synth.attn_inputs(s, seed=77, dtype=torch.bfloat16, with_grad_out=False)
    g = torch.Generator().manual_seed(78)
    alpha = (0.005 * torch.rand(B, steps, H, generator=g)).float()
    Kc = torch.zeros(B, H, w, d, dtype=torch.bfloat16, device="cuda")
    Vc = torch.zeros_like(Kc)
    Uc = torch.zeros(B, H, w, dtype=torch.float32, device="cuda")
    a_dev = alpha.cuda()
    Qd, Kd, Vd = Q.cuda(), K.cuda(), V.cuda()
    for t in range(steps):
        pos = torch.full((B,), t0 + t, dtype=torch.int64, device="cuda")
        o = gb.gfwa_decode(Qd[:, t].contiguous(), Kd[:, t].contiguous(), Vd[:, t].contiguous(),
                           a_dev[:, t].contiguous(), Kc, Vc, Uc, pos)
    torch.cuda.synchronize()
    # before t0 the ring held zeros with U_cache 0 (fully open gates): the first w steps
    # see those zero rows; after w steps only real tokens remain
    U = -np.cumsum(alpha.double().numpy().transpose(0, 2, 1), -1)  # [B, H, steps]
    last = steps - 1
    for t in range(steps - w, steps):
        np.testing.assert_allclose(np64(Uc[:, :, (t0 + t) % w]), U[:, :, t] - U[:, :, last], rtol=0, atol=2e-5)
    ref, _ = oracle.fwd(Q[:, steps - w:], K[:, steps - w:], V[:, steps - w:], U[:, :, steps - w:], w)
    assert np.abs(np64(o) - ref[:, -1]).max() <= TOL_BF16_O
