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
    assert np.allclose(np64(Uc[:, :, t_last % w]), U[:, :, t_last], rtol=1e-6, atol=1e-5)


def test_decode_C5_full_size_sampled():
    """BASELINE configs[4] (C5: B=64, H=32, d=128, w=2048, bf16) with a wrapped,
    pre-filled ring (pos = w + 17); 48 sampled (b, h) rows vs the oracle over
    their token-ordered window."""
    c = synth.CONFIGS["C5"]
    B, H, d, w = c["B"], c["H"], c["d"], c["w"]
    Kc, Vc, a_hist, q, k, v, a_new = synth.decode_inputs(B, H, d, w, seed=c["seed"], device="cuda")
    t = w + 17
    # history tokens t-w .. t-1 live at slot (token mod w); their u from the oracle scan
    U_hist, _ = oracle.gate_prefix(a_hist)            # u of tokens t-w..t-1 (frame: u_{t-w-1} = 0)
    slots = np.arange(t - w, t) % w
    Uc = np.zeros((B, H, w))
    Uc[:, :, slots] = U_hist
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
        u_prev = Uc_used[b, hh, (t - 1) % w]
        ut = u_prev - a_new_np[b, hh]
        u = np.concatenate([Uc_used[b, hh, order], [ut]])
        o_ref, _ = oracle.attend_row(np64(q[b, hh]), keys, vals, u, ut)
        assert np.abs(np64(o[b, hh]) - o_ref).max() <= TOL_BF16_O
    # the replaced slot now holds the new token
    assert torch.equal(Kc_ring[:, :, t % w], k) and torch.equal(Vc_ring[:, :, t % w], v)
