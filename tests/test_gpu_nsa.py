"""GPU parity of the NSA hybrid with GatedFWA as the local branch (App. B,
P:633-703; readings C-28 block-mean compression, C-29 own block + top-n
selection) against the fp64 oracle, through gfwa_nsa_fwd.

The selection is an arg-max decision on fp32 scores: it is checked for validity
against the fp64 scores (every selected block scores within 1e-3 of the best
block left out, C-19: several selections are correct on near-ties), and the
oracle's selected-block attention is evaluated on the kernel's selection."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2512_07782_b200 import binding as gb
from parity import TOL_BF16_O, max_abs, np64

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B,H,N,d,w,blk,nsel", [(1, 2, 300, 128, 96, 16, 4), (2, 3, 520, 64, 200, 32, 5),
                                                 (1, 2, 1024, 128, 512, 64, 16), (1, 1, 40, 64, 8, 16, 3),
                                                 (1, 2, 10, 128, 4, 16, 2)])  # N < block: no complete block
def test_nsa_fwd_matches_oracle(B, H, N, d, w, blk, nsel):
    s = synth.AttnShape(B=B, H=H, N=N, d=d, w=w)
    Q, K, V, _ = synth.attn_inputs(s, seed=N + d, dtype=torch.bfloat16)
    g = torch.Generator().manual_seed(N)
    U = (-torch.cumsum(torch.nn.functional.softplus(torch.randn(B, H, N, generator=g)).double(), -1)).float()
    gates = torch.randn(B, N, H, 3, generator=g)
    O, sv = gb.gfwa_nsa_fwd(Q.cuda(), K.cuda(), V.cuda(), U.cuda(), gates.cuda(), w, block=blk, n_sel=nsel)
    oc, osl, sel, ol = sv["O_cmp"], sv["O_slc"], sv["sel"], sv["O_loc"]
    torch.cuda.synchronize()
    Kc, Vc = oracle.nsa_compress(K, V, blk)
    Ocr, sc = oracle.nsa_cmp(Q, Kc, Vc, blk)
    assert max_abs(oc, Ocr) <= TOL_BF16_O
    # selection: own block first; the others valid against the fp64 scores
    sel = sel.cpu().numpy().astype(np.int64)
    nb = N // blk
    for t in range(N):
        assert np.all(sel[:, :, t, 0] == t // blk)
    ref_sel = oracle.nsa_select(sc, N, blk, nsel)
    n_valid = np.sum(ref_sel[..., 1:] >= 0, -1)
    assert np.array_equal(np.sum(sel[..., 1:] >= 0, -1), n_valid)
    for bb in range(B):
        for hh in range(H):
            for t in range(N):
                picked = [i for i in sel[bb, hh, t, 1:] if i >= 0]
                left = [i for i in range(min(nb, (t + 1) // blk)) if i not in picked and i != t // blk]
                if picked and left:
                    assert min(sc[bb, hh, t, picked]) >= max(sc[bb, hh, t, left]) - 1e-3
    Oslr = oracle.nsa_slc(Q, K, V, sel, blk)
    assert max_abs(osl, Oslr) <= TOL_BF16_O
    Olr, _ = oracle.fwd(Q, K, V, U, w)
    assert max_abs(ol, Olr) <= TOL_BF16_O
    Or = oracle.nsa_combine(Ocr, Oslr, Olr, gates)
    assert max_abs(O, Or) <= TOL_BF16_O


@pytest.mark.parametrize("B,H,N,d,w,blk,nsel", [(1, 2, 300, 128, 96, 16, 4), (2, 2, 260, 64, 70, 32, 3),
                                                 (1, 1, 40, 64, 8, 16, 3), (1, 2, 10, 128, 4, 16, 2)])
def test_nsa_bwd_matches_oracle(B, H, N, d, w, blk, nsel):
    """gfwa_nsa_bwd vs the oracle's chain rule on the kernel's own selection; gradients at
    north_star's bf16 budget (5e-2 abs), dgates likewise."""
    s = synth.AttnShape(B=B, H=H, N=N, d=d, w=w)
    Q, K, V, dO = synth.attn_inputs(s, seed=2 * N + d, dtype=torch.bfloat16)
    g = torch.Generator().manual_seed(N + 1)
    U = (-torch.cumsum(torch.nn.functional.softplus(torch.randn(B, H, N, generator=g)).double(), -1)).float()
    gates = torch.randn(B, N, H, 3, generator=g)
    dev = [x.cuda() for x in (Q, K, V, U, gates, dO)]
    O, sv = gb.gfwa_nsa_fwd(*dev[:5], w, block=blk, n_sel=nsel)
    dQ, dK, dV, dU, dg = gb.gfwa_nsa_bwd(*dev[:5], dev[5], sv, w, block=blk, n_sel=nsel)
    torch.cuda.synchronize()
    sel = sv["sel"].cpu().numpy().astype(np.int64)
    rQ, rK, rV, rU, rg = oracle.nsa_bwd(Q, K, V, U, gates, dO, sel, w, blk)
    from parity import TOL_BF16_GRAD
    for name, got, ref in (("dQ", dQ, rQ), ("dK", dK, rK), ("dV", dV, rV), ("dU", dU, rU), ("dgates", dg, rg)):
        assert max_abs(got, ref) <= TOL_BF16_GRAD, name
