"""One C2 AttnLayer step with the fused epilogue (gfwa_fwd_normgate +
gfwa_bwd_normgate, reading C-27) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2512_07782_b200 import binding as gb  # noqa: E402

c = synth.CONFIGS["C2"]
s = synth.AttnShape(B=c["B"], H=c["H"], N=c["N"], d=c["d"], w=c["w"])
Q, K, V, dY = synth.attn_inputs(s, seed=c["seed"], device="cuda", dtype=torch.bfloat16)
h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=c["seed"], device="cuda")
g = torch.randn(s.B, s.N, s.H, s.d, device="cuda").to(torch.bfloat16)
gamma = torch.ones(s.d, device="cuda")
for _ in range(2):
    U = gb.gfwa_gate_prefix(h, beta)
    Y, O, LSE, Olo, rstd = gb.gfwa_fwd_normgate(Q, K, V, U, g, gamma, s.w, prepare_bwd=True)
    gb.gfwa_bwd_normgate(Q, K, V, U, O, LSE, g, gamma, rstd, dY, s.w, O_lo=Olo, want_dalpha=False)
torch.cuda.synchronize()
