"""One training backward (after a prepared forward) of a workload, for ncu captures."""
import os, sys
import torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2512_07782_b200 import binding as gb
wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
c = synth.CONFIGS[wl]
s = synth.AttnShape(B=c["B"], H=c["H"], N=c["N"], d=c["d"], w=c["w"])
Q, K, V, dO = synth.attn_inputs(s, seed=1, device="cuda", dtype=torch.bfloat16)
h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=2, device="cuda")
U = gb.gfwa_gate_prefix(h, beta)
for _ in range(2):
    O, LSE, Olo = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True, prepare_bwd=True)
    gb.gfwa_bwd(Q, K, V, U, O, LSE, dO, s.w, O_lo=Olo, want_dalpha=False)
torch.cuda.synchronize()
