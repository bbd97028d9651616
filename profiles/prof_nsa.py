import sys, torch
sys.path.insert(0, ".")
import synth
from paper_2512_07782_b200 import binding as gb
s = synth.AttnShape(B=2, H=16, N=4096, d=128, w=512)
Q, K, V, dO = synth.attn_inputs(s, seed=77, device="cuda", dtype=torch.bfloat16)
h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=78, device="cuda")
U = gb.gfwa_gate_prefix(h, beta)
gates = torch.randn(s.B, s.N, s.H, 3, device="cuda")
O, sv = gb.gfwa_nsa_fwd(Q, K, V, U, gates, s.w, 64, 16)
gb.gfwa_nsa_bwd(Q, K, V, U, gates, dO, sv, s.w, 64, 16)
torch.cuda.synchronize()
