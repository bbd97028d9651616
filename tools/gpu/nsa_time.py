"""NSA hybrid timings (bench aux config: B=2, H=16, N=4096, d=128, w=512, block 64, n_sel 16)."""
import os, sys
import torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2512_07782_b200 import binding as gb
s = synth.AttnShape(B=2, H=16, N=4096, d=128, w=512)
Q, K, V, dO = synth.attn_inputs(s, seed=77, device="cuda", dtype=torch.bfloat16)
h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=78, device="cuda")
U = gb.gfwa_gate_prefix(h, beta)
gates = torch.randn(s.B, s.N, s.H, 3, device="cuda")
def t(fn, n=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
O, sv = gb.gfwa_nsa_fwd(Q, K, V, U, gates, s.w, 64, 16)
mf = t(lambda: gb.gfwa_nsa_fwd(Q, K, V, U, gates, s.w, 64, 16))
def fb():
    O, sv = gb.gfwa_nsa_fwd(Q, K, V, U, gates, s.w, 64, 16)
    gb.gfwa_nsa_bwd(Q, K, V, U, gates, dO, sv, s.w, 64, 16)
mfb = t(fb)
print(f"nsa fwd {mf:.3f} ms, fwd+bwd {mfb:.3f} ms", flush=True)
