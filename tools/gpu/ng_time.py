"""Time the fused AttnLayer epilogue calls against the plain ones at C2 (CUDA events)."""
import os, sys
import torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2512_07782_b200 import binding as gb

c = synth.CONFIGS["C2"]
s = synth.AttnShape(B=c["B"], H=c["H"], N=c["N"], d=c["d"], w=c["w"])
Q, K, V, dY = synth.attn_inputs(s, seed=c["seed"], device="cuda", dtype=torch.bfloat16)
h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=c["seed"], device="cuda")
U = gb.gfwa_gate_prefix(h, beta)
g = torch.randn(s.B, s.N, s.H, s.d, device="cuda").to(torch.bfloat16)
gamma = torch.ones(s.d, device="cuda")
Y, O, LSE, Olo, rstd = gb.gfwa_fwd_normgate(Q, K, V, U, g, gamma, s.w, prepare_bwd=True)


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


print("fwd_train      %.1f us" % t(lambda: gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True, prepare_bwd=True)))
print("fwd_normgate   %.1f us" % t(lambda: gb.gfwa_fwd_normgate(Q, K, V, U, g, gamma, s.w, prepare_bwd=True)))
print("bwd            %.1f us" % t(lambda: gb.gfwa_bwd(Q, K, V, U, O, LSE, dY, s.w, O_lo=Olo, want_dalpha=False)))
print("bwd_normgate   %.1f us" % t(lambda: gb.gfwa_bwd_normgate(Q, K, V, U, O, LSE, g, gamma, rstd, dY, s.w, O_lo=Olo,
                                                              want_dalpha=False)))
