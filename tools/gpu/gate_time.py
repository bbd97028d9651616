"""Gate scan timings: probe G (B=4, N=131072, H=32) fwd and bwd, and C2."""
import os, sys
import torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2512_07782_b200 import binding as gb
for wl, (B, N, H) in (("G", (4, 131072, 32)), ("C2", (8, 4096, 16))):
    h, beta = synth.gate_inputs(B, N, H, seed=3, device="cuda")
    h, beta = h.bfloat16(), beta.bfloat16()
    def t(fn, n=50):
        for _ in range(5): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n): fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n
    U = gb.gfwa_gate_prefix(h, beta)
    mf = t(lambda: gb.gfwa_gate_prefix(h, beta))
    mb = t(lambda: gb.gfwa_gate_prefix_bwd(U, h, beta))
    el = B * N * H
    print(f"{wl}: fwd {mf*1e3:.1f} us ({el*8/mf/1e6:.0f} GB/s = {el*8/mf/1e6/6554.6:.3f} of HBM), bwd {mb*1e3:.1f} us", flush=True)
