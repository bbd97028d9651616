"""Training forward (gfwa_fwd_train: O_lo + dQ-accumulator zeroing) timings."""
import os, sys
import torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2512_07782_b200 import binding as gb
for wl in (sys.argv[1:] or ["C2", "C3_w512"]):
    c = synth.CONFIGS[wl]
    s = synth.AttnShape(B=c["B"], H=c["H"], N=c["N"], d=c["d"], w=c["w"])
    Q, K, V, dO = synth.attn_inputs(s, seed=1, device="cuda", dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=2, device="cuda")
    U = gb.gfwa_gate_prefix(h, beta)
    for prep in (False, True):
        for _ in range(3):
            gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True, prepare_bwd=prep)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True, prepare_bwd=prep)
        e1.record(); torch.cuda.synchronize()
        print(f"{wl} train fwd prepare_bwd={prep}: {e0.elapsed_time(e1)/20*1e3:.1f} us", flush=True)
