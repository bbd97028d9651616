"""Forward timings (CUDA events, 20 calls after 3 warm-ups) for the C2/C3 shapes;
GFWA_LIB selects an experiment build."""
import os, sys
import torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2512_07782_b200 import binding as gb
tag = os.environ.get("GFWA_LIB", "default").split("/")[-1]
for wl in (sys.argv[1:] or ["C2", "C3_w512", "C3_w2048", "C3_w128"]):
    c = synth.CONFIGS[wl]
    s = synth.AttnShape(B=c["B"], H=c["H"], N=c["N"], d=c["d"], w=c["w"])
    Q, K, V, dO = synth.attn_inputs(s, seed=1, device="cuda", dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=2, device="cuda")
    U = gb.gfwa_gate_prefix(h, beta)
    for lo in (True, False):
        for _ in range(3):
            gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=lo)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=lo)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        fl = 4.0 * s.N * s.w * s.d * s.B * s.H
        print(f"{tag:22s} {wl:9s} {'train' if lo else 'infer'}: {ms*1e3:7.1f} us {fl/ms/1e9:7.1f} TFLOP/s ({fl/ms/1e9/1627.2:.3f})", flush=True)
