"""d=64 timings (the paper's model head dim) on the tensor-core path."""
import os, sys
import torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2512_07782_b200 import binding as gb
for (B, H, N, w) in ((8, 32, 4096, 512), (1, 64, 8192, 512)):
    s = synth.AttnShape(B=B, H=H, N=N, d=64, w=w)
    Q, K, V, dO = synth.attn_inputs(s, seed=1, device="cuda", dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=2, device="cuda")
    U = gb.gfwa_gate_prefix(h, beta)
    assert gb.gfwa_attn_path(Q, K, V, s.w) == 1
    def t(fn, n=20):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n): fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n
    O, LSE, Olo = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True)
    fl = 4.0 * N * w * 64 * B * H
    mf = t(lambda: gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True))
    mb = t(lambda: gb.gfwa_bwd(Q, K, V, U, O, LSE, dO, s.w, O_lo=Olo, want_dalpha=False), 2) if "--bwd" in sys.argv else float("nan")
    print(f"d64 B{B} H{H} N{N} w{w}: fwd {mf*1e3:.1f} us ({fl/mf/1e9:.0f} TFLOP/s), bwd {mb*1e3:.1f} us ({2.5*fl/mb/1e9:.0f} TFLOP/s)", flush=True)
