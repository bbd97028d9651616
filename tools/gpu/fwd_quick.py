"""Quick forward check + timing of the tensor-core forward against the oracle
(development helper): small shapes element-wise, then C2/C3 timings."""
import sys, os, time
import numpy as np
import torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import oracle, synth
from paper_2512_07782_b200 import binding as gb

def check(s, seed=1):
    Q, K, V, dO = synth.attn_inputs(s, seed=seed, device="cuda", dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, s.nkv, s.H, seed=seed + 1, device="cuda")
    U = gb.gfwa_gate_prefix(h, beta)
    res = []
    for f32 in (False, True):
        O, LSE, Olo = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=f32)
        torch.cuda.synchronize()
        Or, Lr = oracle.fwd(Q, K, V, U, s.w)
        e = np.abs(O.float().cpu().double().numpy() - Or).max()
        el = np.abs(LSE.cpu().double().numpy() - Lr).max()
        e32 = np.abs(O.double().cpu().numpy() + Olo.double().cpu().numpy() - Or).max() if f32 else 0
        res.append((e, el, e32))
    print(s, "err O/LSE/Olo (bf16P, f16P):", res, flush=True)

for s in [synth.AttnShape(B=1, H=2, N=300, d=128, w=96), synth.AttnShape(B=2, H=2, N=1000, d=128, w=512),
          synth.AttnShape(B=1, H=2, N=1, d=128, w=1), synth.AttnShape(B=1, H=3, N=37, d=128, w=33),
          synth.AttnShape(B=1, H=2, N=300, d=128, w=250, N_kv=500), synth.AttnShape(B=1, H=2, N=390, d=128, w=1000),
          synth.AttnShape(B=2, H=2, N=200, d=128, w=1), synth.AttnShape(B=1, H=2, N=777, d=128, w=128)]:
    check(s)

for wl in ["C2", "C3_w512", "C3_w2048", "C3_w128"]:
    c = synth.CONFIGS[wl]
    s = synth.AttnShape(B=c["B"], H=c["H"], N=c["N"], d=c["d"], w=c["w"])
    Q, K, V, dO = synth.attn_inputs(s, seed=1, device="cuda", dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=2, device="cuda")
    U = gb.gfwa_gate_prefix(h, beta)
    for f32 in (False, True):
        for _ in range(3):
            gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=f32)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        n = 20
        for _ in range(n):
            gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=f32)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        fl = 4.0 * s.N * s.w * s.d * s.B * s.H
        print(f"{wl} f32out={f32}: {ms*1e3:.1f} us  {fl/ms/1e9:.1f} TFLOP/s  ({fl/ms/1e9/1627.2:.3f} of peak)", flush=True)
