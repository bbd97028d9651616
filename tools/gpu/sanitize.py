"""Small invocations of every kernel for compute-sanitizer (memcheck / racecheck /
synccheck): gate scan fwd/bwd, tensor-core forward (inference and training),
tensor-core backward, SIMT fp32 path, decode (MHA + GQA)."""
import os, sys
import torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2512_07782_b200 import binding as gb

dev = "cuda"
s = synth.AttnShape(B=1, H=2, N=300, d=128, w=96, N_kv=340)
Q, K, V, dO = synth.attn_inputs(s, seed=1, device=dev, dtype=torch.bfloat16)
h, beta = synth.gate_inputs(s.B, s.nkv, s.H, seed=2, device=dev)
U = gb.gfwa_gate_prefix(h, beta)
for lo in (False, True):
    O, LSE, Olo = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=lo, prepare_bwd=lo)
dQ, dK, dV, dU, da = gb.gfwa_bwd(Q, K, V, U, O, LSE, dO, s.w, O_lo=Olo)
gb.gfwa_gate_prefix_bwd(dU, h, beta)
s32 = synth.AttnShape(B=1, H=2, N=130, d=64, w=40)
Q, K, V, dO = synth.attn_inputs(s32, seed=3, device=dev, dtype=torch.float32)
U32 = gb.gfwa_gate_prefix(*synth.gate_inputs(1, s32.N, 2, seed=4, device=dev))
O, LSE, _ = gb.gfwa_fwd(Q, K, V, U32, s32.w)
gb.gfwa_bwd(Q, K, V, U32, O, LSE, dO, s32.w)
for Hk in (4, 1):
    Kc, Vc, a_hist, q, k, v, a_new = synth.decode_inputs(2, 4, 128, 64, seed=5, device=dev, H_kv=Hk)
    Uc = torch.zeros(2, 4, 64, device=dev)
    pos = torch.full((2,), 70, dtype=torch.int64, device=dev)
    gb.gfwa_decode(q, k, v, a_new, Kc, Vc, Uc, pos)
# persistent kernels with several items per CTA (slot-pool rotation, item boundaries), d = 64 and 128
os.environ["GFWA_BWD_GRID"] = "3"
os.environ["GFWA_FWD_GRID"] = "2"
for d in (64, 128):
    sm = synth.AttnShape(B=1, H=3, N=900, d=d, w=200)
    Q, K, V, dO = synth.attn_inputs(sm, seed=6, device=dev, dtype=torch.bfloat16)
    Um = gb.gfwa_gate_prefix(*synth.gate_inputs(1, sm.N, 3, seed=7, device=dev))
    O, LSE, Olo = gb.gfwa_fwd(Q, K, V, Um, sm.w, want_o_lo=True, prepare_bwd=True)
    gb.gfwa_bwd(Q, K, V, Um, O, LSE, dO, sm.w, O_lo=Olo)
del os.environ["GFWA_BWD_GRID"], os.environ["GFWA_FWD_GRID"]
torch.cuda.synchronize()
print("sanitize workload done")
