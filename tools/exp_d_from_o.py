import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import torch, numpy as np
import oracle, synth
from paper_2512_07782_b200 import binding as gb
from parity import max_abs
from test_gpu_attn import BF16_SHAPES, _U
for s in BF16_SHAPES + [synth.AttnShape(B=1, H=2, N=4096, d=128, w=512)]:
    seed = 3 * s.N + s.w
    Q, K, V, dO = synth.attn_inputs(s, seed=seed, dtype=torch.bfloat16)
    U = _U(s.B, s.H, s.nkv, seed + 1)
    Qd, Kd, Vd, dOd, Ud = (x.cuda() for x in (Q, K, V, dO, U))
    O, LSE, O32 = gb.gfwa_fwd(Qd, Kd, Vd, Ud, s.w, want_o_f32=True)
    g = oracle.bwd(Q, K, V, U, dO, s.w)
    res = []
    for tag, o32 in (("f32", O32), ("bf16", None)):
        dQ, dK, dV, dU, da = gb.gfwa_bwd(Qd, Kd, Vd, Ud, O, LSE, dOd, s.w, O_f32=o32)
        torch.cuda.synchronize()
        res.append(tag + " " + " ".join(f"{k}={max_abs(v, g[k]):.2e}" for k, v in (("dQ", dQ), ("dK", dK), ("dV", dV), ("dU", dU), ("dalpha", da))))
    print(s, *res, sep="\n  ")
