"""C5 GQA decode (B=64, H=32, H_kv=8, w=2048, bf16) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2512_07782_b200 import binding as gb  # noqa: E402

c = synth.CONFIGS["C5_gqa4"]
B, H, Hk, d, w = c["B"], c["H"], c["H_kv"], c["d"], c["w"]
Kc, Vc, a, q, k, v, an = synth.decode_inputs(B, H, d, w, seed=c["seed"], device="cuda", H_kv=Hk)
Uc = -torch.cumsum(a, -1)
pos = torch.full((B,), w + 17, dtype=torch.int64, device="cuda")
for _ in range(3):
    gb.gfwa_decode(q, k, v, an, Kc, Vc, Uc, pos)
torch.cuda.synchronize()
