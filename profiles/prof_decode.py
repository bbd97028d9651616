"""Decode probe C5 (B=64, H=32, d=128, w=2048, bf16 cache) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2512_07782_b200 import binding as gb  # noqa: E402

c = synth.CONFIGS["C5"]
Kc, Vc, a_hist, q, k, v, a_new = synth.decode_inputs(c["B"], c["H"], c["d"], c["w"], seed=c["seed"], device="cuda")
Uc = -torch.cumsum(a_hist, -1)
pos = torch.full((c["B"],), c["w"] + 17, dtype=torch.int64, device="cuda")
for _ in range(3):
    gb.gfwa_decode(q, k, v, a_new, Kc, Vc, Uc, pos)
torch.cuda.synchronize()
