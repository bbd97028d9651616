"""Gate scan fwd + bwd at the LM shapes (C2, C3, one C4 rank at P=8) for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2512_07782_b200 import binding as gb  # noqa: E402

for B, N, H in ((8, 4096, 16), (1, 8192, 32), (1, 16384, 32)):
    h, beta = synth.gate_inputs(B, N, H, seed=1, device="cuda")
    h, beta = h.bfloat16(), beta.bfloat16()
    for _ in range(3):
        U = gb.gfwa_gate_prefix(h, beta)
        gb.gfwa_gate_prefix_bwd(U, h, beta)
torch.cuda.synchronize()
