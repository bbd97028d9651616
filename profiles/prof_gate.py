"""Gate-scan probe G (B=4, N=131072, H=32, bf16) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2512_07782_b200 import binding as gb  # noqa: E402

c = synth.CONFIGS["G"]
h, beta = synth.gate_inputs(c["B"], c["N"], c["H"], seed=c["seed"], device="cuda")
h, beta = h.bfloat16(), beta.bfloat16()
for _ in range(3):
    U = gb.gfwa_gate_prefix(h, beta)
    gb.gfwa_gate_prefix_bwd(U, h, beta)
torch.cuda.synchronize()
