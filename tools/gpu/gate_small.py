"""Gate scan at LM shapes: product (decoupled look-back) vs the one-program-per-head variant."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2512_07782_b200 import binding as gb  # noqa: E402

for B, N, H in ((8, 4096, 16), (1, 8192, 32), (1, 16384, 32)):
    h, beta = synth.gate_inputs(B, N, H, seed=1, device="cuda")
    h, beta = h.bfloat16(), beta.bfloat16()
    for name, fn in (("product", lambda: gb.gfwa_gate_prefix(h, beta)),
                     ("v1", lambda: gb.gfwa_gate_prefix_variant(1, h, beta)),
                     ("v2", lambda: gb.gfwa_gate_prefix_variant(2, h, beta))):
        for _ in range(3):
            fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(10):
                fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(5):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        print(B, N, H, name, round(a.elapsed_time(b) / 50 * 1000, 2), "us (graph replay)")
