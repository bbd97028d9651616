"""One C2 training step (gate -> fwd -> bwd -> gate bwd) for ncu captures.

  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv python profiles/prof_step.py
  ncu --set full --clock-control none --import-source on -k regex:fwd_tc -c 1 \
      -o gpurun_out/fwd python profiles/prof_step.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2512_07782_b200 import binding as gb  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
    c = synth.CONFIGS[wl]
    s = synth.AttnShape(B=c["B"], H=c["H"], N=c["N"], d=c["d"], w=c["w"])
    Q, K, V, dO = synth.attn_inputs(s, seed=c["seed"], device="cuda", dtype=torch.bfloat16)
    h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=c["seed"], device="cuda")
    h, beta = h.bfloat16(), beta.bfloat16()
    for _ in range(2):
        U = gb.gfwa_gate_prefix(h, beta)
        O, LSE, Olo = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True, prepare_bwd=True)
        dQ, dK, dV, dU, _ = gb.gfwa_bwd(Q, K, V, U, O, LSE, dO, s.w, O_lo=Olo, want_dalpha=False)
        gb.gfwa_gate_prefix_bwd(dU, h, beta, want_dalpha=False)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
