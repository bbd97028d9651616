import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, synth
from paper_2512_07782_b200 import binding as gb
c = synth.CONFIGS["C2"]
s = synth.AttnShape(B=c["B"], H=c["H"], N=c["N"], d=c["d"], w=c["w"])
Q, K, V, dO = synth.attn_inputs(s, seed=1, device="cuda", dtype=torch.bfloat16)
h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=1, device="cuda")
U = gb.gfwa_gate_prefix(h, beta)
Z = torch.empty(s.B * s.N * s.H * s.d, dtype=torch.float32, device="cuda")
side = torch.cuda.Stream()
def run(conc, zero):
    ev = torch.cuda.Event()
    if zero and conc:
        ev.record(); side.wait_event(ev)
        with torch.cuda.stream(side): Z.zero_()
    gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True)
    if zero and not conc: Z.zero_()
    if zero and conc:
        e2 = torch.cuda.Event(); e2.record(side); torch.cuda.current_stream().wait_event(e2)
for name, conc, zero in (("fwd alone", False, False), ("fwd then zero", False, True), ("fwd || zero", True, True)):
    for _ in range(3): run(conc, zero)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(20): run(conc, zero)
    b.record(); torch.cuda.synchronize()
    print(name, round(a.elapsed_time(b) / 20 * 1000, 1), "us")
