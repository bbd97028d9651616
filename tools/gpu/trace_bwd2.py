"""Per-role clock64 timeline of the tensor-core backward (diagnostics build:
python paper_2512_07782_b200/_build.py --variant btrace -DGFWA_BWD_TRACE=1).

    GFWA_LIB=paper_2512_07782_b200/variants/libgfwa_btrace.so python tools/gpu/trace_bwd2.py C2
"""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2512_07782_b200 import binding as gb

wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
c = synth.CONFIGS[wl]
s = synth.AttnShape(B=c["B"], H=c["H"], N=c["N"], d=c["d"], w=c["w"])
Q, K, V, dO = synth.attn_inputs(s, seed=1, device="cuda", dtype=torch.bfloat16)
h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=2, device="cuda")
U = gb.gfwa_gate_prefix(h, beta)
O, LSE, Olo = gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True)
for _ in range(3):
    gb.gfwa_bwd(Q, K, V, U, O, LSE, dO, s.w, O_lo=Olo)
torch.cuda.synchronize()
lib = gb.load()
T = 256
buf = np.zeros(296 * 8 * T, dtype=np.int64)
lib.gfwa_debug_bwd_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.gfwa_debug_bwd_trace(buf.ctypes.data, buf.size) == 0
tr = buf.reshape(296, 8, T)
for cta in (150, 200):
    t = tr[cta]
    base = t[5, 2]
    rel = lambda v: int(v - base) if v > 0 else -1  # noqa: E731
    print(f"=== CTA {cta}: start->tmem {rel(t[5,0])}, end {rel(t[5,1])}, dkdv_full {rel(t[4,0])}, epi done {rel(t[4,1])}")
    print(" n | Qload  S_iss  sm_beg  ld_done calc  ds_rdy  bfly_end red_free grad_iss dq_full drained | ld calc st bfly | qfull drnd(n-2)")
    for n in range(12):
        if t[0, 3 * n] == 0:
            break
        row = [rel(t[3, n]), rel(t[1, 2 * n]), rel(t[0, 3 * n]), rel(t[6, 3 * n]), rel(t[6, 3 * n + 1]),
               rel(t[0, 3 * n + 1]), rel(t[6, 3 * n + 2]), rel(t[0, 3 * n + 2]),
               rel(t[1, 2 * n + 1]), rel(t[2, 2 * n]), rel(t[2, 2 * n + 1])]
        d = [row[3] - row[2], row[4] - row[3], row[5] - row[4], row[6] - row[5]]
        print(f"{n:2d} | " + " ".join(f"{v:6d}" for v in row) + " | " + " ".join(f"{v:5d}" for v in d) + f" | {rel(t[7, 2 * n]):6d} {rel(t[7, 2 * n + 1]):6d}")
