"""Per-phase softmax timeline of the persistent forward (diagnostics build
-DGFWA_FWD_TRACE=1): for tile A/B, per key step: s_full wait, pass 1, row-max
exchange, pass 2 (exponentials), the rest (rescale, P store, arrive).

    GFWA_LIB=paper_2512_07782_b200/variants/libgfwa_ftrace.so python tools/gpu/trace_fwd3.py C2
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
for _ in range(3):
    gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=True)
torch.cuda.synchronize()
lib = gb.load()
T = 1024
buf = np.zeros(148 * 8 * T, dtype=np.int64)
lib.gfwa_debug_fwd_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.gfwa_debug_fwd_trace(buf.ctypes.data, buf.size) == 0
tr = buf.reshape(148, 8, T).astype(np.float64)
for x in (0, 1):
    t = tr[:, x, :(T // 6) * 6].reshape(148, T // 6, 6)
    ok = np.all(t > 0, axis=2)
    d = np.diff(t, axis=2)[ok]
    names = ["s_full wait", "pass 1 (max)", "row-max exchange", "pass 2 (exp)", "rest (rescale, arrive)"]
    print(f"tile {'AB'[x]}: median cycles " + ", ".join(f"{n} {np.median(d[:, i]):.0f}" for i, n in enumerate(names)))
    st = t[:, :, 0][ok]
    per = np.diff(t[:, :, 0], axis=1)[ok[:, 1:] & ok[:, :-1]]
    print(f"   step period median {np.median(per):.0f}")
