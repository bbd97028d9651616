"""Per-role clock64 timeline of the persistent forward (diagnostics build:
python paper_2512_07782_b200/_build.py --variant ftrace -DGFWA_FWD_TRACE=1).

    GFWA_LIB=paper_2512_07782_b200/variants/libgfwa_ftrace.so python tools/gpu/trace_fwd2.py C2 [f32]
"""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2512_07782_b200 import binding as gb

wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
f32 = len(sys.argv) > 2 and sys.argv[2] == "f32"
c = synth.CONFIGS[wl]
s = synth.AttnShape(B=c["B"], H=c["H"], N=c["N"], d=c["d"], w=c["w"])
Q, K, V, dO = synth.attn_inputs(s, seed=1, device="cuda", dtype=torch.bfloat16)
h, beta = synth.gate_inputs(s.B, s.N, s.H, seed=2, device="cuda")
U = gb.gfwa_gate_prefix(h, beta)
for _ in range(3):
    gb.gfwa_fwd(Q, K, V, U, s.w, want_o_lo=f32)
torch.cuda.synchronize()
lib = gb.load()
T = 512
buf = np.zeros(148 * 8 * T, dtype=np.int64)
lib.gfwa_debug_fwd_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.gfwa_debug_fwd_trace(buf.ctypes.data, buf.size) == 0
tr = buf.reshape(148, 8, T)
for cta in (0, 77):
    t = tr[cta]
    base = t[t > 0].min()
    rel = lambda v: (v - base) if v > 0 else -1  # noqa: E731
    print(f"=== CTA {cta}")
    for x in (0, 1):
        rows = []
        for k in range(0, 40):
            a, b_, e = t[x, 3 * k], t[x, 3 * k + 1], t[x, 3 * k + 2]
            if e == 0:
                break
            rows.append((rel(a), rel(b_), rel(e), b_ - a, e - b_))
        print(f"softmax {'AB'[x]}: (start, s_ready, done, wait, work)")
        for r in rows[:14]:
            print("   ", r)
        w = np.array([r[3] for r in rows]); k_ = np.array([r[4] for r in rows])
        print(f"   mean wait {w.mean():.0f}  mean work {k_.mean():.0f}  n={len(rows)}")
    pv = [rel(v) for v in t[2, :60:2] if v > 0]
    print("MMA PV issue times:", pv[:16])
    for x in (0, 1):
        print(f"MMA S_{'AB'[x]} issue (by kv index):", [rel(v) for v in t[3 + x, :16] if v > 0])
    print("producer K issue:", [rel(v) for v in t[6, :16] if v > 0])
    print("epilogue (start, data ready, done):", [(rel(t[5, 4 * k]), rel(t[5, 4 * k + 1]), rel(t[5, 4 * k + 2])) for k in range(6) if t[5, 4 * k] > 0])
    last = t[t > 0].max() - base
    print("CTA span cycles:", last)
