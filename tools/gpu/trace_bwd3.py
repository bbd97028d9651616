"""Aggregate per-CTA timeline of the tensor-core backward (diagnostics build
-DGFWA_BWD_TRACE=1): prologue (entry -> first S^T ready), steady step time,
tail (last grad MMA -> exit) and the gap between consecutive CTAs on one SM.

    GFWA_LIB=paper_2512_07782_b200/variants/libgfwa_btrace.so python tools/gpu/trace_bwd3.py C2
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
tr = buf.reshape(296, 8, T).astype(np.float64)
entry, tm, end, smid = tr[:, 5, 2], tr[:, 5, 0], tr[:, 5, 1], tr[:, 5, 3].astype(int)
st0 = tr[:, 0, 0]  # softmax: st_full of step 0 observed
nst = np.array([np.count_nonzero(tr[i, 0, 0::3][:T // 3]) for i in range(296)])
def q(name, v):
    v = v[np.isfinite(v)]
    print(f"{name:40s} p10 {np.percentile(v,10):8.0f}  med {np.median(v):8.0f}  p90 {np.percentile(v,90):8.0f}")
print("steps per CTA (median):", np.median(nst))
q("entry -> tmem/sync", tm - entry)
q("entry -> step0 S^T ready", st0 - entry)
last_st = np.array([tr[i, 0, 3 * (nst[i] - 1)] for i in range(296)])
q("steady: (st(last) - st(0)) / (n-1)", (last_st - st0) / np.maximum(nst - 1, 1))
q("st(last) -> dkdv_full", tr[:, 4, 0] - last_st)
q("dkdv_full -> epilogue done", tr[:, 4, 1] - tr[:, 4, 0])
q("epilogue done -> exit", end - tr[:, 4, 1])
q("entry -> exit", end - entry)
# consecutive CTAs on one SM: gap between the earlier's exit and the later's entry
gaps = []
for sm in np.unique(smid):
    idx = np.where(smid == sm)[0]
    idx = idx[np.argsort(entry[idx])]
    for a, b in zip(idx[:-1], idx[1:]):
        gaps.append(entry[b] - end[a])
if gaps:
    q("exit -> next CTA entry (same SM)", np.array(gaps, dtype=float))
