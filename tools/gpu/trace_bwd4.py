"""Per-step timeline of the persistent tensor-core backward (diagnostics build
-DGFWA_BWD_TRACE=1): producer acquire, S^T issue, softmax start, dQ drain per
global step g of a CTA, and the dK/dV-ready stamp per item.

    GFWA_LIB=paper_2512_07782_b200/variants/libgfwa_btrace.so python tools/gpu/trace_bwd4.py C2
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
T = 512
buf = np.zeros(148 * 12 * T, dtype=np.int64)
lib.gfwa_debug_bwd_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.gfwa_debug_bwd_trace(buf.ctypes.data, buf.size) == 0
tr = buf.reshape(148, 12, T).astype(np.float64)
for cta in (3, 77):
    t = tr[cta]
    base = t[3, 0]
    n = int(np.count_nonzero(t[0]))
    print(f"=== CTA {cta}: {n} steps; columns: g | acq(P) S_issue softmax drain (relative) | dS-dP step deltas")
    for g in list(range(0, min(n, 24))) + list(range(max(24, n - 4), n)):
        row = [t[3, g], t[1, g], t[0, g], t[2, g]]
        rel = [int(v - base) if v > 0 else -1 for v in row]
        d = int(t[0, g] - t[0, g - 1]) if g > 0 else 0
        print(f"{g:4d} | " + " ".join(f"{v:8d}" for v in rel) + f" | sm {d:6d} | S-acq {int(t[1,g]-t[3,g]):6d} sm-S {int(t[0,g]-t[1,g]):6d}")
    ni = int(np.count_nonzero(t[4]))
    print("dkdv_full per item:", [int(v - base) for v in t[4, :min(ni, 6)]])
# aggregate: softmax step-to-step deltas over all CTAs
d = np.diff(tr[:, 0, :], axis=1)
d = d[(tr[:, 0, 1:] > 0) & (tr[:, 0, :-1] > 0)]
S, X, D, M2, R, DR = tr[:, 1], tr[:, 0], tr[:, 2], tr[:, 5], tr[:, 6], tr[:, 7]
def q(nm, v):
    v = v[np.isfinite(v) & (np.abs(v) < 1e6)]
    print(f"{nm:40s} p10 {np.percentile(v,10):6.0f} med {np.median(v):6.0f} p90 {np.percentile(v,90):6.0f}")
ok = lambda *a: np.logical_and.reduce([x > 0 for x in a])
for nm, a, b in (("A st issue -> softmax start", S, X), ("B softmax start -> ds_ready", X, R),
                 ("C ds_ready -> mma2 issue", R, M2), ("D mma2 issue -> drain sees dq_full", M2, D),
                 ("E drain sees -> drained", D, DR)):
    m = ok(a, b)
    q(nm, (b - a)[m])
for nm, a, b in (("WG1 st_full seen - WG0's", X, tr[:, 9]), ("WG1 softmax (warp 4)", tr[:, 9], tr[:, 8]),
                 ("ds_ready warp3 - warp0", R, tr[:, 10]), ("ds_ready warp7 - warp0", R, tr[:, 11]),
                 ("last ds_ready (w0,3,4,7) -> mma2 issue", np.maximum.reduce([R, tr[:, 8], tr[:, 10], tr[:, 11]]), M2)):
    m = ok(a, b)
    q(nm, (b - a)[m])
m = ok(DR[:, :-2], S[:, 2:])
q("F drained(g) -> st(g+2) issue", (S[:, 2:] - DR[:, :-2])[m])
m = ok(S[:, 1:], M2[:, :-1])
q("st(g+1) issue -> mma2(g) issue", (M2[:, :-1] - S[:, 1:])[m])
print("softmax start-to-start: p10 %.0f med %.0f p90 %.0f p99 %.0f mean %.0f" % (np.percentile(d, 10), np.median(d), np.percentile(d, 90), np.percentile(d, 99), d.mean()))
