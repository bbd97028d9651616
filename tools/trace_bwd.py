"""Analyse GFWA_TRACE_BWD dumps: per-step phase timings (clock64 cycles)."""
import sys
import numpy as np
t = np.fromfile(sys.argv[1], dtype=np.int64).reshape(-1, 64).astype(float)
t[t == 0] = np.nan
def stat(name, v):
    v = v[np.isfinite(v)]
    if len(v): print(f"{name:34s} median {np.median(v):9.0f}  p10 {np.percentile(v,10):9.0f}  p90 {np.percentile(v,90):9.0f}")
st, ds, m2, dq, dr = (t[:, o:o + 8] for o in (1, 9, 17, 25, 33))
start = t[:, 0]
stat("start -> first st_full", st[:, 0] - start)
for n in (0, 1, 2, 4):
    stat(f"step{n}: softmax-grad (st->ds)", ds[:, n] - st[:, n])
    stat(f"step{n}: ds -> MMA2 start", m2[:, n] - ds[:, n])
    stat(f"step{n}: MMA2 start -> dq_full", dq[:, n] - m2[:, n])
    stat(f"step{n}: drain (dq_full->drained)", dr[:, n] - dq[:, n])
    stat(f"step{n}: st(n) -> st(n+1)", st[:, n + 1] - st[:, n])
    stat(f"step{n}: drain staging+reduce issue", t[:, 49 + n] - dr[:, n])
    stat(f"step{n}: drain loop (dq_full n -> n+1)", dq[:, n + 1] - dq[:, n])
stat("last MMA2 -> dkdv_full", t[:, 41] - np.nanmax(m2, axis=1))
stat("epilogue", t[:, 42] - t[:, 41])
stat("total", t[:, 42] - start)
s4 = t[:, 1 + 4]
for name, a, b in (("st_full->LDTM done", s4, t[:, 43]), ("compute", t[:, 43], t[:, 44]), ("STTM+STS", t[:, 44], t[:, 45]),
                   ("wait_st+fence+arrive", t[:, 45], t[:, 46]), ("butterfly+partials", t[:, 46], t[:, 47])):
    stat("step4 sg: " + name, b - a)
