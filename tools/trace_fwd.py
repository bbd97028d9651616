"""Analyse GFWA_TRACE_FWD dumps: per-CTA phase timings (clock64 cycles)."""
import sys
import numpy as np
t = np.fromfile(sys.argv[1], dtype=np.int64).reshape(-1, 64)
n = t.shape[0]
start, setup = t[:, 0], t[:, 1]
print("CTAs", n)
def stat(name, v):
    v = v[np.isfinite(v)]
    print(f"{name:28s} median {np.median(v):9.0f}  p10 {np.percentile(v,10):9.0f}  p90 {np.percentile(v,90):9.0f}")
stat("setup (start->sync)", (setup - start).astype(float))
kf = t[:, 2:10].astype(float); kf[kf == 0] = np.nan
stat("first K_full after setup", kf[:, 0] - setup)
for i, base in ((0, 16), (1, 40)):
    sf = t[:, base:base + 8].astype(float); sf[sf == 0] = np.nan
    pr = t[:, base + 8:base + 16].astype(float); pr[pr == 0] = np.nan
    of = t[:, base + 16].astype(float); ep = t[:, base + 17].astype(float)
    stat(f"tile{i}: first S_full - setup", sf[:, 0] - setup)
    stat(f"tile{i}: softmax (S->P) step0", pr[:, 0] - sf[:, 0])
    stat(f"tile{i}: softmax (S->P) step1", pr[:, 1] - sf[:, 1])
    stat(f"tile{i}: P(n)->S(n+1) step0", sf[:, 1] - pr[:, 0])
    stat(f"tile{i}: P(n)->S(n+1) step2", sf[:, 3] - pr[:, 2])
    last = np.nanmax(pr, axis=1)
    stat(f"tile{i}: lastP -> O_full", of - last)
    stat(f"tile{i}: epilogue", ep - of)
    stat(f"tile{i}: total start->epi end", ep - start)
stat("k_full gaps k1-k0", kf[:, 1] - kf[:, 0])
stat("k_full gaps k3-k2", kf[:, 3] - kf[:, 2])
# fine-grained (tile 0, step 1, warps 0 and 3): slot 17 = S_full(step1) for warp 0
sf1 = t[:, 17].astype(float)
for w, off in ((0, 0), (3, 1)):
    a, b_, c, d = (t[:, s + off].astype(float) for s in (10, 12, 14, 34))
    e = t[:, 58 + off].astype(float)
    stat(f"w{w}: S_full->LDTM done", a - sf1)
    stat(f"w{w}: LDTM->own max", e - a)
    stat(f"w{w}: own max->exchange done", b_ - e)
    stat(f"w{w}: max->exp/STTM done", c - b_)
    stat(f"w{w}: exp->wait_st done", d - c)
stat("w3: P arrive - w0 S_full", t[:, 38].astype(float) - sf1)
