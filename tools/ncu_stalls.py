"""Stall-reason breakdown (whole kernel and per SASS index range) from an ncu report."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3]) if len(sys.argv) > 3 else 10**9
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; data = rows[2:]
cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
tot = collections.Counter()
for k, r in enumerate(data):
    if lo <= k < hi:
        for i in cols:
            tot[h[i]] += int(r[i] or 0)
s = sum(tot.values())
for n, c in tot.most_common(12):
    print(f"{n:24s} {c/s*100:5.1f}%")
if len(sys.argv) > 4:  # list top instructions in range
    si = h.index("Warp Stall Sampling (All Samples)"); ni = h.index("Source")
    sel = [(int(r[si] or 0), k, r[ni].strip()[:80], {h[i]: int(r[i] or 0) for i in cols}) for k, r in enumerate(data) if lo <= k < hi]
    for smp, k, src, d in sorted(sel, reverse=True)[:int(sys.argv[4])]:
        top = sorted(d.items(), key=lambda x: -x[1])[:2]
        print(f"{smp:6d} {k:5d} {src:80s} {top}")
