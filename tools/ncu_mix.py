"""Executed-instruction mix and stall samples grouped by opcode from an ncu report."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; data = rows[2:]
si = h.index("Warp Stall Sampling (All Samples)"); ni = h.index("Source"); ei = h.index("Instructions Executed")
ex = collections.Counter(); st = collections.Counter()
for r in data:
    op = r[ni].strip().split()
    if not op: continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0]
    ex[o] += int(r[ei] or 0); st[o] += int(r[si] or 0)
tot = sum(ex.values()); tots = sum(st.values())
print("total warp-instructions executed", tot)
for o, c in ex.most_common(30):
    print(f"{o:12s} {c:12d} {c/tot*100:5.1f}%   stalls {st[o]/tots*100:5.1f}%")
