"""Per-SASS-instruction executed counts and stall samples for the first kernel
in an ncu report; prints the total and the top-N instructions plus a
histogram by opcode."""
import collections, csv, subprocess, sys
rep = sys.argv[1]
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
kern = int(sys.argv[3]) if len(sys.argv) > 3 else 0
starts = [i for i, x in enumerate(r) if x and x[0] == "Kernel Name"] + [len(r)]
print(r[starts[kern]][1][:100])
rows = [x for x in r[starts[kern] + 2:starts[kern + 1]] if len(x) == len(h)]
ie, src, smp = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(x[ie] or 0) for x in rows)
print("total warp instructions", tot)
ops = collections.Counter()
for x in rows:
    op = x[src].strip().split()
    op = [t for t in op if not t.startswith("@")]
    ops[op[0].split(".")[0] if op else "?"] += int(x[ie] or 0)
for o, c in ops.most_common(25):
    print(f"  {o:12s} {c:12d} {c / tot * 100:5.1f}%")
for k, x in sorted(enumerate(rows), key=lambda kx: -int(kx[1][smp] or 0))[:topn]:
    print(f"{k:5d} {int(x[ie] or 0):10d} {int(x[smp] or 0):6d}  {x[src].strip()[:90]}")
