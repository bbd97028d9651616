"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; data = rows[2:]
si = h.index("Warp Stall Sampling (All Samples)"); ni = h.index("Source"); ai = h.index("Address")
tot = sum(int(r[si]) for r in data if r[si].isdigit())
print("total samples", tot)
idx = {r[ai]: k for k, r in enumerate(data)}
for r in sorted(data, key=lambda r: -int(r[si]) if r[si].isdigit() else 0)[:top]:
    print(f"{int(r[si])/tot*100:5.1f}%  {idx[r[ai]]:5d}  {r[ni].strip()[:90]}")
