"""One-page digest of an ncu --set full report (per kernel ID): speed-of-light,
memory, occupancy, tensor-pipe metrics, stall reasons, hottest SASS lines.

  python tools/ncu_digest.py gpurun_out/r01/bwd.ncu-rep [kernel_index] > profiles/r01/bwd_digest.txt
"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
kid = int(sys.argv[2]) if len(sys.argv) > 2 else 0


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


det = list(csv.reader(run("--page", "details", "--csv").splitlines()))
h = det[0]
rows = [r for r in det[1:] if len(r) >= 15 and r[h.index("ID")] == str(kid)]
print("kernel:", rows[0][h.index("Kernel Name")][:150])
keep = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Registers Per Thread",
        "Block Size", "Grid Size", "Dynamic Shared Memory Per Block", "Theoretical Occupancy",
        "Achieved Occupancy", "Waves Per SM"]
seen = set()
for r in rows:
    n = r[h.index("Metric Name")]
    if n in keep and n not in seen:
        seen.add(n)
        print(f"  {n:38s} {r[h.index('Metric Value')]} {r[h.index('Metric Unit')]}")
raw = list(csv.reader(run("--page", "raw", "--csv").splitlines()))
rh, rv = raw[0], raw[2 + kid]
want = ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum")
for i, n in enumerate(rh):
    if any(n.endswith(w) for w in want):
        print(f"  {n:70s} {rv[i]} {raw[1][i]}")
src = list(csv.reader(run("--page", "source", "--csv", "--print-source=sass").splitlines()))
starts = [i for i, x in enumerate(src) if x and x[0] == "Kernel Name"] + [len(src)]
sh = src[starts[kid] + 1]
srows = [x for x in src[starts[kid] + 2:starts[kid + 1]] if len(x) == len(sh)]
cols = [i for i, n in enumerate(sh) if n.startswith("stall_") and "Not Issued" not in n]
tot = collections.Counter()
for x in srows:
    for i in cols:
        tot[sh[i]] += int(x[i] or 0)
S = sum(tot.values())
print("  stall reasons (all samples):", ", ".join(f"{n[6:]} {c * 100 / S:.0f}%" for n, c in tot.most_common(8)))
si, ie, so = sh.index("Warp Stall Sampling (All Samples)"), sh.index("Instructions Executed"), sh.index("Source")
print("  hottest SASS (samples, executions, top stall):")
for k, x in sorted(enumerate(srows), key=lambda kx: -int(kx[1][si] or 0))[:12]:
    top = max(((int(x[i] or 0), sh[i][6:]) for i in cols))
    print(f"    {k:5d} {int(x[si] or 0):6d} {int(x[ie] or 0):9d} {top[1]:12s} {x[so].strip()[:80]}")
