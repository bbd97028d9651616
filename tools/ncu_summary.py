"""Key details-page metrics of one kernel (by ID) from an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]
kid = sys.argv[2] if len(sys.argv) > 2 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
keep = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Issue Slots Busy",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "Block Limit Registers",
        "Block Limit Shared Mem", "Waves Per SM", "Executed Ipc Active", "Mem Busy", "Max Bandwidth")
for row in r[1:]:
    if row[h.index("ID")] != kid:
        continue
    n = row[h.index("Metric Name")]
    if n in keep:
        print(f"{n:38s} {row[h.index('Metric Value')]} {row[h.index('Metric Unit')]}")
