mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gate.py -x -q 2>&1 | tail -2
for geo in "" "5,7" "2,10" "3,10" "2,9" "4,10"; do
GFWA_GATE_GEOM=$geo ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lg.csv python profiles/prof_gate_lm.py > /dev/null 2>&1
echo "geo=$geo"; python - <<'P'
import csv
rows=list(csv.reader(open("gpurun_out/lg.csv"))); h=[r for r in rows if r and r[0]=="ID"][0]
d=[r for r in rows if len(r)==len(h) and r[0]!="ID"]
ts=[(r[h.index("Kernel Name")], float(r[h.index("Metric Value")])/1e3) for r in d if "gate_prefix" in r[h.index("Kernel Name")]]
# 3 shapes x 3 reps x (fwd, bwd)
for i,shape in enumerate(("C2","C3","C4r")):
    blk=ts[i*6:(i+1)*6]
    f=[t for n,t in blk if "gate_prefix_bwd" not in n]; b=[t for n,t in blk if "gate_prefix_bwd" in n]
    print(f"  {shape}: fwd {min(f):6.2f} us  bwd {min(b):6.2f} us")
P
done
