timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python bench.py --no-cpu --steps 10 > gpurun_out/b.log 2>&1; python - <<'P'
import json; d=json.loads(open("gpurun_out/b.log").read().strip().splitlines()[-1]); print(d["ms_breakdown"], d["ms_per_step"], d["value"]); print(d["aux"]["gate_scan_G"]); print(d["aux"]["gate_preproc_compare_G"]); print(d["aux"]["decode_C5_gqa4"])
P
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lg.csv python profiles/prof_gate.py > /dev/null 2>&1; python tools/ncu_launches.py gpurun_out/lg.csv | grep gate
