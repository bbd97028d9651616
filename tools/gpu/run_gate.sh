mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gate.py tests/test_gpu_attn.py tests/test_gpu_dist.py -x -q 2>&1 | tail -2
python bench.py --no-cpu --steps 5 > gpurun_out/b.log 2>&1; python - <<'P'
import json; d=json.loads(open("gpurun_out/b.log").read().strip().splitlines()[-1]); print(d["ms_breakdown"], d["ms_per_step"]); print(d["aux"]["gate_scan_G"]); print(d["aux"]["gate_preproc_compare_G"]["G_elems_per_s"])
P
