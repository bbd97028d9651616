timeout 900 python -m pytest tests/test_gpu_gate.py tests/test_gpu_attn.py::test_end_to_end_from_gate_inputs -x -q 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lg.csv python profiles/prof_gate.py > /dev/null 2>&1; python tools/ncu_launches.py gpurun_out/lg.csv | grep gate
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lg2.csv python profiles/prof_gate_lm.py > /dev/null 2>&1; python tools/ncu_launches.py gpurun_out/lg2.csv | grep gate
