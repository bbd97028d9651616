mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gate.py tests/test_gpu_attn.py tests/test_gpu_graph.py -x -q 2>&1 | tail -2
python tools/time_kernels.py C2 fwd
python tools/time_kernels.py C3_w2048 fwd
GFWA_TRACE_FWD=gpurun_out/fwd.trace python profiles/prof_step.py; python tools/trace_fwd.py gpurun_out/fwd.trace | tail -4; rm -f gpurun_out/fwd.trace
