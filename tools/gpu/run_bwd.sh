mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_dist.py tests/test_gpu_graph.py -x -q 2>&1 | tail -3
python tools/time_kernels.py C2 bwd
GFWA_TRACE_BWD=gpurun_out/bwd.trace python profiles/prof_step.py; python tools/trace_bwd.py gpurun_out/bwd.trace | grep -v "step0\|step2\|step1"; rm -f gpurun_out/bwd.trace
