mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_dist.py tests/test_gpu_graph.py -x -q 2>&1 | tail -2
python tools/time_kernels.py C2 bwd
GFWA_TRACE_BWD=gpurun_out/bwd.trace python profiles/prof_step.py; python tools/trace_bwd.py gpurun_out/bwd.trace | grep "epilogue\|total\|start"; rm -f gpurun_out/bwd.trace
