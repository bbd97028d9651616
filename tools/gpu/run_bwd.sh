mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_dist.py -x -q 2>&1 | tail -1
for i in 1 2 3; do python tools/time_kernels.py C2 bwd; done
GFWA_TRACE_BWD=gpurun_out/bwd.trace python profiles/prof_step.py; python tools/trace_bwd.py gpurun_out/bwd.trace | grep -E "step4|total"; rm -f gpurun_out/bwd.trace
