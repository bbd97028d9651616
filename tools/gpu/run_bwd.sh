mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attn.py -x -q 2>&1 | tail -1
for a in 0 148 296 148 0; do echo "ahead=$a"; GFWA_BWD_PREFETCH=$a python tools/time_kernels.py C2 bwd; GFWA_BWD_PREFETCH=$a python tools/time_kernels.py C3_w512 bwd; done
GFWA_TRACE_BWD=gpurun_out/bwd.trace python profiles/prof_step.py; python tools/trace_bwd.py gpurun_out/bwd.trace | grep "start\|total\|epilogue"; rm -f gpurun_out/bwd.trace
