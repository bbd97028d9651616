for W in C2 C3_w512 C2 C3_w512; do timeout 60 python tools/time_kernels.py $W bwd 2>&1 | tail -1; done
timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_dist.py tests/test_gpu_normgate.py -x -q 2>&1 | tail -2
GFWA_LIB=paper_2512_07782_b200/variants/libgfwa_btrace.so timeout 200 python tools/gpu/trace_bwd4.py C2 2>&1 | grep -E "^ +(9|1[0-4]) \||softmax start"
