for W in C2 C3_w512 C2 C3_w512; do timeout 120 python tools/time_kernels.py $W fwd 2>&1 | tail -1; done
timeout 600 python -m pytest tests/test_gpu_normgate.py tests/test_gpu_attn.py -x -q 2>&1 | tail -2
