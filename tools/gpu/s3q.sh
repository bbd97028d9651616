timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_dist.py -x -q 2>&1 | tail -4
for W in C2 C3_w512; do timeout 120 python tools/time_kernels.py $W bwd 2>&1 | tail -1; done
