timeout 600 python -m pytest tests/test_gpu_normgate.py -x -q 2>&1 | tail -15
timeout 600 python -m pytest tests/test_gpu_attn.py -x -q 2>&1 | tail -2
