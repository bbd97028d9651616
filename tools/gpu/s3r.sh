timeout 600 python -m pytest tests/test_gpu_normgate.py -x -q 2>&1 | tail -2
timeout 300 python - <<'PY'
import sys, torch
sys.path.insert(0, '.')
import bench
print(bench._attn_layer_epilogue(torch.device('cuda')))
PY
