timeout 300 python -m pytest tests/test_gpu_decode.py -q -x 2>&1 | tail -1
python bench.py --no-cpu --steps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['aux']['decode_C5'], d['aux']['decode_C5_gqa4'])"
