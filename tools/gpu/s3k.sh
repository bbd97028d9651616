timeout 600 python -m pytest tests/test_gpu_attn.py -x -q -k "many_items or bf16_path" 2>&1 | tail -3
timeout 300 python bench.py --no-cpu --no-aux 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['ms_breakdown'])"
