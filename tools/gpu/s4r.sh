# Final tree: smoke, full GPU suite, default bench line, C4 N=2 path over gloo (functional).
O=gpurun_out/s4r; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_c2.log 2>&1; grep -c '^{' $O/bench_c2.log
GFWA_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-aux > $O/n2.log 2>&1; echo "n2 rc=$?"; grep -o '"value": [0-9.]*' $O/n2.log | head -2
