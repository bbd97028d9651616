O=gpurun_out/s3m; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1
timeout 600 python bench.py > $O/bench_c2.log 2>&1
tail -3 $O/smoke.log $O/gpu_tests.log
tail -1 $O/bench_c2.log | head -c 3000
