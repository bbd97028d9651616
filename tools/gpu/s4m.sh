# Final check of the session: smoke, full GPU suite, bench lines (C2 with aux incl. the in-kernel halo, C3 w=512).
O=gpurun_out/s4m; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_c2.log 2>&1; tail -c 400 $O/bench_c2.log
timeout 300 python bench.py --workload C3_w512 --no-cpu --no-aux > $O/bench_c3_512.log 2>&1
